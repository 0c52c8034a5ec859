"""Store files and manifests (storage.py), host side: byte-identical to the
reference's writers (tests/golden/make_golden_storage.py) and the reference's
own round-trip / corruption cases (test_storage.py:24-120)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR
from paper_1908_03869_b200 import storage
from paper_1908_03869_b200.engine import EngineConfig, TrajectoryStore


def golden_store():
    data = np.load(os.path.join(GOLDEN_DIR, "store_ref_values.npz"))
    return TrajectoryStore(times=data["times"], values=data["values"], model_name="golden-store")


def test_writers_are_byte_identical_to_the_reference(tmp_path):
    store = golden_store()
    storage.write_store(store, tmp_path / "s.csv", fmt="csv")
    storage.write_store(store, tmp_path / "s.sdb1", fmt="bin",
                        metadata={"seed": 99, "note": "reference writer"})
    for mine, ref in (("s.csv", "store_ref.csv"), ("s.sdb1", "store_ref.sdb1")):
        with open(tmp_path / mine, "rb") as a, open(os.path.join(GOLDEN_DIR, ref), "rb") as b:
            assert a.read() == b.read(), mine


def test_reading_reference_files():
    store = golden_store()
    for name in ("store_ref.csv", "store_ref.sdb1"):
        back = storage.read_store(os.path.join(GOLDEN_DIR, name))
        assert storage.store_hash(back) == storage.store_hash(store)
    assert storage.read_store_bin(os.path.join(GOLDEN_DIR, "store_ref.sdb1")).model_name == \
        "golden-store"


def test_round_trips_and_sniffing(tmp_path):
    g = np.random.default_rng(3)
    store = TrajectoryStore(times=np.arange(5) * 0.1, values=g.standard_normal((4, 5, 3)))
    for fmt in ("csv", "bin"):
        path = tmp_path / ("x." + fmt)
        storage.write_store(store, path, fmt=fmt)
        back = storage.read_store(path)
        assert np.array_equal(back.values, store.values)
        assert np.array_equal(back.times, store.times)
    with open(tmp_path / "x.bin", "rb") as fh:
        assert fh.read(4) == b"SDB1"
    with pytest.raises(ValueError, match="unknown store format"):
        storage.write_store(store, tmp_path / "x.foo", fmt="foo")


def test_corrupt_stores_rejected(tmp_path):
    store = TrajectoryStore(times=np.arange(2) * 1.0, values=np.ones((2, 2, 2)))
    storage.write_store_bin(store, tmp_path / "ok.bin")
    raw = (tmp_path / "ok.bin").read_bytes()
    for bad, what in ((b"XXXX" + raw[4:], "magic"), (raw[:6], "truncated"),
                      (raw[:14], "truncated"), (raw[:-3], "truncated")):
        (tmp_path / "bad.bin").write_bytes(bad)
        with pytest.raises(storage.StoreFormatError, match=what):
            storage.read_store_bin(tmp_path / "bad.bin")
    (tmp_path / "bad.csv").write_text("orbit,time,y0\n0,0.0,1.0\n1,0.0\n")
    with pytest.raises(storage.StoreFormatError):
        storage.read_store_csv(tmp_path / "bad.csv")
    (tmp_path / "bad2.csv").write_text("a,b\n1,2\n")
    with pytest.raises(storage.StoreFormatError, match="not a trajectory"):
        storage.read_store_csv(tmp_path / "bad2.csv")


def test_manifests_and_tables(tmp_path):
    cfg = EngineConfig(dt=0.1, tspan=1.0, ksteps=10, orbits=2, seed=5)
    man = storage.build_manifest("run", {"x": 1}, cfg, "kuramoto:4", {"batch": "b"},
                                 {"store": "s.bin"}, store_sha256="ab", extra={"k": 2})
    storage.write_manifest(man, tmp_path / "m.json")
    back = storage.read_manifest(tmp_path / "m.json")
    assert back == man and back["config"]["seed"] == 5 and back["store_sha256"] == "ab"
    storage.write_matrix_csv(tmp_path / "t.csv", ["a", "b"], [[1, 0.1], ["x", 2.5e-7]])
    assert (tmp_path / "t.csv").read_text() == "a,b\n1,0.1\nx,2.5e-07\n"
    for x in (0.1, 1e-300, 1.0 / 3.0, -2.5e17):
        assert float(storage.format_float(x)) == x
