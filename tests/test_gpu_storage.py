"""The streaming SDB1 writer (storage.run_batch_to_file, sdb_run_to_file):
byte-identical to write_store_bin(run_batch(...)) for the Kuramoto stepper
and a generated program, across device shards and host-pipeline tilings."""

import dataclasses

import numpy as np
import pytest

import paper_1908_03869_b200 as sdb
from paper_1908_03869_b200 import storage
from paper_1908_03869_b200.engine import EngineConfig, run_batch
from paper_1908_03869_b200.model import OrbitBatch

pytestmark = pytest.mark.gpu


def _same_file(tmp_path, model, cfg, batch, meta):
    ref = run_batch(model, cfg, batch)
    storage.write_store_bin(ref, tmp_path / "ref.sdb1", meta)
    fails = storage.run_batch_to_file(model, cfg, batch, tmp_path / "stream.sdb1", meta)
    assert (tmp_path / "ref.sdb1").read_bytes() == (tmp_path / "stream.sdb1").read_bytes()
    assert fails == ref.failures
    return ref


@pytest.mark.parametrize("stream", ["philox", "sfc64"])
def test_stream_to_file_kuramoto(tmp_path, stream, monkeypatch):
    n, m = 16, 777
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.3, seed=2)
    params = batch.params.copy()
    params[500, 3] = np.inf  # a failing orbit (inf frequency: non-finite at step 0)
    batch = OrbitBatch(init=batch.init, params=params)
    cfg = EngineConfig(dt=1e-2, tspan=1.0, ksteps=10, orbits=m, seed=6, stream=stream)
    ref = _same_file(tmp_path, sdb.kuramoto_model(n), cfg, batch, {"run": "k"})
    assert ref.failures and ref.failures[0].orbit == 500
    _same_file(tmp_path, sdb.kuramoto_model(n), dataclasses.replace(cfg, devices=(0, 0, 0)),
               batch, {"run": "k"})
    monkeypatch.setenv("SDEB200_TILES", "5")
    monkeypatch.setenv("SDEB200_PIECE_KB", "16")
    monkeypatch.setenv("SDEB200_HOST_THREADS", "4")
    _same_file(tmp_path, sdb.kuramoto_model(n), cfg, batch, None)
    back = storage.read_store(tmp_path / "stream.sdb1")
    assert sdb.store_hash(back) == sdb.store_hash(ref)


def test_stream_to_file_expression_model(tmp_path):
    model = sdb.model_from_dsl("ou", 3, 5, 3, "p[0]*(p[1] - y[i])", "p[2 + i]*n[i]")
    g = np.random.default_rng(4)
    batch = OrbitBatch(init=g.standard_normal((50, 3)), params=g.uniform(0.1, 0.9, (50, 5)))
    cfg = EngineConfig(dt=0.01, tspan=0.5, ksteps=5, orbits=50, seed=1)
    _same_file(tmp_path, model, cfg, batch, {"model": "ou"})


def test_stream_to_file_ignores_the_in_memory_cap(tmp_path):
    n, m = 4, 64
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.3, seed=2)
    cfg = EngineConfig(dt=0.1, tspan=1.0, ksteps=1, orbits=m, max_store_bytes=100)
    with pytest.raises(sdb.ConfigError):
        run_batch(sdb.kuramoto_model(n), cfg, batch)
    storage.run_batch_to_file(sdb.kuramoto_model(n), cfg, batch, tmp_path / "big.sdb1")
    assert storage.read_store(tmp_path / "big.sdb1").values.shape == (m, 11, n)
