"""CPU-tier tests of the host side: the drop-in API surface, validation that
must happen before any device work (in the reference's order and with its
messages -- /root/reference/pkg/tests/test_engine.py:23-97), the C-ABI
library loading and symbol exports, and loud failure without a GPU."""

import ctypes
import dataclasses
import os
import re

import numpy as np
import pytest

import paper_1908_03869_b200 as sdb
from paper_1908_03869_b200 import _native as nat
from paper_1908_03869_b200.engine import (ConfigError, EngineConfig, iteration_count,
                                          make_desc, partition_orbits, run_batch)
from paper_1908_03869_b200.model import ModelSpec, OrbitBatch, kuramoto_signature

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sdeb200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sdb_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(nat.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(nat.SIGNATURES), "ctypes table out of sync with sdeb200.h"


def test_library_loads_without_gpu():
    lib = nat.lib()
    assert lib.sdb_abi_version() == 2
    assert lib.sdb_device_count() >= 0


def test_descriptor_layout_matches_header():
    # sdb_desc: 8 x int32 + uint64 + double + 4 x int64
    assert ctypes.sizeof(nat.SdbDesc) == 8 * 4 + 8 + 8 + 4 * 8


# ---- reference test_engine.py config tests, re-pointed ------------------------

def test_iteration_count_protocol_values():
    assert iteration_count(400.0, 0.05, 40) == 200
    assert iteration_count(2.0, 0.05, 40) == 1
    assert iteration_count(1.0, 0.0125, 80) == 1
    assert iteration_count(400.0, 0.2, 10) == 200
    with pytest.raises(ConfigError, match="not an integer multiple"):
        iteration_count(400.0, 0.05, 7)
    assert iteration_count(1.0, 0.3, 1, pad=True) == 4
    assert iteration_count(400.0, 0.05, 7, pad=True) == 1143
    with pytest.raises(ConfigError):
        iteration_count(0.0, 0.05, 40)


def test_partition_examples():
    assert partition_orbits(10, 4) == [range(0, 4), range(4, 8), range(8, 10)]
    assert len(partition_orbits(512, 8)) == 64
    assert [i for p in partition_orbits(37, 5) for i in p] == list(range(37))


def test_config_validation_messages():
    with pytest.raises(ConfigError, match="dt must be positive"):
        EngineConfig(dt=0.0, tspan=1.0, ksteps=1, orbits=1)
    with pytest.raises(ConfigError, match="tspan must be positive"):
        EngineConfig(dt=0.1, tspan=-1.0, ksteps=1, orbits=1)
    with pytest.raises(ConfigError, match="ksteps"):
        EngineConfig(dt=0.1, tspan=1.0, ksteps=0, orbits=1)
    with pytest.raises(ConfigError, match="threads"):
        EngineConfig(dt=0.1, tspan=1.0, ksteps=1, orbits=1, threads=0)
    with pytest.raises(ValueError, match="unknown solver"):
        EngineConfig(dt=0.1, tspan=1.0, ksteps=1, orbits=1, solver="milstein")
    with pytest.raises(ConfigError, match="stream"):
        EngineConfig(dt=0.1, tspan=1.0, ksteps=1, orbits=1, stream="mt19937")
    with pytest.raises(ConfigError, match="coupling"):
        EngineConfig(dt=0.1, tspan=1.0, ksteps=1, orbits=1, coupling="fft")
    with pytest.raises(ConfigError, match="lanes"):
        EngineConfig(dt=0.1, tspan=1.0, ksteps=1, orbits=1, lanes=3)


def _batch(n, m):
    return OrbitBatch(init=np.zeros((m, n)), params=np.zeros((m, 2 * n + 1)))


def test_validation_precedes_device_work():
    # these raise the reference's errors even on a machine without a GPU
    m = sdb.kuramoto_model(3)
    with pytest.raises(ConfigError, match="deterministic"):
        run_batch(m, EngineConfig(dt=0.1, tspan=1.0, ksteps=10, orbits=2, solver="rk4"),
                  _batch(3, 2))
    with pytest.raises(ConfigError, match="above the configured cap"):
        run_batch(sdb.kuramoto_model(5),
                  EngineConfig(dt=0.05, tspan=10.0, ksteps=20, orbits=16, max_store_bytes=100),
                  _batch(5, 16))
    with pytest.raises(ConfigError, match="orbits"):
        run_batch(m, EngineConfig(dt=0.1, tspan=1.0, ksteps=10, orbits=5), _batch(3, 4))
    with pytest.raises(ValueError, match="columns"):
        run_batch(sdb.kuramoto_model(4), EngineConfig(dt=0.1, tspan=1.0, ksteps=10, orbits=4),
                  _batch(3, 4))


def test_unsupported_models_raise_not_implemented():
    lam = ModelSpec(name="decay", nequat=1, nparams=0, nnoise=0, drift=lambda t, y, p: -y)
    cfg = EngineConfig(dt=0.1, tspan=1.0, ksteps=10, orbits=1)
    with pytest.raises(NotImplementedError):
        run_batch(lam, cfg, OrbitBatch(init=np.ones((1, 1)), params=np.empty((1, 0))))
    # expression templates are compiled (program.py), not rejected
    assert sdb.model.expression_model(sdb.model_from_dsl("x", 1, 1, 0, "0 - p[0]*y[0]", "0"))
    ode = ModelSpec(name="k0", nequat=2, nparams=5, nnoise=0, drift=sdb.model._kuramoto_drift)
    with pytest.raises(NotImplementedError):
        run_batch(ode, EngineConfig(dt=0.1, tspan=1.0, ksteps=10, orbits=1, solver="ie"),
                  OrbitBatch(init=np.zeros((1, 2)), params=np.zeros((1, 5))))


def test_kuramoto_recognition():
    assert kuramoto_signature(sdb.kuramoto_model(7)) == (7, 7)
    assert kuramoto_signature(sdb.kuramoto_dsl_model(7)) == (7, 7)
    ode = ModelSpec(name="k0", nequat=8, nparams=17, nnoise=0,
                    drift=sdb.model._kuramoto_drift)
    assert kuramoto_signature(ode) == (8, 0)
    dsl0 = sdb.model_from_dsl("k0", 8, 17, 0, sdb.model.KURAMOTO_DRIFT_TEMPLATE, "0")
    assert kuramoto_signature(dsl0) == (8, 0)
    bad = ModelSpec(name="k", nequat=8, nparams=16, nnoise=8, drift=sdb.model._kuramoto_drift,
                    diffusion=sdb.model._kuramoto_diffusion)
    assert kuramoto_signature(bad) is None


def test_model_api_mirrors_reference():
    m = sdb.kuramoto_model(5)
    assert (m.nequat, m.nnoise, m.nparams) == (5, 5, 11)
    assert sdb.kuramoto_model(100).nparams == 201
    with pytest.raises(sdb.ModelDefinitionError):
        sdb.kuramoto_model(0)
    assert sdb.model_from_name("kuramoto:7").nequat == 7
    for bad in ("kuramoto", "kuramoto:", "kuramoto:x", "lorenz:3"):
        with pytest.raises(sdb.ModelDefinitionError):
            sdb.model_from_name(bad)
    with pytest.raises(ValueError):
        OrbitBatch(init=np.zeros((2, 3)), params=np.zeros((3, 5)))


def test_make_desc_fields():
    m = sdb.kuramoto_model(16)
    cfg = EngineConfig(dt=1e-3, tspan=10.0, ksteps=10000, orbits=65536, seed=-5,
                       stream="sfc64", coupling="pairwise", lanes=4)
    d = make_desc(m, cfg, chunks=1, orbits=65536, orbit_offset=7)
    assert (d.nequat, d.nparams, d.nnoise) == (16, 33, 16)
    assert (d.solver, d.stream, d.coupling, d.lanes) == (0, 1, 1, 4)
    assert d.seed == 2 ** 64 - 5
    assert (d.ksteps, d.chunks, d.orbits, d.orbit_offset) == (10000, 1, 65536, 7)


def test_failures_from_steps():
    from paper_1908_03869_b200.engine import failures_from_steps
    f = failures_from_steps(np.array([-1, 0, 7, -1]), ksteps=2, dt=0.5)
    assert [(x.orbit, x.chunk, x.step, x.time) for x in f] == [(1, 0, 0, 0.0), (2, 3, 1, 3.5)]
    assert all("non-finite" in x.reason for x in f)


@pytest.mark.skipif(nat.device_count() > 0, reason="checks the no-GPU behaviour")
def test_device_path_fails_loudly_without_gpu():
    m = sdb.kuramoto_model(2)
    cfg = EngineConfig(dt=0.1, tspan=1.0, ksteps=10, orbits=1)
    with pytest.raises(RuntimeError, match="CUDA device"):
        run_batch(m, cfg, OrbitBatch(init=np.zeros((1, 2)), params=np.zeros((1, 5))))
    with pytest.raises(RuntimeError):
        sdb.rng.normals_for_step(0, 0, 0, 0, 4)


def test_kuramoto_recognised_by_identity_not_name():
    # a user's own callables that happen to share the built-in names (e.g. a
    # phase-lag variant in their own model.py) must not be routed to the stepper
    def _kuramoto_drift(t, y, p):
        return y

    def _kuramoto_diffusion(t, y, p, noise):
        return noise
    _kuramoto_drift.__module__ = _kuramoto_diffusion.__module__ = "model"
    user = ModelSpec(name="lag", nequat=4, nparams=9, nnoise=4, drift=_kuramoto_drift,
                     diffusion=_kuramoto_diffusion)
    assert kuramoto_signature(user) is None
    with pytest.raises(NotImplementedError):
        sdb.model.require_device_model(user)


def test_sharded_run_with_more_ranks_than_orbits_gives_empty_shards():
    # world > orbits: the ranks with nothing to do still join the gather with
    # an empty part instead of raising before the collective (a hang)
    m = sdb.kuramoto_model(3)
    cfg = EngineConfig(dt=0.5, tspan=1.0, ksteps=1, orbits=3)
    batch = OrbitBatch(init=np.zeros((3, 3)), params=np.zeros((3, 7)))
    seen = []

    def gather(part):
        seen.append(part)
        return [part]
    store = sdb.engine.run_batch_sharded(m, cfg, batch, world=4, rank=0, gather=gather)
    assert sdb.engine.shard_bounds(3, 4, 0) == (0, 0)
    assert store.values.shape == (0, 3, 3) and store.failures == []
    assert seen and seen[0][0] == 0 and seen[0][1].shape == (0, 3, 3)
    # an invalid configuration raises on every rank before the collective
    with pytest.raises(sdb.ConfigError):
        sdb.engine.run_batch_sharded(m, dataclasses.replace(cfg, orbits=4), batch, world=4,
                                     rank=0, gather=gather)
    assert len(seen) == 1


def test_run_batch_to_file_checks_indices_before_touching_the_file(tmp_path):
    from paper_1908_03869_b200 import dsl, storage
    path = tmp_path / "keep.sdb1"
    path.write_bytes(b"existing store")
    bad = sdb.model_from_dsl("oob", 2, 1, 0, "p[i] * y[i]", "0")  # p has 1 column, i reaches 1
    cfg = EngineConfig(dt=0.1, tspan=0.2, ksteps=1, orbits=2, solver="euler")
    with pytest.raises(dsl.DomainError):
        storage.run_batch_to_file(bad, cfg, OrbitBatch(init=np.zeros((2, 2)),
                                                       params=np.zeros((2, 1))), path)
    assert path.read_bytes() == b"existing store"


def test_kernel_resource_table_from_ptxas(tmp_path, monkeypatch):
    # the build turns ptxas -v output into the occupancy table the layout
    # autotuner reads instead of loading kernel modules (_build.py)
    from paper_1908_03869_b200 import _build
    obj = tmp_path / "k.o"
    (tmp_path / "k.o.ptxas").write_text(
        "ptxas info    : Compiling entry function "
        "'_ZN4sdeb19kuramoto_run_kernelILi16ELi0ELi0ELi0ELi2EEEvNS_7RunArgsE' for 'sm_100a'\n"
        "ptxas info    : Function properties for x\n"
        "    0 bytes stack frame, 0 bytes spill stores, 0 bytes spill loads\n"
        "ptxas info    : Used 166 registers, used 1 barriers, 24592 bytes smem, 1024 bytes cmem\n")
    out = tmp_path / "table.inc"
    monkeypatch.setattr(_build, "KERNEL_TABLE", str(out))
    _build._write_kernel_table([str(obj)])
    text = out.read_text()
    assert "{16, 0, 0, 0, 2, 166, 24592}," in text and text.rstrip().endswith("};")
    # the real table of this build covers every lane width's default kernel
    real = open(os.path.join(os.path.dirname(_build.LIB), "_obj", "sdeb_kernel_table.inc")).read()
    for J in (1, 2, 4, 8, 16, 3, 5, 15):
        assert "{%d, 0, 0, 0, 0, " % J in real, J
