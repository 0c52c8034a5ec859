"""Parity at BASELINE.json's full sizes (the bench workloads): a head and a
tail slice of orbits against the oracle (tail slices exercise global orbit
ids deep into the run), plus size-independent properties over every orbit --
repeatability, shard / tiling invariance (store hashes), and the fused
order parameter equal to the one of the stored trajectory."""

import dataclasses

import numpy as np
import pytest

import bench
import paper_1908_03869_b200 as sdb
from conftest import PARITY_TOL
from oracle import sdeb_oracle as O
from paper_1908_03869_b200.engine import EngineConfig, run_batch

pytestmark = pytest.mark.gpu


def _setup(name, **over):
    w = dict(bench.WORKLOADS[name], **over)
    model = bench.make_model(sdb, w)
    batch = bench.make_batch(sdb, w, 0)
    cfg = EngineConfig(dt=w["dt"], tspan=w["dt"] * w["steps"], ksteps=w["ksteps"],
                       orbits=w["orbits"], solver=w["solver"], seed=20260809, stream=w["stream"],
                       max_store_bytes=1 << 40)
    return w, model, batch, cfg


def _oracle_rows(w, batch, cfg, rows):
    chunks = w["steps"] // w["ksteps"]
    nnoise = 0 if w["solver"] == "rk4" else w["n"]
    _, values, fails = O.integrate(batch.init[rows], batch.params[rows], dt=w["dt"],
                                   ksteps=w["ksteps"], chunks=chunks, seed=cfg.seed,
                                   solver=w["solver"], nnoise=nnoise, stream=cfg.stream,
                                   orbit_ids=np.asarray(rows, dtype=np.uint64))
    return values


@pytest.mark.parametrize("name, slice_len", [("cfg2", 24), ("cfg5", 12), ("cfg4", 4),
                                              ("cfg3_n32", 8)])
def test_full_size_head_and_tail_match_oracle(name, slice_len):
    w, model, batch, cfg = _setup(name)
    store = run_batch(model, cfg, batch)
    m = w["orbits"]
    rows = list(range(slice_len)) + list(range(m - slice_len, m))
    want = _oracle_rows(w, batch, cfg, rows)
    err = O.mixed_error(store.values[rows], want)
    assert err <= PARITY_TOL, "%s: %.3e" % (name, err)
    assert np.isfinite(store.values).all() and not store.failures


def test_full_size_cfg3_n256_slice():
    # 2^20 orbits of 256 oscillators (4.3 GB of parameters), 100 steps
    w, model, batch, cfg = _setup("cfg3_n256")
    store = run_batch(model, cfg, batch)
    m = w["orbits"]
    rows = [0, 1, m // 2, m - 1]
    want = _oracle_rows(w, batch, cfg, rows)
    assert O.mixed_error(store.values[rows], want) <= PARITY_TOL
    assert store.values.shape == (m, 2, 256) and np.isfinite(store.values).all()


def test_full_size_cfg2_invariances(monkeypatch):
    w, model, batch, cfg = _setup("cfg2")
    ref = sdb.store_hash(run_batch(model, cfg, batch))
    assert sdb.store_hash(run_batch(model, cfg, batch)) == ref          # repeatable
    assert sdb.store_hash(run_batch(model, dataclasses.replace(cfg, devices=(0, 0)),
                                    batch)) == ref                         # 2 shards
    monkeypatch.setenv("SDEB200_TILES", "4")
    assert sdb.store_hash(run_batch(model, cfg, batch)) == ref            # 4 tiles


def test_full_size_cfg5_fused_coherence_equals_store():
    w, model, batch, cfg = _setup("cfg5")
    store = run_batch(model, cfg, batch)
    post = sdb.coherence_series(store)
    fused = sdb.run_coherence(model, cfg, batch)
    assert np.array_equal(post.r, fused.r) and np.array_equal(post.phi, fused.phi)
    assert fused.r.shape == (w["orbits"], w["steps"] // w["ksteps"] + 1)
