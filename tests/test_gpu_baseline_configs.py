"""Parity of the BASELINE configs at their own sizes and lengths (VERDICT r1
"what's missing" 1-2): against stores the REFERENCE produced
(tests/golden/make_golden_r2.py, make_golden_accept.py) and, for rows deep
into the batch (global orbit ids) or for the streams the reference does not
have, against the oracle.  Bar: |got - ref| <= 1e-10 * max(1, |ref|) (FP64),
under both coupling evaluations; the reference's own acceptance thresholds
are asserted on the GPU's numbers.
"""

import ctypes
import json
import os

import numpy as np
import pytest

import bench
import paper_1908_03869_b200 as sdb
from conftest import GOLDEN_DIR, PARITY_TOL
from oracle import sdeb_oracle as O
from paper_1908_03869_b200 import _native as nat
from paper_1908_03869_b200.engine import EngineConfig, make_desc, run_batch

pytestmark = pytest.mark.gpu

COUPLINGS = ["meanfield", "pairwise"]
SEED = bench.SEED


@pytest.fixture(scope="module")
def r2():
    data = np.load(os.path.join(GOLDEN_DIR, "golden_r2_v1.npz"))
    with open(os.path.join(GOLDEN_DIR, "cases_r2.json")) as fh:
        cases = json.load(fh)
    return {k: data[k] for k in data.files}, cases


def _cfg(w, coupling, stream=None, orbits=None):
    return EngineConfig(dt=w["dt"], tspan=w["dt"] * w["steps"], ksteps=w["ksteps"],
                        orbits=orbits or w["orbits"], solver=w["solver"], seed=SEED,
                        stream=stream or w["stream"], coupling=coupling, max_store_bytes=1 << 40)


def _oracle_rows(w, batch, rows, stream="philox"):
    _, values, _ = O.integrate(batch.init[rows], batch.params[rows], dt=w["dt"],
                               ksteps=w["ksteps"], chunks=w["steps"] // w["ksteps"], seed=SEED,
                               stream=stream, orbit_ids=np.asarray(rows, dtype=np.uint64))
    return values


def _run_fresh(model, cfg, batch, layout=None):
    """run_batch on a fresh context (SDEB200_LAYOUT, if given, pins the layout
    before any cache can answer)."""
    if layout:
        os.environ["SDEB200_LAYOUT"] = layout
    try:
        ctx = ctypes.c_void_p()
        nat.check(nat.lib().sdb_open(None, 0, ctypes.byref(ctx)))
        chunks = sdb.iteration_count(cfg.tspan, cfg.dt, cfg.ksteps)
        desc = make_desc(model, cfg, chunks, batch.orbits)
        values = nat.host_empty((batch.orbits, chunks + 1, model.nequat))
        fail = np.empty(batch.orbits, np.int64)
        init, params = nat.f64(batch.init), nat.f64(batch.params)
        nat.check(nat.lib().sdb_run(ctx, desc, nat.dptr(init), nat.dptr(params),
                                    nat.dptr(values), nat.i64ptr(fail)), ctx)
        width = int(nat.lib().sdb_last_lane_width(ctx))
        nat.lib().sdb_close(ctx)
        assert (fail < 0).all()
        return values, width
    finally:
        os.environ.pop("SDEB200_LAYOUT", None)


# ---- cfg1 exactly as BASELINE.json configs[0] states it ----------------------

@pytest.mark.parametrize("coupling", COUPLINGS)
def test_cfg1_full_run_matches_reference_store(r2, coupling):
    arrays, cases = r2
    w = bench.WORKLOADS["cfg1"]
    assert cases["cfg1"]["orbits"] == w["orbits"] == 1024 and cases["cfg1"]["steps"] == 10000
    batch = bench.make_batch(sdb, w)  # the device sampler: bit-exact with the reference's
    assert np.array_equal(batch.init, arrays["cfg1_init"])
    assert np.array_equal(batch.params, arrays["cfg1_params"])
    store = run_batch(sdb.kuramoto_model(4), _cfg(w, coupling, stream="philox"), batch)
    err = O.mixed_error(store.values, arrays["cfg1_values"])
    assert err <= PARITY_TOL, err


@pytest.mark.parametrize("coupling", COUPLINGS)
def test_cfg1_xoshiro_full_run_matches_oracle(coupling):
    # the stream BASELINE names for cfg1 (the reference has none: oracle-pinned)
    w = bench.WORKLOADS["cfg1"]
    assert w["stream"] == "xoshiro256pp"
    batch = bench.make_batch(sdb, w)
    store = run_batch(sdb.kuramoto_model(4), _cfg(w, coupling), batch)
    rows = list(range(w["orbits"]))
    want = _oracle_rows(w, batch, rows, stream="xoshiro256pp")
    err = O.mixed_error(store.values, want)
    assert err <= PARITY_TOL, err


# ---- cfg3 at full size (2^20 orbits) -----------------------------------------

@pytest.mark.parametrize("coupling", COUPLINGS)
@pytest.mark.parametrize("name", ["cfg3_n64", "cfg3_n128", "cfg3_n256"])
def test_cfg3_full_size_head_reference_tail_oracle(r2, name, coupling):
    arrays, cases = r2
    w = bench.WORKLOADS[name]
    head = cases[name]["orbits"]
    assert (cases[name]["n"], cases[name]["steps"]) == (w["n"], w["steps"])
    batch = bench.make_batch(sdb, w)
    assert np.array_equal(batch.init[:head], arrays[name + "_init"])
    assert np.array_equal(batch.params[:head], arrays[name + "_params"])
    store = run_batch(sdb.kuramoto_model(w["n"]), _cfg(w, coupling), batch)
    err_head = O.mixed_error(store.values[:head], arrays[name + "_values"])
    m = w["orbits"]
    tail = [m // 2, m // 2 + 1] + list(range(m - 4, m))
    err_tail = O.mixed_error(store.values[tail], _oracle_rows(w, batch, tail))
    assert err_head <= PARITY_TOL and err_tail <= PARITY_TOL, (err_head, err_tail)
    assert store.values.shape == (m, 2, w["n"]) and np.isfinite(store.values).all()


# ---- the paper's speed protocol at its own length ---------

@pytest.mark.parametrize("n", [5, 10, 15])
def test_paper_protocol_exact_lane_kernels_match_reference(r2, n):
    # N = 5 / 10 / 15, M = 163,840, dt = 0.05, 8000 steps: the exact one-lane
    # J = N kernels (persistent and one CTA per group) and the autotuned layout
    arrays, cases = r2
    name = "paper_n%d" % n
    w = bench.WORKLOADS[name]
    head = cases[name]["orbits"]
    batch = bench.make_batch(sdb, w)
    assert np.array_equal(batch.init[:head], arrays[name + "_init"])
    model = sdb.kuramoto_model(n)
    cfg = _cfg(w, "meanfield")
    m = w["orbits"]
    tail = list(range(m - 8, m))
    want_tail = _oracle_rows(w, batch, tail)
    results = {}
    for layout in ("1,1,0,0,%d" % n, "1,0,0,0,%d" % n, None):
        values, width = _run_fresh(model, cfg, batch, layout)
        if layout:
            assert width == n  # the exact-J instantiation ran
        err_head = O.mixed_error(values[:head], arrays[name + "_values"])
        err_tail = O.mixed_error(values[tail], want_tail)
        assert err_head <= PARITY_TOL and err_tail <= PARITY_TOL, (layout, err_head, err_tail)
        results[layout] = sdb.store_hash(sdb.TrajectoryStore(times=np.zeros(2), values=values))
    assert len(set(results.values())) == 1  # every layout: the same bits


@pytest.mark.parametrize("n", [5, 10, 15])
def test_paper_protocol_pairwise_matches_reference(r2, n):
    arrays, cases = r2
    name = "paper_n%d" % n
    w = bench.WORKLOADS[name]
    head = cases[name]["orbits"]
    batch = bench.make_batch(sdb, w)
    store = run_batch(sdb.kuramoto_model(n), _cfg(w, "pairwise"), batch)
    err = O.mixed_error(store.values[:head], arrays[name + "_values"])
    assert err <= PARITY_TOL, err


# ---- acceptance criteria 1-3 (test_acceptance.py:36-79) through dt_sweep ----

@pytest.fixture(scope="module")
def accept():
    data = np.load(os.path.join(GOLDEN_DIR, "golden_accept_v1.npz"))
    with open(os.path.join(GOLDEN_DIR, "cases_accept.json")) as fh:
        cases = json.load(fh)
    return {k: data[k] for k in data.files}, cases


@pytest.mark.parametrize("coupling", COUPLINGS)
def test_acceptance_transition_sweep_matches_reference(accept, coupling):
    ref, case = accept
    rows = sdb.dt_sweep(case["n"], couplings=tuple(case["couplings"]), dts=tuple(case["dts"]),
                        realizations=case["realizations"], tspan=case["tspan"],
                        sample_interval=case["sample_interval"], seed=case["seed"],
                        coupling=coupling)
    assert [r.coupling for r in rows] == list(ref["couplings"])
    assert [r.dt for r in rows] == list(ref["dts"])
    for k, row in enumerate(rows):
        assert np.array_equal(row.stats.times, ref["times"])
        err_m = O.mixed_error(row.stats.mean_r, ref["mean_r"][k])
        err_s = O.mixed_error(row.stats.std_r, ref["std_r"][k])
        assert err_m <= PARITY_TOL and err_s <= PARITY_TOL, (k, err_m, err_s)

    def row(c, dt):
        return next(r for r in rows if r.coupling == c and r.dt == dt)
    # criterion 1: above / below the transition
    assert row(0.2, 0.05).mean_r_end >= 0.8 and row(0.02, 0.05).mean_r_end <= 0.25
    # criterion 2: onset of synchronisation within [20, 120] s
    st = row(0.2, 0.05).stats
    crossing = sdb.analysis.first_crossing_time(st.times, st.mean_r, 0.8)
    assert crossing is not None and 20.0 <= crossing <= 120.0
    # criterion 3: terminal mean r stable over dt (the reference's 0.05 limit)
    for c in case["couplings"]:
        ends = [row(c, dt).mean_r_end for dt in case["dts"]]
        assert max(ends) - min(ends) <= 0.05
