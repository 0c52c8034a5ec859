"""GPU parity of the analysis row: the device order parameter
(post-hoc kernel and the fused run) against the reference's own outputs
(tests/golden/make_golden_analysis.py) and against each other (bitwise)."""

import dataclasses
import math

import numpy as np
import pytest

import paper_1908_03869_b200 as sdb
from conftest import PARITY_TOL
from oracle import sdeb_oracle as O
from paper_1908_03869_b200 import analysis
from paper_1908_03869_b200.engine import EngineConfig, last_launch_info, run_batch
from paper_1908_03869_b200.model import OrbitBatch

pytestmark = pytest.mark.gpu


def phase_err(a, b):
    """max |wrap(a - b)|: Phi near -pi and +pi are the same angle."""
    d = np.asarray(analysis.wrap_phase(np.asarray(a) - np.asarray(b)))
    return float(np.max(np.abs(d))) if d.size else 0.0


def test_order_parameter_populations(golden_analysis):
    arrays, cases = golden_analysis
    for k in range(cases["populations"]):
        pt = sdb.order_parameter(arrays["pop_%d" % k])
        want = arrays["pop_%d_rphi" % k]
        assert abs(pt.r - want[0]) <= 1e-13
        if want[0] > 1e-9:
            assert phase_err(pt.phi, want[1]) <= 1e-12
    assert sdb.order_parameter(np.full(7, 2.5)).r == 1.0
    assert sdb.order_parameter([0.0, math.pi]).r < 1e-15
    with pytest.raises(ValueError):
        sdb.order_parameter([])


def _golden_store(arrays, cases, name):
    c = cases[name]
    cfg = EngineConfig(dt=c["dt"], tspan=c["tspan"], ksteps=c["ksteps"], orbits=c["orbits"],
                       seed=c["seed"])
    batch = OrbitBatch(init=arrays[name + "_init"], params=arrays[name + "_params"])
    return cfg, batch


@pytest.mark.parametrize("name", ["sync", "incoh", "n5"])
def test_coherence_series_and_stats_match_reference(golden_analysis, name):
    arrays, cases = golden_analysis
    cfg, batch = _golden_store(arrays, cases, name)
    store = run_batch(sdb.kuramoto_model(cases[name]["n"]), cfg, batch)
    assert O.mixed_error(store.values, arrays[name + "_values"]) <= PARITY_TOL
    cs = sdb.coherence_series(store)
    assert O.mixed_error(cs.r, arrays[name + "_r"]) <= PARITY_TOL
    assert phase_err(cs.phi, arrays[name + "_phi"]) <= 1e-9
    st = sdb.ensemble_stats(cs)
    assert O.mixed_error(st.mean_r, arrays[name + "_mean_r"]) <= PARITY_TOL
    assert O.mixed_error(st.std_r, arrays[name + "_std_r"]) <= PARITY_TOL
    assert analysis.first_crossing_time(cs.times, st.mean_r, 0.5) == cases[name]["first_cross"]
    assert O.mixed_error(sdb.kymograph_export(store, 1), arrays[name + "_kymo1"]) <= 1e-9


@pytest.mark.parametrize("coupling", ["meanfield", "pairwise"])
@pytest.mark.parametrize("stream", ["philox", "sfc64"])
@pytest.mark.parametrize("n", [16, 12, 5])
def test_fused_run_equals_coherence_of_store(n, stream, coupling):
    m = 700
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.4, seed=n)
    params = batch.params.copy()
    params[333, 1 + 2] = 1e308  # one failing orbit: NaN coherence from its failure on
    batch = OrbitBatch(init=batch.init, params=params)
    cfg = EngineConfig(dt=1e-2, tspan=3.0, ksteps=25, orbits=m, seed=3, stream=stream,
                       coupling=coupling)
    store = run_batch(sdb.kuramoto_model(n), cfg, batch)
    unfused = sdb.coherence_series(store)
    fused = sdb.run_coherence(sdb.kuramoto_model(n), cfg, batch)
    assert last_launch_info()["launches"] >= 1
    assert np.array_equal(fused.times, unfused.times)
    assert np.array_equal(fused.r, unfused.r, equal_nan=True)
    assert np.array_equal(fused.phi, unfused.phi, equal_nan=True)
    assert fused.failures == store.failures and fused.failures[0].orbit == 333
    assert np.isnan(fused.r[333, -1])


def test_fused_run_shards_and_tiles(monkeypatch):
    n, m = 16, 900
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.3, seed=9)
    cfg = EngineConfig(dt=1e-2, tspan=2.0, ksteps=10, orbits=m, seed=4, stream="xoshiro256pp")
    ref = sdb.run_coherence(sdb.kuramoto_model(n), cfg, batch)
    two = sdb.run_coherence(sdb.kuramoto_model(n), dataclasses.replace(cfg, devices=(0, 0)), batch)
    monkeypatch.setenv("SDEB200_TILES", "3")
    monkeypatch.setenv("SDEB200_PIECE_KB", "20")
    tiled = sdb.run_coherence(sdb.kuramoto_model(n), cfg, batch)
    for other in (two, tiled):
        assert np.array_equal(ref.r, other.r) and np.array_equal(ref.phi, other.phi)


def test_fused_run_for_expression_models_falls_back_to_store_path():
    m = sdb.model_from_dsl("phases", 4, 2, 4, "p[0] + p[1]*sin(y[i])", "0.1*n[i]")
    g = np.random.default_rng(0)
    batch = OrbitBatch(init=g.uniform(-3, 3, (30, 4)), params=g.uniform(0.1, 1.0, (30, 2)))
    cfg = EngineConfig(dt=0.01, tspan=0.5, ksteps=10, orbits=30, seed=2)
    fused = sdb.run_coherence(m, cfg, batch)
    unfused = sdb.coherence_series(run_batch(m, cfg, batch))
    assert np.array_equal(fused.r, unfused.r)


def test_dt_sweep_matches_reference(golden_analysis):
    arrays, cases = golden_analysis
    rows = sdb.dt_sweep(6, couplings=[0.02, 0.2], dts=[0.05, 0.1], realizations=8, tspan=4.0,
                        sample_interval=0.5, seed=21, threads=1)
    assert [(r.coupling, r.dt) for r in rows] == [(c["coupling"], c["dt"])
                                                 for c in cases["dt_sweep"]]
    for k, (row, want) in enumerate(zip(rows, cases["dt_sweep"])):
        assert abs(row.mean_r_end - want["mean_r_end"]) <= PARITY_TOL
        assert abs(row.std_r_end - want["std_r_end"]) <= PARITY_TOL
        assert O.mixed_error(row.stats.mean_r, arrays["sweep_%d_mean" % k]) <= PARITY_TOL
        assert np.array_equal(row.stats.times, arrays["sweep_%d_times" % k])


def test_dt_sweep_cell_equals_engine_path():
    # analysis.py test_dt_sweep_degenerate_cell_matches_ensemble_stats: exact
    rows = sdb.dt_sweep(4, couplings=[0.2], dts=[0.1], realizations=4, tspan=2.0,
                        sample_interval=0.5, seed=11, threads=1)
    cfg = EngineConfig(dt=0.1, tspan=2.0, ksteps=5, orbits=4, seed=11)
    batch = sdb.sample_kuramoto_batch(4, 4, sdb.model.ACCURACY_OMEGA_RANGE,
                                      sdb.model.ACCURACY_NOISE_RANGE, 0.2, cfg.seed)
    stats = sdb.ensemble_stats(sdb.coherence_series(run_batch(sdb.kuramoto_model(4), cfg, batch)))
    assert rows[0].mean_r_end == stats.mean_r[-1]
    assert rows[0].std_r_end == stats.std_r[-1]
    assert rows[0].stats.times[-1] == 2.0
    with pytest.raises(ValueError, match="does not divide"):
        sdb.dt_sweep(3, couplings=[0.2], dts=[0.3], realizations=2, tspan=1.0,
                     sample_interval=0.5, seed=0, threads=1)
