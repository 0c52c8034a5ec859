"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden outputs.

Bars (written per test): integer / index work bit-exact (Philox words,
stream outputs, sampled batches, failure addresses); floating point within
the north_star tolerance |got - ref| <= 1e-10 * max(1, |ref|) (FP64), and
bit-identical across lane layouts, device shards, repeats and ksteps
subsampling (the reference's determinism contract, test_engine.py:145-172).
"""

import dataclasses

import numpy as np
import pytest

import paper_1908_03869_b200 as sdb
from conftest import PARITY_TOL, case_config
from oracle import sdeb_oracle as O
from paper_1908_03869_b200 import rng
from paper_1908_03869_b200.engine import EngineConfig, last_launch_info, run_batch
from paper_1908_03869_b200.model import ModelSpec, OrbitBatch

pytestmark = pytest.mark.gpu

COUPLINGS = ["meanfield", "pairwise"]
STORE_CASES = ["cfg1", "engine5", "engine5_k4", "cfg2", "n33", "n64", "n256", "rk4_8",
               "euler_8", "em0_8", "failures", "pad", "rotator", "accept7"]


def golden_model(case):
    n = case["nequat"]
    if case["nnoise"] == 0:
        return ModelSpec(name=case["model"], nequat=n, nparams=case["nparams"], nnoise=0,
                         drift=sdb.model._kuramoto_drift)
    return sdb.kuramoto_model(n)


def golden_run(arrays, cases, name, **overrides):
    case = cases[name]
    cfg = EngineConfig(**{**case_config(case), **overrides})
    batch = OrbitBatch(init=arrays[name + "_init"], params=arrays[name + "_params"])
    return run_batch(golden_model(case), cfg, batch)


# ---- noise ----------------------------------------------------------------

def test_philox_kats_on_device():
    from test_oracle import PHILOX_KATS
    for counter, key, expected in PHILOX_KATS:
        assert rng.philox_block(rng.CounterKey(key=key, counter=counter)) == expected


def test_philox_words_golden(golden):
    arrays, _ = golden
    kc = arrays["philox_in"]
    words = rng._philox_words(kc[:, 0], kc[:, 1], kc[:, 2], kc[:, 3], kc[:, 4], kc[:, 5])
    assert np.array_equal(np.stack(words, axis=-1), arrays["philox_out"])  # bit-exact


def test_normals_golden(golden):
    arrays, cases = golden
    for idx in range(7):
        c = cases["normals_%d" % idx]
        got = rng.normals_for_orbits(int(c["seed"]), np.array(c["orbits"], np.uint32),
                                     c["chunk"], c["step"], c["m"])
        # device log/sqrt/sincos vs numpy: a few ulp
        # a few ulp of |z| <= ~7: the device log/sqrt/sincos and the exactly reduced
        # angle (sincos_turn) against numpy's
        np.testing.assert_allclose(got, arrays["normals_%d" % idx], rtol=0, atol=1e-14)


def test_normals_prefix_stable_and_reserved_tag():
    full = rng.normals_for_step(7, 1, 0, 5, 12)
    for m in (1, 4, 5, 11):
        assert np.array_equal(rng.normals_for_step(7, 1, 0, 5, m), full[:m])
    with pytest.raises(ValueError):
        rng.normals_for_orbits(11, np.arange(2), rng.SAMPLING_TAG, 0, 4)
    assert rng.normals_for_step(1, 2, 3, 4, 0).shape == (0,)


def test_normals_moments():
    draws = np.concatenate([rng.normals_for_orbits(123, np.arange(2500), 0, s, 4).ravel()
                            for s in range(100)])
    assert abs(draws.mean()) < 0.01 and abs(draws.var() - 1.0) < 0.01


@pytest.mark.parametrize("stream", ["sfc64", "xoshiro256pp"])
def test_stream_raw_bit_exact(stream):
    for seed, orbit, block in [(0, 0, 0), (2 ** 64 - 1, 2 ** 32 - 1, 63), (20260809, 5, 2)]:
        assert np.array_equal(rng.stream_raw(stream, seed, orbit, block, 200),
                              O.stream_raw(stream, seed, orbit, block, 200))


@pytest.mark.parametrize("stream", ["sfc64", "xoshiro256pp"])
def test_stream_normals_match_oracle(stream):
    orbits = np.array([0, 3, 77, 2 ** 32 - 1], np.uint32)
    m, step = 10, 3
    st = O.stream_init(stream, 99, orbits.astype(np.uint64)[:, None],
                       np.arange(3, dtype=np.uint64)[None, :])
    for _ in range(step):
        O.stream_block_words(stream, st)
    want = O.gaussian_from_words(*O.stream_block_words(stream, st), m)
    got = rng.normals_for_orbits(99, orbits, 0, step, m, stream=stream)
    np.testing.assert_allclose(got, want, rtol=0, atol=4e-15)


def test_sampling_bit_exact(golden):
    arrays, _ = golden
    assert np.array_equal(rng.sampling_uniforms(11, np.arange(8), 10), arrays["sampling_uniforms"])
    b = sdb.sample_kuramoto_batch(16, 64, (0.2, 0.4), (0.01, 0.03), 0.25, seed=99)
    assert np.array_equal(b.init, arrays["sample_init"])
    assert np.array_equal(b.params, arrays["sample_params"])
    b = sdb.speed_protocol_batch(4, 32, seed=20260809)
    assert np.array_equal(b.init, arrays["speed_init"])
    assert np.array_equal(b.params, arrays["speed_params"])
    # a shard of a larger batch equals the corresponding rows
    whole = sdb.sample_kuramoto_batch(5, 100, (0.2, 0.4), (0.01, 0.03), 1.0, seed=3)
    part = sdb.sample_kuramoto_batch(5, 40, (0.2, 0.4), (0.01, 0.03), 1.0, seed=3, orbit_offset=60)
    assert np.array_equal(whole.init[60:], part.init)


# ---- drift and single steps --------------------------------------------------

@pytest.mark.parametrize("coupling", COUPLINGS)
@pytest.mark.parametrize("n", [1, 2, 3, 8, 16, 33, 64])
def test_drift_golden(golden, n, coupling):
    arrays, _ = golden
    got = sdb.drift_eval(sdb.kuramoto_model(n), 0.0, arrays["drift_y_%d" % n],
                         arrays["drift_p_%d" % n], coupling=coupling)
    assert O.mixed_error(got, arrays["drift_f_%d" % n]) <= 1e-13


def test_drift_hand_examples():
    m = sdb.kuramoto_model(2)
    f = sdb.drift_eval(m, 0.0, np.array([0.0, np.pi / 2]), np.array([1.0, 0.1, 0.2, 0.0, 0.0]))
    np.testing.assert_allclose(f, [0.6, -0.3], atol=1e-12)
    m4 = sdb.kuramoto_model(4)
    omega = np.array([0.1, 0.2, 0.3, 0.4])
    f = sdb.drift_eval(m4, 0.0, np.full(4, 1.234), np.concatenate([[0.7], omega, np.zeros(4)]))
    np.testing.assert_allclose(f, omega, atol=1e-15)
    assert sdb.drift_eval(sdb.kuramoto_model(1), 0.0, np.array([1.0]),
                          np.array([5.0, 0.25, 0.0]))[0] == 0.25


@pytest.mark.parametrize("coupling", COUPLINGS)
def test_single_steps_match_oracle(coupling):
    g = np.random.default_rng(5)
    for n in (1, 4, 16, 33):
        y = g.uniform(-3, 3, (7, n))
        p = np.column_stack([g.uniform(0, 1, 7), g.uniform(0.2, 0.4, (7, n)),
                             g.uniform(0.01, 0.03, (7, n))])
        noise = g.standard_normal((7, n))
        m = sdb.kuramoto_model(n)
        ode = ModelSpec(name="k0", nequat=n, nparams=2 * n + 1, nnoise=0,
                        drift=sdb.model._kuramoto_drift)
        for got, want in [
            (sdb.euler_maruyama_step(m, 0.0, y, p, 0.01, noise, coupling=coupling),
             O.em_step(y, p, 0.01, noise)),
            (sdb.euler_step(ode, 0.0, y, p, 0.01, coupling=coupling), O.euler_step(y, p, 0.01)),
            (sdb.rk4_step(ode, 0.0, y, p, 0.01, coupling=coupling), O.rk4_step(y, p, 0.01)),
        ]:
            assert O.mixed_error(got, want) <= 1e-13


# ---- full runs against the reference's stores ----------------------------------

@pytest.mark.parametrize("coupling", COUPLINGS)
@pytest.mark.parametrize("name", STORE_CASES)
def test_run_batch_matches_reference_store(golden, name, coupling):
    arrays, cases = golden
    store = golden_run(arrays, cases, name, coupling=coupling)
    assert np.array_equal(store.times, arrays[name + "_times"])
    assert np.array_equal(store.values[:, 0], arrays[name + "_init"])  # sample 0 verbatim
    err = O.mixed_error(store.values, arrays[name + "_values"])
    assert err <= PARITY_TOL, "%s/%s: mixed error %.3e" % (name, coupling, err)
    assert [[f.orbit, f.chunk, f.step, f.time, f.reason] for f in store.failures] == \
        cases[name]["failures"]


@pytest.mark.parametrize("stream", ["sfc64", "xoshiro256pp"])
def test_run_batch_streams_match_oracle(golden, stream):
    arrays, cases = golden
    name = "cfg2"
    store = golden_run(arrays, cases, name, stream=stream)
    cfg = case_config(cases[name])
    chunks = O.iteration_count(cfg["tspan"], cfg["dt"], cfg["ksteps"])
    _, want, fails = O.integrate(arrays[name + "_init"], arrays[name + "_params"], dt=cfg["dt"],
                                 ksteps=cfg["ksteps"], chunks=chunks, seed=cfg["seed"],
                                 stream=stream)
    assert O.mixed_error(store.values, want) <= PARITY_TOL
    assert not fails and not store.failures


# ---- determinism / invariance (bitwise) -----------------------------------------

def _pairwise_lanes(n):
    """csrc/sdeb_kuramoto.cuh pairwise_lanes."""
    p = 1
    while p < n:
        p *= 2
    return 1 if n <= 15 else (p // 8 if p // 8 <= 32 else p // 16)


def _lane_options(n):
    p = 1
    while p < n:
        p *= 2
    return [L for L in (1, 2, 4, 8, 16, 32) if L <= p and p // L <= 16]


@pytest.mark.parametrize("stream", ["philox", "sfc64", "xoshiro256pp"])
@pytest.mark.parametrize("n", [4, 5, 16, 33])
def test_lane_layouts_bit_identical(n, stream):
    batch = sdb.sample_kuramoto_batch(n, 50, (0.2, 0.4), (0.01, 0.1), 0.3, seed=n)
    base = EngineConfig(dt=0.01, tspan=1.0, ksteps=20, orbits=50, seed=11, stream=stream)
    hashes, values = {}, {}
    for coupling in COUPLINGS:
        for L in _lane_options(n):
            store = run_batch(sdb.kuramoto_model(n),
                              dataclasses.replace(base, lanes=L, coupling=coupling), batch)
            hashes[(coupling, L)] = sdb.store_hash(store)
            values[(coupling, L)] = store.values
    # meanfield: one canonical summation tree, bit-identical for every layout
    assert len({h for (c, _), h in hashes.items() if c == "meanfield"}) == 1, hashes
    # pairwise: the antisymmetric tile order depends on (L, J), so run_batch
    # fixes L from n alone (pairwise_lanes); other L agree within the parity bar
    auto = run_batch(sdb.kuramoto_model(n), dataclasses.replace(base, coupling="pairwise"), batch)
    assert sdb.store_hash(auto) == hashes[("pairwise", _pairwise_lanes(n))]
    for L in _lane_options(n):
        assert O.mixed_error(values[("pairwise", L)], auto.values) <= PARITY_TOL, L


@pytest.mark.parametrize("solver", ["rk4", "euler"])
def test_lane_layouts_bit_identical_ode(solver):
    n = 12
    ode = ModelSpec(name="k0", nequat=n, nparams=2 * n + 1, nnoise=0,
                    drift=sdb.model._kuramoto_drift)
    batch = sdb.sample_kuramoto_batch(n, 40, (0.2, 0.4), (0.0, 0.0), 1.5, seed=2)
    base = EngineConfig(dt=0.01, tspan=1.0, ksteps=25, orbits=40, solver=solver)
    hs = {sdb.store_hash(run_batch(ode, dataclasses.replace(base, lanes=L), batch))
          for L in _lane_options(n)}
    assert len(hs) == 1


def test_device_shards_bit_identical():
    # two shards on the same GPU == one shard (the 1/2/4/8-GPU invariance)
    n, m = 16, 333
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.03), 0.2, seed=1)
    base = EngineConfig(dt=1e-3, tspan=0.5, ksteps=50, orbits=m, seed=5, stream="sfc64")
    h1 = sdb.store_hash(run_batch(sdb.kuramoto_model(n), base, batch))
    h2 = sdb.store_hash(run_batch(sdb.kuramoto_model(n),
                                  dataclasses.replace(base, devices=(0, 0)), batch))
    h3 = sdb.store_hash(run_batch(sdb.kuramoto_model(n),
                                  dataclasses.replace(base, devices=(0, 0, 0)), batch))
    assert h1 == h2 == h3


def test_ksteps_subsampling_identity_and_repeatability():
    n, m = 5, 16
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.03), 0.2, seed=7)
    fine = EngineConfig(dt=0.05, tspan=4.0, ksteps=4, orbits=m, seed=3)
    coarse = dataclasses.replace(fine, ksteps=8)
    a = run_batch(sdb.kuramoto_model(n), fine, batch)
    b = run_batch(sdb.kuramoto_model(n), coarse, batch)
    assert np.array_equal(a.values[:, ::2], b.values)
    assert np.array_equal(a.times[::2], b.times)
    again = run_batch(sdb.kuramoto_model(n), fine, batch)
    assert sdb.store_hash(a) == sdb.store_hash(again)
    # threads / chunk_group are scheduling hints only
    for kw in ({"threads": 1}, {"chunk_group": 3}, {"threads": 2, "chunk_group": 100}):
        assert sdb.store_hash(run_batch(sdb.kuramoto_model(n),
                                        dataclasses.replace(fine, **kw), batch)) == \
            sdb.store_hash(a)


def test_identical_rows_diverge_by_orbit_keyed_noise():
    m = sdb.kuramoto_model(3)
    batch = OrbitBatch(init=np.tile([[0.1, -0.4, 1.0]], (2, 1)),
                       params=np.tile([[0.2, 0.3, 0.31, 0.32, 0.02, 0.02, 0.02]], (2, 1)))
    cfg = EngineConfig(dt=0.05, tspan=2.0, ksteps=40, orbits=2, seed=0)
    store = run_batch(m, cfg, batch)
    assert not np.array_equal(store.values[0, 1:], store.values[1, 1:])


def test_phase_sum_conservation():
    # test_engine.py:175-187: with zero noise, sum(theta) - sum(theta0) - sum(omega) t
    # is conserved to 1e-9 over 400 s
    n = 20
    b = sdb.sample_kuramoto_batch(n, 4, (0.2, 0.4), (0.0, 0.0), 0.2, seed=9)
    for coupling in COUPLINGS:
        store = run_batch(sdb.kuramoto_model(n),
                          EngineConfig(dt=0.05, tspan=400.0, ksteps=40, orbits=4, seed=9,
                                       coupling=coupling), b)
        omega_sum = b.params[:, 1:n + 1].sum(axis=-1)
        resid = (store.values.sum(axis=-1) - b.init.sum(axis=-1)[:, None]
                 - omega_sum[:, None] * store.times[None, :])
        assert np.max(np.abs(resid)) < 1e-9


def test_failure_mid_chunk_nan_fill_across_lanes():
    # orbit 1 overflows at step 5 (omega huge, K=0); every lane layout must
    # NaN the whole row from the failing step and record the same address
    n = 8
    init = np.zeros((3, n))
    params = np.zeros((3, 2 * n + 1))
    params[:, 1:n + 1] = 0.1
    params[1, 1 + 6] = 1e308  # oscillator 6 -> inf after 2 steps of dt=1
    cfg = EngineConfig(dt=1.0, tspan=8.0, ksteps=2, orbits=3, seed=1)
    want = O.integrate(init, params, dt=1.0, ksteps=2, chunks=4, seed=1)
    for L in (1, 2, 4, 8):
        store = run_batch(sdb.kuramoto_model(n), dataclasses.replace(cfg, lanes=L),
                          OrbitBatch(init=init, params=params))
        assert O.mixed_error(store.values, want[1]) <= PARITY_TOL
        assert [(f.orbit, f.chunk, f.step, f.time) for f in store.failures] == \
            [f[:4] for f in want[2]]


@pytest.mark.parametrize("n", [1, 31, 128, 511, 512])
def test_edge_sizes_match_oracle(n):
    m = 3
    b = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.03), 0.7, seed=n)
    cfg = EngineConfig(dt=0.01, tspan=0.1, ksteps=5, orbits=m, seed=n)
    want = O.integrate(b.init, b.params, dt=0.01, ksteps=5, chunks=2, seed=n)[1]
    for coupling in COUPLINGS:
        store = run_batch(sdb.kuramoto_model(n), dataclasses.replace(cfg, coupling=coupling), b)
        assert O.mixed_error(store.values, want) <= PARITY_TOL


def test_too_many_oscillators_unsupported():
    b = OrbitBatch(init=np.zeros((1, 513)), params=np.zeros((1, 1027)))
    with pytest.raises(NotImplementedError):
        run_batch(sdb.kuramoto_model(513), EngineConfig(dt=0.1, tspan=0.1, ksteps=1, orbits=1), b)


def test_launch_accounting():
    b = sdb.speed_protocol_batch(4, 64, seed=1)
    run_batch(sdb.kuramoto_model(4), EngineConfig(dt=1e-3, tspan=0.01, ksteps=10, orbits=64,
                                                  lanes=2), b)
    info = last_launch_info()
    assert info["launches"] == 1 and info["lanes"] == 2


def _run_pinned(layout, n, batch, cfg, info=None):
    """run_batch through a fresh context with SDEB200_LAYOUT pinned (info, if
    given, receives the lane width the launch ran with)."""
    import ctypes
    import os

    from paper_1908_03869_b200 import _native as nat
    from paper_1908_03869_b200.engine import make_desc
    os.environ["SDEB200_LAYOUT"] = layout
    try:
        ctx = ctypes.c_void_p()
        nat.check(nat.lib().sdb_open(None, 0, ctypes.byref(ctx)))
        chunks = sdb.iteration_count(cfg.tspan, cfg.dt, cfg.ksteps)
        desc = make_desc(sdb.kuramoto_model(n), cfg, chunks, batch.orbits)
        values = np.empty((batch.orbits, chunks + 1, n))
        fail = np.empty(batch.orbits, np.int64)
        init, params = nat.f64(batch.init), nat.f64(batch.params)
        nat.check(nat.lib().sdb_run(ctx, desc, nat.dptr(init), nat.dptr(params),
                                    nat.dptr(values), nat.i64ptr(fail)), ctx)
        if info is not None:
            info["lane_width"] = int(nat.lib().sdb_last_lane_width(ctx))
        nat.lib().sdb_close(ctx)
        return values, fail
    finally:
        del os.environ["SDEB200_LAYOUT"]


@pytest.mark.parametrize("stream", ["philox", "sfc64", "xoshiro256pp"])
@pytest.mark.parametrize("n", [3, 5, 6, 7, 10, 12, 15])
def test_exact_lane_width_layouts_bit_identical(n, stream):
    # n <= 16 not a power of two also runs J = n oscillators in one lane (no padded slots): the
    # lane tree over n leaves must associate exactly like the canonical tree
    # over next_pow2(n) zero-padded leaves, and the partial last noise block
    # must give the same normals -- same bits as every power-of-two layout
    m = 700
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.3, seed=9)
    params = batch.params.copy()
    params[11, 1 + n - 1] = np.inf  # the last oscillator (partial block) fails
    params[12, 1 + 2] = 1e12       # huge phases: the exact-reduction branch
    batch = OrbitBatch(init=batch.init, params=params)
    cfg = EngineConfig(dt=1e-2, tspan=1.5, ksteps=25, orbits=m, seed=3, stream=stream)
    info = {}
    ref, ref_fail = _run_pinned("1,0,0,0", n, batch, cfg, info)
    assert info["lane_width"] == 1 << (n - 1).bit_length()
    for lay in ("1,0,0,0,%d" % n, "1,1,0,0,%d" % n, "2,0,0,0"):
        got, got_fail = _run_pinned(lay, n, batch, cfg, info)
        if lay.endswith(",%d" % n):
            assert info["lane_width"] == n
        assert np.array_equal(ref, got, equal_nan=True), lay
        assert np.array_equal(ref_fail, got_fail), lay
    assert ref_fail[11] >= 0 and ref_fail[12] < 0
    # the default autotuned run and the fused coherence run agree too
    auto = run_batch(sdb.kuramoto_model(n), cfg, batch)
    assert np.array_equal(auto.values, ref, equal_nan=True)
    coh = sdb.run_coherence(sdb.kuramoto_model(n), cfg, batch)
    series = sdb.coherence_series(auto)
    np.testing.assert_array_equal(coh.r, series.r)


@pytest.mark.parametrize("stream", ["philox", "sfc64"])
@pytest.mark.parametrize("n", [16, 12])
def test_persistent_slab_schedule_bit_identical(n, stream):
    # the work-pulling grid hands each orbit group over between CTAs every
    # 16-step slab (samples every 50 steps fall mid-slab): must be bitwise
    # identical to one CTA per group, for padded and unpadded n
    m = 2000
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.3, seed=4)
    params = batch.params.copy()
    params[7, 1 + 3] = 1e308  # orbit 7 fails mid-run: failure + NaN fill across slabs
    params[7, 0] = 0.0
    batch = OrbitBatch(init=batch.init, params=params)
    cfg = EngineConfig(dt=1e-2, tspan=3.0, ksteps=50, orbits=m, seed=9, stream=stream)
    lanes = 4
    ref, ref_fail = _run_pinned("%d,0,0" % lanes, n, batch, cfg)
    got, got_fail = _run_pinned("%d,1,0" % lanes, n, batch, cfg)
    assert np.array_equal(ref, got, equal_nan=True)
    assert np.array_equal(ref_fail, got_fail) and ref_fail[7] >= 0
    capped, _ = _run_pinned("%d,0,2" % lanes, n, batch, cfg)
    assert np.array_equal(ref, capped, equal_nan=True)


@pytest.mark.parametrize("stream", ["philox", "sfc64"])
def test_host_pipeline_tiling_bit_identical(stream, monkeypatch):
    # sdb_run's host pipeline (orbit tiles x pinned transfer pieces x host copy
    # threads) must not change a single bit, failures and sample 0 included
    from paper_1908_03869_b200.engine import last_launch_info
    n, m = 16, 1501
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.3, seed=11)
    params = batch.params.copy()
    params[1000, 1 + 5] = 1e308  # a failing orbit inside a later tile
    params[1200, 1 + 2] = 1e12   # |theta| >> 2^29: the exact-reduction trig path
    batch = OrbitBatch(init=batch.init, params=params)
    cfg = EngineConfig(dt=1e-2, tspan=2.0, ksteps=20, orbits=m, seed=2, stream=stream)
    ref = run_batch(sdb.kuramoto_model(n), cfg, batch)
    assert ref.failures and ref.failures[0].orbit == 1000
    for tiles, piece_kb, threads in [(3, 100, 4), (7, 40, 1), (2, 65536, 8), (1, 1, 2)]:
        monkeypatch.setenv("SDEB200_TILES", str(tiles))
        monkeypatch.setenv("SDEB200_PIECE_KB", str(piece_kb))
        monkeypatch.setenv("SDEB200_HOST_THREADS", str(threads))
        got = run_batch(sdb.kuramoto_model(n), cfg, batch)
        assert last_launch_info()["tiles"] == tiles
        assert sdb.store_hash(got) == sdb.store_hash(ref)
        assert got.failures == ref.failures
        assert np.array_equal(got.values[:, 0], batch.init)


def test_host_pipeline_large_store_paths(monkeypatch):
    # a store >= 64 MiB takes the streaming-store staging copies, the huge-page
    # allocation and the destination prefault; an odd n makes every row start
    # 8 bytes off a 16-byte boundary.  Same bits as the small-transfer path
    # (plain memcpy into np.empty), reached by running orbit slices
    n, m = 33, 13000
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.3, seed=21)
    params = batch.params.copy()
    params[7777, 1 + 3] = np.inf  # a failing orbit in the middle of a piece
    batch = OrbitBatch(init=batch.init, params=params)
    cfg = EngineConfig(dt=1e-2, tspan=0.2, ksteps=1, orbits=m, seed=4, stream="philox",
                       max_store_bytes=1 << 34)
    model = sdb.kuramoto_model(n)
    big = run_batch(model, cfg, batch)
    assert big.values.nbytes >= 64 << 20
    assert big.failures and big.failures[0].orbit == 7777
    monkeypatch.setenv("SDEB200_PREFAULT", "0")
    assert sdb.store_hash(run_batch(model, cfg, batch)) == sdb.store_hash(big)
    parts = []
    for lo in range(0, m, 3250):
        part = OrbitBatch(init=batch.init[lo:lo + 3250], params=batch.params[lo:lo + 3250])
        parts.append(run_batch(model, dataclasses.replace(cfg, orbits=3250), part,
                               orbit_offset=lo).values)
    assert np.array_equal(np.concatenate(parts), big.values, equal_nan=True)


@pytest.mark.parametrize("stream", ["philox", "sfc64"])
def test_lane_layouts_bit_identical_huge_phases(stream):
    # phases beyond 2^29 take the exact (Payne-Hanek) reduction branch; it must
    # give the same bits in every kernel instantiation (lanes x J)
    n, m = 16, 64
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.3, seed=3)
    params = batch.params.copy()
    params[::3, 1 + 4] = 1e12
    params[1::5, 1:1 + n] = 1e308  # grows through 2^1000 to overflow (fails)
    batch = OrbitBatch(init=batch.init, params=params)
    base = EngineConfig(dt=1e-2, tspan=2.0, ksteps=10, orbits=m, seed=8, stream=stream)
    stores = [run_batch(sdb.kuramoto_model(n), dataclasses.replace(base, lanes=L), batch)
              for L in _lane_options(n)]
    assert len({sdb.store_hash(s) for s in stores}) == 1
    assert {f.orbit for f in stores[0].failures} == set(range(1, m, 5))


def test_concurrent_calls_on_one_context_are_serialised():
    # the cached context is shared by every caller; two host threads
    # running at once must each get exactly their single-threaded result
    import threading
    n, m = 16, 20000
    model = sdb.kuramoto_model(n)
    batches = [sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.3, seed=s)
               for s in (1, 2, 3, 4)]
    cfg = EngineConfig(dt=1e-3, tspan=0.2, ksteps=50, orbits=m, seed=9)
    want = [sdb.store_hash(run_batch(model, cfg, b)) for b in batches]
    got = [None] * len(batches)

    def work(i):
        got[i] = sdb.store_hash(run_batch(model, cfg, batches[i]))
    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(batches))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert got == want


def test_kuramoto_diffusion_eval_on_device_is_the_rounded_product():
    n = 12
    g = np.random.default_rng(4)
    y = g.uniform(-3, 3, (7, n))
    p = g.uniform(-1, 1, (7, 2 * n + 1))
    z = g.standard_normal((7, n))
    want = np.multiply(p[:, n + 1:], z)
    assert np.array_equal(sdb.diffusion_eval(sdb.kuramoto_model(n), 0.0, y, p, z), want)
    assert np.array_equal(sdb.model._kuramoto_diffusion(0.0, y, p, z), want)


def test_layout_autotune_is_bounded_and_persisted():
    # the first call per shape probed the whole run up to 20 times.
    # Now the probe runs on one resident wave, budgeted at ~10% of the run,
    # and its decision is read back from the on-disk cache by a fresh context.
    import ctypes
    import os
    import time

    from paper_1908_03869_b200 import _native as nat
    from paper_1908_03869_b200.engine import make_desc
    n, m, steps = 32, 1 << 18, 400
    batch = sdb.speed_protocol_batch(n, m, seed=3)
    cfg = EngineConfig(dt=1e-3, tspan=steps * 1e-3, ksteps=steps, orbits=m, seed=2)
    desc = make_desc(sdb.kuramoto_model(n), cfg, 1, m)
    values = np.empty((m, 2, n))
    fail = np.empty(m, np.int64)
    init, params = nat.f64(batch.init), nat.f64(batch.params)
    path = os.environ["SDEB200_TUNE_CACHE"]
    rows_before = open(path).read().count("\n") if os.path.exists(path) else 0

    def fresh_run():
        ctx = ctypes.c_void_p()
        nat.check(nat.lib().sdb_open(None, 0, ctypes.byref(ctx)))
        t0 = time.perf_counter()
        nat.check(nat.lib().sdb_run(ctx, desc, nat.dptr(init), nat.dptr(params),
                                    nat.dptr(values), nat.i64ptr(fail)), ctx)
        wall = time.perf_counter() - t0
        tiles = ctypes.c_int32()
        nat.lib().sdb_last_layout(ctx, None, None, None, None, ctypes.byref(tiles))
        # probe launches come on top of one launch per host-pipeline tile
        out = (int(nat.lib().sdb_last_tune_us(ctx)),
               int(nat.lib().sdb_last_launch_count(ctx)) - tiles.value, wall, values.copy())
        nat.lib().sdb_close(ctx)
        return out

    tune_us, launches, wall, first = fresh_run()
    assert launches > 0 and tune_us > 0  # probed (an empty cache for this shape)
    assert tune_us * 1e-6 <= 0.25 * wall, (tune_us, wall)
    assert open(path).read().count("\n") == rows_before + 1  # decision persisted
    tune_us2, launches2, _, second = fresh_run()  # a new context: the disk cache answers
    assert tune_us2 == 0 and launches2 == 0
    assert np.array_equal(first, second)


def test_pinned_inputs_take_the_direct_dma_path_bit_identically(monkeypatch):
    # sdb.pin_batch: inputs in page-locked memory are DMA'd without the host
    # staging copy; results equal the pageable path for every tiling / shard count
    from paper_1908_03869_b200 import _native as nat
    n, m = 32, 40000
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.3, seed=21)
    pinned = sdb.pin_batch(batch)
    assert np.array_equal(pinned.init, batch.init) and np.array_equal(pinned.params, batch.params)
    cfg = EngineConfig(dt=1e-3, tspan=0.1, ksteps=25, orbits=m, seed=4)
    want = sdb.store_hash(run_batch(sdb.kuramoto_model(n), cfg, batch))
    assert sdb.store_hash(run_batch(sdb.kuramoto_model(n), cfg, pinned)) == want
    monkeypatch.setenv("SDEB200_TILES", "3")
    assert sdb.store_hash(run_batch(sdb.kuramoto_model(n), cfg, pinned)) == want
    assert sdb.store_hash(run_batch(sdb.kuramoto_model(n),
                                    dataclasses.replace(cfg, devices=(0, 0)), pinned)) == want
    # a pinned scratch array of any shape
    a = nat.host_pinned((3, 5))
    a[:] = 7.0
    assert a.sum() == 105.0


def test_eight_shards_on_one_gpu_pinned_and_pageable_bit_identical():
    # the host pipeline of an 8-device run (one host thread per shard, shared
    # copy pool) exercised on one GPU: the store equals the one-shard run's
    n, m = 32, 50000
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.3, seed=33)
    cfg = EngineConfig(dt=1e-3, tspan=0.05, ksteps=25, orbits=m, seed=6)
    want = sdb.store_hash(run_batch(sdb.kuramoto_model(n), cfg, batch))
    eight = dataclasses.replace(cfg, devices=(0,) * 8)
    assert sdb.store_hash(run_batch(sdb.kuramoto_model(n), eight, batch)) == want
    assert sdb.store_hash(run_batch(sdb.kuramoto_model(n), eight, sdb.pin_batch(batch))) == want
    assert last_launch_info((0,) * 8)["launches"] >= 8


@pytest.mark.parametrize("stream", ["philox", "sfc64"])
@pytest.mark.parametrize("n", [256, 200, 128])
def test_wide_group_layouts_bit_identical(n, stream):
    # 8-32 lanes per orbit (the cfg3 sizes): the butterfly's canonical tree,
    # the same bits for every layout, and the oracle's values
    batch = sdb.sample_kuramoto_batch(n, 300, (0.2, 0.4), (0.01, 0.1), 0.3, seed=n)
    base = EngineConfig(dt=0.01, tspan=0.5, ksteps=10, orbits=300, seed=12, stream=stream)
    hashes = {L: sdb.store_hash(run_batch(sdb.kuramoto_model(n),
                                          dataclasses.replace(base, lanes=L), batch))
              for L in _lane_options(n)}
    assert len(set(hashes.values())) == 1, hashes
    want = O.integrate(batch.init[:4], batch.params[:4], dt=0.01, ksteps=10, chunks=5, seed=12,
                       stream=stream)[1]
    store = run_batch(sdb.kuramoto_model(n), base, batch)
    assert O.mixed_error(store.values[:4], want) <= PARITY_TOL
