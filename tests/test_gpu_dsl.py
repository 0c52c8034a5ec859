"""GPU parity of runtime-compiled expression-template models (NVRTC programs,
include/sdeb200.h sdb_model_*) against the reference's own stores
(tests/golden/make_golden_dsl.py) and the pinned oracle.

Bars: |got - ref| <= 1e-10 * max(1, |ref|) (north_star, FP64) for values;
failure records (orbit, chunk, step) exact; bit-identical across device
shards, host-pipeline tilings and repeats.
"""

import dataclasses
import math

import numpy as np
import pytest

import paper_1908_03869_b200 as sdb
from conftest import PARITY_TOL
from oracle import sdeb_oracle as O
from paper_1908_03869_b200 import dsl
from paper_1908_03869_b200.dsl import EvalContext
from paper_1908_03869_b200.engine import EngineConfig, last_launch_info, run_batch
from paper_1908_03869_b200.model import OrbitBatch

pytestmark = pytest.mark.gpu

CASES = ["ou", "tdep", "nested", "funcs", "rk4", "euler", "fail", "big", "kuramoto"]


def case_model(case, name):
    return sdb.model_from_dsl(name, case["nequat"], case["nparams"], case["nnoise"],
                              case["drift"], case["diffusion"])


def case_cfg(case, **kw):
    base = dict(dt=case["dt"], tspan=case["dt"] * case["steps"], ksteps=case["ksteps"],
                orbits=case["orbits"], solver=case["solver"], seed=case["seed"])
    base.update(kw)
    return EngineConfig(**base)


def case_batch(arrays, name):
    return OrbitBatch(init=arrays[name + "_init"], params=arrays[name + "_params"])


@pytest.fixture(autouse=True)
def _codegen_for_kuramoto(monkeypatch, request):
    # the "kuramoto" golden goes through the generated program, not the native stepper
    if "kuramoto" in request.node.name:
        monkeypatch.setenv("SDEB200_NO_NATIVE_KURAMOTO", "1")


@pytest.mark.parametrize("name", CASES)
def test_run_batch_matches_reference_store(golden_dsl, name):
    arrays, cases = golden_dsl
    case = cases[name]
    model = case_model(case, name)
    assert sdb.model.expression_model(model)
    store = run_batch(model, case_cfg(case), case_batch(arrays, name))
    assert last_launch_info()["launches"] == 1
    err = O.mixed_error(store.values, arrays[name + "_values"])
    assert err <= PARITY_TOL, "%s: mixed error %.3e" % (name, err)
    assert [[f.orbit, f.chunk, f.step] for f in store.failures] == \
        [f[:3] for f in case["failures"]]
    for got, want in zip(store.failures, case["failures"]):
        assert math.isclose(got.time, want[3], rel_tol=0, abs_tol=1e-15)
        assert got.reason == want[4]
    assert np.array_equal(store.values[:, 0], arrays[name + "_init"])


@pytest.mark.parametrize("name", CASES)
def test_drift_and_diffusion_eval_match_reference(golden_dsl, name):
    arrays, cases = golden_dsl
    case = cases[name]
    model = case_model(case, name)
    y, p = arrays[name + "_eval_y"], arrays[name + "_eval_p"]
    got = sdb.drift_eval(model, 0.37, y, p, strict=False)
    assert O.mixed_error(got, arrays[name + "_drift"]) <= 1e-13
    if case["nnoise"]:
        z = arrays[name + "_eval_noise"]
        got = sdb.diffusion_eval(model, 0.37, y, p, z, strict=False)
        assert O.mixed_error(got, arrays[name + "_diffusion"]) <= 1e-13


@pytest.mark.parametrize("stream", ["sfc64", "xoshiro256pp"])
@pytest.mark.parametrize("name", ["ou", "tdep", "big"])
def test_stateful_streams_match_oracle(golden_dsl, name, stream):
    # the extra streams (not in the reference) against the oracle's restatement
    arrays, cases = golden_dsl
    case = cases[name]
    store = run_batch(case_model(case, name), case_cfg(case, stream=stream),
                      case_batch(arrays, name))
    drift, diffusion = O.expression_model(case["drift"], case["diffusion"])
    _, want, _ = O.integrate(arrays[name + "_init"], arrays[name + "_params"], dt=case["dt"],
                             ksteps=case["ksteps"], chunks=case["steps"] // case["ksteps"],
                             seed=case["seed"], solver="em", nnoise=case["nnoise"],
                             stream=stream, drift=drift, diffusion=diffusion)
    assert O.mixed_error(store.values, want) <= PARITY_TOL


def test_generated_kuramoto_matches_native_stepper(monkeypatch):
    # the same system through the hand-written stepper (pairwise coupling:
    # the reference's term order) and through the generated program
    n, m = 12, 300
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.4, seed=6)
    cfg = EngineConfig(dt=1e-2, tspan=2.0, ksteps=50, orbits=m, seed=8, coupling="pairwise")
    native = run_batch(sdb.kuramoto_dsl_model(n), cfg, batch)
    monkeypatch.setenv("SDEB200_NO_NATIVE_KURAMOTO", "1")
    generated = run_batch(sdb.kuramoto_dsl_model(n), cfg, batch)
    assert O.mixed_error(generated.values, native.values) <= 1e-12


def test_shards_tiles_and_repeats_bit_identical(golden_dsl, monkeypatch):
    arrays, cases = golden_dsl
    case = cases["tdep"]
    model = case_model(case, "tdep")
    m = 301
    g = np.random.default_rng(3)
    batch = OrbitBatch(init=g.uniform(-1, 1, (m, 4)), params=g.uniform(0.05, 0.6, (m, 8)))
    cfg = case_cfg(case, orbits=m, stream="sfc64")
    ref = sdb.store_hash(run_batch(model, cfg, batch))
    assert sdb.store_hash(run_batch(model, cfg, batch)) == ref
    assert sdb.store_hash(run_batch(model, dataclasses.replace(cfg, devices=(0, 0, 0)),
                                    batch)) == ref
    monkeypatch.setenv("SDEB200_TILES", "4")
    monkeypatch.setenv("SDEB200_PIECE_KB", "8")
    assert sdb.store_hash(run_batch(model, cfg, batch)) == ref


def test_ksteps_subsampling_identity(golden_dsl):
    arrays, cases = golden_dsl
    case = cases["ou"]
    model = case_model(case, "ou")
    fine = run_batch(model, case_cfg(case, ksteps=10), case_batch(arrays, "ou"))
    coarse = run_batch(model, case_cfg(case, ksteps=20), case_batch(arrays, "ou"))
    assert np.array_equal(fine.values[:, ::2], coarse.values)


@pytest.mark.parametrize("solver", ["em", "euler", "rk4"])
def test_per_step_api_matches_oracle(golden_dsl, solver):
    arrays, cases = golden_dsl
    name = "tdep"
    case = cases[name]
    model = case_model(case, name)
    y, p = arrays[name + "_eval_y"], arrays[name + "_eval_p"]
    drift, diffusion = O.expression_model(case["drift"], case["diffusion"])
    t, dt = 0.25, 0.01
    if solver == "em":
        z = arrays[name + "_eval_noise"]
        got = sdb.euler_maruyama_step(model, t, y, p, dt, z)
        want = (y + drift(t, y, p) * dt) + np.sqrt(dt) * diffusion(t, y, p, z)
    elif solver == "euler":
        got = sdb.euler_step(model, t, y, p, dt)
        want = y + drift(t, y, p) * dt
    else:
        got = sdb.rk4_step(model, t, y, p, dt)
        half = 0.5 * dt
        k1 = drift(t, y, p)
        k2 = drift(t + half, y + half * k1, p)
        k3 = drift(t + half, y + half * k2, p)
        k4 = drift(t + dt, y + dt * k3, p)
        want = y + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
    assert O.mixed_error(got, want) <= 1e-14


# ---- dsl.evaluate on the device (reference test_dsl.py:24-225) ------------------------

def ctx(y=(0.0,), p=(0.0,), n=None, t=0.0, i=0, N=None):
    y = np.asarray(y, dtype=np.float64)
    return EvalContext(t=t, N=N if N is not None else y.shape[-1], y=y,
                       p=np.asarray(p, dtype=np.float64),
                       n=None if n is None else np.asarray(n, dtype=np.float64), i=i)


def ev(source, **kw):
    return dsl.evaluate(dsl.parse(source), ctx(**kw))


def test_evaluate_arithmetic_and_functions():
    assert ev("2+3*4") == 14.0 and ev("2*3^2") == 18.0 and ev("2^3^2") == 512.0
    assert ev("-2^2") == -4.0 and ev("2^-1") == 0.5 and ev("8/4/2") == 1.0
    assert ev("2 - 3 - 4") == -5.0 and ev("--2") == 2.0
    assert abs(ev("exp(1)") - math.e) < 1e-15
    assert abs(ev("ln(exp(2))") - 2.0) < 1e-12
    assert ev("sqrt(16)") == 4.0 and ev("abs(0-3)") == 3.0
    assert abs(ev("tan(0.5)") - math.tan(0.5)) < 1e-15
    assert ev("sin(y[0]) + 2*p[1]", y=[0.0], p=[0.0, 3.0]) == 6.0
    assert ev("t", t=2.5) == 2.5 and ev("N", y=np.zeros(7), N=7) == 7.0
    assert ev("i", y=np.zeros(3), i=2) == 2.0
    assert ev("sum(j, 1)", y=np.zeros(7), N=7) == 7.0
    assert ev("sum(j, y[i])", y=np.array([2.0, 3.0]), i=1) == 6.0


def test_evaluate_vectorised_batched_and_noise():
    src = "p[i+1] + (p[0]/N)*sum(j, sin(y[j]-y[i])) + 0.5*i"
    y = np.array([0.3, -1.2, 2.5])
    p = np.array([0.7, 0.1, 0.2, 0.3, 0.0, 0.0, 0.0])
    vec = dsl.evaluate(dsl.parse(src), ctx(y=y, p=p, i=None))
    assert vec.shape == (3,)
    want = O.evaluate_expression(src, 0.0, y, p)
    assert O.mixed_error(vec, want) <= 1e-15
    for i in range(3):
        assert abs(vec[i] - ev(src, y=y, p=p, i=i)) < 1e-14
    yb = np.arange(8.0).reshape(2, 4)
    pb = np.array([[2.0], [3.0]])
    out = dsl.evaluate(dsl.parse("p[0]*y[i] + sum(j, y[j])/N"), ctx(y=yb, p=pb, i=None, N=4))
    assert out.shape == (2, 4)
    assert np.array_equal(out, O.evaluate_expression("p[0]*y[i] + sum(j, y[j])/N", 0.0, yb, pb))
    assert ev("p[1+N+i]*n[i]", y=np.zeros(2), p=[1.0, 0.1, 0.2, 0.01, 0.03],
              n=[2.0, -1.0], i=1, N=2) == pytest.approx(-0.03)


def test_evaluate_domain_and_index_errors():
    with pytest.raises(dsl.DomainError):
        ev("1/y[0]", y=[0.0])
    with pytest.raises(dsl.DomainError):
        ev("ln(y[0])", y=[0.0])
    with pytest.raises(dsl.DomainError):
        ev("sqrt(0-1)")
    assert math.isnan(dsl.evaluate(dsl.parse("ln(y[0])"), ctx(y=[-1.0]), strict=False))
    with pytest.raises(dsl.DomainError, match="out of range"):
        ev("y[i+5]", y=np.zeros(3), i=0)
    with pytest.raises(dsl.DomainError, match="out of range"):
        dsl.evaluate(dsl.parse("y[i+1]"), ctx(y=np.zeros(3), i=None))
    assert ev("y[i+1]", y=np.array([1.0, 2.0, 3.0]), i=1) == 3.0
    with pytest.raises(ValueError):
        ev("1", y=np.zeros(2), i=5)


def test_model_file_runs(tmp_path):
    path = tmp_path / "linear.model"
    path.write_text("nequat=2\nnparams=3\nnnoise=2\ndrift: 0 - p[0]*y[i]\n"
                    "diffusion: p[1+i]*n[i]\n", encoding="utf-8")
    model = sdb.model_from_file(path)
    g = np.random.default_rng(1)
    batch = OrbitBatch(init=g.standard_normal((20, 2)), params=g.uniform(0.1, 1.0, (20, 3)))
    cfg = EngineConfig(dt=0.01, tspan=1.0, ksteps=10, orbits=20, seed=4)
    store = run_batch(model, cfg, batch)
    drift, diffusion = O.expression_model("0 - p[0]*y[i]", "p[1+i]*n[i]")
    _, want, _ = O.integrate(batch.init, batch.params, dt=0.01, ksteps=10, chunks=10, seed=4,
                             nnoise=2, drift=drift, diffusion=diffusion)
    assert O.mixed_error(store.values, want) <= PARITY_TOL


@pytest.mark.parametrize("name", ["tdep", "nested", "rk4", "fail", "big"])
def test_lane_groups_bit_identical(golden_dsl, name, monkeypatch):
    # 1..32 lanes per orbit (and the global-scratch columns at 1 lane for
    # "big") give the same bits: each equation is evaluated identically
    arrays, cases = golden_dsl
    case = cases[name]
    model = case_model(case, name)
    hashes = set()
    for lanes in (1, 2, 4, 8, 16, 32):
        monkeypatch.setenv("SDEB200_DSL_LANES", str(lanes))
        store = run_batch(model, case_cfg(case, stream="sfc64" if case["nnoise"] else "philox"),
                          case_batch(arrays, name))
        assert last_launch_info()["lanes"] == lanes
        hashes.add(sdb.store_hash(store))
    assert len(hashes) == 1


def test_global_state_columns_match_shared(monkeypatch):
    # 120 equations at one lane per orbit: the columns do not fit shared
    # memory and live in global scratch
    n = 120
    model = sdb.model_from_dsl("wide", n, 2, n, "p[0]*sum(j, sin(y[j] - y[i]))/N - p[1]*y[i]",
                               "0.1*n[i]")
    g = np.random.default_rng(2)
    m = 50
    batch = OrbitBatch(init=g.uniform(-2, 2, (m, n)), params=g.uniform(0.1, 0.9, (m, 2)))
    cfg = EngineConfig(dt=0.01, tspan=0.2, ksteps=5, orbits=m, seed=3)
    monkeypatch.setenv("SDEB200_DSL_LANES", "1")
    a = run_batch(model, cfg, batch)
    monkeypatch.setenv("SDEB200_DSL_LANES", "32")
    b = run_batch(model, cfg, batch)
    assert sdb.store_hash(a) == sdb.store_hash(b)
    drift, diffusion = O.expression_model("p[0]*sum(j, sin(y[j] - y[i]))/N - p[1]*y[i]",
                                          "0.1*n[i]")
    _, want, _ = O.integrate(batch.init, batch.params, dt=0.01, ksteps=5, chunks=4, seed=3,
                             nnoise=n, drift=drift, diffusion=diffusion)
    assert O.mixed_error(a.values, want) <= PARITY_TOL
