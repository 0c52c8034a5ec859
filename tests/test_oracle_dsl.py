"""Pins the oracle's expression-template restatement (oracle/sdeb_oracle.py,
evaluate_expression / expression_model) against the reference's own run_batch
stores and drift/diffusion evaluations (tests/golden/make_golden_dsl.py)."""

import math

import numpy as np
import pytest

from oracle import sdeb_oracle as O

CASES = ["ou", "tdep", "nested", "funcs", "rk4", "euler", "fail", "big", "kuramoto"]


def run_oracle(arrays, case, name, **kw):
    drift, diffusion = O.expression_model(case["drift"], case["diffusion"])
    chunks = case["steps"] // case["ksteps"]
    return O.integrate(arrays[name + "_init"], arrays[name + "_params"], dt=case["dt"],
                       ksteps=case["ksteps"], chunks=chunks, seed=case["seed"],
                       solver=case["solver"], nnoise=case["nnoise"], drift=drift,
                       diffusion=diffusion, **kw)


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_reference_stores(golden_dsl, name):
    arrays, cases = golden_dsl
    case = cases[name]
    _, values, fails = run_oracle(arrays, case, name)
    # same op order as the reference interpreter: bit-identical on this host
    assert O.mixed_error(values, arrays[name + "_values"]) <= 1e-12
    assert [list(f[:3]) for f in fails] == [f[:3] for f in case["failures"]]
    for got, want in zip(fails, case["failures"]):
        assert math.isclose(got[3], want[3], rel_tol=0, abs_tol=1e-15)


@pytest.mark.parametrize("name", CASES)
def test_oracle_evaluations(golden_dsl, name):
    arrays, cases = golden_dsl
    case = cases[name]
    y, p = arrays[name + "_eval_y"], arrays[name + "_eval_p"]
    got = O.evaluate_expression(case["drift"], 0.37, y, p)
    assert np.array_equal(got, arrays[name + "_drift"], equal_nan=True)
    if case["nnoise"]:
        z = arrays[name + "_eval_noise"]
        got = O.evaluate_expression(case["diffusion"], 0.37, y, p, z)
        assert np.array_equal(got, arrays[name + "_diffusion"], equal_nan=True)


def test_oracle_expression_kuramoto_equals_native_restatement(golden_dsl):
    # the template Kuramoto through the interpreter == the native drift (the
    # reference's DSL-vs-native bitwise property, test_model.py:125-134)
    g = np.random.default_rng(5)
    y, p = g.standard_normal((7, 8)), g.standard_normal((7, 17))
    from_template = O.evaluate_expression("p[i+1] + (p[0]/N) * sum(j, sin(y[j] - y[i]))", 0.0,
                                          y, p)
    assert np.array_equal(from_template, O.kuramoto_drift(y, p))


def test_oracle_shard_offsets_for_expression_models(golden_dsl):
    arrays, cases = golden_dsl
    case = cases["ou"]
    _, whole, _ = run_oracle(arrays, case, "ou")
    ids = np.arange(16, dtype=np.uint64)
    _, part, _ = run_oracle(arrays, case, "ou", orbit_ids=ids, group=5, threads=3)
    assert np.array_equal(whole, part)
