"""Pins the oracle's analysis restatement (analysis.py:72-186) against the
reference's own outputs (tests/golden/make_golden_analysis.py)."""

import numpy as np

from oracle import sdeb_oracle as O


def test_wrap_phase_golden(golden_analysis):
    arrays, _ = golden_analysis
    assert np.array_equal(O.wrap_phase(arrays["wrap_in"]), arrays["wrap_out"])


def test_order_parameter_golden(golden_analysis):
    arrays, cases = golden_analysis
    for k in range(cases["populations"]):
        r, phi = O.order_parameter_arrays(arrays["pop_%d" % k])
        assert np.array_equal(np.array([r, phi]), arrays["pop_%d_rphi" % k])


def test_coherence_and_stats_golden(golden_analysis):
    arrays, _ = golden_analysis
    for name in ("sync", "incoh", "n5"):
        r, phi = O.order_parameter_arrays(arrays[name + "_values"])
        assert np.array_equal(r, arrays[name + "_r"])
        assert np.array_equal(phi, arrays[name + "_phi"])
        mean, std = O.ensemble_mean_std(r)
        assert np.array_equal(mean, arrays[name + "_mean_r"])
        assert np.array_equal(std, arrays[name + "_std_r"])
        assert np.array_equal(O.wrap_phase(arrays[name + "_values"][1]), arrays[name + "_kymo1"])


def test_oracle_run_reproduces_analysis_stores(golden_analysis):
    # the restated loop regenerates the stores the analysis goldens were taken on
    arrays, cases = golden_analysis
    for name in ("sync", "n5"):
        c = cases[name]
        _, values, _ = O.integrate(arrays[name + "_init"], arrays[name + "_params"], dt=c["dt"],
                                   ksteps=c["ksteps"],
                                   chunks=O.iteration_count(c["tspan"], c["dt"], c["ksteps"]),
                                   seed=c["seed"])
        assert O.mixed_error(values, arrays[name + "_values"]) <= 1e-12
