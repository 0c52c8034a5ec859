"""Host-side analysis helpers (small reductions over already-reduced arrays;
analysis.py:72-74, 104-139)."""

import math

import numpy as np
import pytest

from paper_1908_03869_b200 import analysis


def test_wrap_phase_matches_reference_golden(golden_analysis):
    arrays, _ = golden_analysis
    assert np.array_equal(analysis.wrap_phase(arrays["wrap_in"]), arrays["wrap_out"])
    w = analysis.wrap_phase(np.linspace(-20, 20, 1001))
    assert (w >= -math.pi).all() and (w < math.pi).all()


def test_ensemble_stats_and_errors():
    r = np.array([[0.1, 0.5, 0.9], [0.3, 0.5, 0.7]])
    st = analysis.ensemble_stats(r)
    assert np.allclose(st.mean_r, [0.2, 0.5, 0.8]) and np.allclose(st.std_r, [0.1, 0.0, 0.1])
    assert st.count == 2 and np.array_equal(st.times, [0.0, 1.0, 2.0])
    with pytest.raises(ValueError, match="at least 2"):
        analysis.ensemble_stats(r[:1])
    with pytest.raises(ValueError, match="unequal"):
        analysis.ensemble_stats([[0.1, 0.2], [0.3]])
    with pytest.raises(ValueError, match="times length"):
        analysis.ensemble_stats(r, times=[0.0, 1.0])


def test_first_crossing_time():
    t = np.array([0.0, 1.0, 2.0, 3.0])
    assert analysis.first_crossing_time(t, [0.1, 0.4, 0.6, 0.9], 0.5) == 2.0
    assert analysis.first_crossing_time(t, [0.1, 0.2, 0.3, 0.4], 0.5) is None
    assert analysis.STABILITY_DT_VALUES == (0.0125, 0.025, 0.05, 0.1, 0.2)
