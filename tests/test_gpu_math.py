"""Accuracy of the stepper's custom FP64 math (csrc/sdeb_math.cuh) against
numpy/glibc, in units in the last place, over the argument ranges the
stepper uses: unwrapped phases and phase differences (sincos), Box-Muller
uniforms in (0, 1] (log) and radii arguments in [0, 45] (sqrt)."""

import ctypes

import numpy as np
import pytest

from paper_1908_03869_b200 import _native as nat

pytestmark = pytest.mark.gpu


def probe(func, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    ctx = nat.context()
    nat.check(nat.lib().sdb_math_probe(ctx, func, nat.dptr(x), x.size, nat.dptr(out)), ctx)
    return out


def ulp_err(got, ref):
    ref = np.asarray(ref, dtype=np.float64)
    scale = np.spacing(np.maximum(np.abs(ref), np.finfo(np.float64).tiny))
    return np.abs(got - ref) / scale


def test_sincos_accuracy():
    g = np.random.default_rng(0)
    x = np.concatenate([g.uniform(-np.pi, np.pi, 200000), g.uniform(-1e3, 1e3, 200000),
                        g.uniform(-1e6, 1e6, 50000), g.uniform(-1e12, 1e12, 2000),
                        np.arange(-64, 65) * (np.pi / 4), [0.0, -0.0, 1e-300, 5e-324]])
    s, c = probe(0, x), probe(1, x)
    # absolute error bound relative to ulp(1) for results near zero, 2 ulp otherwise
    ds = np.abs(s - np.sin(x))
    dc = np.abs(c - np.cos(x))
    assert np.all((ulp_err(s, np.sin(x)) <= 2) | (ds <= 2.3e-16)), ulp_err(s, np.sin(x)).max()
    assert np.all((ulp_err(c, np.cos(x)) <= 2) | (dc <= 2.3e-16)), ulp_err(c, np.cos(x)).max()
    # documented deviation: sin(-0.0) returns +0.0 (r + r^3*p with p < 0 cannot
    # keep the sign of a zero); only the sign of an exact zero differs
    assert probe(0, np.array([-0.0]))[0] == 0.0


def test_sin_odd_cos_even_bitwise():
    g = np.random.default_rng(1)
    x = g.uniform(-50, 50, 100000)
    assert np.array_equal(probe(0, -x), -probe(0, x))
    assert np.array_equal(probe(1, -x), probe(1, x))


def test_sincos_nonfinite():
    x = np.array([np.inf, -np.inf, np.nan])
    assert np.isnan(probe(0, x)).all() and np.isnan(probe(1, x)).all()


def test_log_accuracy():
    g = np.random.default_rng(2)
    w = g.integers(0, 2 ** 32, 300000, dtype=np.uint64)
    edges = np.array([0, 1, 2, 2 ** 31 - 1, 2 ** 31, 2 ** 32 - 2, 2 ** 32 - 1], dtype=np.uint64)
    u = (np.concatenate([w, edges]).astype(np.float64) + 1.0) * 2.0 ** -32
    got = probe(2, u)
    assert got[-1] == 0.0  # log(1) exactly
    assert ulp_err(got, np.log(u)).max() <= 2
    x = g.uniform(0.5, 50.0, 100000)
    assert ulp_err(probe(2, x), np.log(x)).max() <= 2


def test_sqrt_accuracy():
    g = np.random.default_rng(3)
    x = np.concatenate([g.uniform(0, 45, 300000), [0.0, 4.7e-10, 44.36, 1.0, 4.0]])
    got = probe(3, x)
    assert got[-5] == 0.0
    assert ulp_err(got, np.sqrt(x)).max() <= 1


def test_libdevice_probe_matches_numpy_closely():
    g = np.random.default_rng(4)
    x = g.uniform(-100, 100, 10000)
    assert ulp_err(probe(4, x), np.sin(x)).max() <= 2


def test_box_muller_angle_sincos():
    # sin / cos(2 pi u), u = (w + 1) 2^-32, reduced from the word (sincos_turn)
    g = np.random.default_rng(5)
    w = np.concatenate([g.integers(0, 2 ** 32, 20000), np.arange(0, 3000),
                        2 ** 32 - 1 - np.arange(0, 3000), (np.arange(-3, 4) + 2 ** 31),
                        np.arange(1025) * 2 ** 22 - 1]).astype(np.uint64)
    w = w[w < 2 ** 32].astype(np.float64)
    ang = 2.0 * np.pi * ((w + 1.0) * 2.0 ** -32)
    s, c = probe(7, w), probe(8, w)
    # vs the reference's sin(fl(2 pi u)): the exact angle differs from the rounded
    # one by <= 0.5 ulp(angle) <= 4.5e-16
    assert np.abs(s - np.sin(ang)).max() <= 8e-16
    assert np.abs(c - np.cos(ang)).max() <= 8e-16
