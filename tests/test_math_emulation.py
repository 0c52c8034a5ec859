"""CPU-tier check of the device math algorithms (csrc/sdeb_math.cuh) by exact
emulation: every FMA is evaluated in rational arithmetic and rounded once,
every other op is a plain IEEE double op -- exactly what the sm_100a code
does.  Catches table / constant / reduction mistakes without a GPU; the GPU
tier (test_gpu_math.py) then checks the compiled code itself."""

import math
import os
import re
import struct
from fractions import Fraction

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1908_03869_b200", "csrc")


def _dbl(bits):
    return struct.unpack("<d", struct.pack("<Q", bits & (2 ** 64 - 1)))[0]


def _bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _constants():
    text = open(os.path.join(CSRC, "sdeb_math.cuh")).read()
    body = text[text.index("kMC[MC_COUNT] = {"):]
    body = body[body.index("{") + 1:body.index("};")]
    body = re.sub(r"//[^\n]*", "", body)
    vals = [eval(v.strip()) for v in body.split(",") if v.strip()]  # noqa: S307 (own source)
    names = re.findall(r"MC_[A-Z0-9_]+", text[text.index("enum MathConst"):text.index("MC_COUNT")])
    return dict(zip(names, vals))


def _log_table():
    text = open(os.path.join(CSRC, "sdeb_log_table.cuh")).read()
    return [(_dbl(int(a, 16)), _dbl(int(b, 16)))
            for a, b in re.findall(r"\{0x([0-9A-F]+)ULL, 0x([0-9A-F]+)ULL\}", text)]


C = _constants()
TAB = _log_table()
MAGIC = 6755399441055744.0


def emu_sincos(x):
    t = fma(x, C["MC_TWO_OVER_PI"], MAGIC)
    q = _bits(t) & 0xFFFFFFFF
    q = q - 2 ** 32 if q >= 2 ** 31 else q
    qd = t - MAGIC
    r = fma(-qd, C["MC_PIO2_1"], x)
    r = fma(-qd, C["MC_PIO2_2"], r)
    r = fma(-qd, C["MC_PIO2_3"], r)
    r2 = r * r
    ps = fma(r2, C["MC_S6"], C["MC_S5"])
    for k in ("MC_S4", "MC_S3", "MC_S2", "MC_S1"):
        ps = fma(r2, ps, C[k])
    sr = fma(r2 * r, ps, r)
    pc = fma(r2, C["MC_C6"], C["MC_C5"])
    for k in ("MC_C4", "MC_C3", "MC_C2", "MC_C1"):
        pc = fma(r2, pc, C[k])
    cr = fma(r2 * r2, pc, fma(r2, -0.5, 1.0))
    so, co = (cr, sr) if q & 1 else (sr, cr)
    s = -so if q & 2 else so
    c = -co if (q + 1) & 2 else co
    return s, c


def emu_neg2_log(x):
    """neg2_log_pos (sdeb_math.cuh): -2 ln x from the pre-scaled table."""
    ix = _bits(x)
    tmp = (ix - 0x3FE6000000000000) & (2 ** 64 - 1)
    i = (tmp >> 43) & 511
    k = (tmp - (2 ** 64 if tmp >= 2 ** 63 else 0)) >> 52
    z = _dbl(ix - (tmp & (0xFFF << 52)))
    m2invc, m2logc = TAB[i]
    r = fma(z, m2invc, 2.0)
    p = fma(r, C["MC_LB4"], C["MC_LB3"])
    p = fma(r, p, 2.0 ** -5)
    p = fma(r, p, C["MC_LB1"])
    p = fma(r, p, 0.25)
    lp = fma(r * r, p, r)
    hi = fma(float(k), C["MC_M2LN2_HI"], m2logc)
    lo = fma(float(k), C["MC_M2LN2_LO"], lp)
    return hi + lo


def emu_log(x):
    return -0.5 * emu_neg2_log(x)  # exact rescale (the math probe's log)


def emu_log_unscaled(x):
    """The same table log written in r = z invc - 1 with the unscaled table
    (invc, logc) and series 1/7, -1/6, ...: neg2_log_pos must equal -2 times
    this bit for bit (every intermediate is a power-of-two scaling)."""
    ix = _bits(x)
    tmp = (ix - 0x3FE6000000000000) & (2 ** 64 - 1)
    i = (tmp >> 43) & 511
    k = (tmp - (2 ** 64 if tmp >= 2 ** 63 else 0)) >> 52
    z = _dbl(ix - (tmp & (0xFFF << 52)))
    invc, logc = -0.5 * TAB[i][0], -0.5 * TAB[i][1]
    r = fma(z, invc, -1.0)
    p = fma(r, -1.0 / 6.0, 0.2)
    p = fma(r, p, -0.25)
    p = fma(r, p, 1.0 / 3.0)
    p = fma(r, p, -0.5)
    lp = fma(r * r, p, r)
    hi = fma(float(k), math.log(2.0), logc)
    lo = fma(float(k), 2.31904681384629955842e-17, lp)
    return hi + lo


def ulps(got, ref):
    return abs(got - ref) / math.ulp(ref) if ref != 0 else (0.0 if got == 0 else math.inf)


def test_constants_are_the_intended_values():
    assert C["MC_PIO2_1"] + C["MC_PIO2_2"] == C["MC_PIO2_1"]
    assert Fraction(C["MC_PIO2_1"]) + Fraction(C["MC_PIO2_2"]) + Fraction(C["MC_PIO2_3"]) \
        != Fraction(C["MC_PIO2_1"])
    assert C["MC_M2LN2_HI"] == -2.0 * math.log(2.0)
    assert C["MC_LB4"] == (1.0 / 6.0) / 32
    assert C["MC_LB3"] == 0.2 / 16 and C["MC_LB1"] == (1.0 / 3.0) / 4
    assert C["MC_U32_BIAS"] == 2.0 ** 20 - 2.0 ** -32
    assert len(TAB) == 512 and TAB[319] == (-2.0, 0.0) and TAB[320] == (-2.0, 0.0)  # -2 (invc, logc)


def test_uniform_map_is_exact():
    for w in (0, 1, 2 ** 31 - 1, 2 ** 31, 2 ** 32 - 2, 2 ** 32 - 1, 123456789):
        via_bits = _dbl((0x41300000 << 32) | w) - C["MC_U32_BIAS"]
        assert via_bits == (w + 1.0) * 2.0 ** -32


def test_emulated_sincos_within_2ulp():
    g = np.random.default_rng(0)
    xs = list(g.uniform(-np.pi, np.pi, 1500)) + list(g.uniform(-2e3, 2e3, 1500)) + \
        [k * math.pi / 4 for k in range(-40, 41)] + [0.0, 1e-300, 3.0e8]
    for x in xs:
        s, c = emu_sincos(float(x))
        assert ulps(s, math.sin(x)) <= 2 or abs(s - math.sin(x)) <= 2.3e-16, x
        assert ulps(c, math.cos(x)) <= 2 or abs(c - math.cos(x)) <= 2.3e-16, x


def test_emulated_log_within_1ulp_on_box_muller_uniforms():
    g = np.random.default_rng(1)
    ws = list(g.integers(0, 2 ** 32, 3000)) + [2 ** 32 - 1 - j for j in range(300)] + \
        [2 ** 31 + j - 150 for j in range(300)] + list(range(100))
    for w in ws:
        u = (int(w) + 1.0) * 2.0 ** -32
        assert ulps(emu_log(u), math.log(u)) <= 1.0, w
    assert emu_log(1.0) == 0.0


@pytest.mark.parametrize("x", [0.5, 0.75, 0.99999, 1.0, 1.5, 2.0, 44.0])
def test_emulated_log_general_points(x):
    assert ulps(emu_log(x), math.log(x)) <= 1.0


def _sincos_table():
    text = open(os.path.join(CSRC, "sdeb_sincos_table.cuh")).read()
    return [(_dbl(int(a, 16)), _dbl(int(b, 16)))
            for a, b in re.findall(r"\{0x([0-9A-F]+)ULL, 0x([0-9A-F]+)ULL\}", text)]


SCT = _sincos_table()


def emu_sincos_tab(x):
    t = fma(x, C["MC_TAB_OVER_PI"], MAGIC)
    k = _bits(t) & 0xFFFFFFFF
    kd = t - MAGIC
    r = fma(-kd, C["MC_PITAB_1"], x)
    r = fma(-kd, C["MC_PITAB_2"], r)
    sa, ca = SCT[k & (len(SCT) - 1)]
    r2 = r * r
    ps = fma(r2, C["MC_T_S5"], C["MC_T_S3"])
    sr = fma(r2 * r, ps, r)
    pc = fma(r2, C["MC_T_C4"], -0.5)
    cr = fma(r2, pc, 1.0)
    return fma(sa, cr, ca * sr), fma(ca, cr, -(sa * sr))


def test_table_sincos_constants():
    from decimal import Decimal, getcontext
    getcontext().prec = 50
    pi = Decimal("3.14159265358979323846264338327950288419716939937510582097494")
    split = Decimal(C["MC_PITAB_1"]) + Decimal(C["MC_PITAB_2"])
    assert abs(split - pi / 512) < Decimal(10) ** -34  # |kd| * err < 2^-76 for |x| < 2^29
    assert C["MC_PITAB_1"] == math.pi / 512 and C["MC_TAB_OVER_PI"] == 512 / math.pi
    assert len(SCT) == 1024 and SCT[0] == (0.0, 1.0) and SCT[256] == (1.0, 0.0)
    for k in range(1, 1024):
        assert SCT[1024 - k][0] == -SCT[k][0] and SCT[1024 - k][1] == SCT[k][1]


def test_emulated_table_sincos_within_2ulp_and_odd():
    g = np.random.default_rng(7)
    xs = list(g.uniform(-np.pi, np.pi, 1500)) + list(g.uniform(-2e3, 2e3, 1500)) + \
        list(g.uniform(0, 2 * np.pi, 500)) + [k * math.pi / 512 for k in range(-1200, 1201, 7)] + \
        [(k + 0.5) * math.pi / 512 for k in range(-40, 40)] + \
        [0.0, 1e-300, 3.0e8, 2 * math.pi]
    for x in xs:
        s, c = emu_sincos_tab(float(x))
        assert ulps(s, math.sin(x)) <= 2 or abs(s - math.sin(x)) <= 2.3e-16, x
        assert ulps(c, math.cos(x)) <= 2 or abs(c - math.cos(x)) <= 2.3e-16, x
        ns, nc = emu_sincos_tab(-float(x))
        assert ns == -s and nc == c, x


def emu_sincos_turn(w):
    v = w + 1
    k = (v + 2 ** 21) >> 22
    m = v - (k << 22)
    md = float(m)
    r = md * C["MC_TWO_PI_2M32"]
    sa, ca = SCT[k & (len(SCT) - 1)]
    r2 = r * r
    ps = fma(r2, C["MC_T_S5"], C["MC_T_S3"])
    sr = fma(r2 * r, ps, r)
    pc = fma(r2, C["MC_T_C4"], -0.5)
    cr = fma(r2, pc, 1.0)
    return fma(sa, cr, ca * sr), fma(ca, cr, -(sa * sr))


def test_box_muller_angle_reduction():
    assert C["MC_TWO_PI_2M32"] == 2.0 * math.pi * 2.0 ** -32
    assert C["MC_TURN_BIAS"] == 2.0 ** 52 + 2.0 ** 31
    g = np.random.default_rng(11)
    ws = [int(x) for x in g.integers(0, 2 ** 32, 3000)] + list(range(300)) + \
        [2 ** 32 - 1 - j for j in range(300)] + [k * 2 ** 22 + d for k in range(0, 1024, 37)
                                                for d in (-1, 0, 1, 2 ** 21 - 1, 2 ** 21)]
    for w in ws:
        if not 0 <= w < 2 ** 32:
            continue
        ang = 2.0 * math.pi * ((w + 1.0) * 2.0 ** -32)
        s, c = emu_sincos_turn(w)
        assert abs(s - math.sin(ang)) <= 8e-16 and abs(c - math.cos(ang)) <= 8e-16, w


def test_neg2_log_is_exact_power_of_two_scaling():
    g = np.random.default_rng(11)
    words = list(g.integers(0, 2 ** 32, 4000)) + [0, 1, 2 ** 31, 2 ** 32 - 2, 2 ** 32 - 1]
    xs = [(int(w) + 1.0) * 2.0 ** -32 for w in words] + list(g.uniform(1e-3, 1e3, 2000))
    for x in xs:
        assert emu_neg2_log(x) == -2.0 * emu_log_unscaled(x), x
