// Branch-free FP64 sincos / log / sqrt for the stepper (sm_100a).
//
// Why: ncu on the v1 kernel (profiles/r01/SUMMARY_v1.md) showed the fused
// stepper ISSUE-bound, not FP64-bound: libdevice's sincos/log/sqrt spend
// F2I/I2F.F64 round trips (XU pipe), BSSY/BSYNC-guarded slow paths and
// re-materialised 64-bit constants around ~60 FP64 ops per oscillator-step.
// These versions keep the FP64 work (~20 ops per sincos, ~12 per log) and
// drop almost everything else:
//   - round-to-nearest quadrant by the 1.5*2^52 magic add (no F2I/I2F; the
//     quadrant is the low word of the sum);
//   - 3-part Cody-Waite pi/2 reduction with FMA (exact first step);
//   - fdlibm __kernel_sin/__kernel_cos minimax coefficients on [-pi/4, pi/4];
//   - quadrant rotation by integer select + sign-bit xor on the high word;
//   - log: 128-entry (1/c, -ln(1/c)) table (sdeb_log_table.cuh, generated
//     with 60-digit decimal arithmetic) + degree-8 log1p polynomial;
//   - sqrt: MUFU.RSQ64H seed + one Goldschmidt step + Markstein correction.
// Accuracy (tests/test_gpu_math.py): sincos/log/sqrt within 2 ulp of
// numpy/glibc on the argument ranges the stepper uses.  sin is bitwise odd
// and cos even, which the antisymmetric pairwise tiling relies on.
// |x| >= 2^29 falls back to libdevice sincos (exact Payne-Hanek reduction).
#pragma once
#include "sdeb_cstdint.cuh"

#include "sdeb_log_table.cuh"
#include "sdeb_sincos_table.cuh"

namespace sdeb {

// Polynomial coefficients and reduction constants live in the constant bank:
// DFMA cannot encode a full 64-bit immediate, and as literals ptxas
// re-materialised each one with two UMOVs per use inside the step loop
// (~220 issue slots per iteration in the v2 SASS); from c[] one LDCU.128
// fetches two.  Values that fit a 32-bit high-word immediate (0.5, 1.0,
// 1.5*2^52, ...) stay literals.
enum MathConst : int {
    MC_S1, MC_S2, MC_S3, MC_S4, MC_S5, MC_S6,  // fdlibm k_sin.c (|r| <= pi/4)
    MC_C1, MC_C2, MC_C3, MC_C4, MC_C5, MC_C6,  // fdlibm k_cos.c
    MC_TWO_OVER_PI, MC_PIO2_1, MC_PIO2_2, MC_PIO2_3,
    MC_M2LN2_HI, MC_M2LN2_LO, MC_U32_BIAS,               // -2 ln 2 split; uniform bias
    MC_LB4, MC_LB3, MC_LB1,                              // -2 log1p series in -2r (neg2_log_pos)
    MC_TAB_OVER_PI, MC_PITAB_1, MC_PITAB_2,              // table sincos reduction (pi/512)
    MC_T_S3, MC_T_S5, MC_T_C4,                           // Taylor terms on |r| <= pi/1024
    MC_TURN_BIAS, MC_TWO_PI_2M32,                        // Box-Muller angle (sincos_turn)
    MC_COUNT
};

__constant__ static double kMC[MC_COUNT] = {  // non-const: keeps ptxas from folding them back into UMOV pairs
    -1.66666666666666324348e-01, 8.33333333332248946124e-03, -1.98412698298579493134e-04,
    2.75573137070700676789e-06, -2.50507602534068634195e-08, 1.58969099521155010221e-10,
    4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05,
    -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11,
    6.36619772367581382433e-01,  // 2/pi
    1.5707963267948966,          // fl(pi/2)
    6.123233995736766e-17,       // fl(pi/2 - fl(pi/2))
    -1.4973849048591698e-33,     // next 53 bits of pi/2
    -2 * 6.93147180559945286227e-01,  // -2 fl(ln 2) (exact scaling)
    -2 * 2.31904681384629955842e-17,  // -2 fl(ln 2 - fl(ln 2))
    1048576.0 - 2.3283064365386963e-10,  // 2^20 - 2^-32 (exact)
    0.16666666666666666 / 32,                             // fl(1/6) 2^-5
    0.2 / 16, 0.3333333333333333 / 4,                     // fl(1/5) 2^-4, fl(1/3) 2^-2
    162.97466172610083,          // 512/pi = 4 * fl(128/pi) (exact scaling)
    0.006135923151542565,        // fl(pi/512) = fl(pi) * 2^-9
    2.391888279584674e-19,       // fl(pi/512 - fl(pi/512)) (pi/512 = PITAB_1 + PITAB_2 + O(2^-115))
    -0.16666666666666666, 0.008333333333333333,  // -1/6, 1/120
    0.041666666666666664,                        // 1/24
    4503601774854144.0,                          // 2^52 + 2^31 (biased int -> double)
    1.4629180792671596e-09,                      // fl(2 pi) * 2^-32 (exact scaling)
};

// Table reads.  Translation units that define SDEB_SMEM_TABLES (the fused
// stepper's) stage both tables in static shared memory at kernel start
// (stage_tables()) and read them with LDS: a 32-bit address from the index in
// two integer ops instead of four for the 64-bit global address, and no L1 tag
// traffic.  Everything else reads the global copies through the read-only path.
constexpr size_t kTableSmemBytes = 16 * (kSinCosN + (1 << kLogTableBits));  // both, staged
#ifdef SDEB_SMEM_TABLES
__shared__ double2 s_sincos_tab[kSinCosN];
__shared__ double2 s_log_tab[1 << kLogTableBits];

// Cooperative copy of both tables into shared memory; every thread of the CTA
// must call it (it ends with a barrier).
__device__ __forceinline__ void stage_tables() {
    const double2* gs = reinterpret_cast<const double2*>(kSinCosTable);
    const double2* gl = reinterpret_cast<const double2*>(kLogTable);
    for (int i = threadIdx.x; i < kSinCosN; i += blockDim.x) s_sincos_tab[i] = __ldg(gs + i);
    for (int i = threadIdx.x; i < (1 << kLogTableBits); i += blockDim.x) s_log_tab[i] = __ldg(gl + i);
    __syncthreads();
}

__device__ __forceinline__ double2 sincos_entry(int k) { return s_sincos_tab[k & (kSinCosN - 1)]; }
constexpr size_t kStaticSmemBytes = kTableSmemBytes;
__device__ __forceinline__ double2 log_entry(int i) { return s_log_tab[i]; }
#else
constexpr size_t kStaticSmemBytes = 0;
__device__ __forceinline__ void stage_tables() {}
__device__ __forceinline__ double2 sincos_entry(int k) {
    return __ldg(reinterpret_cast<const double2*>(kSinCosTable[k & (kSinCosN - 1)]));
}
__device__ __forceinline__ double2 log_entry(int i) {
    return __ldg(reinterpret_cast<const double2*>(kLogTable[i]));
}
#endif

constexpr double kRoundMagic = 6755399441055744.0;  // 1.5 * 2^52
constexpr double kSmallArg = 536870912.0;           // 2^29: fast reduction bound

// (w + 1) * 2^-32 (rng.py:121-129) in ONE exact DADD, no I2F conversion.
__device__ __forceinline__ double u32_to_uniform(uint32_t w) {
    return __dsub_rn(__hiloint2double(0x41300000, int(w)), kMC[MC_U32_BIAS]);
}

// w * 2^-32 (rng.py:221, sampling uniforms) in one exact DADD.
__device__ __forceinline__ double u32_to_unit(uint32_t w) {
    return __dsub_rn(__hiloint2double(0x41300000, int(w)), 1048576.0);
}

// sin / cos of r in [-pi/4, pi/4] (slightly beyond is fine), rotated by q*pi/2.
__device__ __forceinline__ void sincos_reduced(double r, int q, double& s, double& c) {
    const double r2 = __dmul_rn(r, r);
    double ps = __fma_rn(r2, kMC[MC_S6], kMC[MC_S5]);
    ps = __fma_rn(r2, ps, kMC[MC_S4]);
    ps = __fma_rn(r2, ps, kMC[MC_S3]);
    ps = __fma_rn(r2, ps, kMC[MC_S2]);
    ps = __fma_rn(r2, ps, kMC[MC_S1]);
    const double sr = __fma_rn(__dmul_rn(r2, r), ps, r);
    double pc = __fma_rn(r2, kMC[MC_C6], kMC[MC_C5]);
    pc = __fma_rn(r2, pc, kMC[MC_C4]);
    pc = __fma_rn(r2, pc, kMC[MC_C3]);
    pc = __fma_rn(r2, pc, kMC[MC_C2]);
    pc = __fma_rn(r2, pc, kMC[MC_C1]);
    const double cr = __fma_rn(__dmul_rn(r2, r2), pc, __fma_rn(r2, -0.5, 1.0));
    const bool swap = (q & 1) != 0;
    const double so = swap ? cr : sr;
    const double co = swap ? sr : cr;
    const int ssign = (q & 2) << 30;        // sin < 0 in quadrants 2, 3
    const int csign = ((q + 1) & 2) << 30;  // cos < 0 in quadrants 1, 2
    s = __hiloint2double(__double2hiint(so) ^ ssign, __double2loint(so));
    c = __hiloint2double(__double2hiint(co) ^ csign, __double2loint(co));
}

// Quadrant form (pi/2 reduction + fdlibm kernels): the v2 stepper's sincos,
// kept as the cross-check for the table form in tests/test_gpu_math.py.
__device__ __forceinline__ void sincos_quadrant(double x, double& s, double& c) {
    const double t = __fma_rn(x, kMC[MC_TWO_OVER_PI], kRoundMagic);
    const int q = __double2loint(t);
    const double qd = __dsub_rn(t, kRoundMagic);
    double r = __fma_rn(-qd, kMC[MC_PIO2_1], x);  // exact for |q| < 2^29
    r = __fma_rn(-qd, kMC[MC_PIO2_2], r);
    r = __fma_rn(-qd, kMC[MC_PIO2_3], r);
    sincos_reduced(r, q, s, c);
}

// Table-driven sincos, |x| < 2^29: x = k*pi/512 + r, |r| <= pi/1024 (3-part
// Cody-Waite, first step exact), (sin, cos)(k*pi/512) from a 1024-entry
// correctly-rounded table indexed by k & 1023 (no quadrant logic), Taylor
// terms to r^5 / r^4 (the next ones are < 2^-60 relative), and the
// angle-addition rotation: 15 FP64 ops + one 16-byte load (the v10 256-entry
// table needed 17, the minimax/quadrant form 22 + ~8 select/sign ops).
// Exactly odd in x (the table is antisymmetric in sin).
__device__ __forceinline__ void sincos_tab(double x, double& s, double& c) {
    const double t = __fma_rn(x, kMC[MC_TAB_OVER_PI], kRoundMagic);
    const int k = __double2loint(t);
    const double kd = __dsub_rn(t, kRoundMagic);
    // two-part Cody-Waite: the split's own error, |kd| * O(2^-115) < 2^-76 for
    // |x| < 2^29, is far below the result's ulp (a third part bought nothing)
    double r = __fma_rn(-kd, kMC[MC_PITAB_1], x);
    r = __fma_rn(-kd, kMC[MC_PITAB_2], r);
    const double2 e = sincos_entry(k);
    const double r2 = __dmul_rn(r, r);
    const double ps = __fma_rn(r2, kMC[MC_T_S5], kMC[MC_T_S3]);
    const double sr = __fma_rn(__dmul_rn(r2, r), ps, r);             // sin r
    const double pc = __fma_rn(r2, kMC[MC_T_C4], -0.5);
    const double cr = __fma_rn(r2, pc, 1.0);                         // cos r
    s = __fma_rn(e.x, cr, __dmul_rn(e.y, sr));                       // sin(a + r)
    c = __fma_rn(e.y, cr, -__dmul_rn(e.x, sr));                      // cos(a + r)
}

// sin / cos of the Box-Muller angle 2*pi*u, u = (w + 1) * 2^-32 (rng.py:183-187),
// reduced in integer arithmetic: v = w + 1 = k*2^22 + m with |m| <= 2^21, so
// 2*pi*u = k*pi/512 + m*(2*pi*2^-32): the table entry k & 1023 and a residual
// r = m * fl(2 pi) * 2^-32 with one rounding (|r| <= pi/1024).  2 FP64 ops
// replace the uniform conversion, the angle product and the 5-op reduction.
// Differs from sin/cos(fl(2*pi*u)) by <= ~1 ulp of the angle (the reference
// rounds the angle first; this evaluates the exact one).
__device__ __forceinline__ void sincos_turn(uint32_t w, double& s, double& c) {
    const uint64_t v = uint64_t(w) + 1u;
    const uint32_t k = uint32_t((v + (1u << 21)) >> 22);            // 0 .. 1024
    const int m = int(int64_t(v) - (int64_t(k) << 22));             // -2^21 .. 2^21
    const double md = __dsub_rn(__hiloint2double(0x43300000, int(uint32_t(m) ^ 0x80000000u)),
                                kMC[MC_TURN_BIAS]);                 // exact
    const double r = __dmul_rn(md, kMC[MC_TWO_PI_2M32]);
    const double2 e = sincos_entry(int(k));
    const double r2 = __dmul_rn(r, r);
    const double ps = __fma_rn(r2, kMC[MC_T_S5], kMC[MC_T_S3]);
    const double sr = __fma_rn(__dmul_rn(r2, r), ps, r);
    const double pc = __fma_rn(r2, kMC[MC_T_C4], -0.5);
    const double cr = __fma_rn(r2, pc, 1.0);
    s = __fma_rn(e.x, cr, __dmul_rn(e.y, sr));
    c = __fma_rn(e.y, cr, -__dmul_rn(e.x, sr));
}

// The stepper's sincos for |x| < 2^29 (NaN/inf propagate to NaN).
__device__ __forceinline__ void sincos_small(double x, double& s, double& c) {
    sincos_tab(x, s, c);
}

// |x| >= 2^29, inf or NaN -- integer test on the high word (ALU, not FP64).
__device__ __forceinline__ bool big_arg(double x) {
    return (__double2hiint(x) & 0x7fffffff) >= 0x41C00000;
}

// Any argument: unwrapped phases beyond 2^29 take libdevice's exact reduction.
__device__ __forceinline__ void sincos_any(double x, double& s, double& c) {
    if (!big_arg(x)) {
        sincos_small(x, s, c);
    } else {
        sincos(x, &s, &c);
    }
}

// J values at once: ONE branch per call site; the fast path carries no
// per-element slow-path code (the stepper's phases are almost never huge).
template <int J>
__device__ __forceinline__ void sincos_vec(const double (&x)[J], double (&s)[J], double (&c)[J]) {
    bool big = false;
#pragma unroll
    for (int q = 0; q < J; ++q) {
        big |= big_arg(x[q]);
        sincos_small(x[q], s[q], c[q]);
    }
    if (big) {
        // rare: only the huge elements are redone with the exact reduction, so
        // a value's bits never depend on its J-vector neighbours (lane
        // layouts stay bit-identical)
#pragma unroll
        for (int q = 0; q < J; ++q)
            if (big_arg(x[q])) sincos(x[q], &s[q], &c[q]);
    }
}

// sincos_vec with the range test already done by the caller: `big` = some
// |x[q]| >= 2^29, inf or NaN (the stepper knows it from the magnitude scan it
// makes for its finiteness check).  Same values element for element.
template <int J>
__device__ __forceinline__ void sincos_vec_hint(const double (&x)[J], double (&s)[J], double (&c)[J],
                                                bool big) {
#pragma unroll
    for (int q = 0; q < J; ++q) sincos_small(x[q], s[q], c[q]);
    if (big) {
#pragma unroll
        for (int q = 0; q < J; ++q)
            if (big_arg(x[q])) sincos(x[q], &s[q], &c[q]);
    }
}

// Largest |x[q]| as the high word of its bits (sign cleared): one integer
// max per element serves both the finiteness test (>= 0x7ff00000) and the
// sincos range test (>= 0x41C00000, big_arg).
template <int J>
__device__ __forceinline__ uint32_t abs_hi_max(const double (&x)[J]) {
    uint32_t m = 0;
#pragma unroll
    for (int q = 0; q < J; ++q) m = max(m, uint32_t(__double2hiint(x[q])) & 0x7fffffffu);
    return m;
}

// -2 ln(x) for a positive normal double: the Box-Muller radius argument
// (rng.py:179, -2.0 * log(u)) with the -2 folded into the table and the
// series.  x = 2^k z, z near c_i; the table holds (-2 invc_i, -2 logc_i) and
// r' = fma(z, -2 invc, 2) = -2 r exactly, where r = z invc - 1 (|r| <= 2^-9).
// In Horner form every intermediate of the series in r' is the series in r
// scaled by a power of two (coefficients a_i (-1/2)^(i+1)), so rounding
// commutes with the scaling and the result equals fl(-2 * ln_table(x)) bit
// for bit -- one DMUL cheaper than scaling afterwards.
__device__ __forceinline__ double neg2_log_pos(double x) {
    const uint64_t ix = uint64_t(__double_as_longlong(x));
    const uint64_t tmp = ix - kLogOff;
    const int i = int((tmp >> (52 - kLogTableBits)) & ((1u << kLogTableBits) - 1));
    const int64_t k = int64_t(tmp) >> 52;
    const double z = __longlong_as_double((long long)(ix - (tmp & (0xFFFull << 52))));
    const double2 e = log_entry(i);  // (-2 invc, -2 logc)
    const double r = __fma_rn(z, e.x, 2.0);  // -2 (z invc - 1)
    const double kd = __dsub_rn(__longlong_as_double((long long)(0x4338000000000000ll + k)),
                                kRoundMagic);
    // -2 log1p(r'/(-2)) = r' + r'^2 (1/4 + r'/12 + r'^2/32 + r'^3/80 + r'^4/192),
    // |r'| <= 2^-8: the next term is < 2^-56.8 relative (tools/gen_log_table.py)
    double p = __fma_rn(r, kMC[MC_LB4], kMC[MC_LB3]);
    p = __fma_rn(r, p, 0.03125);
    p = __fma_rn(r, p, kMC[MC_LB1]);
    p = __fma_rn(r, p, 0.25);
    const double lp = __fma_rn(__dmul_rn(r, r), p, r);
    const double hi = __fma_rn(kd, kMC[MC_M2LN2_HI], e.y);
    const double lo = __fma_rn(kd, kMC[MC_M2LN2_LO], lp);
    return __dadd_rn(hi, lo);
}

// sqrt(x) for x >= 0 (x == 0 -> 0).  The reciprocal-root seed is taken of
// max(x, 2^-1022) -- an integer max on the high word, no FP64 compare and
// selects: x == 0 (the Box-Muller u == 1) then runs the Newton steps with
// g = 0 and returns exactly 0; any x > 0 (normal) is untouched.
__device__ __forceinline__ double sqrt_nonneg(double x) {
    double r;
    const double xs = __hiloint2double(max(__double2hiint(x), 0x00100000), __double2loint(x));
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(xs));
    double g = __dmul_rn(x, r);
    double h = __dmul_rn(0.5, r);
    const double d = __fma_rn(-g, h, 0.5);
    g = __fma_rn(g, d, g);
    h = __fma_rn(h, d, h);
    const double e = __fma_rn(-g, g, x);
    return __fma_rn(e, h, g);
}

}  // namespace sdeb
