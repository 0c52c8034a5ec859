// Kuramoto order parameter on the device (analysis.py:72-82):
//   r e^{i Phi} = (1/N) sum_j e^{i theta_j},  r = min(|z|, 1),
//   Phi = wrap_phase(atan2(Im z, Re z)) in [-pi, pi),  Phi = 0 where r = 0.
// The sums over oscillators use the stepper's canonical tree (P = next_pow2(N)
// leaves, adjacent pairs first, padding leaves +0.0), so the fused in-kernel
// value (sdeb_kuramoto.cuh, out_mode 1) and the post-hoc kernel over a stored
// trajectory are bit-identical.  numpy's complex mean sums in a different
// order: the difference is a few ulp of r (tests: <= 1e-13).
#pragma once
#include "sdeb_math.cuh"

namespace sdeb {

constexpr double kPi = 3.141592653589793;       // math.pi
constexpr double kTwoPiD = 6.283185307179586;   // 2.0 * math.pi

// np.mod(a, b) for doubles (npy_divmod): sign of the divisor, +0.0 for 0.
__device__ __forceinline__ double np_mod(double a, double b) {
    double m = fmod(a, b);
    if (m != 0.0) {
        if ((b < 0.0) != (m < 0.0)) m = __dadd_rn(m, b);
    } else {
        m = copysign(0.0, b);
    }
    return m;
}

// analysis.py:72-74
__device__ __forceinline__ double wrap_phase_d(double x) {
    return __dsub_rn(np_mod(__dadd_rn(x, kPi), kTwoPiD), kPi);
}

// (sum cos, sum sin) over N oscillators -> (r, Phi)
__device__ __forceinline__ void order_param_from_sums(double sum_c, double sum_s, int n, double& r,
                                                      double& phi) {
    const double re = __ddiv_rn(sum_c, double(n)), im = __ddiv_rn(sum_s, double(n));
    const double mag = hypot(re, im);
    r = (mag < 1.0 || mag != mag) ? mag : 1.0;  // np.minimum keeps NaN
    phi = wrap_phase_d(atan2(im, re));
    if (r == 0.0) phi = 0.0;
}

// One thread, one population of N phases: canonical-tree sums via a binary
// counter (merge partial sums left + right whenever a subtree completes).
__device__ __forceinline__ void order_param_row(const double* __restrict__ th, int n, double& r,
                                                double& phi) {
    int P = 1, levels = 0;
    while (P < n) {
        P <<= 1;
        ++levels;
    }
    double sc[32], ss[32];
    for (int j = 0; j < P; ++j) {
        double c = 0.0, s = 0.0;
        if (j < n) sincos_any(th[j], s, c);
        int lv = 0;
        for (int k = j; k & 1; k >>= 1, ++lv) {
            c = __dadd_rn(sc[lv], c);
            s = __dadd_rn(ss[lv], s);
        }
        sc[lv] = c;
        ss[lv] = s;
    }
    order_param_from_sums(sc[levels], ss[levels], n, r, phi);
}

}  // namespace sdeb
