// Device template of the runtime-compiled expression-template models (the
// paper's mechanism: the user's system is turned into GPU source at run time,
// PAPER.md:88-113; the reference's interpreter is dsl.py:441-571).
//
// sdeb_dsl.cu generates one translation unit per (model, kind):
//
//     #define SDB_N / SDB_NP / SDB_NN / SDB_KIND / SDB_LANES / SDB_UNROLL / SDB_GLOBAL_STATE
//     #include "sdeb_dsl_kernel.cuh"
//     __device__ double sdb_drift(int i, double t, const DVec& y, const double* p) {...}
//     __device__ double sdb_diffusion(int i, double t, const DVec& y,
//                                     const double* p, const DVec& n) {...}
//
// and NVRTC compiles it for sm_100a.  A group of SDB_LANES threads integrates
// one orbit (equations split across its lanes); N is a compile-time constant.
// The vector the templates index (y, and the step's normals n) sits in a
// per-orbit shared-memory column, since template indices are runtime values
// (y[j] inside sum(j, .)); the per-equation temporaries (f, g, RK4 stages)
// are indexed by the unrolled equation loop only and live in registers.  Arithmetic is
// IEEE double with the reference's operation order (explicit _rn intrinsics,
// --fmad=false), sum(j, .) uses numpy's pairwise order (Appendix B of
// SURVEY.md), and the noise is the fused Philox / sfc64 / xoshiro256++ +
// Box-Muller of the Kuramoto stepper.
#pragma once
#include "sdeb_dsl_args.h"
#include "sdeb_rng.cuh"

#ifndef SDB_N
#error "SDB_N must be defined by the generated program"
#endif

namespace sdeb {

constexpr int kDslNB = (SDB_NN + 3) / 4 > 0 ? (SDB_NN + 3) / 4 : 1;  // 4-normal blocks
constexpr int kDslNZ = SDB_NN > 0 ? 4 * kDslNB : 0;                   // normals per step
constexpr double kDslN = double(SDB_N);
constexpr int kDslUnroll = SDB_UNROLL;  // equation loops: unrolled for small systems, else 1

// A per-thread vector with a stride: shared memory columns (stride = the CTA
// width, conflict-free) or, for very large systems, a global scratch column
// (stride = rows, coalesced).  The generated code indexes it like an array.
struct DVec {
    double* base;
    int64_t stride;
    __device__ __forceinline__ double& operator[](int k) const { return base[int64_t(k) * stride]; }
};

// ---- expression helpers used by the generated code -------------------------

// numpy's pairwise add.reduce over j in [LO, LO + CNT) (numpy
// pairwise_sum_DOUBLE): < 8 terms sequential from 0.0; <= 128: eight strided
// accumulators, a fixed tree, then the tail; larger: split at a multiple of 8.
template <int LO, int CNT, class F>
__device__ __forceinline__ double pw_sum(F&& f) {
    if constexpr (CNT < 8) {
        double r = 0.0;
#pragma unroll
        for (int k = 0; k < CNT; ++k) r = __dadd_rn(r, f(LO + k));
        return r;
    } else if constexpr (CNT <= 128) {
        double r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = f(LO + k);
        constexpr int body = CNT - CNT % 8;
#pragma unroll 1
        for (int i = 8; i < body; i += 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], f(LO + i + k));
        }
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll
        for (int i = body; i < CNT; ++i) res = __dadd_rn(res, f(LO + i));
        return res;
    } else {
        constexpr int half = CNT / 2 - (CNT / 2) % 8;
        return __dadd_rn(pw_sum<LO, half>(f), pw_sum<LO + half, CNT - half>(f));
    }
}

template <class F>
__device__ __forceinline__ double dsl_sum(F&& f) {
    return pw_sum<0, SDB_N>(f);
}

// sum(j, sin(a_j)) and sum(j, cos(a_j)) in one pass (one sincos per term),
// each in numpy's pairwise order: the factored meanfield form of the
// generated code (sdeb_dsl.cu Gen::factored).
template <int LO, int CNT, bool EXACT, class F>
__device__ __forceinline__ void pw_sum_sincos(F&& f, bool& big, double& ss, double& sc,
                                              double* keep_s = nullptr, double* keep_c = nullptr) {
    auto sc_of = [&](int j, double& s, double& c) {
        const double x = f(j);
        if constexpr (EXACT) {
            if (big_arg(x)) {
                sincos(x, &s, &c);
            } else {
                sincos_small(x, s, c);
            }
        } else {
            big |= big_arg(x);
            sincos_small(x, s, c);
        }
        if (keep_s) {  // the equation-side values (sum(j, sin(y[j] - y[i])) form)
            keep_s[j] = s;
            keep_c[j] = c;
        }
    };
    if constexpr (CNT < 8) {
        ss = 0.0;
        sc = 0.0;
#pragma unroll
        for (int k = 0; k < CNT; ++k) {
            double s, c;
            sc_of(LO + k, s, c);
            ss = __dadd_rn(ss, s);
            sc = __dadd_rn(sc, c);
        }
    } else if constexpr (CNT <= 128) {
        double rs[8], rc[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) sc_of(LO + k, rs[k], rc[k]);
        constexpr int body = CNT - CNT % 8;
#pragma unroll 1
        for (int i = 8; i < body; i += 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                double s, c;
                sc_of(LO + i + k, s, c);
                rs[k] = __dadd_rn(rs[k], s);
                rc[k] = __dadd_rn(rc[k], c);
            }
        }
        ss = __dadd_rn(__dadd_rn(__dadd_rn(rs[0], rs[1]), __dadd_rn(rs[2], rs[3])),
                       __dadd_rn(__dadd_rn(rs[4], rs[5]), __dadd_rn(rs[6], rs[7])));
        sc = __dadd_rn(__dadd_rn(__dadd_rn(rc[0], rc[1]), __dadd_rn(rc[2], rc[3])),
                       __dadd_rn(__dadd_rn(rc[4], rc[5]), __dadd_rn(rc[6], rc[7])));
#pragma unroll
        for (int i = body; i < CNT; ++i) {
            double s, c;
            sc_of(LO + i, s, c);
            ss = __dadd_rn(ss, s);
            sc = __dadd_rn(sc, c);
        }
    } else {
        constexpr int half = CNT / 2 - (CNT / 2) % 8;
        double s1, c1, s2, c2;
        pw_sum_sincos<LO, half, EXACT>(f, big, s1, c1, keep_s, keep_c);
        pw_sum_sincos<LO + half, CNT - half, EXACT>(f, big, s2, c2, keep_s, keep_c);
        ss = __dadd_rn(s1, s2);
        sc = __dadd_rn(c1, c2);
    }
}

template <bool EXACT, class F>
__device__ __forceinline__ void dsl_sum_sincos(F&& f, bool& big, double& ss, double& sc) {
    pw_sum_sincos<0, SDB_N, EXACT>(f, big, ss, sc);
}

template <bool EXACT, class F>
__device__ __forceinline__ void dsl_sum_sincos_keep(F&& f, bool& big, double& ss, double& sc,
                                                    double* keep_s, double* keep_c) {
    pw_sum_sincos<0, SDB_N, EXACT>(f, big, ss, sc, keep_s, keep_c);
}

// |x| >= 2^29 (or inf/NaN): libdevice's exact reduction, out of line so the
// unrolled model code stays small.
__device__ __noinline__ double2 dsl_sincos_big(double x) {
    double2 r;
    sincos(x, &r.x, &r.y);
    return r;
}

// sin / cos in the generated code.  The fast instantiation is branch- and
// call-free (table sincos, valid for |x| < 2^29) and only flags a huge, inf
// or NaN argument; a step that flagged anything is recomputed with EXACT =
// true (libdevice's exact reduction for those arguments).  Keeping the call
// out of the hot code keeps the coefficients in registers across the sums.
template <bool EXACT>
__device__ __forceinline__ double dsl_sin(double x, bool& big) {
    if constexpr (EXACT) {
        if (big_arg(x)) return dsl_sincos_big(x).x;
    } else {
        big |= big_arg(x);
    }
    double s, c;
    sincos_small(x, s, c);
    return s;
}

template <bool EXACT>
__device__ __forceinline__ double dsl_cos(double x, bool& big) {
    if constexpr (EXACT) {
        if (big_arg(x)) return dsl_sincos_big(x).y;
    } else {
        big |= big_arg(x);
    }
    double s, c;
    sincos_small(x, s, c);
    return c;
}

__device__ __forceinline__ double dsl_sq(double x) { return __dmul_rn(x, x); }

// ---- the model (defined by the generated code after this header) ------------

// Each template comes as a prologue computing the values that do not depend
// on the equation (hoisted sums, H) once per evaluation, and the per-equation
// function reading them.
template <bool EXACT>
__device__ __forceinline__ void sdb_drift_pre(double t, const DVec& y, const double* __restrict__ p,
                                              bool& big, double (&H)[SDB_DRIFT_H]);
template <bool EXACT>
__device__ __forceinline__ double sdb_drift(int i, double t, const DVec& y,
                                           const double* __restrict__ p, bool& big,
                                           const double (&H)[SDB_DRIFT_H]);
template <bool EXACT>
__device__ __forceinline__ void sdb_diffusion_pre(double t, const DVec& y,
                                                  const double* __restrict__ p, const DVec& n,
                                                  bool& big, double (&H)[SDB_DIFF_H]);
template <bool EXACT>
__device__ __forceinline__ double sdb_diffusion(int i, double t, const DVec& y,
                                               const double* __restrict__ p, const DVec& n,
                                               bool& big, const double (&H)[SDB_DIFF_H]);

__device__ __forceinline__ bool dsl_finite(double x) {
    return (__double2hiint(x) & 0x7ff00000) != 0x7ff00000;
}

// ---- lane groups -------------------------------------------------------------
// kL = SDB_LANES consecutive threads of a warp integrate one orbit; lane l owns
// equations i = l, l + kL, l + 2 kL, ... (kEPL of them).  The vector the
// templates index (y, the normals) is the orbit's shared column; every step
// reads it in one phase and writes it in the next, separated by __syncwarp
// (groups never straddle warps).  Each equation is evaluated exactly as with
// one lane, so every kL gives bit-identical results.
constexpr int kL = SDB_LANES;
constexpr int kEPL = (SDB_N + kL - 1) / kL;   // equations per lane
constexpr int kBPL = (kDslNB + kL - 1) / kL;  // 4-normal blocks per lane

// Group barrier.  One lane per orbit shares nothing, so the fence (which
// also makes the compiler re-load the parameters after it) is skipped.
__device__ __forceinline__ void dsl_sync() {
    if constexpr (kL > 1) __syncwarp();
}

// "Any lane of the warp flagged a huge argument" (warp-uniform at kL > 1;
// at kL = 1 each orbit redoes only its own step).
__device__ __forceinline__ bool dsl_any(bool flag) {
    if constexpr (kL > 1) {
        return __any_sync(0xffffffffu, flag);
    } else {
        return flag;
    }
}

template <bool EXACT>
__device__ __forceinline__ void dsl_drift_vec(int lane, double t, const DVec& y,
                                              const double* __restrict__ p, double (&f)[kEPL],
                                              bool& big) {
    double H[SDB_DRIFT_H];
    sdb_drift_pre<EXACT>(t, y, p, big, H);
#pragma unroll kDslUnroll
    for (int q = 0; q < kEPL; ++q) {
        const int i = lane + q * kL;
        f[q] = (i < SDB_N) ? sdb_drift<EXACT>(i, t, y, p, big, H) : 0.0;
    }
}

// one em step (solvers.py:70-71): ynew = (y + f*dt) + sqrt(dt) * g
template <bool EXACT>
__device__ __forceinline__ void dsl_em_pass(int lane, double t, double dt, double sqrt_dt,
                                            const DVec& y, const double* __restrict__ p,
                                            const DVec& nz, double (&ynew)[kEPL], bool& big) {
    double f[kEPL];
    dsl_drift_vec<EXACT>(lane, t, y, p, f, big);
    double G[SDB_DIFF_H];
    sdb_diffusion_pre<EXACT>(t, y, p, nz, big, G);
#pragma unroll kDslUnroll
    for (int q = 0; q < kEPL; ++q) {
        const int i = lane + q * kL;
        if (i < SDB_N) {
            const double g = sdb_diffusion<EXACT>(i, t, y, p, nz, big, G);
            ynew[q] = __dadd_rn(__dadd_rn(y[i], __dmul_rn(f[q], dt)), __dmul_rn(sqrt_dt, g));
        } else {
            ynew[q] = 0.0;
        }
    }
}

__device__ __forceinline__ void dsl_em(int lane, double t, double dt, double sqrt_dt, const DVec& y,
                                       const double* __restrict__ p, const DVec& nz,
                                       double (&ynew)[kEPL]) {
    bool big = false;
    dsl_em_pass<false>(lane, t, dt, sqrt_dt, y, p, nz, ynew, big);
    if (dsl_any(big)) dsl_em_pass<true>(lane, t, dt, sqrt_dt, y, p, nz, ynew, big);
}

// one euler step (solvers.py:74-77): ynew = y + f*dt
template <bool EXACT>
__device__ __forceinline__ void dsl_euler_pass(int lane, double t, double dt, const DVec& y,
                                               const double* __restrict__ p, double (&ynew)[kEPL],
                                               bool& big) {
    double f[kEPL];
    dsl_drift_vec<EXACT>(lane, t, y, p, f, big);
#pragma unroll kDslUnroll
    for (int q = 0; q < kEPL; ++q) {
        const int i = lane + q * kL;
        ynew[q] = (i < SDB_N) ? __dadd_rn(y[i], __dmul_rn(f[q], dt)) : 0.0;
    }
}

__device__ __forceinline__ void dsl_euler(int lane, double t, double dt, const DVec& y,
                                          const double* __restrict__ p, double (&ynew)[kEPL]) {
    bool big = false;
    dsl_euler_pass<false>(lane, t, dt, y, p, ynew, big);
    if (dsl_any(big)) dsl_euler_pass<true>(lane, t, dt, y, p, ynew, big);
}

// one classical RK4 step in the reference's order (solvers.py:80-88):
// y + (dt/6) * (((k1 + 2 k2) + 2 k3) + k4).  The stage states are written
// into the shared column the drift reads; the step's start state is yk (this
// lane's equations, registers) and ynew is returned uncommitted.
template <bool EXACT>
__device__ __forceinline__ void dsl_rk4_pass(int lane, double t, double dt, const DVec& y,
                                             const double* __restrict__ p,
                                             const double (&yk)[kEPL], double (&ynew)[kEPL],
                                             bool& big) {
    const double half = __dmul_rn(0.5, dt);
    const double th = __dadd_rn(t, half);
    double k[kEPL], acc[kEPL];
    dsl_drift_vec<EXACT>(lane, t, y, p, k, big);
    dsl_sync();
#pragma unroll kDslUnroll
    for (int q = 0; q < kEPL; ++q) {
        const int i = lane + q * kL;
        acc[q] = k[q];
        if (i < SDB_N) y[i] = __dadd_rn(yk[q], __dmul_rn(half, k[q]));
    }
    dsl_sync();
    dsl_drift_vec<EXACT>(lane, th, y, p, k, big);
    dsl_sync();
#pragma unroll kDslUnroll
    for (int q = 0; q < kEPL; ++q) {
        const int i = lane + q * kL;
        acc[q] = __dadd_rn(acc[q], __dmul_rn(2.0, k[q]));
        if (i < SDB_N) y[i] = __dadd_rn(yk[q], __dmul_rn(half, k[q]));
    }
    dsl_sync();
    dsl_drift_vec<EXACT>(lane, th, y, p, k, big);
    dsl_sync();
#pragma unroll kDslUnroll
    for (int q = 0; q < kEPL; ++q) {
        const int i = lane + q * kL;
        acc[q] = __dadd_rn(acc[q], __dmul_rn(2.0, k[q]));
        if (i < SDB_N) y[i] = __dadd_rn(yk[q], __dmul_rn(dt, k[q]));
    }
    dsl_sync();
    dsl_drift_vec<EXACT>(lane, __dadd_rn(t, dt), y, p, k, big);
    const double dt6 = __ddiv_rn(dt, 6.0);
#pragma unroll kDslUnroll
    for (int q = 0; q < kEPL; ++q) {
        acc[q] = __dadd_rn(acc[q], k[q]);
        ynew[q] = __dadd_rn(yk[q], __dmul_rn(dt6, acc[q]));
    }
}

__device__ __forceinline__ void dsl_rk4(int lane, double t, double dt, const DVec& y,
                                        const double* __restrict__ p, double (&ynew)[kEPL]) {
    double yk[kEPL];
#pragma unroll kDslUnroll
    for (int q = 0; q < kEPL; ++q) {
        const int i = lane + q * kL;
        yk[q] = (i < SDB_N) ? y[i] : 0.0;
    }
    bool big = false;
    dsl_rk4_pass<false>(lane, t, dt, y, p, yk, ynew, big);
    if (dsl_any(big)) {
        dsl_sync();  // every lane is past its last stage read
#pragma unroll kDslUnroll
        for (int q = 0; q < kEPL; ++q) {
            const int i = lane + q * kL;
            if (i < SDB_N) y[i] = yk[q];
        }
        dsl_sync();
        dsl_rk4_pass<true>(lane, t, dt, y, p, yk, ynew, big);
    }
}

// Write the step's result into the shared column after every lane finished
// reading it.  check: isfinite(y).all(-1) over the orbit (OR across the
// group); a failing orbit records its first step and becomes NaN
// (engine.py:244-261).
__device__ __forceinline__ void dsl_commit(int lane, const DVec& y, double (&ynew)[kEPL], bool check,
                                           int64_t& fail, uint64_t step) {
    dsl_sync();
    if (check) {
        bool bad = false;
#pragma unroll
        for (int q = 0; q < kEPL; ++q) {
            const int i = lane + q * kL;
            bad |= (i < SDB_N) && !dsl_finite(ynew[q]);
        }
#pragma unroll
        for (int o = 1; o < kL; o <<= 1) bad |= __shfl_xor_sync(0xffffffffu, int(bad), o) != 0;
        if (bad) {
            if (fail < 0) fail = int64_t(step);
#pragma unroll
            for (int q = 0; q < kEPL; ++q) ynew[q] = __longlong_as_double(0x7ff8000000000000ll);
        }
    }
#pragma unroll kDslUnroll
    for (int q = 0; q < kEPL; ++q) {
        const int i = lane + q * kL;
        if (i < SDB_N) y[i] = ynew[q];
    }
    dsl_sync();
}

}  // namespace sdeb

// ---- the kernel ------------------------------------------------------------------
// CTA = 128 threads = 128/kL orbit slots.  The per-orbit columns (y, the
// step's normals) live in dynamic shared memory, [words][slots] per CTA, or
// (SDB_GLOBAL_STATE) in the global scratch [words][grid * slots].  Tail
// threads past the last orbit mirror it into their own column and write
// nothing, so every warp runs the same sequence of __syncwarp.

#ifndef SDB_MINB
#define SDB_MINB 1
#endif
extern "C" __global__ void __launch_bounds__(128, SDB_MINB) sdb_dsl_main(const sdeb::DslArgs a) {
    using namespace sdeb;
    extern __shared__ double dsl_smem[];
    constexpr int kSlots = 128 / kL;
    stage_tables();  // sincos / log tables into shared memory (SDEB_SMEM_TABLES)
    const int lane = int(threadIdx.x) % kL;
    const int slot = int(threadIdx.x) / kL;
    const int64_t orbit = int64_t(blockIdx.x) * kSlots + slot;
    const bool active = orbit < a.rows;
    const int64_t row = active ? orbit : a.rows - 1;
#if SDB_GLOBAL_STATE
    const int64_t cols = int64_t(gridDim.x) * kSlots;
    const DVec y{a.scratch + int64_t(blockIdx.x) * kSlots + slot, cols};
    const DVec nz{a.scratch + int64_t(SDB_N) * cols + int64_t(blockIdx.x) * kSlots + slot, cols};
#else
    const DVec y{dsl_smem + slot, int64_t(kSlots)};
    const DVec nz{dsl_smem + int64_t(SDB_N) * kSlots + slot, int64_t(kSlots)};
#endif
    const double* __restrict__ p = a.params + row * SDB_NP;
#pragma unroll kDslUnroll
    for (int q = 0; q < kEPL; ++q) {
        const int i = lane + q * kL;
        if (i < SDB_N) y[i] = a.state_in[row * SDB_N + i];
    }
#if SDB_NN > 0
    if (a.noise != nullptr) {
#pragma unroll 1
        for (int k = lane; k < SDB_NN; k += kL) nz[k] = a.noise[row * SDB_NN + k];
    }
#endif
    dsl_sync();

#if SDB_KIND == 8 || SDB_KIND == 9  // drift_eval / diffusion_eval
    bool big = false;  // evaluation is not a hot loop: always the exact form
#if SDB_KIND == 8
    double H[SDB_DRIFT_H];
    sdb_drift_pre<true>(a.t, y, p, big, H);
#else
    double H[SDB_DIFF_H];
    sdb_diffusion_pre<true>(a.t, y, p, nz, big, H);
#endif
#pragma unroll kDslUnroll
    for (int q = 0; q < kEPL; ++q) {
        const int i = lane + q * kL;
#if SDB_KIND == 8
        if (i < SDB_N && active) a.values[row * SDB_N + i] = sdb_drift<true>(i, a.t, y, p, big, H);
#else
        if (i < SDB_N && active)
            a.values[row * SDB_N + i] = sdb_diffusion<true>(i, a.t, y, p, nz, big, H);
#endif
    }
#elif SDB_KIND >= 5  // one caller-driven step
    double ynew[kEPL];
#if SDB_KIND == 5
    dsl_em(lane, a.t, a.dt, a.sqrt_dt, y, p, nz, ynew);
#elif SDB_KIND == 6
    dsl_euler(lane, a.t, a.dt, y, p, ynew);
#else
    dsl_rk4(lane, a.t, a.dt, y, p, ynew);
#endif
#pragma unroll kDslUnroll
    for (int q = 0; q < kEPL; ++q) {
        const int i = lane + q * kL;
        if (i < SDB_N && active) a.state_out[row * SDB_N + i] = ynew[q];
    }
#else  // run_batch's chunk x step loop (engine.py:231-262)
    constexpr bool kStateful = SDB_KIND == 1 || SDB_KIND == 2;
    const uint32_t orbit_g = uint32_t(a.orbit_offset + row);
    const bool fresh = a.fresh != 0;
    int64_t fail = (fresh || a.fail_step == nullptr) ? -1 : a.fail_step[row];
    StreamState rs[kBPL];  // block b = lane + r*kL
    if constexpr (kStateful) {
#pragma unroll
        for (int r = 0; r < kBPL; ++r) {
            const int b = lane + r * kL;
            if (b >= kDslNB) {
                rs[r] = StreamState{0, 0, 0, 0};
            } else if (fresh) {
                rs[r] = stream_init<SDB_KIND>(a.seed, uint64_t(orbit_g), uint64_t(b));
            } else {
                const uint64_t* q = a.rng_state + (row * kDslNB + b) * 4;
                rs[r] = StreamState{q[0], q[1], q[2], q[3]};
            }
        }
    }
    const uint32_t seed_lo = uint32_t(a.seed), seed_hi = uint32_t(a.seed >> 32);
    (void)seed_lo;
    (void)seed_hi;
    const uint64_t ks = uint64_t(a.ksteps);
    uint64_t step = uint64_t(a.chunk_begin) * ks;
    double ynew[kEPL];
#pragma unroll 1
    for (int64_t c = a.chunk_begin; c < a.chunk_end; ++c) {
#pragma unroll 1
        for (uint64_t l = 0; l < ks; ++l, ++step) {
            const double t = __dmul_rn(double(step), a.dt);  // t = step_index * dt
#if SDB_KIND <= 2
            // the step's normals: this lane's 4-normal blocks into the column
#pragma unroll
            for (int r = 0; r < kBPL; ++r) {
                const int b = lane + r * kL;
                if (b < kDslNB) {
                    Words4 w;
                    if constexpr (SDB_KIND == 0) {
                        w = philox4x32_10(seed_hi, uint32_t(step >> 32), uint32_t(step),
                                          uint32_t(b), seed_lo, orbit_g);
                    } else {
                        w = stream_block<SDB_KIND>(rs[r]);
                    }
                    double z0, z1, z2, z3;
                    box_muller_pair(w.w0, w.w1, z0, z1);
                    box_muller_pair(w.w2, w.w3, z2, z3);
                    nz[4 * b] = z0;
                    nz[4 * b + 1] = z1;
                    nz[4 * b + 2] = z2;
                    nz[4 * b + 3] = z3;
                }
            }
            dsl_sync();
            dsl_em(lane, t, a.dt, a.sqrt_dt, y, p, nz, ynew);
#elif SDB_KIND == 3
            dsl_euler(lane, t, a.dt, y, p, ynew);
#else
            dsl_rk4(lane, t, a.dt, y, p, ynew);
#endif
            dsl_commit(lane, y, ynew, true, fail, step);
        }
        if (active) {
            double* out = a.values + (row * a.vstride + (c - a.chunk_begin)) * SDB_N;
#pragma unroll kDslUnroll
            for (int q = 0; q < kEPL; ++q) {
                const int i = lane + q * kL;
                if (i < SDB_N) out[i] = y[i];
            }
        }
    }
    if (active) {
#pragma unroll kDslUnroll
        for (int q = 0; q < kEPL; ++q) {
            const int i = lane + q * kL;
            if (i < SDB_N && a.state_out != nullptr) a.state_out[row * SDB_N + i] = y[i];
        }
        if (a.fail_step != nullptr && lane == 0) a.fail_step[row] = fail;
        if constexpr (kStateful) {
#pragma unroll
            for (int r = 0; r < kBPL; ++r) {
                const int b = lane + r * kL;
                if (b < kDslNB) {
                    uint64_t* q = a.rng_state + (row * kDslNB + b) * 4;
                    q[0] = rs[r].s0;
                    q[1] = rs[r].s1;
                    q[2] = rs[r].s2;
                    q[3] = rs[r].s3;
                }
            }
        }
    }
#endif
}
