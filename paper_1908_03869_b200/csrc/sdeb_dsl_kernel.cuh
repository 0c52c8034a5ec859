// Device template of the runtime-compiled expression-template models (the
// paper's mechanism: the user's system is turned into GPU source at run time,
// PAPER.md:88-113; the reference's interpreter is dsl.py:441-571).
//
// sdeb_dsl.cu generates one translation unit per (model, kind):
//
//     #define SDB_N / SDB_NP / SDB_NN / SDB_KIND / SDB_UNROLL / SDB_GLOBAL_STATE
//     #include "sdeb_dsl_kernel.cuh"
//     __device__ double sdb_drift(int i, double t, const DVec& y, const double* p) {...}
//     __device__ double sdb_diffusion(int i, double t, const DVec& y,
//                                     const double* p, const DVec& n) {...}
//
// and NVRTC compiles it for sm_100a.  One thread integrates one orbit; N is a
// compile-time constant.  The vector the templates index (y, and the step's
// normals n) sits in a per-thread shared-memory column, since template
// indices are runtime values (y[j] inside sum(j, .)); the per-equation
// temporaries (f, g, RK4 stages) are indexed by the unrolled equation loop
// only and live in registers for SDB_UNROLL = N.  Arithmetic is
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
constexpr int kDslUnroll = SDB_UNROLL;  // equation loops: N for small systems (registers), else 1

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

// |x| >= 2^29 (or inf/NaN): libdevice's exact reduction, out of line so the
// unrolled model code stays small.
__device__ __noinline__ double2 dsl_sincos_big(double x) {
    double2 r;
    sincos(x, &r.x, &r.y);
    return r;
}

__device__ __forceinline__ double dsl_sin(double x) {
    if (big_arg(x)) return dsl_sincos_big(x).x;
    double s, c;
    sincos_small(x, s, c);
    return s;
}

__device__ __forceinline__ double dsl_cos(double x) {
    if (big_arg(x)) return dsl_sincos_big(x).y;
    double s, c;
    sincos_small(x, s, c);
    return c;
}

__device__ __forceinline__ double dsl_sq(double x) { return __dmul_rn(x, x); }

// ---- the model (defined by the generated code after this header) ------------

__device__ __forceinline__ double sdb_drift(int i, double t, const DVec& y,
                                           const double* __restrict__ p);
__device__ __forceinline__ double sdb_diffusion(int i, double t, const DVec& y,
                                               const double* __restrict__ p, const DVec& n);

__device__ __forceinline__ bool dsl_finite(double x) {
    return (__double2hiint(x) & 0x7ff00000) != 0x7ff00000;
}

__device__ __forceinline__ void dsl_drift_vec(double t, const DVec& y, const double* __restrict__ p,
                                              double (&f)[SDB_N]) {
#pragma unroll kDslUnroll
    for (int i = 0; i < SDB_N; ++i) f[i] = sdb_drift(i, t, y, p);
}

// y <- (y + f*dt) + sqrt(dt) * g   (solvers.py:70-71)
__device__ __forceinline__ void dsl_em(double t, double dt, double sqrt_dt, const DVec& y,
                                       const double* __restrict__ p, const DVec& nz) {
    double f[SDB_N], g[SDB_N];
    dsl_drift_vec(t, y, p, f);
#pragma unroll kDslUnroll
    for (int i = 0; i < SDB_N; ++i) g[i] = sdb_diffusion(i, t, y, p, nz);
#pragma unroll kDslUnroll
    for (int i = 0; i < SDB_N; ++i)
        y[i] = __dadd_rn(__dadd_rn(y[i], __dmul_rn(f[i], dt)), __dmul_rn(sqrt_dt, g[i]));
}

// y <- y + f*dt   (solvers.py:74-77)
__device__ __forceinline__ void dsl_euler(double t, double dt, const DVec& y,
                                          const double* __restrict__ p) {
    double f[SDB_N];
    dsl_drift_vec(t, y, p, f);
#pragma unroll kDslUnroll
    for (int i = 0; i < SDB_N; ++i) y[i] = __dadd_rn(y[i], __dmul_rn(f[i], dt));
}

// classical RK4 in the reference's order (solvers.py:80-88):
// y + (dt/6) * (((k1 + 2 k2) + 2 k3) + k4).  `y` is the vector the drift
// reads (stage states are written into it); the state itself is kept in yk.
__device__ __forceinline__ void dsl_rk4(double t, double dt, const DVec& y,
                                        const double* __restrict__ p) {
    const double half = __dmul_rn(0.5, dt);
    const double th = __dadd_rn(t, half);
    double k[SDB_N], acc[SDB_N], yk[SDB_N];
#pragma unroll kDslUnroll
    for (int i = 0; i < SDB_N; ++i) yk[i] = y[i];
    dsl_drift_vec(t, y, p, k);
#pragma unroll kDslUnroll
    for (int i = 0; i < SDB_N; ++i) {
        acc[i] = k[i];
        y[i] = __dadd_rn(yk[i], __dmul_rn(half, k[i]));
    }
    dsl_drift_vec(th, y, p, k);
#pragma unroll kDslUnroll
    for (int i = 0; i < SDB_N; ++i) {
        acc[i] = __dadd_rn(acc[i], __dmul_rn(2.0, k[i]));
        y[i] = __dadd_rn(yk[i], __dmul_rn(half, k[i]));
    }
    dsl_drift_vec(th, y, p, k);
#pragma unroll kDslUnroll
    for (int i = 0; i < SDB_N; ++i) {
        acc[i] = __dadd_rn(acc[i], __dmul_rn(2.0, k[i]));
        y[i] = __dadd_rn(yk[i], __dmul_rn(dt, k[i]));
    }
    dsl_drift_vec(__dadd_rn(t, dt), y, p, k);
    const double dt6 = __ddiv_rn(dt, 6.0);
#pragma unroll kDslUnroll
    for (int i = 0; i < SDB_N; ++i) {
        acc[i] = __dadd_rn(acc[i], k[i]);
        y[i] = __dadd_rn(yk[i], __dmul_rn(dt6, acc[i]));
    }
}

}  // namespace sdeb

// ---- the kernel ------------------------------------------------------------------
// Per thread: the state vector y and the step's normals live in a strided
// column (DVec) -- dynamic shared memory of blockDim.x * (N + NZ) doubles, or
// (SDB_GLOBAL_STATE) the global scratch [N + NZ][rows].

extern "C" __global__ void __launch_bounds__(128) sdb_dsl_main(const sdeb::DslArgs a) {
    using namespace sdeb;
    extern __shared__ double dsl_smem[];
    const int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (row >= a.rows) return;
#if SDB_GLOBAL_STATE
    const DVec y{a.scratch + row, a.rows};
    const DVec nz{a.scratch + int64_t(SDB_N) * a.rows + row, a.rows};
#else
    const DVec y{dsl_smem + threadIdx.x, int64_t(blockDim.x)};
    const DVec nz{dsl_smem + int64_t(SDB_N) * blockDim.x + threadIdx.x, int64_t(blockDim.x)};
#endif
    const double* __restrict__ p = a.params + row * SDB_NP;
#pragma unroll kDslUnroll
    for (int i = 0; i < SDB_N; ++i) y[i] = a.state_in[row * SDB_N + i];
#if SDB_NN > 0
    if (a.noise != nullptr) {
#pragma unroll 1
        for (int k = 0; k < SDB_NN; ++k) nz[k] = a.noise[row * SDB_NN + k];
    }
#endif

#if SDB_KIND == 8 || SDB_KIND == 9  // drift_eval / diffusion_eval
#pragma unroll kDslUnroll
    for (int i = 0; i < SDB_N; ++i)
        a.values[row * SDB_N + i] = SDB_KIND == 8 ? sdb_drift(i, a.t, y, p)
                                                  : sdb_diffusion(i, a.t, y, p, nz);
#elif SDB_KIND >= 5  // one caller-driven step
#if SDB_KIND == 5
    dsl_em(a.t, a.dt, a.sqrt_dt, y, p, nz);
#elif SDB_KIND == 6
    dsl_euler(a.t, a.dt, y, p);
#else
    dsl_rk4(a.t, a.dt, y, p);
#endif
#pragma unroll kDslUnroll
    for (int i = 0; i < SDB_N; ++i) a.state_out[row * SDB_N + i] = y[i];
#else  // run_batch's chunk x step loop (engine.py:231-262)
    constexpr bool kStateful = SDB_KIND == 1 || SDB_KIND == 2;
    const uint32_t orbit_g = uint32_t(a.orbit_offset + row);
    const bool fresh = a.fresh != 0;
    int64_t fail = (fresh || a.fail_step == nullptr) ? -1 : a.fail_step[row];
    StreamState rs[kDslNB];
    if constexpr (kStateful) {
#pragma unroll
        for (int b = 0; b < kDslNB; ++b) {
            if (fresh) {
                rs[b] = stream_init<SDB_KIND>(a.seed, uint64_t(orbit_g), uint64_t(b));
            } else {
                const uint64_t* q = a.rng_state + (row * kDslNB + b) * 4;
                rs[b] = StreamState{q[0], q[1], q[2], q[3]};
            }
        }
    }
    const uint32_t seed_lo = uint32_t(a.seed), seed_hi = uint32_t(a.seed >> 32);
    (void)seed_lo;
    (void)seed_hi;
    const uint64_t ks = uint64_t(a.ksteps);
    uint64_t step = uint64_t(a.chunk_begin) * ks;
#pragma unroll 1
    for (int64_t c = a.chunk_begin; c < a.chunk_end; ++c) {
#pragma unroll 1
        for (uint64_t l = 0; l < ks; ++l, ++step) {
            const double t = __dmul_rn(double(step), a.dt);  // t = step_index * dt
#if SDB_KIND <= 2
#pragma unroll
            for (int b = 0; b < kDslNB; ++b) {
                Words4 w;
                if constexpr (SDB_KIND == 0) {
                    w = philox4x32_10(seed_hi, uint32_t(step >> 32), uint32_t(step), uint32_t(b),
                                      seed_lo, orbit_g);
                } else {
                    w = stream_block<SDB_KIND>(rs[b]);
                }
                double z0, z1, z2, z3;
                box_muller_pair(w.w0, w.w1, z0, z1);
                box_muller_pair(w.w2, w.w3, z2, z3);
                nz[4 * b] = z0;
                nz[4 * b + 1] = z1;
                nz[4 * b + 2] = z2;
                nz[4 * b + 3] = z3;
            }
            dsl_em(t, a.dt, a.sqrt_dt, y, p, nz);
#elif SDB_KIND == 3
            dsl_euler(t, a.dt, y, p);
#else
            dsl_rk4(t, a.dt, y, p);
#endif
            // isfinite(y).all(-1); first failure recorded, row -> NaN (engine.py:244-261)
            bool bad = false;
#pragma unroll kDslUnroll
            for (int i = 0; i < SDB_N; ++i) bad |= !dsl_finite(y[i]);
            if (bad) {
                if (fail < 0) fail = int64_t(step);
#pragma unroll kDslUnroll
                for (int i = 0; i < SDB_N; ++i) y[i] = __longlong_as_double(0x7ff8000000000000ll);
            }
        }
        double* out = a.values + (row * a.vstride + (c - a.chunk_begin)) * SDB_N;
#pragma unroll kDslUnroll
        for (int i = 0; i < SDB_N; ++i) out[i] = y[i];
    }
    if (a.state_out != nullptr) {
#pragma unroll kDslUnroll
        for (int i = 0; i < SDB_N; ++i) a.state_out[row * SDB_N + i] = y[i];
    }
    if (a.fail_step != nullptr) a.fail_step[row] = fail;
    if constexpr (kStateful) {
#pragma unroll
        for (int b = 0; b < kDslNB; ++b) {
            uint64_t* q = a.rng_state + (row * kDslNB + b) * 4;
            q[0] = rs[b].s0;
            q[1] = rs[b].s1;
            q[2] = rs[b].s2;
            q[3] = rs[b].s3;
        }
    }
#endif
}
