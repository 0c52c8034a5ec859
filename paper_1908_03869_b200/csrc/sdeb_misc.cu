// Noise-stream and batch-sampling kernels behind the rng.py / model.py
// entry points of the C ABI (sdb_philox_words, sdb_normals, sdb_stream_raw,
// sdb_sampling_uniforms, sdb_sample_kuramoto).  They share every device
// function with the fused stepper, so what these return is exactly what the
// stepper consumes.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "sdeb_misc.h"
#include "sdeb_analysis.cuh"
#include "sdeb_rng.cuh"

namespace sdeb {

__global__ void philox_words_kernel(const uint32_t* __restrict__ in, int64_t count,
                                    uint32_t* __restrict__ out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint32_t* k = in + 6 * i;  // (k0, k1, c0, c1, c2, c3)
    const Words4 w = philox4x32_10(k[2], k[3], k[4], k[5], k[0], k[1]);
    uint32_t* o = out + 4 * i;
    o[0] = w.w0;
    o[1] = w.w1;
    o[2] = w.w2;
    o[3] = w.w3;
}

// rng.normals_for_orbits (rng.py:150-188): one thread per (row, block).
template <int STREAM>
__global__ void normals_kernel(uint64_t seed, const uint32_t* __restrict__ orbits, int64_t count,
                               uint32_t chunk, uint32_t step, int m, double* __restrict__ out) {
    const int nblocks = (m + 3) / 4;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= count * nblocks) return;
    const int64_t row = t / nblocks;
    const int b = int(t % nblocks);
    Words4 w;
    if constexpr (STREAM == 0) {
        w = philox4x32_10(uint32_t(seed >> 32), chunk, step, uint32_t(b), uint32_t(seed),
                          orbits[row]);
    } else {
        StreamState s = stream_init<STREAM>(seed, orbits[row], uint64_t(b));
        const uint64_t steps = (uint64_t(chunk) << 32) | step;
        for (uint64_t k = 0; k < steps; ++k) stream_block<STREAM>(s);
        w = stream_block<STREAM>(s);
    }
    double z[4];
    box_muller_pair(w.w0, w.w1, z[0], z[1]);
    box_muller_pair(w.w2, w.w3, z[2], z[3]);
    for (int k = 0; k < 4; ++k) {
        const int col = 4 * b + k;
        if (col < m) out[row * m + col] = z[k];
    }
}

template <int STREAM>
__global__ void stream_raw_kernel(uint64_t seed, uint64_t orbit, uint64_t block, int64_t count,
                                  uint64_t* __restrict__ out) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    StreamState s = stream_init<STREAM>(seed, orbit, block);
    for (int64_t k = 0; k < count; ++k) out[k] = stream_next<STREAM>(s);
}

// rng.sampling_uniforms (rng.py:200-222): counter (seed_hi, TAG, 0, block), u = w * 2^-32.
__global__ void sampling_kernel(uint64_t seed, const uint32_t* __restrict__ orbits, int64_t count,
                                int ncols, double* __restrict__ out) {
    const int nblocks = (ncols + 3) / 4;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= count * nblocks) return;
    const int64_t row = t / nblocks;
    const int b = int(t % nblocks);
    const Words4 w = philox4x32_10(uint32_t(seed >> 32), kSamplingTag, 0u, uint32_t(b),
                                   uint32_t(seed), orbits[row]);
    const uint32_t ws[4] = {w.w0, w.w1, w.w2, w.w3};
    for (int k = 0; k < 4; ++k) {
        const int col = 4 * b + k;
        if (col < ncols) out[row * ncols + col] = __dmul_rn(double(ws[k]), kTwoNeg32);
    }
}

// model.sample_kuramoto_batch (model.py:262-269):
//   theta0 = -pi + (2pi * u); omega = lo + (hi - lo) * u; s = lo + (hi - lo) * u.
__global__ void sample_kuramoto_kernel(int n, uint64_t seed, const uint32_t* __restrict__ orbits,
                                       int64_t count, double omega_lo, double omega_w,
                                       double noise_lo, double noise_w, double coupling,
                                       double* __restrict__ init, double* __restrict__ params) {
    const int ncols = 3 * n;
    const int nblocks = (ncols + 3) / 4;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= count * nblocks) return;
    const int64_t row = t / nblocks;
    const int b = int(t % nblocks);
    const Words4 w = philox4x32_10(uint32_t(seed >> 32), kSamplingTag, 0u, uint32_t(b),
                                   uint32_t(seed), orbits[row]);
    const uint32_t ws[4] = {w.w0, w.w1, w.w2, w.w3};
    double* prow = params + row * (2 * n + 1);
    if (b == 0) prow[0] = coupling;
    for (int k = 0; k < 4; ++k) {
        const int col = 4 * b + k;
        if (col >= ncols) break;
        const double u = __dmul_rn(double(ws[k]), kTwoNeg32);
        if (col < n) {
            init[row * n + col] = __dadd_rn(-CUDART_PI, __dmul_rn(kTwoPi, u));
        } else if (col < 2 * n) {
            prow[1 + (col - n)] = __dadd_rn(omega_lo, __dmul_rn(omega_w, u));
        } else {
            prow[1 + n + (col - 2 * n)] = __dadd_rn(noise_lo, __dmul_rn(noise_w, u));
        }
    }
}

// DFMA throughput probe: 8 independent chains per thread keep the FP64 pipe
// issue-bound (DFMA latency is hidden by ILP x resident warps).
__global__ void __launch_bounds__(256) fp64_peak_kernel(int iters, double seed, double* out) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 1e-7 + k;
    const double m = 0.9999999, c = 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = __fma_rn(a[k], m, c);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.678) out[0] = s;  // keep the chains live
}

cudaError_t launch_fp64_peak(int blocks, int iters, double* out, cudaStream_t st) {
    fp64_peak_kernel<<<blocks, 256, 0, st>>>(iters, 1.0, out);
    return cudaGetLastError();
}

__global__ void math_probe_kernel(int func, const double* __restrict__ x, int64_t count,
                                  double* __restrict__ out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const double v = x[i];
    double s, c, r = 0.0;
    switch (func) {
        case 0: sincos_any(v, s, c); r = s; break;
        case 1: sincos_any(v, s, c); r = c; break;
        case 2: r = __dmul_rn(-0.5, neg2_log_pos(v)); break;  // exact rescale
        case 3: r = sqrt_nonneg(v); break;
        case 4: r = sin(v); break;
        case 5: r = cos(v); break;
        case 6: r = log(v); break;
        // Box-Muller angle: x carries the 32-bit word w (exactly, as a double)
        case 7: sincos_turn(uint32_t(v), s, c); r = s; break;
        case 8: sincos_turn(uint32_t(v), s, c); r = c; break;
        default: r = CUDART_NAN;
    }
    out[i] = r;
}

static unsigned grid_for(int64_t items, int block) { return unsigned((items + block - 1) / block); }

cudaError_t launch_math_probe(int func, const double* x, int64_t count, double* out,
                              cudaStream_t st) {
    math_probe_kernel<<<grid_for(count, 256), 256, 0, st>>>(func, x, count, out);
    return cudaGetLastError();
}

cudaError_t launch_philox_words(const uint32_t* in, int64_t count, uint32_t* out, cudaStream_t st) {
    philox_words_kernel<<<grid_for(count, 256), 256, 0, st>>>(in, count, out);
    return cudaGetLastError();
}

cudaError_t launch_normals(int stream, uint64_t seed, const uint32_t* orbits, int64_t count,
                           uint32_t chunk, uint32_t step, int m, double* out, cudaStream_t st) {
    const int64_t items = count * int64_t((m + 3) / 4);
    const unsigned g = grid_for(items, 128);
    if (stream == 0) {
        normals_kernel<0><<<g, 128, 0, st>>>(seed, orbits, count, chunk, step, m, out);
    } else if (stream == 1) {
        normals_kernel<1><<<g, 128, 0, st>>>(seed, orbits, count, chunk, step, m, out);
    } else {
        normals_kernel<2><<<g, 128, 0, st>>>(seed, orbits, count, chunk, step, m, out);
    }
    return cudaGetLastError();
}

cudaError_t launch_stream_raw(int stream, uint64_t seed, uint64_t orbit, uint64_t block,
                              int64_t count, uint64_t* out, cudaStream_t st) {
    if (stream == 1) {
        stream_raw_kernel<1><<<1, 32, 0, st>>>(seed, orbit, block, count, out);
    } else {
        stream_raw_kernel<2><<<1, 32, 0, st>>>(seed, orbit, block, count, out);
    }
    return cudaGetLastError();
}

cudaError_t launch_sampling(uint64_t seed, const uint32_t* orbits, int64_t count, int ncols,
                            double* out, cudaStream_t st) {
    sampling_kernel<<<grid_for(count * ((ncols + 3) / 4), 128), 128, 0, st>>>(seed, orbits, count,
                                                                               ncols, out);
    return cudaGetLastError();
}

cudaError_t launch_sample_kuramoto(int n, uint64_t seed, const uint32_t* orbits, int64_t count,
                                   double omega_lo, double omega_w, double noise_lo,
                                   double noise_w, double coupling, double* init, double* params,
                                   cudaStream_t st) {
    sample_kuramoto_kernel<<<grid_for(count * ((3 * n + 3) / 4), 128), 128, 0, st>>>(
        n, seed, orbits, count, omega_lo, omega_w, noise_lo, noise_w, coupling, init, params);
    return cudaGetLastError();
}

// analysis.py:77-82 over a stored trajectory: one thread per population.
__global__ void order_parameter_kernel(const double* __restrict__ th, int n, int64_t rows,
                                       double* __restrict__ r, double* __restrict__ phi) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    double rr, pp;
    order_param_row(th + i * n, n, rr, pp);
    r[i] = rr;
    phi[i] = pp;
}

cudaError_t launch_order_parameter(const double* th, int n, int64_t rows, double* r, double* phi,
                                   cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    order_parameter_kernel<<<unsigned((rows + 127) / 128), 128, 0, st>>>(th, n, rows, r, phi);
    return cudaGetLastError();
}

}  // namespace sdeb
