// Launch wrappers for the rng / sampling kernels (sdeb_misc.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace sdeb {

cudaError_t launch_philox_words(const uint32_t* in, int64_t count, uint32_t* out, cudaStream_t st);
cudaError_t launch_normals(int stream, uint64_t seed, const uint32_t* orbits, int64_t count,
                           uint32_t chunk, uint32_t step, int m, double* out, cudaStream_t st);
cudaError_t launch_stream_raw(int stream, uint64_t seed, uint64_t orbit, uint64_t block,
                              int64_t count, uint64_t* out, cudaStream_t st);
cudaError_t launch_sampling(uint64_t seed, const uint32_t* orbits, int64_t count, int ncols,
                            double* out, cudaStream_t st);
cudaError_t launch_sample_kuramoto(int n, uint64_t seed, const uint32_t* orbits, int64_t count,
                                   double omega_lo, double omega_w, double noise_lo,
                                   double noise_w, double coupling, double* init, double* params,
                                   cudaStream_t st);

// Order parameter (r, Phi) of `rows` populations of n phases (analysis.py:77-82).
cudaError_t launch_order_parameter(const double* th, int n, int64_t rows, double* r, double* phi,
                                   cudaStream_t st);

// FP64 DFMA-throughput probe: blocks x 256 threads x iters x 128 DFMA.
cudaError_t launch_fp64_peak(int blocks, int iters, double* out, cudaStream_t st);
cudaError_t launch_math_probe(int func, const double* x, int64_t count, double* out,
                              cudaStream_t st);

}  // namespace sdeb
