// Per-J launch dispatch; included by sdeb_kuramoto_j{1,2,4,8,16}.cu so the
// instantiations compile in parallel.
#pragma once
#include "sdeb_kuramoto.cuh"

namespace sdeb {

template <int J, int S, int R, int C>
static cudaError_t launch_one(const RunArgs& a, cudaStream_t st) {
    const int64_t threads = a.orbits * int64_t(a.lanes);
    const unsigned grid = unsigned((threads + kBlock - 1) / kBlock);
    const size_t smem = pairwise_smem_bytes(J, C);
    kuramoto_run_kernel<J, S, R, C><<<grid, kBlock, smem, st>>>(a);
    return cudaGetLastError();
}

template <int J, int C>
static cudaError_t launch_coupling(const RunArgs& a, int solver, int stream, cudaStream_t st) {
    if (solver == KS_RK4) return launch_one<J, KS_RK4, KS_NONE, C>(a, st);
    if (solver == KS_DRIFT) return launch_one<J, KS_DRIFT, KS_NONE, C>(a, st);
    switch (stream) {
        case KS_PHILOX: return launch_one<J, KS_EM, KS_PHILOX, C>(a, st);
        case KS_SFC64: return launch_one<J, KS_EM, KS_SFC64, C>(a, st);
        case KS_XOSHIRO: return launch_one<J, KS_EM, KS_XOSHIRO, C>(a, st);
        case KS_NONE: return launch_one<J, KS_EM, KS_NONE, C>(a, st);
        case KS_EXPLICIT: return launch_one<J, KS_EM, KS_EXPLICIT, C>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

template <int J>
cudaError_t launch_kuramoto_j(const RunArgs& a, int solver, int stream, int coupling,
                              cudaStream_t st) {
    if (coupling == KC_PAIRWISE) return launch_coupling<J, KC_PAIRWISE>(a, solver, stream, st);
    return launch_coupling<J, KC_MEANFIELD>(a, solver, stream, st);
}

}  // namespace sdeb
