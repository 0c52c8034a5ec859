// Per-J launch dispatch; included by sdeb_kuramoto_j{1,2,4,8,16}.cu so the
// instantiations compile in parallel.
#pragma once
#include "sdeb_kuramoto.cuh"

namespace sdeb {

template <int J, int S, int R, int C, int M>
static cudaError_t launch_one(const RunArgs& a, cudaStream_t st) {
    const int64_t threads = a.orbits * int64_t(a.lanes);
    const unsigned grid = unsigned((threads + kBlock - 1) / kBlock);
    const size_t need = pairwise_smem_bytes(J, C);
    const size_t smem = need > size_t(a.smem_pad) ? need : size_t(a.smem_pad);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kuramoto_run_kernel<J, S, R, C, M>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem));
        if (e != cudaSuccess) return e;
    }
    kuramoto_run_kernel<J, S, R, C, M><<<grid, kBlock, smem, st>>>(a);
    return cudaGetLastError();
}

template <int J, int S, int R, int C, int M>
static cudaError_t occupancy_one(size_t smem, int* blocks) {
    const size_t need = pairwise_smem_bytes(J, C);
    if (smem < need) smem = need;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kuramoto_run_kernel<J, S, R, C, M>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem));
        if (e != cudaSuccess) return e;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, kuramoto_run_kernel<J, S, R, C, M>,
                                                         kBlock, smem);
}

// Visits the kernel instantiation for (solver, stream, coupling, tight) with
// op.template run<J, S, R, C, M>().  Tight variants exist for the meanfield
// em / rk4 paths at J in {4, 8}.
template <int J, class Op>
static cudaError_t dispatch(int solver, int stream, int coupling, int tight, Op&& op) {
    constexpr int MT = tight_minb<J>();
    const bool t = tight && MT > 1 && coupling == KC_MEANFIELD;
#define SDEB_PICK(S, R, C)                                                      \
    return t ? op.template run<J, S, R, C, (C == KC_MEANFIELD ? MT : 1)>()     \
             : op.template run<J, S, R, C, 1>()
    if (coupling == KC_PAIRWISE) {
        if (solver == KS_RK4) SDEB_PICK(KS_RK4, KS_NONE, KC_PAIRWISE);
        if (solver == KS_DRIFT) SDEB_PICK(KS_DRIFT, KS_NONE, KC_PAIRWISE);
        switch (stream) {
            case KS_PHILOX: SDEB_PICK(KS_EM, KS_PHILOX, KC_PAIRWISE);
            case KS_SFC64: SDEB_PICK(KS_EM, KS_SFC64, KC_PAIRWISE);
            case KS_XOSHIRO: SDEB_PICK(KS_EM, KS_XOSHIRO, KC_PAIRWISE);
            case KS_NONE: SDEB_PICK(KS_EM, KS_NONE, KC_PAIRWISE);
            case KS_EXPLICIT: SDEB_PICK(KS_EM, KS_EXPLICIT, KC_PAIRWISE);
            default: return cudaErrorInvalidValue;
        }
    }
    if (solver == KS_RK4) SDEB_PICK(KS_RK4, KS_NONE, KC_MEANFIELD);
    if (solver == KS_DRIFT) return op.template run<J, KS_DRIFT, KS_NONE, KC_MEANFIELD, 1>();
    switch (stream) {
        case KS_PHILOX: SDEB_PICK(KS_EM, KS_PHILOX, KC_MEANFIELD);
        case KS_SFC64: SDEB_PICK(KS_EM, KS_SFC64, KC_MEANFIELD);
        case KS_XOSHIRO: SDEB_PICK(KS_EM, KS_XOSHIRO, KC_MEANFIELD);
        case KS_NONE: SDEB_PICK(KS_EM, KS_NONE, KC_MEANFIELD);
        case KS_EXPLICIT: return op.template run<J, KS_EM, KS_EXPLICIT, KC_MEANFIELD, 1>();
        default: return cudaErrorInvalidValue;
    }
#undef SDEB_PICK
}

struct LaunchOp {
    const RunArgs& a;
    cudaStream_t st;
    template <int J, int S, int R, int C, int M>
    cudaError_t run() const {
        return launch_one<J, S, R, C, M>(a, st);
    }
};

struct OccupancyOp {
    size_t smem;
    int* blocks;
    template <int J, int S, int R, int C, int M>
    cudaError_t run() const {
        return occupancy_one<J, S, R, C, M>(smem, blocks);
    }
};

template <int J>
cudaError_t launch_kuramoto_j(const RunArgs& a, int solver, int stream, int coupling, int tight,
                              cudaStream_t st) {
    return dispatch<J>(solver, stream, coupling, tight, LaunchOp{a, st});
}

template <int J>
cudaError_t occupancy_kuramoto_j(int solver, int stream, int coupling, int tight, size_t smem,
                                 int* blocks) {
    return dispatch<J>(solver, stream, coupling, tight, OccupancyOp{smem, blocks});
}

}  // namespace sdeb
