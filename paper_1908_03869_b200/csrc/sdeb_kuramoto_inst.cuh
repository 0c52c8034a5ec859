// Per-J launch dispatch; included by sdeb_kuramoto_j{1,2,4,8,16}.cu so the
// instantiations compile in parallel.
#pragma once
#include "sdeb_kuramoto.cuh"

namespace sdeb {

template <int J, int S, int R, int C, int P>
static cudaError_t launch_one(const RunArgs& a, cudaStream_t st) {
    const int64_t threads = a.orbits * int64_t(a.lanes);
    const unsigned grid = a.persistent > 0 ? unsigned(a.persistent)
                                           : unsigned((threads + kBlock - 1) / kBlock);
    constexpr size_t need = own_smem_bytes<J, S, R, C, P>();
    size_t smem = size_t(a.smem_pad);
    if constexpr (need > 0) smem = smem < need ? need : smem;
    // static shared memory (the staged math tables) counts against the 48 KB
    // default too: opt in whenever the sum exceeds it
    if (smem + kStaticSmemBytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kuramoto_run_kernel<J, S, R, C, P>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem));
        if (e != cudaSuccess) return e;
    }
    kuramoto_run_kernel<J, S, R, C, P><<<grid, kBlock, smem, st>>>(a);
    return cudaGetLastError();
}

// Largest shared memory one CTA may use on the current device (opt-in).
static inline size_t smem_optin_bytes() {
    int dev = 0, optin = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
        return 48 * 1024;
    return size_t(optin);
}

template <int J, int S, int R, int C, int P>
static cudaError_t occupancy_one(size_t smem, int* blocks) {
    constexpr size_t need = own_smem_bytes<J, S, R, C, P>();
    if constexpr (need > 0) smem = smem < need ? need : smem;
    // the kernel's own static shared memory (tables + scheduling slot) plus the
    // dynamic request must fit the opt-in limit, else no CTA can be resident
    cudaFuncAttributes fa{};
    cudaError_t ea = cudaFuncGetAttributes(&fa, kuramoto_run_kernel<J, S, R, C, P>);
    if (ea != cudaSuccess) return ea;
    if (smem + fa.sharedSizeBytes > smem_optin_bytes()) {
        *blocks = 0;
        return cudaSuccess;
    }
    if (smem + kStaticSmemBytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kuramoto_run_kernel<J, S, R, C, P>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem));
        if (e != cudaSuccess) return e;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, kuramoto_run_kernel<J, S, R, C, P>,
                                                         kBlock, smem);
}

// Visits the kernel instantiation for (solver, stream, coupling, variant)
// with op.template run<J, S, R, C, V>() (V: 0 unpadded, 1 padded, 2 unpadded
// register-capped; +4: samples are the order parameter, kVarCoherence).
// The explicit-noise / drift entry points always use the padded form; capped
// variants exist where tight_minb<J>() > 1 (meanfield only).
template <int J, class Op>
static cudaError_t dispatch(int solver, int stream, int coupling, int variant, Op&& op) {
    if (variant == 2 && !has_var2<J>()) variant = 0;
#define SDEB_PICK(S, R)                                                          \
    switch (variant) {                                                           \
        case 0: return op.template run<J, S, R, KC_MEANFIELD, 0>();              \
        case 1: return op.template run<J, S, R, KC_MEANFIELD, 1>();              \
        case 4: return op.template run<J, S, R, KC_MEANFIELD, 4>();              \
        case 5: return op.template run<J, S, R, KC_MEANFIELD, 5>();              \
        default: return op.template run<J, S, R, KC_MEANFIELD, (has_var2<J>() ? 2 : 0)>(); \
    }
#define SDEB_PAIR(S, R)                                                          \
    switch (variant) {                                                           \
        case 0: case 2: return op.template run<J, S, R, KC_PAIRWISE, 0>();       \
        case 4: return op.template run<J, S, R, KC_PAIRWISE, 4>();               \
        case 5: return op.template run<J, S, R, KC_PAIRWISE, 5>();               \
        default: return op.template run<J, S, R, KC_PAIRWISE, 1>();              \
    }
    if (coupling == KC_PAIRWISE) {
        if (solver == KS_RK4) SDEB_PAIR(KS_RK4, KS_NONE);
        if (solver == KS_DRIFT) return op.template run<J, KS_DRIFT, KS_NONE, KC_PAIRWISE, 1>();
        switch (stream) {
            case KS_PHILOX: SDEB_PAIR(KS_EM, KS_PHILOX);
            case KS_SFC64: SDEB_PAIR(KS_EM, KS_SFC64);
            case KS_XOSHIRO: SDEB_PAIR(KS_EM, KS_XOSHIRO);
            case KS_NONE: SDEB_PAIR(KS_EM, KS_NONE);
            case KS_EXPLICIT: return op.template run<J, KS_EM, KS_EXPLICIT, KC_PAIRWISE, 1>();
            default: return cudaErrorInvalidValue;
        }
    }
    if (solver == KS_RK4) SDEB_PICK(KS_RK4, KS_NONE);
    if (solver == KS_DRIFT) return op.template run<J, KS_DRIFT, KS_NONE, KC_MEANFIELD, 1>();
    switch (stream) {
        case KS_PHILOX: SDEB_PICK(KS_EM, KS_PHILOX);
        case KS_SFC64: SDEB_PICK(KS_EM, KS_SFC64);
        case KS_XOSHIRO: SDEB_PICK(KS_EM, KS_XOSHIRO);
        case KS_NONE: SDEB_PICK(KS_EM, KS_NONE);
        case KS_EXPLICIT: return op.template run<J, KS_EM, KS_EXPLICIT, KC_MEANFIELD, 1>();
        default: return cudaErrorInvalidValue;
    }
#undef SDEB_PICK
#undef SDEB_PAIR
}

struct LaunchOp {
    const RunArgs& a;
    cudaStream_t st;
    template <int J, int S, int R, int C, int P>
    cudaError_t run() const {
        return launch_one<J, S, R, C, P>(a, st);
    }
};

struct OccupancyOp {
    size_t smem;
    int* blocks;
    template <int J, int S, int R, int C, int P>
    cudaError_t run() const {
        return occupancy_one<J, S, R, C, P>(smem, blocks);
    }
};

template <int J>
cudaError_t launch_kuramoto_j(const RunArgs& a, int solver, int stream, int coupling,
                              int padded, cudaStream_t st) {
    return dispatch<J>(solver, stream, coupling, padded, LaunchOp{a, st});
}

template <int J>
cudaError_t occupancy_kuramoto_j(int solver, int stream, int coupling, int padded, size_t smem,
                                 int* blocks) {
    return dispatch<J>(solver, stream, coupling, padded, OccupancyOp{smem, blocks});
}

}  // namespace sdeb
