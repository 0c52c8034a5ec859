// C ABI (include/sdeb200.h): contexts, validation, sharding, layout
// autotune, host<->device staging.  The reference equivalent is run_batch's
// driver (engine.py:184-277) and its thread pool over contiguous orbit
// groups (engine.py:145-150, 265-274): here the groups are per-device shards
// driven by one host thread each, and the per-group Python step loop is the
// fused kernel of sdeb_kuramoto.cuh.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <sys/mman.h>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/sdeb200.h"
#include "sdeb_dsl.h"
#include "sdeb_kuramoto.cuh"
#include "sdeb_misc.h"

namespace {

thread_local std::string g_thread_error;

struct DevBuf {
    void* ptr = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(bytes, 256);
        cudaError_t e = cudaMalloc(&ptr, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(ptr);
    }
};

// Pinned host staging slot (grow-only) + the event of the last DMA that used it.
struct PinBuf {
    void* ptr = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    cudaError_t ensure(size_t bytes) {
        if (!ev) {
            cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
        if (bytes <= cap) return cudaSuccess;
        if (ptr) {
            cudaError_t e = cudaEventSynchronize(ev);
            if (e != cudaSuccess) return e;
            cudaFreeHost(ptr);
        }
        ptr = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(bytes, 1 << 20);
        cudaError_t e = cudaHostAlloc(&ptr, want, cudaHostAllocPortable);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (ev) cudaEventSynchronize(ev);
        if (ptr) cudaFreeHost(ptr);
        if (ev) cudaEventDestroy(ev);
        ptr = nullptr;
        ev = nullptr;
        cap = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(ptr);
    }
};

constexpr int kPinSlots = 2;

struct Slot {
    int device = 0;
    cudaStream_t stream = nullptr;  // kernels
    cudaStream_t h2d = nullptr;     // host-buffer runs: input DMA
    cudaStream_t d2h = nullptr;     // host-buffer runs: output DMA
    cudaEvent_t ev_in = nullptr;
    std::vector<cudaEvent_t> ev_tile;  // end of each tile's kernel
    PinBuf pin_in[kPinSlots], pin_out[kPinSlots];
    PinBuf pin_warm;  // one small page-locked block opened with the context
    DevBuf init, params, values, state, fail, rng;
    DevBuf t_values, t_state, t_fail, t_rng, t_work;  // autotune scratch
    DevBuf work;  // persistent mode: item counter + per-group slab counters
    DevBuf scratch;  // expression-template programs with global state columns
    int64_t launches = 0;
    int32_t lanes = 0;
    int32_t persistent = 0;
    int32_t ctas_per_sm = 0;
    int32_t tight = 0;
    int32_t lane_width = 0;  // oscillators per lane (J) of the last launch
    int32_t tiles = 0;  // orbit tiles of the last host-buffer run
    int64_t tune_us = 0;  // autotune probe time of the current call
    // end of the last launch that used this slot's scratch (state, rng, work),
    // and the stream it ran on: a launch on another stream waits for it first
    cudaEvent_t done = nullptr;
    cudaStream_t done_stream = nullptr;
    std::string error;
};

// One launch layout: lanes per orbit, persistent work-pulling grid or one
// CTA per CTA-group, dynamic shared memory used to cap resident CTAs per SM
// (wave shaping), and the resident CTAs per SM it runs at.
struct Layout {
    int lanes = 0;
    int persistent = 0;
    int smem = 0;
    int ctas_per_sm = 0;
    int tight = 0;  // VAR 2: register-capped J in {4, 8}, or J = 16 with step constants in smem
    int J = 0;      // oscillators per lane; 0 = next_pow2(n) / lanes
    int exact = 1;  // 0: ctas_per_sm estimated from the build's resource table
};

// Registers / static shared memory of every stepper instantiation (ptxas -v at
// build time, _build.py): occupancy without loading a kernel module.
struct KernelRes {
    short J, solver, stream, coupling, variant, regs;
    int smem;
};
#include "sdeb_kernel_table.inc"

using TuneKey = std::tuple<int, int, int, int, int, int64_t, int, int>;

}  // namespace

struct sdb_ctx {
    std::vector<Slot> slots;
    std::string error;
    int64_t launches = 0;
    int32_t last_lanes = 0;
    int32_t last_persistent = 0;
    int32_t last_ctas_per_sm = 0;
    int32_t last_tight = 0;
    int32_t last_lane_width = 0;
    int32_t last_tiles = 0;
    int64_t last_tune_us = 0;
    std::map<TuneKey, Layout> tune;
    std::mutex mu;  // guards tune and error: shard threads of one run share the context
    // Serialises the public entry points on one context: its slots' device
    // buffers and pinned staging are reused by every call, so two host
    // threads calling sdb_run* at once must take turns (the reference's
    // run_batch is reentrant; so is this one, per context).
    std::mutex call_mu;
};

namespace {

sdb_status fail_with(sdb_ctx* ctx, sdb_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (ctx) {
        std::lock_guard<std::mutex> lock(ctx->mu);
        ctx->error = buf;
    }
    g_thread_error = buf;
    return st;
}

// Held for the duration of one public call on a context (sdb_ctx::call_mu);
// starts the call with no error recorded for this thread or the context.
struct CallScope {
    std::unique_lock<std::mutex> lock;
    explicit CallScope(sdb_ctx* ctx) : lock(ctx->call_mu) {
        g_thread_error.clear();
        std::lock_guard<std::mutex> l(ctx->mu);
        ctx->error.clear();
    }
};

#define SDB_ENTRY(ctx)                                                               \
    if (!(ctx)) return fail_with(nullptr, SDB_ERR_ARGUMENT, "null context");        \
    CallScope call_scope__(ctx)

sdb_status cuda_fail(sdb_ctx* ctx, cudaError_t e, const char* what) {
    return fail_with(ctx, SDB_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorString(e),
                     cudaGetErrorName(e));
}

sdb_status cuda_fail_if(sdb_ctx* ctx, cudaError_t e) {
    return e == cudaSuccess ? SDB_OK : cuda_fail(ctx, e, "autotune scratch");
}

#define SDB_CUDA(ctx, expr)                                      \
    do {                                                         \
        cudaError_t e__ = (expr);                                \
        if (e__ != cudaSuccess) return cuda_fail(ctx, e__, #expr); \
    } while (0)

int next_pow2(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    return p;
}

int ilog2(int x) {
    int l = 0;
    while ((1 << l) < x) ++l;
    return l;
}

// Lane widths J whose kernel module this process has launched from: the first
// launch from a module pays its (lazy) load, ~6-45 ms on B200 (measured,
// tools/module_load_probe.py), which the layout probe budgets for.
std::atomic<uint32_t> g_loaded_j{0};

cudaError_t launch_run_j(const sdeb::RunArgs& a, int J, int solver, int stream, int coupling,
                         int padded, cudaStream_t st);

cudaError_t launch_run(const sdeb::RunArgs& a, int J, int solver, int stream, int coupling,
                       int padded, cudaStream_t st) {
    const cudaError_t e = launch_run_j(a, J, solver, stream, coupling, padded, st);
    if (e == cudaSuccess && J >= 0 && J < 32) g_loaded_j.fetch_or(1u << J);
    return e;
}

bool module_loaded(int J) { return J >= 0 && J < 32 && (g_loaded_j.load() >> J) & 1u; }

cudaError_t launch_run_j(const sdeb::RunArgs& a, int J, int solver, int stream, int coupling,
                         int padded, cudaStream_t st) {
    switch (J) {
        case 1: return sdeb::launch_kuramoto_j<1>(a, solver, stream, coupling, padded, st);
        case 2: return sdeb::launch_kuramoto_j<2>(a, solver, stream, coupling, padded, st);
        case 4: return sdeb::launch_kuramoto_j<4>(a, solver, stream, coupling, padded, st);
        case 8: return sdeb::launch_kuramoto_j<8>(a, solver, stream, coupling, padded, st);
        case 16: return sdeb::launch_kuramoto_j<16>(a, solver, stream, coupling, padded, st);
        case 3: return sdeb::launch_kuramoto_j<3>(a, solver, stream, coupling, padded, st);
        case 5: return sdeb::launch_kuramoto_j<5>(a, solver, stream, coupling, padded, st);
        case 6: return sdeb::launch_kuramoto_j<6>(a, solver, stream, coupling, padded, st);
        case 7: return sdeb::launch_kuramoto_j<7>(a, solver, stream, coupling, padded, st);
        case 9: return sdeb::launch_kuramoto_j<9>(a, solver, stream, coupling, padded, st);
        case 10: return sdeb::launch_kuramoto_j<10>(a, solver, stream, coupling, padded, st);
        case 11: return sdeb::launch_kuramoto_j<11>(a, solver, stream, coupling, padded, st);
        case 12: return sdeb::launch_kuramoto_j<12>(a, solver, stream, coupling, padded, st);
        case 13: return sdeb::launch_kuramoto_j<13>(a, solver, stream, coupling, padded, st);
        case 14: return sdeb::launch_kuramoto_j<14>(a, solver, stream, coupling, padded, st);
        case 15: return sdeb::launch_kuramoto_j<15>(a, solver, stream, coupling, padded, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t occupancy_run(int J, int solver, int stream, int coupling, int padded, size_t smem,
                          int* blocks) {
    switch (J) {
        case 1: return sdeb::occupancy_kuramoto_j<1>(solver, stream, coupling, padded, smem, blocks);
        case 2: return sdeb::occupancy_kuramoto_j<2>(solver, stream, coupling, padded, smem, blocks);
        case 4: return sdeb::occupancy_kuramoto_j<4>(solver, stream, coupling, padded, smem, blocks);
        case 8: return sdeb::occupancy_kuramoto_j<8>(solver, stream, coupling, padded, smem, blocks);
        case 16: return sdeb::occupancy_kuramoto_j<16>(solver, stream, coupling, padded, smem, blocks);
        case 3: return sdeb::occupancy_kuramoto_j<3>(solver, stream, coupling, padded, smem, blocks);
        case 5: return sdeb::occupancy_kuramoto_j<5>(solver, stream, coupling, padded, smem, blocks);
        case 6: return sdeb::occupancy_kuramoto_j<6>(solver, stream, coupling, padded, smem, blocks);
        case 7: return sdeb::occupancy_kuramoto_j<7>(solver, stream, coupling, padded, smem, blocks);
        case 9: return sdeb::occupancy_kuramoto_j<9>(solver, stream, coupling, padded, smem, blocks);
        case 10: return sdeb::occupancy_kuramoto_j<10>(solver, stream, coupling, padded, smem, blocks);
        case 11: return sdeb::occupancy_kuramoto_j<11>(solver, stream, coupling, padded, smem, blocks);
        case 12: return sdeb::occupancy_kuramoto_j<12>(solver, stream, coupling, padded, smem, blocks);
        case 13: return sdeb::occupancy_kuramoto_j<13>(solver, stream, coupling, padded, smem, blocks);
        case 14: return sdeb::occupancy_kuramoto_j<14>(solver, stream, coupling, padded, smem, blocks);
        case 15: return sdeb::occupancy_kuramoto_j<15>(solver, stream, coupling, padded, smem, blocks);
        default: return cudaErrorInvalidValue;
    }
}


// Resident CTAs per SM of an instantiation from the build's resource table
// (registers in 256-register warp allocations, static shared memory + 1 KB
// per CTA of the SM's opt-in maximum, 16 warps... the 32-CTA and 64-warp
// limits), or -1 when the table has no entry.  An estimate for ordering
// candidates: a layout that is launched is re-checked with the CUDA
// occupancy query (finalize_layout), which the persistent grid relies on.
int table_occupancy(int device, int J, int solver, int stream, int coupling, int variant) {
    for (int pass = 0; pass < 2; ++pass) {
        const int want = pass == 0 ? variant : (variant == 2 ? 0 : -1);
        if (want < 0) break;
        for (const KernelRes* r = kKernelRes; r->J != 0; ++r) {
            if (r->J != J || r->solver != solver || r->stream != stream ||
                r->coupling != coupling || r->variant != want)
                continue;
            int sm_smem = 0, regs_sm = 0;
            cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
            cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, device);
            const int per_warp = ((int(r->regs) * 32 + 255) / 256) * 256;
            const int warps = per_warp > 0 ? regs_sm / per_warp : 64;
            const int by_regs = std::min(warps, 64) / (sdeb::kBlock / 32);
            const int by_smem = sm_smem / (r->smem + 1024);
            return std::max(0, std::min({by_regs, by_smem, 32}));
        }
    }
    return -1;
}

// Kernel kind for a validated descriptor.
void kernel_kind(const sdb_desc& d, int* solver, int* stream) {
    if (d.solver == SDB_SOLVER_RK4) {
        *solver = sdeb::KS_RK4;
        *stream = sdeb::KS_NONE;
    } else if (d.solver == SDB_SOLVER_EM && d.nnoise > 0) {
        *solver = sdeb::KS_EM;
        *stream = d.stream;  // KS_PHILOX/SFC64/XOSHIRO share the ABI values
    } else {
        *solver = sdeb::KS_EM;  // euler, or em on a noise-free model (solvers.py:63-71)
        *stream = sdeb::KS_NONE;
    }
}

constexpr int kMaxLanes = 32;
constexpr int kMaxJ = 16;
constexpr int kMaxN = kMaxLanes * kMaxJ;

sdb_status validate(sdb_ctx* ctx, const sdb_desc* d) {
    if (!d) return fail_with(ctx, SDB_ERR_ARGUMENT, "null descriptor");
    if (d->model != SDB_MODEL_KURAMOTO)
        return fail_with(ctx, SDB_ERR_UNSUPPORTED, "only the Kuramoto model has a device path");
    if (d->nequat < 1) return fail_with(ctx, SDB_ERR_ARGUMENT, "nequat must be >= 1");
    if (d->nequat > kMaxN)
        return fail_with(ctx, SDB_ERR_UNSUPPORTED, "nequat=%d above the device limit %d", d->nequat,
                         kMaxN);
    if (d->nnoise != 0 && d->nnoise != d->nequat)
        return fail_with(ctx, SDB_ERR_UNSUPPORTED, "Kuramoto needs nnoise == nequat or 0");
    if (d->nparams < d->nequat + 1 || (d->nnoise > 0 && d->nparams != 2 * d->nequat + 1))
        return fail_with(ctx, SDB_ERR_ARGUMENT, "nparams=%d does not fit Kuramoto(n=%d, nnoise=%d)",
                         d->nparams, d->nequat, d->nnoise);
    if (d->solver != SDB_SOLVER_EM && d->solver != SDB_SOLVER_EULER && d->solver != SDB_SOLVER_RK4)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "unknown solver %d", d->solver);
    if (d->solver != SDB_SOLVER_EM && d->nnoise > 0)
        return fail_with(ctx, SDB_ERR_CONFIG,
                         "solver is deterministic but the model has %d noise terms", d->nnoise);
    if (d->stream < SDB_STREAM_PHILOX || d->stream > SDB_STREAM_XOSHIRO256PP)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "unknown stream %d", d->stream);
    if (d->coupling != SDB_COUPLING_MEANFIELD && d->coupling != SDB_COUPLING_PAIRWISE)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "unknown coupling %d", d->coupling);
    if (!(d->dt > 0.0)) return fail_with(ctx, SDB_ERR_CONFIG, "dt must be positive");
    if (d->ksteps < 1) return fail_with(ctx, SDB_ERR_CONFIG, "ksteps must be >= 1");
    if (d->chunks < 1) return fail_with(ctx, SDB_ERR_CONFIG, "chunks must be >= 1");
    if (d->orbits < 1) return fail_with(ctx, SDB_ERR_CONFIG, "orbits must be >= 1");
    if (d->orbit_offset < 0 || d->orbit_offset + d->orbits > (int64_t(1) << 32))
        return fail_with(ctx, SDB_ERR_CONFIG, "global orbit ids must fit in 32 bits");
    if (d->chunks > INT64_MAX / d->ksteps)
        return fail_with(ctx, SDB_ERR_CONFIG, "total step count does not fit in 63 bits");
    const int P = next_pow2(d->nequat);
    if (d->lanes != 0) {
        const int L = d->lanes;
        if (L < 1 || L > kMaxLanes || (L & (L - 1)) || L > P || P / L > kMaxJ)
            return fail_with(ctx, SDB_ERR_ARGUMENT, "lanes=%d is not a valid layout for n=%d", L,
                             d->nequat);
    }
    return SDB_OK;
}

std::vector<int> candidate_lanes(int n) {
    const int P = next_pow2(n);
    std::vector<int> out;
    for (int L = 1; L <= kMaxLanes && L <= P; L <<= 1)
        if (P / L <= kMaxJ) out.push_back(L);
    return out;
}

sdeb::RunArgs make_args(const sdb_desc& d, int lanes) {
    sdeb::RunArgs a{};
    a.n = d.nequat;
    a.nparams = d.nparams;
    a.nnoise = d.nnoise;
    a.lanes = lanes;
    a.log2lanes = ilog2(lanes);
    a.orbits = d.orbits;
    a.orbit_offset = d.orbit_offset;
    a.seed = d.seed;
    a.dt = d.dt;
    a.sqrt_dt = std::sqrt(d.dt);  // np.sqrt(dt), IEEE correctly rounded
    a.half_dt = 0.5 * d.dt;
    a.dt6 = d.dt / 6.0;
    a.ksteps = d.ksteps;
    a.chunk_begin = 0;
    a.chunk_end = d.chunks;
    a.vstride = d.chunks;
    a.fresh = 1;
    a.check_finite = 1;
    a.groups = (d.orbits * lanes + sdeb::kBlock - 1) / sdeb::kBlock;  // one CTA per group
    return a;
}

size_t rng_words(const sdb_desc& d, int64_t rows) {
    const bool stateful = d.solver == SDB_SOLVER_EM && d.nnoise > 0 &&
                          (d.stream == SDB_STREAM_SFC64 || d.stream == SDB_STREAM_XOSHIRO256PP);
    return stateful ? size_t(rows) * size_t((d.nnoise + 3) / 4) * 4 : 0;
}

// Shared memory that caps a kernel at `cap` resident CTAs per SM.
int smem_for_cap(int device, int cap) {
    int per_sm = 0;
    cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    const int reserved = 1024;  // per-CTA reservation on sm_100
    // the stepper's static shared memory (staged math tables) is part of the budget
    return std::max(0, per_sm / cap - reserved - int(sdeb::kTableSmemBytes)) & ~255;
}

// Dynamic shared memory that holds a kernel at exactly `cap` CTAs per SM:
// smem_for_cap's estimate, stepped down 256 B at a time until the occupancy
// calculator agrees (the kernel's own static shared memory and allocation
// granularity are not known exactly up front).  0 if no size works.
int fit_smem_for_cap(int device, int J, int solver, int stream, int coupling, int variant,
                     int cap) {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    for (int smem = smem_for_cap(device, cap), tries = 0; smem > 0 && tries < 16;
         smem -= 256, ++tries) {
        if (smem > optin) continue;
        int got = 0;
        if (occupancy_run(J, solver, stream, coupling, variant, size_t(smem), &got) != cudaSuccess) {
            cudaGetLastError();  // not sticky: drop it so later launches see a clean slate
            return 0;
        }
        if (got == cap) return smem;
        if (got < cap) continue;  // still too large per CTA
        return 0;                 // more CTAs than asked: smaller sizes only add more
    }
    return 0;
}

// Kernel instantiation variant: 1 padded (n < next_pow2(n)), else 0, or 2
// for the register-capped unpadded form.
int kernel_variant(const sdb_desc& d, int lanes, int J, int tight) {
    if (d.nequat < lanes * J) return 1;
    return tight ? 2 : 0;
}

// Oscillators per lane of a layout.
int layout_J(const sdb_desc& d, const Layout& l) {
    return l.J ? l.J : next_pow2(d.nequat) / l.lanes;
}

// n <= 16 that is not a power of two (e.g. the paper's N = 5, 10, 15) also
// runs one lane per orbit with J = n: no padded oscillators (n = 5 in a
// power-of-two span wastes 3/8 of the sincos, sums and updates).  Same bits
// as the padded layouts: the stride-doubling lane tree over n leaves
// associates exactly like the canonical tree over next_pow2(n) leaves with
// zero padding, and the noise blocks and Box-Muller pairs are the same.
int exact_J(const sdb_desc& d) {
    const bool fits = d.nequat >= 3 && d.nequat <= kMaxJ && d.nequat != next_pow2(d.nequat);
    const bool one_lane = d.lanes == 1 ||
                          (d.lanes == 0 && (d.coupling == SDB_COUPLING_MEANFIELD ||
                                            sdeb::pairwise_lanes(d.nequat) == 1));
    return (fits && one_lane) ? d.nequat : 0;
}

int64_t cta_groups(const sdb_desc& d, int lanes) {
    return (d.orbits * lanes + sdeb::kBlock - 1) / sdeb::kBlock;
}

// Persistent mode: slabs sized so the resident grid sees >= 32 rounds of
// work items (the end-of-run imbalance is then < ~3%), and >= 16 steps each.
int64_t slab_steps_for(int64_t total_steps, int64_t groups, int64_t grid) {
    const int64_t rounds = 32;
    const int64_t nslabs = std::max<int64_t>(1, (rounds * grid + groups - 1) / groups);
    return std::max<int64_t>(16, (total_steps + nslabs - 1) / nslabs);
}

// Candidate layouts per lanes-per-orbit: natural occupancy; CTA-per-SM caps
// below it that turn a ragged last wave into full ones; and the persistent
// work-pulling grid (whenever the CTA-groups exceed one wave).
sdb_status candidate_layouts(sdb_ctx* ctx, const Slot& s, const sdb_desc& d, int kind_solver,
                             int kind_stream, std::vector<Layout>* out) {
    const int P = next_pow2(d.nequat);
    int sms = 0;
    SDB_CUDA(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s.device));
    std::vector<int> lanes_list;
    if (d.lanes != 0) {
        lanes_list.push_back(d.lanes);
    } else if (d.coupling == SDB_COUPLING_PAIRWISE) {
        // the pairwise sum's order depends on (L, J): one lane count per n
        lanes_list.push_back(sdeb::pairwise_lanes(d.nequat));
    } else {
        for (int L : candidate_lanes(d.nequat)) lanes_list.push_back(L);
    }
    // (L, J) pairs: the power-of-two span for every lane count, plus the exact
    // one-lane layout where n has one (exact_J)
    std::vector<std::pair<int, int>> shapes;
    for (int L : lanes_list) shapes.emplace_back(L, P / L);
    if (const int XJ = exact_J(d)) shapes.emplace_back(1, XJ);
    for (const auto& shape : shapes) {
      const int L = shape.first, J = shape.second;
      const int XJ = J == P / L ? 0 : J;  // Layout::J (0 = the power-of-two span)
      const bool can_tight = d.nequat == P && d.coupling == SDB_COUPLING_MEANFIELD &&
                             (J == 4 || J == 8 || (J == 16 && kind_solver == sdeb::KS_EM &&
                                                    kind_stream != sdeb::KS_NONE));
      for (int tight = 0; tight <= (can_tight ? 1 : 0); ++tight) {
        const int padded = kernel_variant(d, L, J, tight);
        // a kernel whose module this process has not loaded: estimate its
        // occupancy from the build's resource table rather than loading the
        // module (~20-40 ms lazily) for a layout the probe may never run
        int occ = -1;
        if (!module_loaded(J))
            occ = table_occupancy(s.device, J, kind_solver, kind_stream, d.coupling, padded);
        const int exact = occ < 0 ? 1 : 0;
        if (exact)
            SDB_CUDA(ctx, occupancy_run(J, kind_solver, kind_stream, d.coupling, padded, 0, &occ));
        if (occ < 1) continue;
        const int64_t ctas = cta_groups(d, L);
        out->push_back(Layout{L, 0, 0, occ, tight, XJ, exact});
        if (ctas > int64_t(sms) * occ) out->push_back(Layout{L, 1, 0, occ, tight, XJ, exact});
        if (tight || !exact) continue;  // wave-shaping caps need the exact query
        for (int cap = occ - 1; cap >= 1 && cap >= occ - 4; --cap) {
            const double waves_cap = double(ctas) / (double(sms) * cap);
            const double waves_occ = double(ctas) / (double(sms) * occ);
            const double eff_cap = waves_cap / std::ceil(waves_cap);
            const double eff_occ = waves_occ / std::ceil(waves_occ);
            if (eff_cap <= eff_occ + 0.02) continue;
            const int smem = fit_smem_for_cap(s.device, J, kind_solver, kind_stream, d.coupling,
                                              padded, cap);
            if (smem > 0) out->push_back(Layout{L, 0, smem, cap, 0, XJ});
        }
      }
    }
    return SDB_OK;
}

// Replace a table-estimated occupancy by the CUDA occupancy query (this loads
// the kernel, which is about to run): the persistent grid must be exactly the
// resident CTAs.
sdb_status finalize_layout(sdb_ctx* ctx, const sdb_desc& d, Layout* lay) {
    if (lay->exact) return SDB_OK;
    int kind_solver, kind_stream;
    kernel_kind(d, &kind_solver, &kind_stream);
    const int J = lay->J ? lay->J : next_pow2(d.nequat) / lay->lanes;
    int occ = 0;
    SDB_CUDA(ctx, occupancy_run(J, kind_solver, kind_stream, d.coupling,
                                kernel_variant(d, lay->lanes, J, lay->tight), size_t(lay->smem),
                                &occ));
    if (occ < 1) return fail_with(ctx, SDB_ERR_CUDA, "layout L=%d J=%d cannot be resident",
                                  lay->lanes, J);
    lay->ctas_per_sm = occ;
    lay->exact = 1;
    return SDB_OK;
}

// Fill the layout-dependent launch arguments; zeroes the persistent-mode
// counters on `st` (one memset) when needed.
sdb_status configure_layout(sdb_ctx* ctx, const Slot& s, DevBuf& work, const sdb_desc& d,
                            const Layout& lay, int64_t total_steps, cudaStream_t st,
                            sdeb::RunArgs* a) {
    a->smem_pad = lay.smem;
    a->groups = cta_groups(d, lay.lanes);
    a->persistent = 0;
    if (lay.persistent) {
        int sms = 0;
        SDB_CUDA(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s.device));
        const int64_t grid = int64_t(sms) * lay.ctas_per_sm;
        const size_t bytes = sizeof(uint64_t) + size_t(a->groups) * sizeof(unsigned);
        SDB_CUDA(ctx, work.ensure(bytes));
        SDB_CUDA(ctx, cudaMemsetAsync(work.ptr, 0, bytes, st));
        a->persistent = int(grid);
        a->slab_steps = slab_steps_for(total_steps, a->groups, grid);
        a->work_counter = work.as<uint64_t>();
        a->slab_done = reinterpret_cast<unsigned*>(work.as<char>() + sizeof(uint64_t));
    }
    return SDB_OK;
}

// One device's contiguous shard [r0, r0+rows) of a host-buffer run.
// SDEB200_TRACE=1: per-phase wall-clock of host-buffer runs on stderr (adds
// stream synchronisations between phases; for diagnosis only).
bool trace_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SDEB200_TRACE");
        return e && *e && *e != '0';
    }();
    return on;
}

double now_ms();

// ---- layout selection ------------------------------------------------------
//
// Every layout gives bit-identical results (canonical summation tree, exact
// slab hand-off), so choosing one only affects speed.  The choice costs at
// most ~10% of the run it is made for, and is remembered on disk:
//   1. in-memory cache per context, then the on-disk cache (SDEB200_TUNE_CACHE,
//      default ~/.cache/sdeb200/layouts-v2.tsv) keyed by GPU, driver, build
//      and shape;
//   2. otherwise the candidates are ordered by a cost model (prior_cost) and
//      probed on ONE resident wave of orbits (every SM full, so the per-wave
//      step time is the steady state of a long run) for a differential pair
//      of step counts; the full-run time of each candidate is then predicted
//      from its wave count (ragged last wave for one CTA per group, the
//      fractional count for the persistent grid).  Probe step counts are
//      sized so the whole probe stays within ~10% of the predicted run; when
//      that budget is too small to resolve a candidate, the prior order
//      decides the rest.

// Cost-model ordering of the candidates (smaller is better): FP64 work per
// thread-step of a lane (J oscillators incl. padding, log2(L) butterfly levels
// of the two coupling sums), at the SM throughput the resident warps can
// sustain (latency hiding saturates at ~8 warps/SM, measured r02), times the
// wave count of the launch mode.  Only an ordering for the probe and, when a
// short run leaves no budget to probe more (cold module loads count), the
// decision itself.
double prior_cost(const sdb_desc& d, const Layout& l, int J, int sms) {
    const int L = l.lanes;
    const double lane_work = double(J) * 40.0 + 6.0 * ilog2(L) + 12.0;
    const double warps = double(l.ctas_per_sm) * sdeb::kBlock / 32.0;
    const double eff = std::min(1.0, warps / 8.0);  // J=16 at 8 warps/SM ran as fast as at 12
    const double per_wave = double(sms) * l.ctas_per_sm;
    const double ctas = double(cta_groups(d, L));
    const double waves = l.persistent ? std::max(1.0, 1.01 * ctas / per_wave)
                                      : std::ceil(ctas / per_wave);
    // a wave's duration is one CTA's: lane_work per step per thread over the
    // SM's share of the pipe (per_wave CTAs run side by side)
    return waves * lane_work * double(l.ctas_per_sm) / eff;
}

std::string disk_cache_path() {
    const char* e = std::getenv("SDEB200_TUNE_CACHE");
    if (e) return (*e == '\0' || std::strcmp(e, "0") == 0) ? std::string() : std::string(e);
    const char* xdg = std::getenv("XDG_CACHE_HOME");
    const char* home = std::getenv("HOME");
    std::string base = (xdg && *xdg) ? std::string(xdg) : (home && *home ? std::string(home) + "/.cache" : "");
    return base.empty() ? std::string() : base + "/sdeb200/layouts-v2.tsv";
}

// Key of one tuning decision: the device and software it was measured on
// (name, SM count, driver, this build) and the launch shape.
std::string disk_key(int device, const sdb_desc& d, int kind_solver, int kind_stream) {
    // attribute queries, not cudaGetDeviceProperties (which costs tens of ms
    // on this driver -- a cold call would pay it): compute capability, SM
    // count, memory and clock identify the GPU model well enough for a cache
    int sms = 0, major = 0, minor = 0, clock = 0, driver = 0;
    size_t free_b = 0, total_b = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    cudaDeviceGetAttribute(&clock, cudaDevAttrClockRate, device);
    cudaMemGetInfo(&free_b, &total_b);
    cudaDriverGetVersion(&driver);
    const int64_t total = d.chunks * d.ksteps;
    char buf[512];
    std::snprintf(buf, sizeof(buf), "mem%lluGB-clk%d|sm%d|cc%d.%d|drv%d|abi%d|%s %s|n%d|s%d|r%d|c%d|L%d|M%lld|T%lld",
                  (unsigned long long)(total_b >> 30), clock, sms, major, minor, driver,
                  SDB_ABI_VERSION, __DATE__, __TIME__, d.nequat, kind_solver, kind_stream,
                  d.coupling, d.lanes, (long long)d.orbits,
                  (long long)std::min<int64_t>(total, int64_t(1) << 20));
    std::string k(buf);
    for (char& c : k)
        if (c == '\t' || c == '\n') c = ' ';
    return k;
}

std::mutex g_disk_mu;
bool g_disk_loaded = false;
std::map<std::string, Layout> g_disk;

void disk_load_locked() {
    if (g_disk_loaded) return;
    g_disk_loaded = true;
    const std::string path = disk_cache_path();
    if (path.empty()) return;
    FILE* f = std::fopen(path.c_str(), "r");
    if (!f) return;
    char line[1024];
    while (std::fgets(line, sizeof(line), f)) {
        char* tab = std::strchr(line, '\t');
        if (!tab) continue;
        *tab = '\0';
        Layout l;
        if (std::sscanf(tab + 1, "%d,%d,%d,%d,%d,%d", &l.lanes, &l.persistent, &l.smem,
                        &l.ctas_per_sm, &l.tight, &l.J) == 6 && l.lanes > 0)
            g_disk[line] = l;  // later lines win
    }
    std::fclose(f);
}

bool disk_lookup(const std::string& key, Layout* out) {
    std::lock_guard<std::mutex> lock(g_disk_mu);
    disk_load_locked();
    auto it = g_disk.find(key);
    if (it == g_disk.end()) return false;
    *out = it->second;
    return true;
}

void disk_store(const std::string& key, const Layout& l) {
    std::lock_guard<std::mutex> lock(g_disk_mu);
    disk_load_locked();
    g_disk[key] = l;
    const std::string path = disk_cache_path();
    if (path.empty()) return;
    const size_t slash = path.rfind('/');
    if (slash != std::string::npos && slash > 0) {  // mkdir -p of the parent
        for (size_t i = 1; i <= slash; ++i)
            if (path[i] == '/' || i == slash) ::mkdir(path.substr(0, i == slash ? slash : i).c_str(), 0755);
    }
    char row[1200];
    const int len = std::snprintf(row, sizeof(row), "%s\t%d,%d,%d,%d,%d,%d\n", key.c_str(),
                                  l.lanes, l.persistent, l.smem, l.ctas_per_sm, l.tight, l.J);
    const int fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_APPEND | O_CLOEXEC, 0644);
    if (fd < 0) return;  // a read-only home only costs the next process a probe
    if (len > 0 && len < int(sizeof(row))) {
        ssize_t w = ::write(fd, row, size_t(len));
        (void)w;
    }
    ::close(fd);
}

// Probe the candidates (see the section comment) and return the best.
sdb_status probe_layouts(sdb_ctx* ctx, Slot& s, const sdb_desc& d, int kind_solver,
                         int kind_stream, const double* d_init, const double* d_params,
                         cudaStream_t st, std::vector<Layout>& cands, Layout* best_out) {
    int sms = 148;
    SDB_CUDA(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s.device));
    const int64_t total = d.chunks * d.ksteps;
    std::stable_sort(cands.begin(), cands.end(), [&](const Layout& a, const Layout& b) {
        return prior_cost(d, a, layout_J(d, a), sms) < prior_cost(d, b, layout_J(d, b), sms);
    });
    // one resident wave of the largest-occupancy candidate bounds the scratch
    int64_t wave_rows_max = 1;
    for (const Layout& l : cands)
        wave_rows_max = std::max<int64_t>(
            wave_rows_max, int64_t(sms) * l.ctas_per_sm * (sdeb::kBlock / l.lanes));
    const int64_t rows_cap = std::min<int64_t>(d.orbits, wave_rows_max);
    SDB_CUDA(ctx, s.t_values.ensure(size_t(rows_cap) * d.nequat * sizeof(double)));
    SDB_CUDA(ctx, s.t_state.ensure(size_t(rows_cap) * d.nequat * sizeof(double)));
    SDB_CUDA(ctx, s.t_fail.ensure(size_t(rows_cap) * sizeof(int64_t)));
    SDB_CUDA(ctx, s.t_rng.ensure(std::max<size_t>(rng_words(d, rows_cap), 4) * sizeof(uint64_t)));
    cudaEvent_t e0, e1;
    SDB_CUDA(ctx, cudaEventCreate(&e0));
    SDB_CUDA(ctx, cudaEventCreate(&e1));
    // one launch of `steps` steps over the candidate's wave: ms (best of 2)
    auto timed = [&](const Layout& lay, int64_t rows, int64_t steps, float* ms_out) -> sdb_status {
        sdb_desc pd = d;
        pd.orbits = rows;
        sdeb::RunArgs a = make_args(pd, lay.lanes);
        a.state_in = d_init;
        a.params = d_params;
        a.state_out = nullptr;
        a.values = s.t_values.as<double>();
        a.vstride = 1;
        a.fail_step = s.t_fail.as<int64_t>();
        a.rng_state = nullptr;
        a.ksteps = steps;
        a.chunk_end = 1;
        a.smem_pad = lay.smem;
        a.groups = cta_groups(pd, lay.lanes);
        a.persistent = 0;  // one wave: every CTA-group resident at once
        const int J = layout_J(d, lay);
        float best = 1e30f;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0, st);
            cudaError_t e = launch_run(a, J, kind_solver, kind_stream, d.coupling,
                                       kernel_variant(d, lay.lanes, J, lay.tight), st);
            cudaEventRecord(e1, st);
            if (e == cudaSuccess) e = cudaEventSynchronize(e1);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "autotune launch");
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
            s.launches += 1;
        }
        *ms_out = best;
        return SDB_OK;
    };
    // predicted full-run ms of a layout from its per-wave step time
    auto predict = [&](const Layout& l, double wave_step_ms, int64_t rows) {
        if (rows >= d.orbits) return wave_step_ms * double(total);  // the probe was the run
        const double per_wave = double(sms) * l.ctas_per_sm;
        const double ctas = double(cta_groups(d, l.lanes));
        // one CTA per group: the ragged last wave costs a whole one; the
        // persistent grid balances to the fractional count (+1%: slab hand-offs)
        const double waves = l.persistent ? 1.01 * ctas / per_wave : std::ceil(ctas / per_wave);
        return wave_step_ms * double(total) * std::max(1.0, waves);
    };
    sdb_status rc = SDB_OK;
    double spent_ms = 0.0, budget_ms = -1.0;
    int64_t p1 = 32;  // first probe: the cost model's favourite, 32 + 64 steps
    double best_pred = 1e300;
    Layout best = cands[0];
    // the probe runs every candidate as one resident wave of one CTA per
    // group, so a persistent layout and its one-CTA-per-group twin measure the
    // same launch: time it once, predict both (no noise-driven mode flips)
    std::map<std::tuple<int, int, int, int, int>, double> measured;
    std::vector<std::pair<double, size_t>> ranked;  // (predicted ms, candidate) of probed ones
    constexpr double kModuleLoadMs = 40.0;  // first launch from a not yet loaded module
    // SDEB200_TUNE=thorough: probe every candidate (module loads and budget
    // ignored) -- for long-lived processes and benchmarks that amortise a
    // complete search; SDEB200_TUNE_BUDGET: the probe's fraction of the run
    static const bool thorough = [] {
        const char* e = std::getenv("SDEB200_TUNE");
        return e && std::strcmp(e, "thorough") == 0;
    }();
    static const double budget_frac = [] {
        const char* e = std::getenv("SDEB200_TUNE_BUDGET");
        const double v = e ? std::atof(e) : 0.1;
        return v > 0.0 ? v : 0.1;
    }();
    for (size_t ci = 0; ci < cands.size() && rc == SDB_OK; ++ci) {
        // a candidate in a module this process has not loaded yet costs its
        // load on top of the probe: only within the budget (never the first)
        if (!thorough && ci > 0 && !module_loaded(layout_J(d, cands[ci])) &&
            spent_ms + kModuleLoadMs > budget_ms)
            continue;
        rc = finalize_layout(ctx, d, &cands[ci]);
        if (rc != SDB_OK) break;
        const Layout& lay = cands[ci];
        const int64_t rows =
            std::min<int64_t>(d.orbits, int64_t(sms) * lay.ctas_per_sm * (sdeb::kBlock / lay.lanes));
        if (rows > rows_cap) {  // the exact occupancy exceeded the table's estimate
            rc = cuda_fail_if(ctx, s.t_values.ensure(size_t(rows) * d.nequat * sizeof(double)));
            if (rc == SDB_OK) rc = cuda_fail_if(ctx, s.t_fail.ensure(size_t(rows) * sizeof(int64_t)));
            if (rc != SDB_OK) break;
        }
        float t1 = 0.f, t2 = 0.f;
        const auto mkey = std::make_tuple(lay.lanes, layout_J(d, lay), lay.tight, lay.smem,
                                          lay.ctas_per_sm);
        // thorough search of a batch smaller than one wave (the probe is the
        // run itself, latency-bound): longer probes, a few-microsecond step
        // otherwise drowns in launch noise (cfg1: 1,024 orbits)
        if (thorough && rows >= d.orbits)
            p1 = std::max<int64_t>(p1, std::min<int64_t>(total / 10, 2048));
        double step_ms;
        auto hit = measured.find(mkey);
        if (hit != measured.end()) {
            step_ms = hit->second;
        } else {
            const double w0 = now_ms();
            rc = timed(lay, rows, p1, &t1);
            if (rc != SDB_OK) break;
            rc = timed(lay, rows, 2 * p1, &t2);
            if (rc != SDB_OK) break;
            spent_ms += now_ms() - w0;  // wall time: launches, module loads, syncs
            // differential step time; if timing noise swallowed the difference,
            // the plain average of the longer probe (launch overhead included)
            step_ms = t2 > t1 ? double(t2 - t1) / double(p1) : double(t2) / double(2 * p1);
            step_ms = std::max(1e-9, step_ms);
            measured[mkey] = step_ms;
        }
        const double pred = predict(lay, step_ms, rows);
        if (trace_enabled())
            std::fprintf(stderr, "[sdeb200] tune n=%d L=%d J=%d pers=%d ctas=%d tight=%d: "
                                 "%.5f ms/step/wave (%lld rows, %lld steps) -> %.3f ms predicted\n",
                         d.nequat, lay.lanes, layout_J(d, lay), lay.persistent, lay.ctas_per_sm,
                         lay.tight, step_ms, (long long)rows, (long long)p1, pred);
        if (pred < best_pred) {
            best_pred = pred;
            best = lay;
        }
        if (budget_ms < 0.0 && t2 > 0.f) {
            // 10% of the predicted run for the whole probe (the first
            // candidate's load and probe included); the remaining candidates
            // share what is left (3 p steps each, 2 repetitions)
            budget_ms = budget_frac * pred;
            const double left = budget_ms - spent_ms;
            const double per_cand = left / double(std::max<size_t>(1, cands.size() - 1));
            const double per_step = double(t2) / double(2 * p1);  // launch overhead included
            const int64_t p = int64_t(per_cand / (6.0 * std::max(1e-6, per_step)));
            if (p < 16) {
                // too short a run to resolve more layouts: keep the cost-model
                // order, probing as many of the next ones as the budget allows
                p1 = 16;
            } else {
                p1 = std::min<int64_t>(p, 2048);
            }
        }
        if (!thorough && ci + 1 < cands.size() && spent_ms >= budget_ms) break;
        ranked.emplace_back(pred, ci);
    }
    // thorough mode, stage 2: the three best predictions re-timed as they will
    // really run -- every orbit, the real grid mode and slab size -- on a
    // differential pair of step counts (the one-wave model misjudged
    // neighbours by a few percent, e.g. cfg3 n=32 L2 J16 vs L4 J8)
    if (thorough && rc == SDB_OK && ranked.size() > 1 && d.orbits > rows_cap) {
        std::sort(ranked.begin(), ranked.end());
        const int64_t p2 = std::min<int64_t>(total, std::max<int64_t>(32, total / 10));
        const size_t need_v = size_t(d.orbits) * d.nequat * sizeof(double);
        rc = cuda_fail_if(ctx, s.t_values.ensure(need_v));
        if (rc == SDB_OK) rc = cuda_fail_if(ctx, s.t_fail.ensure(size_t(d.orbits) * sizeof(int64_t)));
        if (rc == SDB_OK) rc = cuda_fail_if(ctx, s.t_state.ensure(need_v));
        if (rc == SDB_OK)
            rc = cuda_fail_if(ctx, s.t_rng.ensure(std::max<size_t>(rng_words(d, d.orbits), 4) *
                                                  sizeof(uint64_t)));
        // runs predicted to take <= 300 ms are timed at their own length (best
        // of two): the differential form drops per-launch costs that differ
        // between layouts (cfg3 n=256: the shared-constant J=16 layout won the
        // differential and ran 2.6 % slower, profiles/r02/p2u)
        const bool direct = ranked.front().first <= 300.0;
        double best_full = 1e300;
        for (size_t r = 0; r < ranked.size() && r < 3 && rc == SDB_OK; ++r) {
            const Layout& lay = cands[ranked[r].second];
            float tt[2] = {0.f, 0.f};
            tt[0] = tt[1] = 1e30f;
            // (p2, 2 p2, p2, 2 p2): the best of two launches per length
            for (int rep = 0; rep < 4 && rc == SDB_OK; ++rep) {
                if (direct && (rep & 1)) continue;
                const int64_t steps = direct ? total : (rep & 1) == 0 ? p2 : 2 * p2;
                sdeb::RunArgs a = make_args(d, lay.lanes);
                a.state_in = d_init;
                a.params = d_params;
                a.values = s.t_values.as<double>();
                a.vstride = 1;
                a.fail_step = s.t_fail.as<int64_t>();
                a.ksteps = steps;
                a.chunk_end = 1;
                rc = configure_layout(ctx, s, s.t_work, d, lay, total, st, &a);
                if (rc != SDB_OK) break;
                a.state_out = nullptr;
                a.rng_state = nullptr;
                if (a.persistent > 0 && a.slab_steps < steps) {
                    a.state_out = s.t_state.as<double>();
                    a.rng_state = s.t_rng.as<uint64_t>();
                }
                const int J = layout_J(d, lay);
                cudaEventRecord(e0, st);
                cudaError_t e = launch_run(a, J, kind_solver, kind_stream, d.coupling,
                                           kernel_variant(d, lay.lanes, J, lay.tight), st);
                cudaEventRecord(e1, st);
                if (e == cudaSuccess) e = cudaEventSynchronize(e1);
                if (e != cudaSuccess) {
                    rc = cuda_fail(ctx, e, "autotune launch");
                    break;
                }
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                tt[rep & 1] = std::min(tt[rep & 1], ms);
                s.launches += 1;
            }
            if (rc != SDB_OK) break;
            const double full = direct ? double(tt[0])
                                : (tt[1] > tt[0] ? double(tt[1] - tt[0]) / double(p2)
                                                 : double(tt[1]) / double(2 * p2)) * double(total);
            if (trace_enabled())
                std::fprintf(stderr, "[sdeb200] tune stage 2 L=%d J=%d pers=%d ctas=%d: %.3f ms "
                                     "predicted from a full-grid run of %lld steps\n",
                             lay.lanes, layout_J(d, lay), lay.persistent, lay.ctas_per_sm, full,
                             (long long)(direct ? total : p2));
            if (full < best_full) {
                best_full = full;
                best = lay;
            }
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    // full-grid stage-2 scratch can be GBs (cfg3 n=256: 4 GB): give it back
    for (DevBuf* b : {&s.t_values, &s.t_state, &s.t_rng, &s.t_fail})
        if (b->cap > (size_t(256) << 20)) b->release();
    if (rc != SDB_OK) return rc;
    *best_out = best;
    return SDB_OK;
}

// Pick the launch layout: cached, pinned (SDEB200_LAYOUT), single candidate,
// or timed on a short probe into scratch buffers.  Every layout gives
// bit-identical results (canonical summation tree, exact slab hand-off), so
// this only affects speed.
sdb_status choose_layout(sdb_ctx* ctx, Slot& s, const sdb_desc& d, const double* d_init,
                         const double* d_params, cudaStream_t st, Layout* out) {
    int kind_solver, kind_stream;
    kernel_kind(d, &kind_solver, &kind_stream);
    const int64_t total = d.chunks * d.ksteps;
    const TuneKey key{s.device, d.nequat, kind_solver, kind_stream, d.coupling, d.orbits,
                      int(std::min<int64_t>(total, 1 << 20)), d.lanes};
    {
        std::lock_guard<std::mutex> lock(ctx->mu);
        auto it = ctx->tune.find(key);
        if (it != ctx->tune.end()) {
            *out = it->second;
            return SDB_OK;
        }
    }
    // SDEB200_LAYOUT="lanes,persistent,ctas_per_sm[,tight]" pins the layout
    // (profiling runs must not capture autotune probes); ctas_per_sm 0 =
    // natural occupancy.
    if (const char* env = std::getenv("SDEB200_LAYOUT")) {
        int L = 0, pers = 0, cap = 0, tight = 0, xj = 0;
        if (std::sscanf(env, "%d,%d,%d,%d,%d", &L, &pers, &cap, &tight, &xj) >= 1 && L > 0) {
            // 5th field: J (only the exact one-lane layout, J == n, is accepted)
            xj = (xj > 0 && L == 1 && xj == exact_J(d)) ? xj : 0;
            const int J = xj ? xj : next_pow2(d.nequat) / L;
            const int var = kernel_variant(d, L, J, tight);
            int occ = 0;
            SDB_CUDA(ctx, occupancy_run(J, kind_solver, kind_stream, d.coupling, var, 0, &occ));
            const int smem = (cap > 0 && !pers && cap < occ)
                                 ? fit_smem_for_cap(s.device, J, kind_solver, kind_stream,
                                                    d.coupling, var, cap)
                                 : 0;
            Layout lay{L, pers, smem, (cap > 0 && cap < occ && smem > 0) ? cap : occ, tight, xj};
            {
                std::lock_guard<std::mutex> lock(ctx->mu);
                ctx->tune[key] = lay;
            }
            *out = lay;
            return SDB_OK;
        }
    }
    std::vector<Layout> cands;
    const double tc0 = trace_enabled() ? now_ms() : 0.0;
    sdb_status rc = candidate_layouts(ctx, s, d, kind_solver, kind_stream, &cands);
    if (rc != SDB_OK) return rc;
    if (cands.empty()) return fail_with(ctx, SDB_ERR_CUDA, "no launchable layout for n=%d", d.nequat);
    const double tc1 = trace_enabled() ? now_ms() : 0.0;
    const std::string dkey = disk_key(s.device, d, kind_solver, kind_stream);
    if (trace_enabled())
        std::fprintf(stderr, "[sdeb200] layout search: %zu candidates in %.3f ms, cache key in "
                             "%.3f ms\n", cands.size(), tc1 - tc0, now_ms() - tc1);
    Layout lay_disk;
    if (disk_lookup(dkey, &lay_disk)) {
        for (const Layout& c : cands) {  // only a shape this build can still launch
            if (c.lanes == lay_disk.lanes && c.tight == lay_disk.tight && c.J == lay_disk.J) {
                Layout use = lay_disk;  // incl. a wave-shaping smem cap; occupancy re-queried
                use.exact = 0;
                rc = finalize_layout(ctx, d, &use);
                if (rc != SDB_OK) return rc;
                std::lock_guard<std::mutex> lock(ctx->mu);
                ctx->tune[key] = use;
                *out = use;
                return SDB_OK;
            }
        }
    }
    Layout best_l = cands[0];
    if (cands.size() > 1) {
        const double t0 = now_ms();
        rc = probe_layouts(ctx, s, d, kind_solver, kind_stream, d_init, d_params, st, cands,
                           &best_l);
        s.tune_us += int64_t(1e3 * (now_ms() - t0));
        if (rc != SDB_OK) return rc;
    }
    rc = finalize_layout(ctx, d, &best_l);
    if (rc != SDB_OK) return rc;
    {
        std::lock_guard<std::mutex> lock(ctx->mu);
        ctx->tune[key] = best_l;
    }
    disk_store(dkey, best_l);
    *out = best_l;
    return SDB_OK;
}

// One launch of an expression-template program over d.orbits rows (one
// thread per orbit; no layout autotune).
sdb_status launch_model(sdb_ctx* ctx, Slot& s, const sdb_desc& d, sdb_model* m,
                        const double* d_init, const double* d_params, double* d_values,
                        int64_t* d_fail, cudaStream_t st) {
    const int nb = std::max(1, (m->nnoise + 3) / 4);
    SDB_CUDA(ctx, s.state.ensure(size_t(d.orbits) * d.nequat * sizeof(double)));
    int kind = sdeb::DK_RUN_EULER;
    if (d.solver == SDB_SOLVER_RK4) {
        kind = sdeb::DK_RUN_RK4;
    } else if (d.solver == SDB_SOLVER_EM && m->nnoise > 0) {
        kind = d.stream == SDB_STREAM_SFC64 ? sdeb::DK_RUN_SFC64
             : d.stream == SDB_STREAM_XOSHIRO256PP ? sdeb::DK_RUN_XOSHIRO : sdeb::DK_RUN_PHILOX;
        if (kind != sdeb::DK_RUN_PHILOX)
            SDB_CUDA(ctx, s.rng.ensure(size_t(d.orbits) * nb * 4 * sizeof(uint64_t)));
    }
    sdeb::DslArgs a{};
    a.state_in = d_init;
    a.params = d_params;
    a.state_out = s.state.as<double>();
    a.values = d_values;
    a.fail_step = d_fail;
    a.rng_state = s.rng.as<uint64_t>();
    a.rows = d.orbits;
    a.orbit_offset = d.orbit_offset;
    a.vstride = d.chunks;
    a.ksteps = d.ksteps;
    a.chunk_begin = 0;
    a.chunk_end = d.chunks;
    a.seed = d.seed;
    a.dt = d.dt;
    a.sqrt_dt = std::sqrt(d.dt);
    a.fresh = 1;
    const bool factor = d.coupling == SDB_COUPLING_MEANFIELD;
    if (const size_t words =
            sdeb_dsl::scratch_doubles(m, sdeb_dsl::lanes_for(m, factor), d.orbits)) {
        SDB_CUDA(ctx, s.scratch.ensure(words * sizeof(double)));
        a.scratch = s.scratch.as<double>();
    }
    std::string err;
    // the meanfield setting lets the generated program factor
    // sum(j, sin|cos(A_j - B)); pairwise keeps the literal form
    cudaError_t e = sdeb_dsl::launch(m, kind, a, st, &err, factor);
    if (e != cudaSuccess) return fail_with(ctx, SDB_ERR_CUDA, "%s", err.c_str());
    s.launches += 1;
    s.lanes = sdeb_dsl::lanes_for(m, factor);
    s.persistent = 0;
    s.ctas_per_sm = 0;
    s.tight = 0;
    s.lane_width = 0;
    return SDB_OK;
}

sdb_status launch_device_ordered(sdb_ctx* ctx, Slot& s, const sdb_desc& d, sdb_model* m,
                                 const double* d_init, const double* d_params, double* d_values,
                                 int64_t* d_fail, cudaStream_t st, int out_mode);

// out_mode 0: samples of the state, d_values [orbits][chunks][n]; 1 (Kuramoto
// only): the order parameter, d_values [orbits][2][chunks + 1] (r, Phi planes)
// with sample 0.
sdb_status launch_device(sdb_ctx* ctx, Slot& s, const sdb_desc& d, sdb_model* m,
                         const double* d_init, const double* d_params, double* d_values,
                         int64_t* d_fail, cudaStream_t st, int out_mode = 0) {
    // the slot's scratch (continuation state, stream states, persistent
    // counters, autotune buffers) may still be in use by a launch on another
    // stream: order this one after it
    if (!s.done) SDB_CUDA(ctx, cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    if (s.done_stream != nullptr && s.done_stream != st) SDB_CUDA(ctx, cudaStreamWaitEvent(st, s.done, 0));
    sdb_status rc0 = launch_device_ordered(ctx, s, d, m, d_init, d_params, d_values, d_fail, st,
                                           out_mode);
    if (rc0 != SDB_OK) return rc0;
    SDB_CUDA(ctx, cudaEventRecord(s.done, st));
    s.done_stream = st;
    return SDB_OK;
}

sdb_status launch_device_ordered(sdb_ctx* ctx, Slot& s, const sdb_desc& d, sdb_model* m,
                                 const double* d_init, const double* d_params, double* d_values,
                                 int64_t* d_fail, cudaStream_t st, int out_mode) {
    if (m) {
        if (out_mode != 0)
            return fail_with(ctx, SDB_ERR_UNSUPPORTED,
                             "fused order parameter is implemented for the Kuramoto stepper");
        return launch_model(ctx, s, d, m, d_init, d_params, d_values, d_fail, st);
    }
    Layout lay;
    sdb_status rc = choose_layout(ctx, s, d, d_init, d_params, st, &lay);
    if (rc != SDB_OK) return rc;
    int kind_solver, kind_stream;
    kernel_kind(d, &kind_solver, &kind_stream);
    sdeb::RunArgs a = make_args(d, lay.lanes);
    a.state_in = d_init;
    a.params = d_params;
    a.values = d_values;
    a.fail_step = d_fail;
    rc = configure_layout(ctx, s, s.work, d, lay, d.chunks * d.ksteps, st, &a);
    if (rc != SDB_OK) return rc;
    // continuation state and stream states are only read back by a later slab
    // of a persistent grid: a launch whose groups finish in one pass (one CTA
    // per group, or one slab) writes neither -- 2 GB of HBM writes at cfg3
    // n=256
    a.state_out = nullptr;
    a.rng_state = nullptr;
    if (a.persistent > 0 && a.slab_steps < d.chunks * d.ksteps) {
        SDB_CUDA(ctx, s.state.ensure(size_t(d.orbits) * d.nequat * sizeof(double)));
        const size_t rw = rng_words(d, d.orbits);
        if (rw) SDB_CUDA(ctx, s.rng.ensure(rw * sizeof(uint64_t)));
        a.state_out = s.state.as<double>();
        a.rng_state = s.rng.as<uint64_t>();
    }
    const int J = layout_J(d, lay);
    int variant = kernel_variant(d, lay.lanes, J, out_mode ? 0 : lay.tight);
    if (out_mode) {
        variant += sdeb::kVarCoherence;  // same layout, order-parameter samples
        a.vstride = d.chunks + 1;
    }
    cudaError_t e = launch_run(a, J, kind_solver, kind_stream, d.coupling, variant, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "kuramoto_run_kernel launch");
    s.launches += 1;
    s.lanes = lay.lanes;
    s.persistent = lay.persistent;
    s.ctas_per_sm = lay.ctas_per_sm;
    s.tight = lay.tight;
    s.lane_width = J;
    return SDB_OK;
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return (e && *e) ? std::atoi(e) : dflt;
}

// Persistent host workers for the pipeline's copies (spawning a std::thread
// per piece cost ~50 us each, ~0.8 ms per 16-way copy).  Jobs are ranges of
// one parallel_rows call; the caller runs a share itself and waits.
class CopyPool {
  public:
    static CopyPool& get() {
        static CopyPool pool;
        return pool;
    }
    // run fn(t) for t in [1, n) on the workers and fn(0) here; returns when all done
    template <class F>
    void run(int n, F& fn) {
        // one job at a time: shard threads of a multi-device run take turns
        std::lock_guard<std::mutex> serial(run_mu_);
        std::unique_lock<std::mutex> lock(mu_);
        while (workers_.size() < size_t(n - 1)) workers_.emplace_back([this] { loop(); });
        job_ = [&fn](int t) { fn(t); };
        pending_ = n - 1;
        next_ = 1;
        total_ = n;
        ++generation_;
        lock.unlock();
        cv_.notify_all();
        fn(0);
        lock.lock();
        done_cv_.wait(lock, [this] { return pending_ == 0; });
        job_ = nullptr;
    }

  private:
    CopyPool() = default;
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lock(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lock(mu_);
            cv_.wait(lock, [&] { return stop_ || (generation_ != seen && next_ < total_); });
            if (stop_) return;
            const int t = next_++;
            if (next_ >= total_) seen = generation_;
            auto job = job_;
            lock.unlock();
            job(t);
            lock.lock();
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    std::mutex run_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<std::thread> workers_;
    std::function<void(int)> job_;
    int pending_ = 0, next_ = 0, total_ = 0;
    uint64_t generation_ = 0;
    bool stop_ = false;
};

// Host copy of rows [0, rows) split over up to `threads` workers (the calling
// thread takes the first range).  Pageable numpy destinations fault their
// pages in on first touch; spreading the copy spreads the faults too.  Each
// range ends with a store fence, so streaming stores (copy_bytes) are
// globally visible before the pool reports the job done.
template <class F>
void parallel_rows(int64_t rows, size_t bytes, int threads, F&& fn) {
    const int64_t want = std::min<int64_t>(threads, int64_t(bytes >> 18));  // >= 256 KiB each
    const int nt = int(std::max<int64_t>(1, std::min<int64_t>(want, rows)));
    auto part = [&](int t) {
        fn(rows * t / nt, rows * (t + 1) / nt);
#if defined(__SSE2__)
        _mm_sfence();
#endif
    };
    if (nt == 1) {
        part(0);
        return;
    }
    CopyPool::get().run(nt, part);
}

// Bulk host copy for the staging legs.  `stream` = non-temporal stores: the
// GB-sized legs are not re-read by the copying thread, so skipping the
// destination's read-for-ownership and cache fill raises the copy rate
// (B200 host, 16 threads: 72 -> 80 GB/s into touched pages, 19 -> 28 GB/s
// into fresh 4 KiB pages; tools/host_copy_bench.cpp).  Small runs keep plain
// memcpy so their outputs stay cache-resident for the caller.
inline void copy_bytes(void* dst, const void* src, size_t bytes, bool stream) {
#if defined(__SSE2__)
    if (stream && bytes >= 256) {
        char* d = static_cast<char*>(dst);
        const char* s = static_cast<const char*>(src);
        const size_t head = (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15;
        std::memcpy(d, s, head);
        d += head;
        s += head;
        bytes -= head;
        size_t i = 0;
        for (; i + 64 <= bytes; i += 64) {
            const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
            const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
            const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
            const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
            _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
            _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
            _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
            _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
        }
        std::memcpy(d + i, s + i, bytes - i);
        return;
    }
#endif
    (void)stream;
    std::memcpy(dst, src, bytes);
}

// transfers at least this large (per shard and direction) use streaming stores
constexpr size_t kStreamCopyBytes = size_t(64) << 20;

// Fault in the pages of [lo, hi) of a caller's store without changing their
// contents (MADV_POPULATE_WRITE, Linux 5.14+), else by writing one byte per
// page inside the range -- only ever called on rows no drain has written yet.
// A fresh store's first-touch faults are the drain's dominant cost (the
// pinned -> fresh copy runs at 19-38 GB/s, into touched pages at 80 GB/s);
// doing them while the host would otherwise block on a kernel or a DMA takes
// them off the critical path.
void prefault_range(char* lo, char* hi) {
    if (hi <= lo) return;
    constexpr uintptr_t kPage = 4096;
#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif
    static std::atomic<bool> no_madvise{false};
    const uintptr_t a = (reinterpret_cast<uintptr_t>(lo) + kPage - 1) & ~(kPage - 1);
    const uintptr_t b = reinterpret_cast<uintptr_t>(hi) & ~(kPage - 1);
    if (b > a && !no_madvise.load(std::memory_order_relaxed)) {
        if (::madvise(reinterpret_cast<void*>(a), b - a, MADV_POPULATE_WRITE) == 0) return;
        if (errno == EINVAL) no_madvise.store(true, std::memory_order_relaxed);
    }
    for (char* q = lo; q < hi;) {
        *reinterpret_cast<volatile char*>(q) = 0;
        q = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(q) & ~(kPage - 1)) + kPage);
    }
}

int host_copy_threads(int /*shards*/) {
    const int hw = int(std::max(1u, std::thread::hardware_concurrency()));
    // every hardware thread, whatever the shard count: the copies are bound by
    // page faults / memory traffic (cfg3 n=256 e2e 393 -> 303 ms going from 8 to
    // 16 threads on a 16-thread host), and the pool runs one piece at a time.
    // One process per GPU (torchrun sets LOCAL_WORLD_SIZE): a share each.
    const int procs = std::max(1, env_int("LOCAL_WORLD_SIZE", 1));
    return std::max(1, env_int("SDEB200_HOST_THREADS", std::min(32, std::max(1, hw / procs))));
}

// True when [p, p + bytes) lies in page-locked memory the driver knows
// (cudaHostAlloc / cudaHostRegister): the DMA engines can read it directly.
bool is_pinned_range(const void* p, size_t bytes) {
    if (!p || bytes == 0) return false;
    const char* lo = static_cast<const char*>(p);
    for (const char* q : {lo, lo + bytes - 1}) {
        cudaPointerAttributes attr{};
        if (cudaPointerGetAttributes(&attr, q) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (attr.type != cudaMemoryTypeHost) return false;
    }
    return true;
}

// Orbit tiles of a host-buffer shard: copies of tile t+1 / t-1 overlap the
// kernel of tile t.  A tile must keep the kernel well fed (>= ~8 waves of
// resident threads at a typical lanes-per-orbit, 2 for transfer-heavy runs)
// and be worth a pipeline stage (>= 32 MB of transfers); at most 8.
// SDEB200_TILES overrides.
int64_t shard_tiles(const sdb_desc& d, int64_t rows, int device) {
    const int forced = env_int("SDEB200_TILES", 0);
    if (forced > 0) return std::min<int64_t>(forced, rows);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int64_t lanes_est = std::min(32, std::max(1, next_pow2(d.nequat) / 4));
    const double io = double(rows) * double(d.nequat + d.nparams + d.chunks * d.nequat) * 8.0;
    // transfer-heavy runs (>= 1 GB moved) accept tiles of >= 2 waves: hiding the
    // kernel under the transfers pays more than a short tile's tail (cfg5
    // e2e 95 -> 86-90 ms at 4 tiles); otherwise >= 8 waves per tile
    const int64_t waves = io >= 1e9 ? 2 : 8;
    const int64_t min_rows = waves * sms * 768 / lanes_est;
    int64_t t = std::min<int64_t>(rows / std::max<int64_t>(1, min_rows), int64_t(io / 32e6));
    return std::max<int64_t>(1, std::min<int64_t>(8, t));
}

// One device's contiguous shard [r0, r0+rows) of a host-buffer run, as a
// pipeline over orbit tiles and transfer pieces (<= SDEB200_PIECE_KB, 64 MiB):
//   inputs  host rows -> pinned slot (parallel memcpy) -> DMA on s.h2d
//   kernel  tile t on s.stream after its inputs landed
//   outputs DMA on s.d2h after the tile's kernel -> pinned slot -> host rows,
//           written as [init row | samples 1..k] (engine.py:213-214)
// Pinned slots alternate (kPinSlots each way); a slot is refilled only after
// the DMA that last used it completed.  Input staging of tile t+1 is issued
// before the outputs of tile t are drained, so host copies, both DMA
// directions and the kernels overlap.  Results are identical for any tiling:
// noise is keyed by global orbit id and orbits are independent.
// pwrite the whole buffer (retrying short writes); false on error.
bool pwrite_all(int fd, const void* buf, size_t bytes, int64_t offset) {
    const char* p = static_cast<const char*>(buf);
    while (bytes > 0) {
        const ssize_t w = ::pwrite(fd, p, bytes, off_t(offset));
        if (w < 0) {
            if (errno == EINTR) continue;
            return false;
        }
        p += w;
        bytes -= size_t(w);
        offset += w;
    }
    return true;
}

// Where a host-buffer run's store goes: the caller's (M, k+1, n) array, or
// (fd >= 0) an SDB1 file whose value section starts at byte `offset`.
struct OutSink {
    double* values = nullptr;
    int fd = -1;
    int64_t offset = 0;
};

sdb_status run_shard(sdb_ctx* ctx, Slot& s, sdb_desc d, sdb_model* m, int64_t r0, int64_t rows,
                     const double* init, const double* params, const OutSink& sink, int64_t* fail,
                     int shards, int out_mode) {
    double* values = sink.values;
    std::atomic<int> write_errno{0};
    SDB_CUDA(ctx, cudaSetDevice(s.device));
    const bool tr = trace_enabled();
    const double t0 = tr ? now_ms() : 0.0;
    const int n = d.nequat;
    const int64_t np_ = d.nparams;
    const int64_t k = d.chunks;
    const int threads = host_copy_threads(shards);
    d.orbit_offset += r0;
    d.orbits = rows;
    const double ta = tr ? now_ms() : 0.0;
    SDB_CUDA(ctx, s.init.ensure(size_t(rows) * n * sizeof(double)));
    SDB_CUDA(ctx, s.params.ensure(size_t(rows) * np_ * sizeof(double)));
    // device words per row: samples 1..k of the state, or (r, Phi) of samples 0..k
    const int64_t width = out_mode ? (k + 1) * 2 : k * n;
    SDB_CUDA(ctx, s.values.ensure(size_t(rows) * width * sizeof(double)));
    SDB_CUDA(ctx, s.fail.ensure(size_t(rows) * sizeof(int64_t)));
    if (!s.ev_in) SDB_CUDA(ctx, cudaEventCreateWithFlags(&s.ev_in, cudaEventDisableTiming));
    const double alloc_ms = tr ? now_ms() - ta : 0.0;
    double pin_ms = 0.0, launch_ms = 0.0;  // pinned-slot growth, launch_device (incl. autotune)

    const int64_t tiles = shard_tiles(d, rows, s.device);
    const size_t piece_cap = size_t(std::max(1, env_int("SDEB200_PIECE_KB", 65536))) << 10;
    const size_t in_row = size_t(n + np_) * sizeof(double);
    const size_t out_row = size_t(width + 1) * sizeof(double);  // samples + fail word
    // pinned input staging is only ever read by the DMA engine: streaming stores
    // always (SDEB200_NT_IN=0 restores the size threshold, for A/B runs)
    const bool nt_in = env_int("SDEB200_NT_IN", 1) != 0 || size_t(rows) * in_row >= kStreamCopyBytes;
    const bool nt_out = size_t(rows) * out_row >= kStreamCopyBytes;
    // pieces of ~1/8 of a tile (4 MiB .. piece_cap): even a one-tile run then
    // overlaps each piece's host copy with the neighbouring piece's DMA
    const size_t piece_div = size_t(std::max(1, env_int("SDEB200_PIECE_DIV", 8)));
    auto piece_rows = [&](size_t row_bytes) {
        const size_t tile_bytes = size_t((rows + tiles - 1) / tiles) * row_bytes;
        const size_t want =
            std::min(piece_cap, std::max(size_t(4) << 20, tile_bytes / piece_div));
        return std::max<int64_t>(1, int64_t(want / row_bytes));
    };
    const int64_t in_piece = piece_rows(in_row);
    const int64_t out_piece = piece_rows(out_row);
    double* d_init = s.init.as<double>();
    double* d_params = s.params.as<double>();
    double* d_values = s.values.as<double>();
    int64_t* d_fail = s.fail.as<int64_t>();
    int in_next = 0, out_next = 0;
    double host_in_ms = 0.0, host_out_ms = 0.0, wait_ms = 0.0;

    struct Pending {
        int slot;
        int64_t a, rows;  // shard-local rows
    };
    std::vector<Pending> pending;  // FIFO of issued output pieces
    size_t head = 0;

    // Destination prefault (see prefault_range): while the next piece's DMA
    // (or the kernel before it) is still running, fault in the store pages of
    // rows no drain has reached yet, 32 MiB at a time (stores >= 4 MiB), and
    // write their sample 0 (the initial state, host data).
    // SDEB200_PREFAULT=0 turns it off.
    const int64_t row_words = out_mode ? width : (k + 1) * n;
    const size_t store_bytes = size_t(rows) * size_t(row_words) * sizeof(double);
    const bool prefault =
        values && store_bytes >= (size_t(4) << 20) && env_int("SDEB200_PREFAULT", 1) != 0;
    const int64_t pf_rows = std::max<int64_t>(1, int64_t((size_t(32) << 20) / (row_words * 8)));
    int64_t pf_next = 0;  // shard-local rows below this are populated (or drained)
    int64_t init_next = 0;  // shard-local rows below this have sample 0 written
    double prefault_ms = 0.0;

    auto drain_one = [&]() -> sdb_status {
        const Pending p = pending[head++];
        PinBuf& pb = s.pin_out[p.slot];
        if (prefault) {
            const double f0 = now_ms();
            pf_next = std::max(pf_next, p.a);  // rows below p.a are drained already
            while (pf_next < rows && cudaEventQuery(pb.ev) == cudaErrorNotReady) {
                const int64_t a = pf_next, b = std::min(rows, a + pf_rows);
                char* base = reinterpret_cast<char*>(values + (r0 + a) * row_words);
                const size_t span = size_t(b - a) * size_t(row_words) * sizeof(double);
                parallel_rows(int64_t(threads), span, threads, [&](int64_t x, int64_t y) {
                    prefault_range(base + span * size_t(x) / size_t(threads),
                                   base + span * size_t(y) / size_t(threads));
                });
                if (!out_mode) {  // sample 0 (the initial state) needs no device data
                    parallel_rows(b - a, size_t(b - a) * n * sizeof(double), threads,
                                  [&](int64_t x, int64_t y) {
                        for (int64_t r = a + x; r < a + y; ++r)
                            copy_bytes(values + (r0 + r) * row_words, init + (r0 + r) * n,
                                       size_t(n) * sizeof(double), nt_out);
                    });
                    init_next = b;
                }
                pf_next = b;
            }
            prefault_ms += now_ms() - f0;
        }
        const double w0 = now_ms();
        SDB_CUDA(ctx, cudaEventSynchronize(pb.ev));
        const double w1 = now_ms();
        const double* src = pb.as<double>();
        const int64_t* fsrc = reinterpret_cast<const int64_t*>(src + p.rows * width);
        parallel_rows(p.rows, size_t(p.rows) * out_row, threads, [&](int64_t a, int64_t b) {
            if (sink.fd >= 0) {  // rows [a, b) of the piece are contiguous in the file
                const size_t row_words = size_t(k + 1) * n;
                std::vector<double> buf(size_t(b - a) * row_words);
                for (int64_t r = a; r < b; ++r) {
                    double* dst = buf.data() + size_t(r - a) * row_words;
                    std::memcpy(dst, init + (r0 + p.a + r) * n, size_t(n) * sizeof(double));
                    std::memcpy(dst + n, src + r * k * n, size_t(k) * n * sizeof(double));
                }
                const int64_t at = sink.offset + (r0 + p.a + a) * int64_t(row_words * sizeof(double));
                if (!pwrite_all(sink.fd, buf.data(), buf.size() * sizeof(double), at))
                    write_errno.store(errno ? errno : EIO);
                return;
            }
            for (int64_t r = a; r < b; ++r) {
                const int64_t g = r0 + p.a + r;
                if (out_mode) {
                    copy_bytes(values + g * width, src + r * width, size_t(width) * sizeof(double),
                               nt_out);
                    continue;
                }
                double* dst = values + g * (k + 1) * n;
                if (p.a + r >= init_next)  // else written while the host waited
                    copy_bytes(dst, init + g * n, size_t(n) * sizeof(double), nt_out);
                copy_bytes(dst + n, src + r * k * n, size_t(k) * n * sizeof(double), nt_out);
            }
        });
        std::memcpy(fail + r0 + p.a, fsrc, size_t(p.rows) * sizeof(int64_t));
        wait_ms += w1 - w0;
        host_out_ms += now_ms() - w1;
        return SDB_OK;
    };

    // inputs in page-locked memory (sdb_host_alloc): one DMA per tile straight
    // from the caller's rows, no host copy
    const bool pinned_in = is_pinned_range(init + r0 * n, size_t(rows) * n * sizeof(double)) &&
                           is_pinned_range(params + r0 * np_, size_t(rows) * np_ * sizeof(double));
    auto stage_inputs = [&](int64_t a, int64_t b) -> sdb_status {
        if (pinned_in) {
            SDB_CUDA(ctx, cudaMemcpyAsync(d_init + a * n, init + (r0 + a) * n,
                                          size_t(b - a) * n * sizeof(double),
                                          cudaMemcpyHostToDevice, s.h2d));
            SDB_CUDA(ctx, cudaMemcpyAsync(d_params + a * np_, params + (r0 + a) * np_,
                                          size_t(b - a) * np_ * sizeof(double),
                                          cudaMemcpyHostToDevice, s.h2d));
            return SDB_OK;
        }
        for (int64_t p0 = a; p0 < b; p0 += in_piece) {
            const int64_t pr = std::min(in_piece, b - p0);
            PinBuf& pb = s.pin_in[in_next];
            in_next = (in_next + 1) % kPinSlots;
            const double p0t = tr ? now_ms() : 0.0;
            SDB_CUDA(ctx, pb.ensure(size_t(pr) * in_row));
            if (tr) pin_ms += now_ms() - p0t;
            const double w0 = now_ms();
            SDB_CUDA(ctx, cudaEventSynchronize(pb.ev));  // the slot's previous DMA is done
            const double w1 = now_ms();
            double* pin_init = pb.as<double>();
            double* pin_par = pin_init + pr * n;
            const double* h_init = init + (r0 + p0) * n;
            const double* h_par = params + (r0 + p0) * np_;
            parallel_rows(pr, size_t(pr) * in_row, threads, [&](int64_t x, int64_t y) {
                copy_bytes(pin_init + x * n, h_init + x * n, size_t(y - x) * n * sizeof(double), nt_in);
                copy_bytes(pin_par + x * np_, h_par + x * np_, size_t(y - x) * np_ * sizeof(double),
                           nt_in);
            });
            wait_ms += w1 - w0;
            host_in_ms += now_ms() - w1;
            SDB_CUDA(ctx, cudaMemcpyAsync(d_init + p0 * n, pin_init, size_t(pr) * n * sizeof(double),
                                          cudaMemcpyHostToDevice, s.h2d));
            SDB_CUDA(ctx, cudaMemcpyAsync(d_params + p0 * np_, pin_par,
                                          size_t(pr) * np_ * sizeof(double),
                                          cudaMemcpyHostToDevice, s.h2d));
            SDB_CUDA(ctx, cudaEventRecord(pb.ev, s.h2d));
        }
        return SDB_OK;
    };

    while (s.ev_tile.size() < size_t(tiles)) {
        cudaEvent_t e;
        SDB_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        s.ev_tile.push_back(e);
    }

    auto launch_tile = [&](int64_t t, int64_t a, int64_t b) -> sdb_status {
        SDB_CUDA(ctx, cudaEventRecord(s.ev_in, s.h2d));
        SDB_CUDA(ctx, cudaStreamWaitEvent(s.stream, s.ev_in, 0));
        sdb_desc td = d;
        td.orbit_offset = d.orbit_offset + a;
        td.orbits = b - a;
        const double l0 = tr ? now_ms() : 0.0;
        sdb_status rc = launch_device(ctx, s, td, m, d_init + a * n, d_params + a * np_,
                                      d_values + a * width, d_fail + a, s.stream, out_mode);
        if (tr) launch_ms += now_ms() - l0;
        if (rc != SDB_OK) return rc;
        SDB_CUDA(ctx, cudaEventRecord(s.ev_tile[t], s.stream));
        return SDB_OK;
    };

    auto issue_outputs = [&](int64_t t, int64_t a, int64_t b) -> sdb_status {
        SDB_CUDA(ctx, cudaStreamWaitEvent(s.d2h, s.ev_tile[t], 0));
        for (int64_t p0 = a; p0 < b; p0 += out_piece) {
            const int64_t pr = std::min(out_piece, b - p0);
            // a slot is free once the piece that used it has been drained
            while (pending.size() - head >= size_t(kPinSlots)) {
                sdb_status rc = drain_one();
                if (rc != SDB_OK) return rc;
            }
            const int slot = out_next;
            out_next = (out_next + 1) % kPinSlots;
            PinBuf& pb = s.pin_out[slot];
            const double p0t = tr ? now_ms() : 0.0;
            SDB_CUDA(ctx, pb.ensure(size_t(pr) * out_row));
            if (tr) pin_ms += now_ms() - p0t;
            double* dst = pb.as<double>();
            SDB_CUDA(ctx, cudaMemcpyAsync(dst, d_values + p0 * width,
                                          size_t(pr) * width * sizeof(double),
                                          cudaMemcpyDeviceToHost, s.d2h));
            SDB_CUDA(ctx, cudaMemcpyAsync(dst + pr * width, d_fail + p0,
                                          size_t(pr) * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                          s.d2h));
            SDB_CUDA(ctx, cudaEventRecord(pb.ev, s.d2h));
            pending.push_back(Pending{slot, p0, pr});
        }
        return SDB_OK;
    };

    auto lo = [&](int64_t t) { return rows * t / tiles; };
    sdb_status rc = stage_inputs(lo(0), lo(1));
    if (rc == SDB_OK) rc = launch_tile(0, lo(0), lo(1));
    for (int64_t t = 0; t < tiles && rc == SDB_OK; ++t) {
        if (t + 1 < tiles) {  // queue tile t+1 before draining tile t
            rc = stage_inputs(lo(t + 1), lo(t + 2));
            if (rc == SDB_OK) rc = launch_tile(t + 1, lo(t + 1), lo(t + 2));
        }
        if (rc == SDB_OK) rc = issue_outputs(t, lo(t), lo(t + 1));
    }
    while (rc == SDB_OK && head < pending.size()) rc = drain_one();
    if (rc == SDB_OK && write_errno.load() != 0)
        rc = fail_with(ctx, SDB_ERR_CUDA, "writing the store file failed: %s",
                       std::strerror(write_errno.load()));
    if (rc != SDB_OK) {
        cudaStreamSynchronize(s.h2d);  // leave no DMA in flight into pinned slots
        cudaStreamSynchronize(s.stream);
        cudaStreamSynchronize(s.d2h);
        return rc;
    }
    s.tiles = int32_t(tiles);
    if (tr) {
        std::fprintf(stderr,
                     "[sdeb200] dev %d rows %lld tiles %lld: total %.3f ms, host-in %.3f ms, "
                     "host-out %.3f ms, waits %.3f ms, prefault %.3f ms, device alloc %.3f ms, "
                     "pinned alloc %.3f ms, launch calls %.3f ms, tune %.3f ms (%.1f MB in, "
                     "%.1f MB out)\n",
                     s.device, (long long)rows, (long long)tiles, now_ms() - t0, host_in_ms,
                     host_out_ms, wait_ms, prefault_ms, alloc_ms, pin_ms, launch_ms,
                     s.tune_us * 1e-3, double(rows) * in_row / 1e6, double(rows) * out_row / 1e6);
    }
    return rc;
}

// Scoped device buffer for the context-free utility entry points.
struct TmpBuf {
    void* p = nullptr;
    ~TmpBuf() {
        if (p) cudaFree(p);
    }
};

sdb_status utility_prologue(sdb_ctx* ctx) {
    if (!ctx || ctx->slots.empty()) return fail_with(ctx, SDB_ERR_ARGUMENT, "null context");
    SDB_CUDA(ctx, cudaSetDevice(ctx->slots[0].device));
    return SDB_OK;
}


sdb_status validate_model(sdb_ctx* ctx, const sdb_desc* d, const sdb_model* m) {
    if (!d) return fail_with(ctx, SDB_ERR_ARGUMENT, "null descriptor");
    if (!m) return fail_with(ctx, SDB_ERR_ARGUMENT, "null model");
    if (d->model != SDB_MODEL_EXPRESSION)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "descriptor model must be SDB_MODEL_EXPRESSION");
    if (d->nequat != m->nequat || d->nparams != m->nparams || d->nnoise != m->nnoise)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "descriptor dimensions (%d, %d, %d) do not match "
                         "the model (%d, %d, %d)", d->nequat, d->nparams, d->nnoise, m->nequat,
                         m->nparams, m->nnoise);
    if (d->solver != SDB_SOLVER_EM && d->solver != SDB_SOLVER_EULER && d->solver != SDB_SOLVER_RK4)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "unknown solver %d", d->solver);
    if (d->solver != SDB_SOLVER_EM && d->nnoise > 0)
        return fail_with(ctx, SDB_ERR_CONFIG,
                         "solver is deterministic but the model has %d noise terms", d->nnoise);
    if (d->stream < SDB_STREAM_PHILOX || d->stream > SDB_STREAM_XOSHIRO256PP)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "unknown stream %d", d->stream);
    if (!(d->dt > 0.0)) return fail_with(ctx, SDB_ERR_CONFIG, "dt must be positive");
    if (d->ksteps < 1) return fail_with(ctx, SDB_ERR_CONFIG, "ksteps must be >= 1");
    if (d->chunks < 1) return fail_with(ctx, SDB_ERR_CONFIG, "chunks must be >= 1");
    if (d->orbits < 1) return fail_with(ctx, SDB_ERR_CONFIG, "orbits must be >= 1");
    if (d->orbit_offset < 0 || d->orbit_offset + d->orbits > (int64_t(1) << 32))
        return fail_with(ctx, SDB_ERR_CONFIG, "global orbit ids must fit in 32 bits");
    if (d->chunks > INT64_MAX / d->ksteps)
        return fail_with(ctx, SDB_ERR_CONFIG, "total step count does not fit in 63 bits");
    return SDB_OK;
}

// Host-buffer run over all of the context's devices (validated descriptor).
sdb_status run_host(sdb_ctx* ctx, const sdb_desc& d, sdb_model* m, const double* init,
                    const double* params, double* values, int64_t* fail_step, int out_mode = 0,
                    int fd = -1, int64_t file_offset = 0) {
    if (!init || !params || (!values && fd < 0) || !fail_step)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "null host buffer");
    OutSink sink;
    sink.values = values;
    sink.fd = fd;
    sink.offset = file_offset;
    const int64_t nslots = int64_t(ctx->slots.size());
    const int64_t used = std::min<int64_t>(nslots, d.orbits);
    std::vector<sdb_status> status(used, SDB_OK);
    std::vector<std::thread> threads;
    for (Slot& s : ctx->slots) {
        s.launches = 0;
        s.tune_us = 0;
        s.error.clear();
    }
    // contiguous shards [g*M/G, (g+1)*M/G)
    auto shard = [&](int64_t g) {
        const int64_t r0 = g * d.orbits / used, r1 = (g + 1) * d.orbits / used;
        status[g] = run_shard(ctx, ctx->slots[g], d, m, r0, r1 - r0, init, params, sink,
                              fail_step, int(used), out_mode);
    };
    if (used == 1) {
        shard(0);
    } else {
        for (int64_t g = 0; g < used; ++g) threads.emplace_back(shard, g);
        for (auto& t : threads) t.join();
    }
    ctx->launches = 0;
    ctx->last_tune_us = 0;
    for (int64_t g = 0; g < used; ++g) {
        ctx->launches += ctx->slots[g].launches;
        ctx->last_tune_us = std::max(ctx->last_tune_us, ctx->slots[g].tune_us);
    }
    ctx->last_lanes = ctx->slots[0].lanes;
    ctx->last_persistent = ctx->slots[0].persistent;
    ctx->last_ctas_per_sm = ctx->slots[0].ctas_per_sm;
    ctx->last_tight = ctx->slots[0].tight;
    ctx->last_lane_width = ctx->slots[0].lane_width;
    ctx->last_tiles = ctx->slots[0].tiles;
    for (int64_t g = 0; g < used; ++g) {
        if (status[g] != SDB_OK) {
            // a shard thread recorded the message: make it this thread's too
            std::lock_guard<std::mutex> lock(ctx->mu);
            g_thread_error = ctx->error;
            return status[g];
        }
    }
    return SDB_OK;
}

// Device-buffer run on the first device (validated descriptor).
sdb_status run_dev(sdb_ctx* ctx, const sdb_desc& d, sdb_model* m, const double* d_init,
                   const double* d_params, double* d_values, int64_t* d_fail_step, void* stream,
                   int out_mode = 0) {
    if (!d_init || !d_params || !d_values || !d_fail_step)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "null device buffer");
    Slot& s = ctx->slots[0];
    SDB_CUDA(ctx, cudaSetDevice(s.device));
    s.launches = 0;
    s.tune_us = 0;
    sdb_status rc = launch_device(ctx, s, d, m, d_init, d_params, d_values, d_fail_step,
                                  static_cast<cudaStream_t>(stream), out_mode);
    ctx->launches = s.launches;
    ctx->last_tune_us = s.tune_us;
    ctx->last_lanes = s.lanes;
    ctx->last_persistent = s.persistent;
    ctx->last_ctas_per_sm = s.ctas_per_sm;
    ctx->last_tight = s.tight;
    ctx->last_lane_width = s.lane_width;
    ctx->last_tiles = 0;
    return rc;
}

// Row-wise program (eval / one step) over host arrays: y [count][N], p
// [count][NP], noise [count][NN] or null, out [count][N].
sdb_status model_rows(sdb_ctx* ctx, sdb_model* m, int kind, double t, double dt, int64_t count,
                      const double* y, const double* p, const double* noise, double* out) {
    sdb_status rc = utility_prologue(ctx);
    if (rc != SDB_OK) return rc;
    if (count < 0 || !y || !p || !out) return fail_with(ctx, SDB_ERR_ARGUMENT, "bad row arrays");
    if (count == 0) return SDB_OK;
    const size_t n = size_t(m->nequat), np_ = size_t(m->nparams), nn = size_t(m->nnoise);
    TmpBuf dy, dp, dn, dout;
    SDB_CUDA(ctx, cudaMalloc(&dy.p, count * n * sizeof(double)));
    SDB_CUDA(ctx, cudaMalloc(&dp.p, count * std::max<size_t>(np_, 1) * sizeof(double)));
    SDB_CUDA(ctx, cudaMalloc(&dout.p, count * n * sizeof(double)));
    SDB_CUDA(ctx, cudaMemcpy(dy.p, y, count * n * sizeof(double), cudaMemcpyHostToDevice));
    if (np_) SDB_CUDA(ctx, cudaMemcpy(dp.p, p, count * np_ * sizeof(double), cudaMemcpyHostToDevice));
    if (noise && nn) {
        SDB_CUDA(ctx, cudaMalloc(&dn.p, count * nn * sizeof(double)));
        SDB_CUDA(ctx, cudaMemcpy(dn.p, noise, count * nn * sizeof(double), cudaMemcpyHostToDevice));
    }
    sdeb::DslArgs a{};
    a.state_in = static_cast<const double*>(dy.p);
    a.params = static_cast<const double*>(dp.p);
    a.noise = static_cast<const double*>(dn.p);
    a.state_out = static_cast<double*>(dout.p);
    a.values = static_cast<double*>(dout.p);
    a.rows = count;
    a.t = t;
    a.dt = dt;
    a.sqrt_dt = dt > 0.0 ? std::sqrt(dt) : 0.0;
    TmpBuf scratch;
    if (const size_t words = sdeb_dsl::scratch_doubles(m, sdeb_dsl::lanes_for(m, false), count)) {
        SDB_CUDA(ctx, cudaMalloc(&scratch.p, words * sizeof(double)));
        a.scratch = static_cast<double*>(scratch.p);
    }
    std::string err;
    cudaError_t e = sdeb_dsl::launch(m, kind, a, nullptr, &err);
    if (e != cudaSuccess) return fail_with(ctx, SDB_ERR_CUDA, "%s", err.c_str());
    SDB_CUDA(ctx, cudaMemcpy(out, dout.p, count * n * sizeof(double), cudaMemcpyDeviceToHost));
    ctx->launches = 1;
    return SDB_OK;
}

}  // namespace

extern "C" {

int sdb_abi_version(void) { return SDB_ABI_VERSION; }

int sdb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

sdb_status sdb_open(const int* devices, int ndevices, sdb_ctx** out) {
    if (!out) return fail_with(nullptr, SDB_ERR_ARGUMENT, "null output pointer");
    *out = nullptr;
    int count = sdb_device_count();
    if (count < 1) return fail_with(nullptr, SDB_ERR_CUDA, "no CUDA device is visible");
    std::vector<int> devs;
    if (devices == nullptr || ndevices <= 0) {
        devs.push_back(0);
    } else {
        devs.assign(devices, devices + ndevices);
    }
    auto* ctx = new sdb_ctx();
    for (int dev : devs) {
        if (dev < 0 || dev >= count) {
            delete ctx;
            return fail_with(nullptr, SDB_ERR_ARGUMENT, "device %d out of range (%d visible)", dev,
                             count);
        }
        Slot s;
        s.device = dev;
        cudaError_t e = cudaSetDevice(dev);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s.h2d, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s.d2h, cudaStreamNonBlocking);
        // the process's first page-locked allocation carries a fixed setup
        // cost (tens of ms on the B200 host): pay it with the context, one
        // small block; the staging slots are sized by the first run that uses
        // them (growing a slot later frees the old block, which synchronises)
        if (e == cudaSuccess && env_int("SDEB200_PIN_WARM", 1) != 0)
            e = s.pin_warm.ensure(1);
        if (e != cudaSuccess) {
            s.pin_warm.release();
            sdb_close(ctx);
            return cuda_fail(nullptr, e, "sdb_open");
        }
        ctx->slots.push_back(s);
    }
    *out = ctx;
    return SDB_OK;
}

void sdb_close(sdb_ctx* ctx) {
    if (!ctx) return;
    for (Slot& s : ctx->slots) {
        cudaSetDevice(s.device);
        for (DevBuf* b : {&s.init, &s.params, &s.values, &s.state, &s.fail, &s.rng, &s.work, &s.scratch,
                          &s.t_values, &s.t_state, &s.t_fail, &s.t_rng, &s.t_work})
            b->release();
        for (PinBuf* b : {&s.pin_in[0], &s.pin_in[1], &s.pin_out[0], &s.pin_out[1], &s.pin_warm})
            b->release();
        if (s.ev_in) cudaEventDestroy(s.ev_in);
        if (s.done) cudaEventDestroy(s.done);
        for (cudaEvent_t e : s.ev_tile) cudaEventDestroy(e);
        for (cudaStream_t st : {s.stream, s.h2d, s.d2h})
            if (st) cudaStreamDestroy(st);
    }
    delete ctx;
}

// The calling thread's last error (every failing call records it there, also
// when a shard thread failed); the context's as a fallback.
const char* sdb_last_error(const sdb_ctx* ctx) {
    if (!g_thread_error.empty() || !ctx) return g_thread_error.c_str();
    return ctx->error.c_str();
}

int64_t sdb_last_launch_count(const sdb_ctx* ctx) { return ctx ? ctx->launches : 0; }
int32_t sdb_last_lanes(const sdb_ctx* ctx) { return ctx ? ctx->last_lanes : 0; }

int32_t sdb_last_lane_width(const sdb_ctx* ctx) { return ctx ? ctx->last_lane_width : 0; }

int64_t sdb_last_tune_us(const sdb_ctx* ctx) { return ctx ? ctx->last_tune_us : 0; }

sdb_status sdb_host_alloc(int64_t bytes, void** out) {
    if (!out || bytes < 0) return fail_with(nullptr, SDB_ERR_ARGUMENT, "bad host allocation");
    *out = nullptr;
    cudaError_t e = cudaHostAlloc(out, size_t(std::max<int64_t>(bytes, 1)), cudaHostAllocPortable);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaHostAlloc");
    return SDB_OK;
}

void sdb_host_free(void* ptr) {
    if (ptr) cudaFreeHost(ptr);
}

void sdb_last_layout(const sdb_ctx* ctx, int32_t* lanes, int32_t* persistent,
                     int32_t* ctas_per_sm, int32_t* variant, int32_t* tiles) {
    if (variant) *variant = ctx ? ctx->last_tight : 0;
    if (tiles) *tiles = ctx ? ctx->last_tiles : 0;
    if (lanes) *lanes = ctx ? ctx->last_lanes : 0;
    if (persistent) *persistent = ctx ? ctx->last_persistent : 0;
    if (ctas_per_sm) *ctas_per_sm = ctx ? ctx->last_ctas_per_sm : 0;
}

sdb_status sdb_run(sdb_ctx* ctx, const sdb_desc* desc, const double* init, const double* params,
                   double* values, int64_t* fail_step) {
    SDB_ENTRY(ctx);
    sdb_status rc = validate(ctx, desc);
    if (rc != SDB_OK) return rc;
    return run_host(ctx, *desc, nullptr, init, params, values, fail_step);
}

sdb_status sdb_run_device(sdb_ctx* ctx, const sdb_desc* desc, const double* d_init,
                          const double* d_params, double* d_values, int64_t* d_fail_step,
                          void* stream) {
    SDB_ENTRY(ctx);
    sdb_status rc = validate(ctx, desc);
    if (rc != SDB_OK) return rc;
    return run_dev(ctx, *desc, nullptr, d_init, d_params, d_values, d_fail_step, stream);
}

/* ---- streaming store writer (storage.py:108-131) ------------------------- */

sdb_status sdb_run_to_file(sdb_ctx* ctx, sdb_model* model, const sdb_desc* desc,
                           const double* init, const double* params, const char* path,
                           int64_t offset, int64_t* fail_step) {
    SDB_ENTRY(ctx);
    sdb_status rc = model ? validate_model(ctx, desc, model) : validate(ctx, desc);
    if (rc != SDB_OK) return rc;
    if (!path || offset < 0) return fail_with(ctx, SDB_ERR_ARGUMENT, "bad store file arguments");
    const int fd = ::open(path, O_WRONLY | O_CLOEXEC);
    if (fd < 0) return fail_with(ctx, SDB_ERR_CUDA, "opening %s: %s", path, std::strerror(errno));
    rc = run_host(ctx, *desc, model, init, params, nullptr, fail_step, 0, fd, offset);
    if (::close(fd) != 0 && rc == SDB_OK)
        rc = fail_with(ctx, SDB_ERR_CUDA, "closing %s: %s", path, std::strerror(errno));
    return rc;
}

/* ---- analysis (analysis.py) ---------------------------------------------- */

sdb_status sdb_run_coherence(sdb_ctx* ctx, const sdb_desc* desc, const double* init,
                             const double* params, double* r_phi, int64_t* fail_step) {
    SDB_ENTRY(ctx);
    sdb_status rc = validate(ctx, desc);
    if (rc != SDB_OK) return rc;
    return run_host(ctx, *desc, nullptr, init, params, r_phi, fail_step, 1);
}

sdb_status sdb_run_coherence_device(sdb_ctx* ctx, const sdb_desc* desc, const double* d_init,
                                    const double* d_params, double* d_r_phi, int64_t* d_fail_step,
                                    void* stream) {
    SDB_ENTRY(ctx);
    sdb_status rc = validate(ctx, desc);
    if (rc != SDB_OK) return rc;
    return run_dev(ctx, *desc, nullptr, d_init, d_params, d_r_phi, d_fail_step, stream, 1);
}

sdb_status sdb_order_parameter(sdb_ctx* ctx, int32_t n, int64_t rows, const double* phases,
                               double* r, double* phi) {
    SDB_ENTRY(ctx);
    sdb_status rc = utility_prologue(ctx);
    if (rc != SDB_OK) return rc;
    if (n < 1 || rows < 0 || !phases || !r || !phi)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "bad order-parameter arguments");
    if (rows == 0) return SDB_OK;
    TmpBuf dth, dr, dphi;
    SDB_CUDA(ctx, cudaMalloc(&dth.p, size_t(rows) * n * sizeof(double)));
    SDB_CUDA(ctx, cudaMalloc(&dr.p, size_t(rows) * sizeof(double)));
    SDB_CUDA(ctx, cudaMalloc(&dphi.p, size_t(rows) * sizeof(double)));
    SDB_CUDA(ctx, cudaMemcpy(dth.p, phases, size_t(rows) * n * sizeof(double),
                             cudaMemcpyHostToDevice));
    SDB_CUDA(ctx, sdeb::launch_order_parameter(static_cast<const double*>(dth.p), n, rows,
                                               static_cast<double*>(dr.p),
                                               static_cast<double*>(dphi.p), nullptr));
    SDB_CUDA(ctx, cudaMemcpy(r, dr.p, size_t(rows) * sizeof(double), cudaMemcpyDeviceToHost));
    SDB_CUDA(ctx, cudaMemcpy(phi, dphi.p, size_t(rows) * sizeof(double), cudaMemcpyDeviceToHost));
    ctx->launches = 1;
    return SDB_OK;
}

/* ---- expression-template models ------------------------------------------ */

sdb_status sdb_model_create(int32_t nequat, int32_t nparams, int32_t nnoise, const char* drift,
                            const char* diffusion, sdb_model** out) {
    if (!out || !drift || !diffusion)
        return fail_with(nullptr, SDB_ERR_ARGUMENT, "null model argument");
    *out = nullptr;
    if (nequat < 1 || nparams < 0 || nnoise < 0)
        return fail_with(nullptr, SDB_ERR_ARGUMENT, "bad model dimensions (%d, %d, %d)", nequat,
                         nparams, nnoise);
    auto* m = new sdb_model();
    m->nequat = nequat;
    m->nparams = nparams;
    m->nnoise = nnoise;
    m->drift_text = drift;
    m->diffusion_text = diffusion;
    std::string err;
    if (!sdeb_dsl::generate(m, &err)) {
        delete m;
        return fail_with(nullptr, SDB_ERR_ARGUMENT, "%s", err.c_str());
    }
    *out = m;
    return SDB_OK;
}

void sdb_model_free(sdb_model* m) { delete m; }

int64_t sdb_model_source(const sdb_model* m, int32_t kind, char* buf, int64_t cap) {
    if (!m || kind < 0 || (kind & 255) >= sdeb::DK_COUNT || kind > 511) return -1;
    const bool factor = (kind & 256) != 0;
    const std::string src = sdeb_dsl::program_source(m, kind & 255, sdeb_dsl::lanes_for(m, factor),
                                                     factor);
    if (buf && cap > 0) {
        const size_t n = std::min<size_t>(src.size(), size_t(cap - 1));
        std::memcpy(buf, src.data(), n);
        buf[n] = '\0';
    }
    return int64_t(src.size());
}

sdb_status sdb_model_build(sdb_model* m, int32_t kind) {
    if (!m || kind < 0 || (kind & 255) >= sdeb::DK_COUNT || kind > 511)
        return fail_with(nullptr, SDB_ERR_ARGUMENT, "bad model or program kind");
    std::string err;
    const bool factor = (kind & 256) != 0;
    cudaError_t e = sdeb_dsl::compile_only(m, kind & 255, sdeb_dsl::lanes_for(m, factor), factor,
                                           &err);
    if (e != cudaSuccess) return fail_with(nullptr, SDB_ERR_CUDA, "%s", err.c_str());
    return SDB_OK;
}

sdb_status sdb_run_model(sdb_ctx* ctx, sdb_model* m, const sdb_desc* desc, const double* init,
                         const double* params, double* values, int64_t* fail_step) {
    SDB_ENTRY(ctx);
    sdb_status rc = validate_model(ctx, desc, m);
    if (rc != SDB_OK) return rc;
    return run_host(ctx, *desc, m, init, params, values, fail_step);
}

sdb_status sdb_run_model_device(sdb_ctx* ctx, sdb_model* m, const sdb_desc* desc,
                                const double* d_init, const double* d_params, double* d_values,
                                int64_t* d_fail_step, void* stream) {
    SDB_ENTRY(ctx);
    sdb_status rc = validate_model(ctx, desc, m);
    if (rc != SDB_OK) return rc;
    return run_dev(ctx, *desc, m, d_init, d_params, d_values, d_fail_step, stream);
}

sdb_status sdb_model_eval(sdb_ctx* ctx, sdb_model* m, int32_t which, double t, int64_t count,
                          const double* y, const double* p, const double* noise, double* out) {
    SDB_ENTRY(ctx);
    if (!m) return fail_with(ctx, SDB_ERR_ARGUMENT, "null model");
    if (which != 0 && which != 1) return fail_with(ctx, SDB_ERR_ARGUMENT, "which must be 0 or 1");
    if (which == 1 && m->nnoise > 0 && !noise)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "diffusion needs a noise array");
    return model_rows(ctx, m, which == 0 ? sdeb::DK_EVAL_DRIFT : sdeb::DK_EVAL_DIFFUSION, t, 0.0,
                      count, y, p, which == 1 ? noise : nullptr, out);
}

sdb_status sdb_model_step(sdb_ctx* ctx, sdb_model* m, int32_t solver, double t, double dt,
                          int64_t count, const double* y, const double* p, const double* noise,
                          double* out) {
    SDB_ENTRY(ctx);
    if (!m) return fail_with(ctx, SDB_ERR_ARGUMENT, "null model");
    if (!(dt > 0.0)) return fail_with(ctx, SDB_ERR_ARGUMENT, "dt must be positive");
    int kind;
    if (solver == SDB_SOLVER_RK4) {
        kind = sdeb::DK_STEP_RK4;
    } else if (solver == SDB_SOLVER_EM && m->nnoise > 0) {
        if (!noise) return fail_with(ctx, SDB_ERR_ARGUMENT, "em step needs a noise array");
        kind = sdeb::DK_STEP_EM;
    } else if (solver == SDB_SOLVER_EM || solver == SDB_SOLVER_EULER) {
        kind = sdeb::DK_STEP_EULER;
    } else {
        return fail_with(ctx, SDB_ERR_ARGUMENT, "unknown solver %d", solver);
    }
    return model_rows(ctx, m, kind, t, dt, count, y, p, kind == sdeb::DK_STEP_EM ? noise : nullptr,
                      out);
}

sdb_status sdb_philox_words(sdb_ctx* ctx, const uint32_t* in, int64_t count, uint32_t* out) {
    SDB_ENTRY(ctx);
    sdb_status rc = utility_prologue(ctx);
    if (rc != SDB_OK) return rc;
    if (count <= 0) return SDB_OK;
    TmpBuf din, dout;
    SDB_CUDA(ctx, cudaMalloc(&din.p, size_t(count) * 6 * sizeof(uint32_t)));
    SDB_CUDA(ctx, cudaMalloc(&dout.p, size_t(count) * 4 * sizeof(uint32_t)));
    SDB_CUDA(ctx, cudaMemcpy(din.p, in, size_t(count) * 6 * sizeof(uint32_t), cudaMemcpyHostToDevice));
    SDB_CUDA(ctx, sdeb::launch_philox_words(static_cast<uint32_t*>(din.p), count,
                                            static_cast<uint32_t*>(dout.p), nullptr));
    SDB_CUDA(ctx, cudaMemcpy(out, dout.p, size_t(count) * 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    return SDB_OK;
}

sdb_status sdb_normals(sdb_ctx* ctx, int32_t stream, uint64_t seed, const uint32_t* orbits,
                       int64_t count, uint32_t chunk, uint32_t step, int32_t m, double* out) {
    SDB_ENTRY(ctx);
    sdb_status rc = utility_prologue(ctx);
    if (rc != SDB_OK) return rc;
    if (stream < SDB_STREAM_PHILOX || stream > SDB_STREAM_XOSHIRO256PP)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "unknown stream %d", stream);
    if (m < 0) return fail_with(ctx, SDB_ERR_ARGUMENT, "noise count must be >= 0");
    if (stream == SDB_STREAM_PHILOX && chunk == sdeb::kSamplingTag)
        return fail_with(ctx, SDB_ERR_ARGUMENT,
                         "counter word 0x%08X is reserved for sampling streams", chunk);
    if (count <= 0 || m == 0) return SDB_OK;
    TmpBuf dorb, dout;
    SDB_CUDA(ctx, cudaMalloc(&dorb.p, size_t(count) * sizeof(uint32_t)));
    SDB_CUDA(ctx, cudaMalloc(&dout.p, size_t(count) * m * sizeof(double)));
    SDB_CUDA(ctx, cudaMemcpy(dorb.p, orbits, size_t(count) * sizeof(uint32_t), cudaMemcpyHostToDevice));
    SDB_CUDA(ctx, sdeb::launch_normals(stream, seed, static_cast<uint32_t*>(dorb.p), count, chunk,
                                       step, m, static_cast<double*>(dout.p), nullptr));
    SDB_CUDA(ctx, cudaMemcpy(out, dout.p, size_t(count) * m * sizeof(double), cudaMemcpyDeviceToHost));
    return SDB_OK;
}

sdb_status sdb_stream_raw(sdb_ctx* ctx, int32_t stream, uint64_t seed, uint64_t orbit,
                          uint64_t block, int64_t count, uint64_t* out) {
    SDB_ENTRY(ctx);
    sdb_status rc = utility_prologue(ctx);
    if (rc != SDB_OK) return rc;
    if (stream != SDB_STREAM_SFC64 && stream != SDB_STREAM_XOSHIRO256PP)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "stream %d has no state", stream);
    if (count <= 0) return SDB_OK;
    TmpBuf dout;
    SDB_CUDA(ctx, cudaMalloc(&dout.p, size_t(count) * sizeof(uint64_t)));
    SDB_CUDA(ctx, sdeb::launch_stream_raw(stream, seed, orbit, block, count,
                                          static_cast<uint64_t*>(dout.p), nullptr));
    SDB_CUDA(ctx, cudaMemcpy(out, dout.p, size_t(count) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return SDB_OK;
}

sdb_status sdb_sampling_uniforms(sdb_ctx* ctx, uint64_t seed, const uint32_t* orbits,
                                 int64_t count, int32_t ncols, double* out) {
    SDB_ENTRY(ctx);
    sdb_status rc = utility_prologue(ctx);
    if (rc != SDB_OK) return rc;
    if (ncols < 0) return fail_with(ctx, SDB_ERR_ARGUMENT, "count must be >= 0");
    if (count <= 0 || ncols == 0) return SDB_OK;
    TmpBuf dorb, dout;
    SDB_CUDA(ctx, cudaMalloc(&dorb.p, size_t(count) * sizeof(uint32_t)));
    SDB_CUDA(ctx, cudaMalloc(&dout.p, size_t(count) * ncols * sizeof(double)));
    SDB_CUDA(ctx, cudaMemcpy(dorb.p, orbits, size_t(count) * sizeof(uint32_t), cudaMemcpyHostToDevice));
    SDB_CUDA(ctx, sdeb::launch_sampling(seed, static_cast<uint32_t*>(dorb.p), count, ncols,
                                        static_cast<double*>(dout.p), nullptr));
    SDB_CUDA(ctx, cudaMemcpy(out, dout.p, size_t(count) * ncols * sizeof(double), cudaMemcpyDeviceToHost));
    return SDB_OK;
}

sdb_status sdb_sample_kuramoto(sdb_ctx* ctx, int32_t n, uint64_t seed, const uint32_t* orbits,
                               int64_t count, double omega_lo, double omega_hi, double noise_lo,
                               double noise_hi, double coupling, double* init, double* params) {
    SDB_ENTRY(ctx);
    sdb_status rc = utility_prologue(ctx);
    if (rc != SDB_OK) return rc;
    if (n < 1) return fail_with(ctx, SDB_ERR_ARGUMENT, "need at least one oscillator");
    if (count <= 0) return SDB_OK;
    TmpBuf dorb, dinit, dpar;
    SDB_CUDA(ctx, cudaMalloc(&dorb.p, size_t(count) * sizeof(uint32_t)));
    SDB_CUDA(ctx, cudaMalloc(&dinit.p, size_t(count) * n * sizeof(double)));
    SDB_CUDA(ctx, cudaMalloc(&dpar.p, size_t(count) * (2 * n + 1) * sizeof(double)));
    SDB_CUDA(ctx, cudaMemcpy(dorb.p, orbits, size_t(count) * sizeof(uint32_t), cudaMemcpyHostToDevice));
    SDB_CUDA(ctx, sdeb::launch_sample_kuramoto(
                      n, seed, static_cast<uint32_t*>(dorb.p), count, omega_lo,
                      omega_hi - omega_lo, noise_lo, noise_hi - noise_lo, coupling,
                      static_cast<double*>(dinit.p), static_cast<double*>(dpar.p), nullptr));
    SDB_CUDA(ctx, cudaMemcpy(init, dinit.p, size_t(count) * n * sizeof(double), cudaMemcpyDeviceToHost));
    SDB_CUDA(ctx, cudaMemcpy(params, dpar.p, size_t(count) * (2 * n + 1) * sizeof(double),
                             cudaMemcpyDeviceToHost));
    return SDB_OK;
}

static sdb_status per_step(sdb_ctx* ctx, int kind_solver, int kind_stream, int32_t n,
                           int32_t nparams, int32_t nnoise, int32_t coupling, int64_t count,
                           double dt, const double* y, const double* p, const double* noise,
                           double* out) {
    SDB_ENTRY(ctx);
    sdb_status rc = utility_prologue(ctx);
    if (rc != SDB_OK) return rc;
    if (n < 1 || n > kMaxN) return fail_with(ctx, SDB_ERR_UNSUPPORTED, "nequat=%d unsupported", n);
    if (nparams < n + 1 || (nnoise > 0 && nparams < 2 * n + 1))
        return fail_with(ctx, SDB_ERR_ARGUMENT, "nparams=%d does not fit Kuramoto(n=%d)", nparams, n);
    if (coupling != SDB_COUPLING_MEANFIELD && coupling != SDB_COUPLING_PAIRWISE)
        return fail_with(ctx, SDB_ERR_ARGUMENT, "unknown coupling %d", coupling);
    if (count <= 0) return SDB_OK;
    TmpBuf dy, dp, dn, dout;
    SDB_CUDA(ctx, cudaMalloc(&dy.p, size_t(count) * n * sizeof(double)));
    SDB_CUDA(ctx, cudaMalloc(&dp.p, size_t(count) * nparams * sizeof(double)));
    SDB_CUDA(ctx, cudaMalloc(&dout.p, size_t(count) * n * sizeof(double)));
    SDB_CUDA(ctx, cudaMemcpy(dy.p, y, size_t(count) * n * sizeof(double), cudaMemcpyHostToDevice));
    SDB_CUDA(ctx, cudaMemcpy(dp.p, p, size_t(count) * nparams * sizeof(double), cudaMemcpyHostToDevice));
    if (kind_stream == sdeb::KS_EXPLICIT) {
        SDB_CUDA(ctx, cudaMalloc(&dn.p, size_t(count) * n * sizeof(double)));
        SDB_CUDA(ctx, cudaMemcpy(dn.p, noise, size_t(count) * n * sizeof(double), cudaMemcpyHostToDevice));
    }
    const int P = next_pow2(n);
    const int L = std::max(1, P / kMaxJ);
    sdb_desc d{};
    d.nequat = n;
    d.nparams = nparams;
    d.nnoise = nnoise;
    d.dt = dt;
    d.ksteps = 1;
    d.chunks = 1;
    d.orbits = count;
    sdeb::RunArgs a = make_args(d, L);
    a.state_in = static_cast<double*>(dy.p);
    a.params = static_cast<double*>(dp.p);
    a.noise = static_cast<double*>(dn.p);
    a.values = static_cast<double*>(dout.p);
    a.vstride = 1;
    a.check_finite = 0;
    SDB_CUDA(ctx, launch_run(a, P / L, kind_solver, kind_stream, coupling, 1, nullptr));
    SDB_CUDA(ctx, cudaMemcpy(out, dout.p, size_t(count) * n * sizeof(double), cudaMemcpyDeviceToHost));
    return SDB_OK;
}

sdb_status sdb_drift(sdb_ctx* ctx, int32_t n, int32_t nparams, int32_t coupling, int64_t count,
                     const double* y, const double* p, double* f) {
    return per_step(ctx, sdeb::KS_DRIFT, sdeb::KS_NONE, n, nparams, 0, coupling, count, 1.0, y, p,
                    nullptr, f);
}

sdb_status sdb_step(sdb_ctx* ctx, int32_t solver, int32_t n, int32_t nparams, int32_t nnoise,
                    int32_t coupling, int64_t count, double dt, const double* y, const double* p,
                    const double* noise, double* out) {
    if (!(dt > 0.0)) return fail_with(ctx, SDB_ERR_ARGUMENT, "dt must be positive");
    if (solver == SDB_SOLVER_EM && nnoise > 0) {
        if (!noise) return fail_with(ctx, SDB_ERR_ARGUMENT, "em step needs a noise array");
        return per_step(ctx, sdeb::KS_EM, sdeb::KS_EXPLICIT, n, nparams, nnoise, coupling, count,
                        dt, y, p, noise, out);
    }
    if (solver == SDB_SOLVER_RK4)
        return per_step(ctx, sdeb::KS_RK4, sdeb::KS_NONE, n, nparams, 0, coupling, count, dt, y, p,
                        nullptr, out);
    if (solver == SDB_SOLVER_EM || solver == SDB_SOLVER_EULER)
        return per_step(ctx, sdeb::KS_EM, sdeb::KS_NONE, n, nparams, 0, coupling, count, dt, y, p,
                        nullptr, out);
    return fail_with(ctx, SDB_ERR_ARGUMENT, "unknown solver %d", solver);
}

sdb_status sdb_fp64_peak(sdb_ctx* ctx, double* ops_per_s, double* ms_out) {
    SDB_ENTRY(ctx);
    sdb_status rc = utility_prologue(ctx);
    if (rc != SDB_OK) return rc;
    int sms = 0;
    SDB_CUDA(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->slots[0].device));
    const int blocks = sms * 8;  // 8 x 256 threads = 64 warps per SM
    const int iters = 2000;
    TmpBuf dout;
    SDB_CUDA(ctx, cudaMalloc(&dout.p, sizeof(double)));
    cudaEvent_t e0, e1;
    SDB_CUDA(ctx, cudaEventCreate(&e0));
    SDB_CUDA(ctx, cudaEventCreate(&e1));
    SDB_CUDA(ctx, sdeb::launch_fp64_peak(blocks, iters / 10, static_cast<double*>(dout.p), nullptr));
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0, nullptr);
        sdeb::launch_fp64_peak(blocks, iters, static_cast<double*>(dout.p), nullptr);
        cudaEventRecord(e1, nullptr);
        SDB_CUDA(ctx, cudaEventSynchronize(e1));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    SDB_CUDA(ctx, cudaGetLastError());
    const double ops = double(blocks) * 256.0 * double(iters) * 128.0;
    if (ops_per_s) *ops_per_s = ops / (double(best) * 1e-3);
    if (ms_out) *ms_out = best;
    return SDB_OK;
}

sdb_status sdb_math_probe(sdb_ctx* ctx, int32_t func, const double* x, int64_t count,
                          double* out) {
    SDB_ENTRY(ctx);
    sdb_status rc = utility_prologue(ctx);
    if (rc != SDB_OK) return rc;
    if (func < 0 || func > 8) return fail_with(ctx, SDB_ERR_ARGUMENT, "unknown math probe %d", func);
    if (count <= 0) return SDB_OK;
    TmpBuf dx, dout;
    SDB_CUDA(ctx, cudaMalloc(&dx.p, size_t(count) * sizeof(double)));
    SDB_CUDA(ctx, cudaMalloc(&dout.p, size_t(count) * sizeof(double)));
    SDB_CUDA(ctx, cudaMemcpy(dx.p, x, size_t(count) * sizeof(double), cudaMemcpyHostToDevice));
    SDB_CUDA(ctx, sdeb::launch_math_probe(func, static_cast<double*>(dx.p), count,
                                          static_cast<double*>(dout.p), nullptr));
    SDB_CUDA(ctx, cudaMemcpy(out, dout.p, size_t(count) * sizeof(double), cudaMemcpyDeviceToHost));
    return SDB_OK;
}

}  // extern "C"
