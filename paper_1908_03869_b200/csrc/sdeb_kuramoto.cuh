// Fused Kuramoto ensemble stepper for sm_100a.
//
// Replaces the reference's chunk x step loop (engine.py:223-263) with the
// noise draw (rng.py:150-188), the drift (model.py:188-196), the diffusion
// (model.py:199-201) and the em/euler/rk4 update (solvers.py:63-88) fused
// into ONE persistent-per-orbit kernel: state, parameters and stateful RNG
// words stay in registers for all steps of a launch; HBM sees one read of
// init/params and one n-vector write per sample.
//
// Layout ("lane groups"): each orbit is owned by L = lanes consecutive
// threads of a warp (L in {1,2,..,32}); lane l owns oscillators
// [l*J, l*J+J) with L*J = P = next_pow2(n).  Sums over oscillators use ONE
// canonical binary tree over the P leaves (adjacent leaves first, padding
// leaves = +0.0): in-lane levels in registers, upper levels by
// __shfl_xor_sync.  IEEE addition is commutative, so every (L, J) layout
// produces bit-identical results -- the host may autotune the layout freely
// (results never depend on it, nor on shard boundaries or GPU count).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <math_constants.h>

#include "sdeb_analysis.cuh"
#include "sdeb_rng.cuh"

namespace sdeb {

constexpr int kBlock = 128;

enum SolverKind : int { KS_EM = 0, KS_RK4 = 2, KS_DRIFT = 3 };
// S_NONE: deterministic (euler, or em with nnoise=0); S_EXPLICIT: caller-given noise
enum StreamKind : int { KS_PHILOX = 0, KS_SFC64 = 1, KS_XOSHIRO = 2, KS_NONE = 3, KS_EXPLICIT = 4 };
enum CouplingKind : int { KC_MEANFIELD = 0, KC_PAIRWISE = 1 };

struct RunArgs {
    const double* state_in;   // [orbits][n] state at chunk_begin (init on the first launch)
    const double* params;     // [orbits][nparams]
    const double* noise;      // [orbits][n] explicit noise (KS_EXPLICIT) or null
    double* state_out;        // [orbits][n] state at chunk_end (may be null)
    double* values;           // sample of chunk c, row r: values[(r*vstride + c-chunk_begin)*n + i]
    int64_t* fail_step;       // [orbits] first non-finite absolute step or -1 (may be null)
    uint64_t* rng_state;      // [orbits][nblocks][4] for stateful streams (null: not saved)
    int64_t orbits, orbit_offset, vstride;
    int64_t ksteps, chunk_begin, chunk_end;
    uint64_t seed;
    double dt, sqrt_dt, half_dt, dt6;
    int n, nparams, nnoise, lanes, log2lanes;
    int fresh;                // 1: fail=-1 and seed stateful streams in-kernel
    int check_finite;         // 1: run_batch failure semantics; 0: raw per-step API
    int smem_pad;             // dynamic shared memory per CTA (caps CTAs/SM; 0 = none)
    int persistent;           // > 0: grid size of the work-pulling (slab, CTA-group) mode
    int64_t groups;           // CTA-groups = ceil(orbits * lanes / kBlock)
    int64_t slab_steps;       // steps per work item (persistent mode)
    uint64_t* work_counter;   // persistent: zeroed item counter
    unsigned* slab_done;      // persistent: [groups] published slabs, zeroed
};

__device__ __forceinline__ bool finite_bits(double x) {
    return (__double2hiint(x) & 0x7ff00000) != 0x7ff00000;
}

__device__ __forceinline__ int64_t fail_combine(int64_t a, int64_t b) {
    return a < 0 ? b : (b < 0 ? a : (a < b ? a : b));
}

// Canonical in-lane tree: level s combines leaves (q, q+s) for q % 2s == 0.
template <int J>
__device__ __forceinline__ double lane_tree_sum(double (&v)[J]) {
#pragma unroll
    for (int s = 1; s < J; s <<= 1) {
#pragma unroll
        for (int q = 0; q + s < J; q += 2 * s) v[q] = __dadd_rn(v[q], v[q + s]);
    }
    return v[0];
}

__device__ __forceinline__ double group_sum(double x, int lanes) {
    for (int o = 1; o < lanes; o <<= 1) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

// Both coupling sums over the orbit's lanes, upper levels of the canonical
// tree, as one unrolled butterfly with warp-uniform exits: a runtime-bounded
// loop per sum cost ~9 issue slots per level (divergence checks, moves, loop
// control) around its 2 SHFLs.
__device__ __forceinline__ void xor_level(double& a, double& b, int o) {
    const double pa = __shfl_xor_sync(0xffffffffu, a, o);
    const double pb = __shfl_xor_sync(0xffffffffu, b, o);
    a = __dadd_rn(a, pa);
    b = __dadd_rn(b, pb);
}

__device__ __forceinline__ void group_sum2(double& a, double& b, int lanes) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        if (o >= lanes) break;  // warp-uniform exit
        xor_level(a, b, o);
    }
}

__device__ __forceinline__ int64_t group_fail(int64_t f, int lanes) {
    for (int o = 1; o < lanes; o <<= 1) {
        const long long other = __shfl_xor_sync(0xffffffffu, (long long)f, o);
        f = fail_combine(f, other);
    }
    return f;
}

// ---- drift f_i = omega_i + (K/n) * S_i (model.py:193-196) -----------------

// MEANFIELD: S_i = cos(y_i) * sum_j sin(y_j) - sin(y_i) * sum_j cos(y_j).
// PADDED (n < L*J): padding leaves (whose y stays 0) are forced to +0.0 in
// the sums; the unpadded instantiation (n a power of two: every BASELINE
// config) carries no per-oscillator predicates at all.
template <int J, bool PADDED>
__device__ __forceinline__ void meanfield_sums(const double (&y)[J], int base, int n, int lanes,
                                               double (&S)[J]) {
    double sn[J], cs[J], ts[J], tc[J];
    sincos_vec<J>(y, sn, cs);
#pragma unroll
    for (int q = 0; q < J; ++q) {
        if (PADDED && base + q >= n) {
            sn[q] = 0.0;
            cs[q] = 0.0;
        }
        ts[q] = sn[q];
        tc[q] = cs[q];
    }
    double a = lane_tree_sum<J>(ts);
    double b = lane_tree_sum<J>(tc);
    group_sum2(a, b, lanes);
#pragma unroll
    for (int q = 0; q < J; ++q) {
        // two rounded products, not an FMA: the self term cos*sin - sin*cos
        // then cancels exactly (n=1 gives S == 0, like sin(0) == 0)
        S[q] = __dsub_rn(__dmul_rn(cs[q], a), __dmul_rn(sn[q], b));
    }
}

template <int J, bool PADDED>
__device__ __forceinline__ void drift_meanfield(const double (&y)[J], const double (&om)[J],
                                                double kn, int base, int n, int lanes,
                                                double (&f)[J]) {
    double S[J];
    meanfield_sums<J, PADDED>(y, base, n, lanes, S);
#pragma unroll
    for (int q = 0; q < J; ++q) f[q] = __dadd_rn(om[q], __dmul_rn(kn, S[q]));
}

// The stepping form: c0_i + scale*S_i with the scale folded into the two
// group sums, fma(cos y_i, scale*sum sin, fma(-sin y_i, scale*sum cos, c0_i))
// -- 2 FP64 ops per oscillator instead of 4 (+2 per lane).  A reassociation
// of the reference's (ω + (K/n) S) by a few ulp (folded
// update); drift_eval keeps the exact form above.
template <int J, bool PADDED, class C0>
__device__ __forceinline__ void meanfield_folded_acc(const double (&y)[J], C0&& c0, double scale,
                                                     int base, int n, int lanes,
                                                     double (&out)[J], int big_hint = -1) {
    double sn[J], cs[J], ts[J], tc[J];
    if (big_hint < 0) {
        sincos_vec<J>(y, sn, cs);
    } else {
        sincos_vec_hint<J>(y, sn, cs, big_hint != 0);
    }
#pragma unroll
    for (int q = 0; q < J; ++q) {
        if (PADDED && base + q >= n) {
            sn[q] = 0.0;
            cs[q] = 0.0;
        }
        ts[q] = sn[q];
        tc[q] = cs[q];
    }
    double a = lane_tree_sum<J>(ts);
    double b = lane_tree_sum<J>(tc);
    group_sum2(a, b, lanes);
    const double sa = __dmul_rn(scale, a), sb = __dmul_rn(scale, b);
#pragma unroll
    for (int q = 0; q < J; ++q) out[q] = __fma_rn(cs[q], sa, __fma_rn(-sn[q], sb, c0(q)));
}

template <int J, bool PADDED>
__device__ __forceinline__ void meanfield_folded(const double (&y)[J], const double (&c0)[J],
                                                 double scale, int base, int n, int lanes,
                                                 double (&out)[J], int big_hint = -1) {
    meanfield_folded_acc<J, PADDED>(y, [&](int q) { return c0[q]; }, scale, base, n, lanes, out,
                                    big_hint);
}

// PAIRWISE: S_i = sum_{j != i} sin(fl(y_j - y_i)), every term computed as
// the reference computes it (model.py:193-195), each unordered pair ONCE:
// fl(a - b) == -fl(b - a) and the table sin is exactly odd, so the term of
// row j is the negated term of row i (the diagonal sin(0) = 0 is skipped).
//
// Lane l of an orbit's L lanes owns oscillators [lJ, lJ + J) (registers).
// The pairs form L x L tiles of J x J terms:
//   * tile (l, l) (the lane's own block): J(J-1)/2 terms, j-sequential per row;
//   * round d = 1 .. L/2-1: lane l takes tile (l, l+d) -- the partner's block
//     arrives by __shfl_sync, each term goes to the lane's row sum and,
//     negated, to a column sum that is shuffled back to the partner (the
//     partner receives from lane l-d: every unordered block pair is covered
//     once, by the lane at the smaller cyclic distance);
//   * round L/2 (the two lanes are each other's partners): the tile is split
//     in a checkerboard, lane l computing the pairs with (q + r + h) even
//     (h = the upper half's 1), through a one-slot rotation of the partner's
//     block so both halves run the same instruction stream; the column sums
//     are exchanged with __shfl_xor_sync.
// Per lane (L J)(L J - 1) / (2 L) terms: the n^2 / 2 of the antisymmetric sum,
// balanced, with 4J SHFL.64 per round and no shared memory.  The summation
// order is fixed by (L, J); run_batch derives the pairwise layout from n alone
// (pairwise_lanes), so results do not depend on GPU count, shards, tiles or
// grid mode.  Within 1e-15 relative of the reference's numpy order.
// sin of any argument, out of line: the rare huge-phase path of the pairwise
// tiles calls it per term (inlining libdevice's reduction into J^2 unrolled
// terms multiplied the code and the compile time).
static __device__ __noinline__ double pair_sin_exact(double x) {
    double s, c;
    sincos_any(x, s, c);
    (void)c;
    return s;
}

template <bool SLOW>
__device__ __forceinline__ double pair_sin(double x) {
    if constexpr (SLOW) {
        return pair_sin_exact(x);
    } else {
        double s, c;
        sincos_small(x, s, c);  // the cos half is dead code
        (void)c;
        return s;
    }
}

template <int J, bool PADDED, bool SLOW>
__device__ __forceinline__ void pair_tile_diag(const double (&y)[J], int base, int n,
                                               double (&S)[J]) {
#pragma unroll
    for (int i = 0; i < J; ++i) {
#pragma unroll
        for (int j = i + 1; j < J; ++j) {
            double d = __dsub_rn(y[j], y[i]);
            if (PADDED && base + j >= n) d = 0.0;  // j > i: covers an invalid i too
            const double t = pair_sin<SLOW>(d);
            S[i] = __dadd_rn(S[i], t);
            S[j] = __dsub_rn(S[j], t);
        }
    }
}

template <int J, bool PADDED, bool SLOW>
__device__ __forceinline__ void pair_tile_full(const double (&y)[J], const double (&ym)[J],
                                               int base, int pbase, int n, double (&S)[J],
                                               double (&C)[J]) {
#pragma unroll
    for (int r = 0; r < J; ++r) C[r] = 0.0;
    // J > 8 only runs for explicit lane counts (pairwise_lanes uses J <= 8 for
    // multi-lane layouts): rolled row loop there, to bound code size
#pragma unroll(J <= 8 ? J : 1)
    for (int q = 0; q < J; ++q) {
#pragma unroll
        for (int r = 0; r < J; ++r) {
            double d = __dsub_rn(ym[r], y[q]);
            if (PADDED && (base + q >= n || pbase + r >= n)) d = 0.0;
            const double t = pair_sin<SLOW>(d);
            S[q] = __dadd_rn(S[q], t);
            C[r] = __dsub_rn(C[r], t);
        }
    }
}

// The checkerboard half of tile (l, partner) for the half round: pairs
// (q, r) with r == q + h (mod 2); ymr[s] = ym[(s + h) % J] so that r = s + h
// and both halves loop over s = q + 2k (mod J) with no divergence.
template <int J, bool PADDED, bool SLOW>
__device__ __forceinline__ void pair_tile_half(const double (&y)[J], const double (&ym)[J], int h,
                                               int base, int pbase, int n, double (&S)[J],
                                               double (&C)[J]) {
    double ymr[J], Cr[J];
    bool vr[J];
#pragma unroll
    for (int s = 0; s < J; ++s) {
        ymr[s] = h ? ym[(s + 1) % J] : ym[s];
        vr[s] = !PADDED || pbase + ((s + h) % J) < n;
        Cr[s] = 0.0;
    }
#pragma unroll(J <= 8 ? J : 1)
    for (int q = 0; q < J; ++q) {
#pragma unroll
        for (int k = 0; k < J / 2; ++k) {
            const int sidx = (q + 2 * k) % J;
            double d = __dsub_rn(ymr[sidx], y[q]);
            if (PADDED && (base + q >= n || !vr[sidx])) d = 0.0;
            const double t = pair_sin<SLOW>(d);
            S[q] = __dadd_rn(S[q], t);
            Cr[sidx] = __dsub_rn(Cr[sidx], t);
        }
    }
#pragma unroll
    for (int r = 0; r < J; ++r) C[r] = h ? Cr[(r + J - 1) % J] : Cr[r];
}

template <int J, bool PADDED, bool SLOW>
__device__ __forceinline__ void pair_sums(const double (&y)[J], int base, int n, int lanes,
                                          double (&S)[J]) {
#pragma unroll
    for (int q = 0; q < J; ++q) S[q] = 0.0;
    pair_tile_diag<J, PADDED, SLOW>(y, base, n, S);
    const int lane = int(threadIdx.x) & (lanes - 1);
    const int half = lanes >> 1;
    for (int d = 1; d < half; ++d) {  // full tiles (lanes >= 4)
        double ym[J], C[J];
        const int src = (lane + d) & (lanes - 1);
#pragma unroll
        for (int r = 0; r < J; ++r) ym[r] = __shfl_sync(0xffffffffu, y[r], src, lanes);
        pair_tile_full<J, PADDED, SLOW>(y, ym, base, src * J, n, S, C);
        const int from = (lane - d) & (lanes - 1);
#pragma unroll
        for (int q = 0; q < J; ++q)
            S[q] = __dadd_rn(S[q], __shfl_sync(0xffffffffu, C[q], from, lanes));
    }
    if (half > 0) {  // the half round (lanes >= 2)
        double ym[J], C[J];
#pragma unroll
        for (int r = 0; r < J; ++r) ym[r] = __shfl_xor_sync(0xffffffffu, y[r], half);
        const int h = lane >= half ? 1 : 0;
        if constexpr (J >= 2) {
            pair_tile_half<J, PADDED, SLOW>(y, ym, h, base, (lane ^ half) * J, n, S, C);
        } else {  // one oscillator per lane: the lower lane takes the single pair
            double d = __dsub_rn(ym[0], y[0]);
            if (PADDED && (base >= n || (lane ^ half) * J >= n)) d = 0.0;
            const double t = h ? 0.0 : pair_sin<SLOW>(d);
            S[0] = __dadd_rn(S[0], t);
            C[0] = -t;
        }
#pragma unroll
        for (int q = 0; q < J; ++q)
            S[q] = __dadd_rn(S[q], __shfl_xor_sync(0xffffffffu, C[q], half));
    }
}

template <int J, bool PADDED>
__device__ __forceinline__ void drift_pairwise(const double (&y)[J], const double (&om)[J],
                                               double kn, int base, int n, int lanes,
                                               double* /*sh*/, double* /*shs*/, double (&f)[J]) {
    // |y| < 2^28 everywhere in the warp keeps every difference inside the fast
    // sin's range; otherwise the whole warp takes the exact reduction (same
    // bits for the small arguments, so the vote never changes a result)
    bool big = false;
#pragma unroll
    for (int q = 0; q < J; ++q) big |= (__double2hiint(y[q]) & 0x7fffffff) >= 0x41B00000;
    double S[J];
    if (__any_sync(0xffffffffu, big)) {
        pair_sums<J, PADDED, true>(y, base, n, lanes, S);
    } else {
        pair_sums<J, PADDED, false>(y, base, n, lanes, S);
    }
#pragma unroll
    for (int q = 0; q < J; ++q) {
        f[q] = (base + q < n) ? __dadd_rn(om[q], __dmul_rn(kn, S[q])) : 0.0;
    }
}

template <int J, int COUPLING, bool PADDED>
__device__ __forceinline__ void drift(const double (&y)[J], const double (&om)[J], double kn,
                                      int base, int n, int lanes, double* sh, double* shs,
                                      double (&f)[J]) {
    if constexpr (COUPLING == KC_MEANFIELD) {
        drift_meanfield<J, PADDED>(y, om, kn, base, n, lanes, f);
    } else {
        drift_pairwise<J, PADDED>(y, om, kn, base, n, lanes, sh, shs, f);
    }
}

// RK4 stage drift: the folded meanfield form, or the exact pairwise one.
template <int J, int COUPLING, bool PADDED>
__device__ __forceinline__ void rk4_drift(const double (&y)[J], const double (&om)[J], double kn,
                                          int base, int n, int lanes, double* sh, double* shs,
                                          double (&f)[J]) {
    if constexpr (COUPLING == KC_MEANFIELD) {
        meanfield_folded<J, PADDED>(y, om, kn, base, n, lanes, f);
    } else {
        drift_pairwise<J, PADDED>(y, om, kn, base, n, lanes, sh, shs, f);
    }
}

// Order parameter of the orbit (analysis.py:77-82) from its lanes' phases:
// the canonical-tree sums of cos / sin (as drift_meanfield), every lane gets
// (r, Phi).  Used at sample time when the run stores coherence instead of y.
template <int J, bool PADDED>
__device__ __forceinline__ void group_order_param(const double (&y)[J], int base, int n, int lanes,
                                                  double& r, double& phi) {
    double sn[J], cs[J];
    sincos_vec<J>(y, sn, cs);
#pragma unroll
    for (int q = 0; q < J; ++q) {
        if (PADDED && base + q >= n) {
            sn[q] = 0.0;
            cs[q] = 0.0;
        }
    }
    double ss = lane_tree_sum<J>(sn), sc = lane_tree_sum<J>(cs);
    group_sum2(ss, sc, lanes);
    order_param_from_sums(sc, ss, n, r, phi);
}

// ---- noise for one step (rng.py:150-188 / DESIGN.md streams) ---------------

// Noise blocks a lane draws per step.  J not a power of two (the exact
// one-lane layouts of n <= 16) ends in a partial block.
template <int J>
__host__ __device__ constexpr int blocks_per_lane() {
    return J >= 3 ? (J + 3) / 4 : 1;
}

// Draws the step's normals pair by pair and hands each to apply(q, z) as
// soon as it exists, so at most one Box-Muller pair is live at a time (the
// v2 kernel materialised z[J] next to the drift's sin/cos arrays: 124
// registers at J=4).
template <int J, int STREAM, bool PADDED, class Apply>
__device__ __forceinline__ void step_noise_apply(const RunArgs& a, int64_t row, uint32_t orbit_g,
                                                 uint64_t step, int base,
                                                 StreamState (&rs)[blocks_per_lane<J>()],
                                                 Apply&& apply) {
    if constexpr (STREAM == KS_EXPLICIT) {
#pragma unroll
        for (int q = 0; q < J; ++q)
            if (base + q < a.n) apply(q, a.noise[row * a.n + base + q]);
    } else {
        const uint32_t seed_lo = uint32_t(a.seed), seed_hi = uint32_t(a.seed >> 32);
        const uint32_t step_hi = uint32_t(step >> 32), step_lo = uint32_t(step);
        const int nn = a.nnoise;
        if constexpr (J >= 3) {
            // unpadded with J % 4 == 0: n = L*J, whole blocks, no checks.  Any
            // other J >= 3 (lane 0 of a one-lane orbit, J == n) ends in a partial
            // block: the reference draws it whole and keeps the first n normals
            constexpr bool kWhole = !PADDED && J % 4 == 0;
            // all of the step's blocks first: independent integer chains side
            // by side, then the Box-Muller pairs (Philox: paper N=10 -4 %, cfg3
            // / cfg5 -0.2..0.5 %; sfc64: cfg2 at L=2 -3 %).  A padded lane's
            // surplus Philox block is unused; a stream block past the last noise
            // term holds a zero state that is never saved, so advancing it is
            // harmless.
            Words4 ws[blocks_per_lane<J>()];
#pragma unroll
            for (int t = 0; t < blocks_per_lane<J>(); ++t) {
                if constexpr (STREAM == KS_PHILOX) {
                    ws[t] = philox4x32_10(seed_hi, step_hi, step_lo, uint32_t(base / 4 + t), seed_lo,
                                          orbit_g);
                } else {
                    ws[t] = stream_block<STREAM>(rs[t]);
                }
            }
#pragma unroll
            for (int t = 0; t < blocks_per_lane<J>(); ++t) {
                const int b = base / 4 + t;
                if (kWhole || 4 * b < nn) {
                    const Words4 w = ws[t];
                    double z0, z1;
                    box_muller_pair(w.w0, w.w1, z0, z1);
                    apply(4 * t, z0);
                    if (4 * t + 1 < J) apply(4 * t + 1, z1);
                    if (4 * t + 2 < J && (kWhole || 4 * b + 2 < nn)) {
                        box_muller_pair(w.w2, w.w3, z0, z1);
                        apply(4 * t + 2, z0);
                        if (4 * t + 3 < J) apply(4 * t + 3, z1);
                    }
                }
            }
        } else {
            // J in {1, 2}: the lane's oscillators sit inside one block shared
            // with neighbouring lanes; each lane derives the same words.
            const int b = base / 4;
            if (base < nn) {
                Words4 w;
                if constexpr (STREAM == KS_PHILOX) {
                    w = philox4x32_10(seed_hi, step_hi, step_lo, uint32_t(b), seed_lo, orbit_g);
                } else {
                    w = stream_block<STREAM>(rs[0]);
                }
                const bool second = (base >> 1) & 1;
                const uint32_t wa = second ? w.w2 : w.w0, wb = second ? w.w3 : w.w1;
                double z0, z1;
                box_muller_pair(wa, wb, z0, z1);
                if constexpr (J == 2) {
                    apply(0, z0);
                    apply(1, z1);
                } else {
                    apply(0, (base & 1) ? z1 : z0);
                }
            }
        }
    }
}

// ---- the fused run kernel ----------------------------------------------------

// One work item: CTA-group `cg` (kBlock/L orbits) advanced over the absolute
// steps [s0, s1).  first = this item starts the run (state from state_in,
// rng seeded / loaded per a.fresh); otherwise the state saved by the previous
// slab is resumed from state_out / rng_state / fail_step.  Saving and resuming
// are exact, so any slab split gives bit-identical results.
// COH: samples are the orbit's order parameter instead of its phases
// (analysis.py coherence_series fused into the run): per orbit row a plane of
// r then a plane of Phi, values[row*2*vstride + {0, vstride} + 1 + c-chunk_begin],
// sample 0 (the initial state) at offset 0.
template <int J, int SOLVER, int STREAM, int COUPLING, bool PADDED, bool COH = false,
          bool CSM = false>
__device__ __forceinline__ void run_item(const RunArgs& a, int64_t cg, uint64_t s0, uint64_t s1,
                                         bool first, double* sh, double* shs) {
    constexpr bool kStochastic = (SOLVER == KS_EM) && (STREAM != KS_NONE);
    constexpr bool kStateful = kStochastic && (STREAM == KS_SFC64 || STREAM == KS_XOSHIRO);
    constexpr int NB = blocks_per_lane<J>();

    const int64_t gtid = cg * kBlock + threadIdx.x;
    const int lanes = a.lanes;
    const int64_t group = gtid >> a.log2lanes;
    const int lane = int(gtid & (lanes - 1));
    const bool active = group < a.orbits;
    const int64_t row = active ? group : a.orbits - 1;  // idle tail groups mirror the last row
    const int n = a.n;
    const int base = lane * J;
    const uint32_t orbit_g = uint32_t(a.orbit_offset + row);

    double y[J], om[J], sg[J];
    const double* prow = a.params + row * a.nparams;
    const double kn = __ddiv_rn(__ldg(prow), double(n));  // np.divide(p[...,0:1], float(n))
    const double* src = first ? a.state_in : a.state_out;
#pragma unroll
    for (int q = 0; q < J; ++q) {
        const int i = base + q;
        const bool valid = i < n;
        y[q] = valid ? src[row * n + i] : 0.0;
        om[q] = valid ? __ldg(prow + 1 + i) : 0.0;
        sg[q] = (kStochastic && valid) ? __ldg(prow + 1 + n + i) : 0.0;
    }

    // folded step constants of the meanfield EM form (see the step below).
    // CSM: kept in this thread's shared-memory column (re-read where a step
    // uses them; volatile, never hoisted back) instead of 4J registers, which
    // the sincos / Box-Muller chains of a step can then use for ILP
    double omdt[J], sgs[J];
    const double kndt = __dmul_rn(kn, a.dt);
    volatile double* cst = sh + threadIdx.x;  // CSM: [2J][kBlock]
#pragma unroll
    for (int q = 0; q < J; ++q) {
        omdt[q] = __dmul_rn(om[q], a.dt);
        sgs[q] = __dmul_rn(a.sqrt_dt, sg[q]);
        if constexpr (CSM) {
            cst[q * kBlock] = omdt[q];
            cst[(J + q) * kBlock] = sgs[q];
        }
    }

    if constexpr (SOLVER == KS_DRIFT) {
        double f[J];
        drift<J, COUPLING, PADDED>(y, om, kn, base, n, lanes, sh, shs, f);
        if (active) {
#pragma unroll
            for (int q = 0; q < J; ++q)
                if (base + q < n) a.values[row * n + base + q] = f[q];
        }
        return;
    } else {
        const bool fresh = first && a.fresh;
        int64_t fail = (fresh || a.fail_step == nullptr) ? -1 : a.fail_step[row];
        const int nblocks = (a.nnoise + 3) / 4;

        StreamState rs[NB];
        if constexpr (kStateful) {
#pragma unroll
            for (int t = 0; t < NB; ++t) {
                const int b = base / 4 + t;
                if (b < nblocks) {
                    if (fresh) {
                        rs[t] = stream_init<STREAM>(a.seed, uint64_t(orbit_g), uint64_t(b));
                    } else {
                        const uint64_t* p = a.rng_state + (row * nblocks + b) * 4;
                        rs[t] = StreamState{p[0], p[1], p[2], p[3]};
                    }
                } else {
                    rs[t] = StreamState{0, 0, 0, 0};
                }
            }
        }

        if (COH && fresh && s0 == 0) {  // coherence of the initial state
            double r, phi;
            group_order_param<J, PADDED>(y, base, n, lanes, r, phi);
            if (active && lane == 0) {
                double* o = a.values + row * a.vstride * 2;
                o[0] = r;
                o[a.vstride] = phi;
            }
        }
        const double dt = a.dt;
        const uint64_t ks = uint64_t(a.ksteps);
        // meanfield EM: |y| scanned once per step (after the update), shared by
        // the failure test and the next step's sincos range test
        constexpr bool kMagScan = SOLVER == KS_EM && kStochastic && COUPLING == KC_MEANFIELD;
        uint32_t hmax = abs_hi_max<J>(y);
        // Segments between chunk ends: the sample write sits outside the hot
        // inner loop (a branch inside it cost ~40 registers of scheduling).
        uint64_t chunk = s0 / ks;                // the chunk s0 lies in (one division per item)
        uint64_t next_sample = (chunk + 1) * ks;  // exclusive end of s0's chunk
        uint64_t step = s0;
        while (step < s1) {
          const uint64_t seg_end = next_sample < s1 ? next_sample : s1;
          for (; step < seg_end; ++step) {
            if constexpr (SOLVER == KS_EM) {
                double f[J];
                if constexpr (kStochastic && COUPLING == KC_MEANFIELD) {
                    // the meanfield form, with the step constants folded:
                    // fma(sqrt(dt)*s_i, N_i, y + (omega*dt + (K/n*dt)*S)) -- the
                    // reference's (y + f*dt) + sqrt(dt)*(s_i*N_i) reassociated,
                    // (K/n)*dt folded into the sums, the noise product unrounded
                    // (a few ulp per step): 4 FP64 ops instead of 10
                    double inc[J];
                    meanfield_folded_acc<J, PADDED>(
                        y, [&](int q) { return CSM ? cst[q * kBlock] : omdt[q]; }, kndt, base, n,
                        lanes, inc, hmax >= 0x41C00000u ? 1 : 0);
                    step_noise_apply<J, STREAM, PADDED>(
                        a, row, orbit_g, step, base, rs, [&](int q, double z) {
                            const double sq = CSM ? cst[(J + q) * kBlock] : sgs[q];
                            y[q] = __fma_rn(sq, z, __dadd_rn(y[q], inc[q]));
                        });
                } else if constexpr (kStochastic) {
                    drift<J, COUPLING, PADDED>(y, om, kn, base, n, lanes, sh, shs, f);
                    // (y + f*dt) + sqrt(dt) * (s_i * N_i)   (solvers.py:70-71, model.py:201)
                    step_noise_apply<J, STREAM, PADDED>(
                        a, row, orbit_g, step, base, rs, [&](int q, double z) {
                            const double g = __dmul_rn(sg[q], z);
                            y[q] = __dadd_rn(__dadd_rn(y[q], __dmul_rn(f[q], dt)),
                                             __dmul_rn(a.sqrt_dt, g));
                        });
                } else {
                    drift<J, COUPLING, PADDED>(y, om, kn, base, n, lanes, sh, shs, f);
#pragma unroll
                    for (int q = 0; q < J; ++q) y[q] = __dadd_rn(y[q], __dmul_rn(f[q], dt));
                }
            } else {  // KS_RK4 (solvers.py:80-88)
                double k[J], acc[J], ys[J];
                rk4_drift<J, COUPLING, PADDED>(y, om, kn, base, n, lanes, sh, shs, k);  // k1
#pragma unroll
                for (int q = 0; q < J; ++q) {
                    acc[q] = k[q];
                    ys[q] = __dadd_rn(y[q], __dmul_rn(a.half_dt, k[q]));
                }
                rk4_drift<J, COUPLING, PADDED>(ys, om, kn, base, n, lanes, sh, shs, k);  // k2
#pragma unroll
                for (int q = 0; q < J; ++q) {
                    acc[q] = __dadd_rn(acc[q], __dmul_rn(2.0, k[q]));
                    ys[q] = __dadd_rn(y[q], __dmul_rn(a.half_dt, k[q]));
                }
                rk4_drift<J, COUPLING, PADDED>(ys, om, kn, base, n, lanes, sh, shs, k);  // k3
#pragma unroll
                for (int q = 0; q < J; ++q) {
                    acc[q] = __dadd_rn(acc[q], __dmul_rn(2.0, k[q]));
                    ys[q] = __dadd_rn(y[q], __dmul_rn(dt, k[q]));
                }
                rk4_drift<J, COUPLING, PADDED>(ys, om, kn, base, n, lanes, sh, shs, k);  // k4
#pragma unroll
                for (int q = 0; q < J; ++q) {
                    acc[q] = __dadd_rn(acc[q], k[q]);
                    y[q] = __dadd_rn(y[q], __dmul_rn(a.dt6, acc[q]));
                }
            }
            // isfinite(y).all(-1) per orbit; first failure recorded, row -> NaN
            // (engine.py:244-261).  Lanes record independently; the group
            // minimum is the orbit's first failing step.  Padding oscillators
            // stay 0, so no validity predicate is needed.
            bool bad;
            if constexpr (kMagScan) {
                // one magnitude scan: the finiteness test here and the next
                // step's sincos range test (hmax)
                hmax = abs_hi_max<J>(y);
                bad = hmax >= 0x7ff00000u;
            } else {
                bad = false;
#pragma unroll
                for (int q = 0; q < J; ++q) bad |= !finite_bits(y[q]);
            }
            // a warp vote keeps the (rare) NaN fill out of the issue stream:
            // as predicated code it cost ~11 slots every step
            if (__any_sync(0xffffffffu, bad)) {
                if (bad && a.check_finite) {
                    if (fail < 0) fail = int64_t(step);
#pragma unroll
                    for (int q = 0; q < J; ++q) y[q] = CUDART_NAN;
                    hmax = 0x7ff80000u;
                }
            }
            }
            if (step == next_sample) {
                // one sample per chunk (engine.py:262)
                next_sample += ks;
                const int64_t gf = group_fail(fail, lanes);
                if (gf >= 0 && a.check_finite) {
#pragma unroll
                    for (int q = 0; q < J; ++q) y[q] = CUDART_NAN;
                }
                const int64_t c = int64_t(chunk++);  // == step / ks - 1, without a 64-bit division
                if constexpr (COH) {
                    double r, phi;
                    group_order_param<J, PADDED>(y, base, n, lanes, r, phi);
                    if (active && lane == 0) {
                        double* o = a.values + row * a.vstride * 2 + 1 + (c - a.chunk_begin);
                        o[0] = r;
                        o[a.vstride] = phi;
                    }
                } else if (active) {
                    double* out = a.values + (row * a.vstride + (c - a.chunk_begin)) * n + base;
                    bool stored = false;
                    if constexpr (!PADDED && J % 2 == 0) {
                        // unpadded rows: the lane's J doubles as 16-byte stores
                        if ((reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
                            for (int q = 0; q < J; q += 2)
                                *reinterpret_cast<double2*>(out + q) = make_double2(y[q], y[q + 1]);
                            stored = true;
                        }
                    }
                    if (!stored) {
#pragma unroll
                        for (int q = 0; q < J; ++q)
                            if (base + q < n) out[q] = y[q];
                    }
                }
            }
        }

        const int64_t gf = group_fail(fail, lanes);
        if (active) {
            if (a.state_out != nullptr) {
#pragma unroll
                for (int q = 0; q < J; ++q)
                    if (base + q < n) a.state_out[row * n + base + q] = gf >= 0 ? CUDART_NAN : y[q];
            }
            if (a.fail_step != nullptr && lane == 0) a.fail_step[row] = gf;
            if constexpr (kStateful) {
                if (a.rng_state != nullptr && base % 4 == 0) {
#pragma unroll
                    for (int t = 0; t < NB; ++t) {
                        const int b = base / 4 + t;
                        if (b < nblocks) {
                            uint64_t* p = a.rng_state + (row * nblocks + b) * 4;
                            p[0] = rs[t].s0;
                            p[1] = rs[t].s1;
                            p[2] = rs[t].s2;
                            p[3] = rs[t].s3;
                        }
                    }
                }
            }
        }
    }
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" : : "l"(p), "r"(v) : "memory");
}

// Non-persistent: CTA b advances CTA-group b over the whole launch range.
// Persistent (a.persistent): a grid of exactly the resident CTAs pulls work
// items w = slab * groups + cg from a global counter; slab k of a group waits
// (acquire) for slab k-1 to be published (release).  The smallest in-flight
// item's predecessor is always complete, so this cannot deadlock, and the
// run ends within one slab of perfectly balanced: no partially-filled last
// wave (the v3 profile lost ~13-23% to wave quantisation).
// VAR: 0 = unpadded (n == lanes * J, no per-oscillator predicates),
// 1 = padded, 2 = unpadded with registers capped (tight_minb<J>() CTAs/SM):
// more resident warps against fewer registers; the autotuner decides.
// VAR + kVarCoherence (4, 5): the same with order-parameter samples.
constexpr int kVarCoherence = 4;
template <int J>
__host__ __device__ constexpr int tight_minb() {
    return J == 4 ? 6 : (J == 8 ? 4 : 1);
}

// Instantiations with a VAR = 2 form: the register-capped J = 4 / 8 steppers,
// and the J = 16 meanfield EM stepper with its step constants in shared
// memory (CSM: 166 registers, 3 CTAs/SM for Philox) -- the autotuner picks
// between it and the register-resident form per workload (cfg3 n=256 +1.3%,
// cfg5 -2.8%: profiles/r02/experiments.md).
template <int J>
__host__ __device__ constexpr bool has_var2() {
    return tight_minb<J>() > 1 || J == 16;
}

// Dynamic shared memory a kernel instantiation needs for itself (none: the
// pairwise tiles live in registers; measured and dropped in r02: step
// constants in shared memory for J = 16, profiles/r02/experiments.md).
#ifndef SDEB_CSM16
#define SDEB_CSM16 1
#endif
template <int J, int SOLVER, int STREAM, int COUPLING, int VAR>
__host__ __device__ constexpr bool uses_const_smem() {
    return SDEB_CSM16 && J == 16 && VAR == 2 && SOLVER == KS_EM && STREAM != KS_NONE &&
           STREAM != KS_EXPLICIT && COUPLING == KC_MEANFIELD;
}

template <int J, int SOLVER, int STREAM, int COUPLING, int VAR>
__host__ __device__ constexpr size_t own_smem_bytes() {
    return uses_const_smem<J, SOLVER, STREAM, COUPLING, VAR>()
               ? size_t(2) * J * kBlock * sizeof(double)
               : 0;
}

template <int J, int SOLVER, int STREAM, int COUPLING, int VAR>
__global__ void __launch_bounds__(kBlock, (VAR == 2 && tight_minb<J>() > 1 ? tight_minb<J>() : 0))
    kuramoto_run_kernel(const RunArgs a) {
    constexpr bool PADDED = (VAR & 1) != 0;
    constexpr bool COH = VAR >= kVarCoherence;
    stage_tables();
    extern __shared__ double smem[];
    double* sh = smem;                  // spare: no instantiation uses dynamic smem
    double* shs = smem + J * kBlock;
    const uint64_t begin = uint64_t(a.chunk_begin) * uint64_t(a.ksteps);
    const uint64_t end = uint64_t(a.chunk_end) * uint64_t(a.ksteps);
    // One run_item call site for both modes (two inlined copies cost ~40
    // registers): the non-persistent mode is the one-item-per-CTA special case.
    __shared__ int64_t item;
    const bool persistent = a.persistent > 0;
    const uint64_t slab = persistent ? uint64_t(a.slab_steps) : end - begin;
    const int64_t nslabs = persistent ? int64_t((end - begin + slab - 1) / slab) : 1;
    const int64_t total = nslabs * a.groups;
    int64_t w = blockIdx.x;
    for (;;) {
        if (persistent) {
            if (threadIdx.x == 0)
                item = int64_t(atomicAdd(reinterpret_cast<unsigned long long*>(a.work_counter), 1ull));
            __syncthreads();
            w = item;
            __syncthreads();
        }
        if (w >= total) break;
        const int64_t cg = w % a.groups;
        const int64_t k = w / a.groups;
        if (k > 0 && threadIdx.x == 0) {
            while (ld_acquire(a.slab_done + cg) < unsigned(k)) __nanosleep(256);
        }
        if (persistent) __syncthreads();
        const uint64_t s0 = begin + uint64_t(k) * slab;
        const uint64_t s1 = s0 + slab < end ? s0 + slab : end;
        run_item<J, SOLVER, STREAM, COUPLING, PADDED, COH,
                 uses_const_smem<J, SOLVER, STREAM, COUPLING, VAR>()>(a, cg, s0, s1, k == 0, sh,
                                                                      shs);
        if (!persistent) break;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) st_release(a.slab_done + cg, unsigned(k + 1));
    }
}

// Host-side dispatch (sdeb_kuramoto_j*.cu instantiate per J).  padded=0 selects
// the predicate-free instantiation (requires n == lanes * J).
template <int J>
cudaError_t launch_kuramoto_j(const RunArgs& a, int solver, int stream, int coupling,
                              int padded, cudaStream_t st);
// Resident CTAs per SM of that kernel at the given dynamic shared memory.
template <int J>
cudaError_t occupancy_kuramoto_j(int solver, int stream, int coupling, int padded, size_t smem,
                                 int* blocks);

// The pairwise coupling's lane count for n oscillators: one lane per orbit up
// to n = 15 (J = n, the whole antisymmetric triangle in registers), else
// blocks of J = 8 (J = 16 beyond n = 256), L = next_pow2(n) / J.  A function
// of n alone: the pairwise summation order depends on (L, J).
inline int pairwise_lanes(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    if (n <= 15) return 1;
    return p / 8 <= 32 ? p / 8 : p / 16;
}

}  // namespace sdeb
