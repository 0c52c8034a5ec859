// Device noise generators and the Gaussian transform.
//
// Philox-4x32-10 and the (w+1)*2^-32 / Box-Muller transform follow the
// reference exactly (rng.py:31-45, 74-142, 150-188 under
// /root/reference/pkg/src/sdebatch): the integer words are bit-exact; the
// normals differ from numpy's only by the device log/sqrt/sincos rounding.
// SplitMix64 / sfc64 / xoshiro256++ are the extra per-(orbit, block) streams
// DESIGN.md defines ("Noise streams"); they are not in the reference.
#pragma once
#include "sdeb_cstdint.cuh"

#include "sdeb_math.cuh"

namespace sdeb {

constexpr double kTwoPi = 6.283185307179586;      // 2.0 * math.pi (rng.py:45)
constexpr double kTwoNeg32 = 2.3283064365386963e-10;  // 2**-32 (rng.py:44)
constexpr uint32_t kSamplingTag = 0xFFFFFFFFu;       // rng.py:42

struct Words4 {
    uint32_t w0, w1, w2, w3;
};

// rng.py:74-90 / 93-118: x0'=hi(M1*x2)^x1^k0, x1'=lo(M1*x2), x2'=hi(M0*x0)^x3^k1, x3'=lo(M0*x0)
__host__ __device__ __forceinline__ Words4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                         uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
#else
        const uint64_t p0 = uint64_t(0xD2511F53u) * c0, p1 = uint64_t(0xCD9E8D57u) * c2;
        const uint32_t hi0 = uint32_t(p0 >> 32), lo0 = uint32_t(p0);
        const uint32_t hi1 = uint32_t(p1 >> 32), lo1 = uint32_t(p1);
#endif
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return Words4{c0, c1, c2, c3};
}

// to_uniform (rng.py:121-129): (w + 1.0) * 2^-32, exact in double.
__device__ __forceinline__ double to_uniform(uint32_t w) { return u32_to_uniform(w); }

// One Box-Muller pair in the reference's form (rng.py:179-187):
// r = sqrt(-2 ln u_a); (r cos(2 pi u_b), r sin(2 pi u_b)).  The angle's sincos
// is reduced in integer arithmetic from the word itself (sincos_turn).
__device__ __forceinline__ void box_muller_pair(uint32_t wa, uint32_t wb, double& z0, double& z1) {
    const double ua = u32_to_uniform(wa);
    const double r = sqrt_nonneg(neg2_log_pos(ua));  // sqrt(-2 ln u)
    double s, c;
    sincos_turn(wb, s, c);
    z0 = __dmul_rn(r, c);
    z1 = __dmul_rn(r, s);
}

// ---- SplitMix64 seeding + sfc64 / xoshiro256++ ----------------------------

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) {
    return (x << k) | (x >> (64 - k));
}

struct StreamState {
    uint64_t s0, s1, s2, s3;
};

// numpy sfc64_next: s = (a, b, c, counter)
__host__ __device__ __forceinline__ uint64_t sfc64_next(StreamState& s) {
    const uint64_t tmp = s.s0 + s.s1 + s.s3;
    s.s3 += 1;
    s.s0 = s.s1 ^ (s.s1 >> 11);
    s.s1 = s.s2 + (s.s2 << 3);
    s.s2 = rotl64(s.s2, 24) + tmp;
    return tmp;
}

__host__ __device__ __forceinline__ uint64_t xoshiro256pp_next(StreamState& s) {
    const uint64_t result = rotl64(s.s0 + s.s3, 23) + s.s0;
    const uint64_t t = s.s1 << 17;
    s.s2 ^= s.s0;
    s.s3 ^= s.s1;
    s.s1 ^= s.s2;
    s.s0 ^= s.s3;
    s.s2 ^= t;
    s.s3 = rotl64(s.s3, 45);
    return result;
}

template <int STREAM>
__host__ __device__ __forceinline__ uint64_t stream_next(StreamState& s) {
    if constexpr (STREAM == 1) {
        return sfc64_next(s);
    } else {
        return xoshiro256pp_next(s);
    }
}

// Per-(orbit, block) origin: mix64(seed ^ mix64((orbit<<32 | block) ^ salt)),
// then SplitMix64 outputs o1..o4.  sfc64: (o1, o2, o3, 1) + 12 discarded
// outputs (numpy's sfc64_set_seed); xoshiro256++: (o1, o2, o3, o4).
template <int STREAM>
__host__ __device__ __forceinline__ StreamState stream_init(uint64_t seed, uint64_t orbit,
                                                            uint64_t block) {
    const uint64_t id = (orbit << 32) | (block & 0xFFFFFFFFull);
    uint64_t x = mix64(seed ^ mix64(id ^ 0x243F6A8885A308D3ull));
    uint64_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        x += 0x9E3779B97F4A7C15ull;
        o[k] = mix64(x);
    }
    StreamState s;
    if constexpr (STREAM == 1) {
        s = StreamState{o[0], o[1], o[2], 1ull};
#pragma unroll 1
        for (int k = 0; k < 12; ++k) sfc64_next(s);
    } else {
        s = StreamState{o[0], o[1], o[2], o[3]};
    }
    return s;
}

// One 4-word block from a stateful stream: two outputs split (lo32, hi32).
template <int STREAM>
__host__ __device__ __forceinline__ Words4 stream_block(StreamState& s) {
    const uint64_t a = stream_next<STREAM>(s);
    const uint64_t b = stream_next<STREAM>(s);
    return Words4{uint32_t(a), uint32_t(a >> 32), uint32_t(b), uint32_t(b >> 32)};
}

}  // namespace sdeb
