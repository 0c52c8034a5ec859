/* Independent C restatement of the noise generators -- TEST INFRASTRUCTURE ONLY.
 *
 * Cross-checks the numpy restatement in sdeb_oracle.py and the device code in
 * paper_1908_03869_b200/csrc/sdeb_rng.cuh.  Loaded by tests/ via ctypes from
 * oracle/_build/liboracle_streams.so (built by oracle/Makefile or
 * __graft_entry__.build()).
 *
 *  - Philox-4x32-10: the reference's only generator
 *    (/root/reference/pkg/src/sdebatch/rng.py:74-90).
 *  - SplitMix64, sfc64 (numpy's sfc64_next / sfc64_set_seed) and xoshiro256++
 *    (Blackman & Vigna, published algorithm): NOT in the reference; the
 *    per-(orbit, block) stream layout is the one DESIGN.md defines.
 */
#include <stdint.h>
#include <string.h>

void oracle_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * x0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * x2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ x1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ x3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        x0 = n0; x1 = n1; x2 = n2; x3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static uint64_t sfc64_next(uint64_t s[4]) {
    uint64_t tmp = s[0] + s[1] + s[3]++;
    s[0] = s[1] ^ (s[1] >> 11);
    s[1] = s[2] + (s[2] << 3);
    s[2] = rotl(s[2], 24) + tmp;
    return tmp;
}

static uint64_t xoshiro_next(uint64_t s[4]) {
    uint64_t result = rotl(s[0] + s[3], 23) + s[0];
    uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
}

/* stream: 1 = sfc64, 2 = xoshiro256++ (the sdeb200.h enum values). */
void oracle_stream_init(int stream, uint64_t seed, uint64_t orbit, uint64_t block, uint64_t s[4]) {
    uint64_t id = (orbit << 32) | (block & 0xFFFFFFFFull);
    uint64_t x = mix64(seed ^ mix64(id ^ 0x243F6A8885A308D3ull));
    uint64_t o[4];
    for (int k = 0; k < 4; ++k) { x += 0x9E3779B97F4A7C15ull; o[k] = mix64(x); }
    if (stream == 1) {
        s[0] = o[0]; s[1] = o[1]; s[2] = o[2]; s[3] = 1;
        for (int k = 0; k < 12; ++k) sfc64_next(s);
    } else {
        memcpy(s, o, sizeof(o));
    }
}

void oracle_stream_raw(int stream, uint64_t seed, uint64_t orbit, uint64_t block,
                       int64_t count, uint64_t* out) {
    uint64_t s[4];
    oracle_stream_init(stream, seed, orbit, block, s);
    for (int64_t k = 0; k < count; ++k) out[k] = stream == 1 ? sfc64_next(s) : xoshiro_next(s);
}

/* Raw outputs from an explicit state (for KATs: numpy-seeded sfc64, {1,2,3,4} xoshiro). */
void oracle_stream_raw_from_state(int stream, const uint64_t state[4], int64_t count, uint64_t* out) {
    uint64_t s[4];
    memcpy(s, state, sizeof(s));
    for (int64_t k = 0; k < count; ++k) out[k] = stream == 1 ? sfc64_next(s) : xoshiro_next(s);
}

void oracle_sfc64_set_seed(const uint64_t seed3[3], uint64_t s[4]) {
    s[0] = seed3[0]; s[1] = seed3[1]; s[2] = seed3[2]; s[3] = 1;
    for (int k = 0; k < 12; ++k) sfc64_next(s);
}
