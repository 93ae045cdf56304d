/*
 * TEST INFRASTRUCTURE (oracle side) -- not part of the shipped product.
 *
 * Counter-based random stream shared by every CPU checker under oracle/:
 *   - the stream-shim build of the UNMODIFIED reference sampler
 *     (oracle/shim/epochbc/rng.hpp shadows /root/reference/proj/include/epochbc/rng.hpp:30-52)
 *   - the plain-C restatement (oracle/ebc_oracle.c).
 *
 * The reference's own Rng is std::mt19937_64 + libstdc++ distributions
 * (rng.hpp:41-51), whose engine-output -> variate mapping is implementation
 * defined.  SURVEY.md section 8c replaces it ON BOTH SIDES by Philox-4x32-10
 * (Salmon et al., SC'11, "Parallel random numbers: as easy as 1, 2, 3") so a
 * sample's draws depend only on (seed, phase tag, global sample index, draw #).
 *
 * Stream definition (must be byte-identical in the CUDA product, which carries
 * its own independent implementation in paper_1910_11039_b200/csrc/philox.cuh):
 *   key     = (seed & 0xffffffff, seed >> 32)
 *   counter = (draw, tag, index & 0xffffffff, index >> 32)
 *   next_u64()      = out[0] | out[1] << 32 of that block; draw += 1
 *   next_below(b)   = Lemire multiply-shift with rejection (unbiased):
 *                       m = x*b (128 bit); if lo64(m) < b { t = (-b) % b;
 *                       while lo64(m) < t redraw }  return hi64(m)
 *   next_double()   = (next_u64() >> 11) * 2^-53
 */
#ifndef EBC_ORACLE_PHILOX_H
#define EBC_ORACLE_PHILOX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint32_t key[2];
    uint32_t tag;
    uint32_t idx_lo, idx_hi;
    uint32_t draw;
} ebc_stream;

static inline void ebc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static inline void ebc_stream_init(ebc_stream *s, uint64_t seed, uint32_t tag, uint64_t index) {
    s->key[0] = (uint32_t)seed;
    s->key[1] = (uint32_t)(seed >> 32);
    s->tag = tag;
    s->idx_lo = (uint32_t)index;
    s->idx_hi = (uint32_t)(index >> 32);
    s->draw = 0;
}

static inline uint64_t ebc_stream_u64(ebc_stream *s) {
    uint32_t ctr[4] = {s->draw, s->tag, s->idx_lo, s->idx_hi};
    uint32_t out[4];
    ebc_philox4x32_10(ctr, s->key, out);
    s->draw += 1;
    return (uint64_t)out[0] | ((uint64_t)out[1] << 32);
}

static inline uint64_t ebc_stream_below(ebc_stream *s, uint64_t bound) {
    unsigned __int128 m = (unsigned __int128)ebc_stream_u64(s) * bound;
    uint64_t lo = (uint64_t)m;
    if (lo < bound) {
        uint64_t t = (0 - bound) % bound;
        while (lo < t) {
            m = (unsigned __int128)ebc_stream_u64(s) * bound;
            lo = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

static inline double ebc_stream_double(ebc_stream *s) {
    return (double)(ebc_stream_u64(s) >> 11) * (1.0 / 9007199254740992.0);
}

#ifdef __cplusplus
}
#endif
#endif
