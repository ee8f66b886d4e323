// amz_rng.cuh -- numpy-compatible random streams for device (and host key setup).
//
// The reference draws every level from
//   Generator(Philox(SeedSequence(entropy, spawn_key=key)))      (rng.py:43-50)
// so bit-exact levels on the GPU need numpy's exact stream consumption:
//   * SeedSequence: 4-word pool, hashmix/mix over the assembled entropy words, then
//     generate_state(2, uint64) -> Philox key; counter starts at 0.
//   * Philox4x64-10; the bit generator hands out the 4 u64 of a block in order
//     (pre-incrementing counter[0] before each block).
//   * next_uint32 returns the pending upper half of the previous 64-bit draw if any,
//     else takes a fresh u64, returns its low half and keeps the high half pending.
//     random() takes a fresh u64 and leaves the pending half alone.
//   * integers(0, n), n < 2^32: 32-bit Lemire rejection on next_uint32.
//   * permutation: Fisher-Yates from the top with masked-rejection random_interval.
// The device never hashes the full key: the host absorbs the common key prefix once
// (amz_seed_t) and each lane mixes only its suffix words (1-2 words).
#pragma once
#include <stdint.h>

#include "../../include/amaze_b200.h"

#if defined(__CUDACC__)
#define AMZ_HD __host__ __device__ __forceinline__
#else
#define AMZ_HD inline
#endif

namespace amz {

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

AMZ_HD uint32_t ss_hashmix(uint32_t v, uint32_t &hc) {
    v ^= hc;
    hc *= kMultA;
    v *= hc;
    return v ^ (v >> 16);
}

AMZ_HD uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = kMixL * x - kMixR * y;
    return r ^ (r >> 16);
}

// words[0..3] initialise the pool (absent words hash as 0), then cross-mix.
AMZ_HD void seed_init(amz_seed_t &s, const uint32_t *w, int n) {
    s.hash_const = kInitA;
    for (int i = 0; i < 4; i++) s.pool[i] = ss_hashmix(i < n ? w[i] : 0u, s.hash_const);
    for (int a = 0; a < 4; a++)
        for (int b = 0; b < 4; b++)
            if (a != b) s.pool[b] = ss_mix(s.pool[b], ss_hashmix(s.pool[a], s.hash_const));
    s.n_words = 4;
}

// Every word past the 4th is mixed into all pool words in turn.
AMZ_HD void seed_absorb(amz_seed_t &s, uint32_t w) {
#pragma unroll
    for (int d = 0; d < 4; d++) s.pool[d] = ss_mix(s.pool[d], ss_hashmix(w, s.hash_const));
    s.n_words++;
}

AMZ_HD void seed_key(const amz_seed_t &s, uint64_t &k0, uint64_t &k1) {
    uint32_t h = kInitB, o[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        uint32_t v = s.pool[i] ^ h;
        h *= kMultB;
        v *= h;
        o[i] = v ^ (v >> 16);
    }
    k0 = (uint64_t)o[0] | ((uint64_t)o[1] << 32);
    k1 = (uint64_t)o[2] | ((uint64_t)o[3] << 32);
}

AMZ_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// Philox4x64-10 on counter (c0, 0, 0, 0): the upper counter words stay 0 for any
// stream shorter than 2^64 blocks, so only c0 is carried.
AMZ_HD void philox_block(uint64_t c0, uint64_t k0, uint64_t k1, uint64_t &o0, uint64_t &o1,
                         uint64_t &o2, uint64_t &o3) {
    uint64_t x0 = c0, x1 = 0, x2 = 0, x3 = 0;
#pragma unroll
    for (int r = 0; r < 10; r++) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ull;
            k1 += 0xBB67AE8584CAA73Bull;
        }
        const uint64_t m0 = 0xD2E7470EE14C6C93ull, m1 = 0xCA5A826395121157ull;
        uint64_t h0 = mulhi64(m0, x0), l0 = m0 * x0;
        uint64_t h1 = mulhi64(m1, x2), l1 = m1 * x2;
        uint64_t n0 = h1 ^ x1 ^ k0, n2 = h0 ^ x3 ^ k1;
        x0 = n0;
        x1 = l1;
        x2 = n2;
        x3 = l0;
    }
    o0 = x0;
    o1 = x1;
    o2 = x2;
    o3 = x3;
}

// numpy's Philox bit generator + the Generator methods the reference calls.
struct Stream {
    uint64_t k0, k1, ctr;
    uint64_t b0, b1, b2, b3;
    uint32_t pos;  // next u64 of the block to hand out (4 = exhausted)
    uint32_t half;
    bool has_half;

    AMZ_HD void init(uint64_t key0, uint64_t key1) {
        k0 = key0;
        k1 = key1;
        ctr = 0;
        pos = 4;
        has_half = false;
        half = 0;
        b0 = b1 = b2 = b3 = 0;
    }
    AMZ_HD void init(const amz_seed_t &s) {
        uint64_t a, b;
        seed_key(s, a, b);
        init(a, b);
    }
    AMZ_HD uint64_t next64() {
        if (pos >= 4) {
            ++ctr;
            philox_block(ctr, k0, k1, b0, b1, b2, b3);
            pos = 0;
        }
        uint64_t v = pos == 0 ? b0 : pos == 1 ? b1 : pos == 2 ? b2 : b3;
        ++pos;
        return v;
    }
    AMZ_HD uint32_t next32() {
        if (has_half) {
            has_half = false;
            return half;
        }
        uint64_t v = next64();
        has_half = true;
        half = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
    // Generator.random(): 53-bit double in [0, 1)
    AMZ_HD double random() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
    // Generator.integers(0, n) for 1 <= n < 2^32 (Lemire, 32-bit)
    AMZ_HD uint32_t below(uint32_t n) {
        if (n <= 1u) return 0u;
        uint64_t m = (uint64_t)next32() * n;
        uint32_t left = (uint32_t)m;
        if (left < n) {
            uint32_t thresh = (0u - n) % n;
            while (left < thresh) {
                m = (uint64_t)next32() * n;
                left = (uint32_t)m;
            }
        }
        return (uint32_t)(m >> 32);
    }
    // random_interval(max), 1 <= max < 2^32 (masked rejection)
    AMZ_HD uint32_t interval(uint32_t max) {
#if defined(__CUDA_ARCH__)
        uint32_t mask = 0xFFFFFFFFu >> __clz(max);
#else
        uint32_t mask = 0xFFFFFFFFu >> __builtin_clz(max);
#endif
        uint32_t v;
        do {
            v = next32() & mask;
        } while (v > max);
        return v;
    }
};

// Host: numpy _int_to_uint32_array + SeedSequence assembly of a key prefix.
inline int seed_prefix_host(const uint32_t *run, int n_run, const uint32_t *key, int n_key, amz_seed_t &out) {
    uint32_t w[4] = {0, 0, 0, 0};
    int n0 = n_run < 4 ? 4 : n_run;  // padded because the final spawn key is non-empty
    for (int i = 0; i < 4; i++) {
        int idx = i;
        if (idx < n_run)
            w[i] = run[idx];
        else if (idx < n0)
            w[i] = 0u;
        else
            w[i] = key[idx - n0];
    }
    // total words available so far
    int total = n0 + n_key;
    seed_init(out, w, total < 4 ? total : 4);
    for (int i = 4; i < total; i++) {
        uint32_t v = i < n_run ? run[i] : (i < n0 ? 0u : key[i - n0]);
        seed_absorb(out, v);
    }
    out.n_words = (uint32_t)total;
    return 0;
}

}  // namespace amz
