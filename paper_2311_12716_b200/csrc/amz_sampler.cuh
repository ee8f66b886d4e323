// amz_sampler.cuh -- warp-cooperative sample_random_level (amaze/generator.py:36-52).
//
// One level per warp, bit-identical to numpy's stream consumption:
//   * the level's Philox4x64-10 blocks are counter-indexed, so lane b computes block
//     b+1 and the warp stages the first kNB blocks (kNB*8 u32 words) in shared memory;
//     words past that are computed on demand (numpy's next_uint32 order: lo, hi of each
//     u64, u64s in block order);
//   * integers(0, n) (Lemire) draws run as uniform scalar code;
//   * the Fisher-Yates of permutation(ni) needs, per step i, the first draw at or after
//     the stream position whose masked value is <= i.  The warp tests 32 consecutive
//     words at once (ballot + find-first), so a step costs a handful of dependent
//     instructions instead of a rejection loop;
//   * instead of materialising the permuted array, every lane tracks the final
//     positions of its (up to 4) elements under the transpositions (i, j_i); the wall
//     mask is then "elements whose final position < n_walls" (an OR-reduction), and
//     the goal/agent are the elements at two final positions (a ballot).
#pragma once
#include <stdint.h>

#include "amz_level.cuh"

namespace amz {

constexpr int kWNB = 28;  // staged Philox blocks (224 words; a 13x13 level uses ~172 on average)
constexpr int kWNW = kWNB * 8;

struct WarpStream {
    const uint32_t *sw;  // this warp's staged words [kWNW]
    uint64_t k0, k1;

    __device__ __forceinline__ uint32_t word(uint32_t q) const {
        if (q < (uint32_t)kWNW) return sw[q];
        uint64_t o0, o1, o2, o3;
        philox_block((uint64_t)(q >> 3) + 1ull, k0, k1, o0, o1, o2, o3);
        const uint32_t j = (q & 7u) >> 1;
        const uint64_t v = j == 0 ? o0 : j == 1 ? o1 : j == 2 ? o2 : o3;
        return (q & 1u) ? (uint32_t)(v >> 32) : (uint32_t)v;
    }
    // Generator.integers(0, n) on next_uint32 (uniform across the warp)
    __device__ __forceinline__ uint32_t below(uint32_t &p, uint32_t n) const {
        if (n <= 1u) return 0u;
        uint64_t m = (uint64_t)word(p++) * n;
        uint32_t left = (uint32_t)m;
        if (left < n) {
            const uint32_t thresh = (0u - n) % n;
            while (left < thresh) {
                m = (uint64_t)word(p++) * n;
                left = (uint32_t)m;
            }
        }
        return (uint32_t)(m >> 32);
    }
};

__device__ __forceinline__ void warp_stage_stream(uint64_t k0, uint64_t k1, uint32_t *sw) {
    const int lane = threadIdx.x & 31;
    if (lane < kWNB) {
        uint64_t o0, o1, o2, o3;
        philox_block((uint64_t)lane + 1ull, k0, k1, o0, o1, o2, o3);
        uint4 *d = reinterpret_cast<uint4 *>(sw + 8 * lane);
        d[0] = make_uint4((uint32_t)o0, (uint32_t)(o0 >> 32), (uint32_t)o1, (uint32_t)(o1 >> 32));
        d[1] = make_uint4((uint32_t)o2, (uint32_t)(o2 >> 32), (uint32_t)o3, (uint32_t)(o3 >> 32));
    }
    __syncwarp();
}

// All 32 lanes call with the same key; every lane returns the same level.
// `sw` = this warp's 16-byte aligned scratch of kWNW words.
__device__ __forceinline__ void warp_sample_level(uint64_t k0, uint64_t k1, const Geo &G, uint32_t *sw, Mask &mask,
                                                  int &ar, int &ac, int &ad, int &gr, int &gc) {
    const int lane = threadIdx.x & 31;
    warp_stage_stream(k0, k1, sw);
    const WarpStream S{sw, k0, k1};
    uint32_t p = 0;
    const uint32_t nw = S.below(p, (uint32_t)G.budget + 1u);
    // final positions of the elements this lane owns (lane, lane+32, lane+64, lane+96)
    int pos0 = lane, pos1 = lane + 32, pos2 = lane + 64, pos3 = lane + 96;
    uint32_t wb = p, w = S.word(wb + lane);
    for (int i = G.ni - 1; i >= 1; i--) {
        const uint32_t mk = 0xFFFFFFFFu >> __clz(i);
        int j;
        while (true) {
            const int o = (int)(p - wb);
            const bool ok = lane >= o && (w & mk) <= (uint32_t)i;
            const unsigned b = __ballot_sync(0xFFFFFFFFu, ok);
            if (b) {
                const int f = __ffs(b) - 1;
                j = (int)(__shfl_sync(0xFFFFFFFFu, w, f) & mk);
                p = wb + f + 1;
                break;
            }
            wb += 32;
            w = S.word(wb + lane);
        }
        pos0 = pos0 == i ? j : (pos0 == j ? i : pos0);
        pos1 = pos1 == i ? j : (pos1 == j ? i : pos1);
        pos2 = pos2 == i ? j : (pos2 == j ? i : pos2);
        pos3 = pos3 == i ? j : (pos3 == j ? i : pos3);
    }
    // walls: elements whose final position is below n_walls
    const int ni = G.ni;
    const uint32_t b0 = (lane < ni && pos0 < (int)nw) ? 1u : 0u;
    const uint32_t b1 = (lane + 32 < ni && pos1 < (int)nw) ? 1u : 0u;
    const uint32_t b2 = (lane + 64 < ni && pos2 < (int)nw) ? 1u : 0u;
    const uint32_t b3 = (lane + 96 < ni && pos3 < (int)nw) ? 1u : 0u;
    mask.w[0] = __ballot_sync(0xFFFFFFFFu, b0);
    mask.w[1] = __ballot_sync(0xFFFFFFFFu, b1);
    mask.w[2] = __ballot_sync(0xFFFFFFFFu, b2);
    mask.w[3] = __ballot_sync(0xFFFFFFFFu, b3);
    // goal = free[gk], agent = (free without goal)[ak]; free = final positions nw..ni-1
    const uint32_t nfree = (uint32_t)ni - nw;
    const uint32_t gk = S.below(p, nfree);
    const uint32_t ak = S.below(p, nfree - 1u);
    ad = (int)S.below(p, 4u);
    const int pg = (int)(nw + gk), pa = (int)(nw + (ak < gk ? ak : ak + 1u));
    auto elem_at = [&](int target) {
        int e = -1;
        if (lane < ni && pos0 == target) e = lane;
        if (lane + 32 < ni && pos1 == target) e = lane + 32;
        if (lane + 64 < ni && pos2 == target) e = lane + 64;
        if (lane + 96 < ni && pos3 == target) e = lane + 96;
        const unsigned b = __ballot_sync(0xFFFFFFFFu, e >= 0);
        return __shfl_sync(0xFFFFFFFFu, e, __ffs(b) - 1);
    };
    const int goal = elem_at(pg), agent = elem_at(pa);
    gr = goal / G.iw + 1;
    gc = goal % G.iw + 1;
    ar = agent / G.iw + 1;
    ac = agent % G.iw + 1;
}

}  // namespace amz

namespace amz {

// ---------------------------------------------------------------------------------
// Staged SIMT sampler: every lane whose bit is set in `need` samples its OWN level.
// The whole warp first computes the Philox blocks of all requesting lanes round-robin
// (block b of requesting lane L is one work item) into per-lane word columns of `sw`
// ([kSNW][LPW], word q of lane L at q*LPW + L); then each requesting lane runs the
// sequential Fisher-Yates over its staged words, continuing with inline blocks in the
// rare case the level needs more than kSNB blocks.  Cost per batch of W levels:
// ceil(28W/32) Philox blocks per thread + one Fisher-Yates (SIMT over the W lanes).
// ---------------------------------------------------------------------------------
constexpr int kSNB = 24;
constexpr int kSNW = kSNB * 8;

struct LaneStream {
    const uint32_t *w;
    int stride;
    uint32_t p;
    uint64_t k0, k1;
    uint64_t cb;
    uint64_t c0, c1, c2, c3;

    __device__ __forceinline__ uint32_t next32() {
        if (p < (uint32_t)kSNW) return w[(p++) * stride];
        const uint64_t blk = p >> 3;
        if (cb != blk + 1) {
            philox_block(blk + 1, k0, k1, c0, c1, c2, c3);
            cb = blk + 1;
        }
        const uint32_t j = (p & 7u) >> 1;
        const uint64_t v = j == 0 ? c0 : j == 1 ? c1 : j == 2 ? c2 : c3;
        const bool hi = p & 1u;
        p++;
        return hi ? (uint32_t)(v >> 32) : (uint32_t)v;
    }
    __device__ __forceinline__ uint32_t below(uint32_t n) {
        if (n <= 1u) return 0u;
        uint64_t m = (uint64_t)next32() * n;
        uint32_t left = (uint32_t)m;
        if (left < n) {
            const uint32_t thresh = (0u - n) % n;
            while (left < thresh) {
                m = (uint64_t)next32() * n;
                left = (uint32_t)m;
            }
        }
        return (uint32_t)(m >> 32);
    }
    __device__ __forceinline__ uint32_t interval(uint32_t max) {
        const uint32_t mk = 0xFFFFFFFFu >> __clz(max);
        uint32_t v;
        do {
            v = next32() & mk;
        } while (v > max);
        return v;
    }
};

// sample_random_level over any 32-bit draw source (amaze/generator.py:36-52);
// `perm` is this lane's ni-byte column (stride `ps`).
template <class Src>
__device__ __forceinline__ void sample_level_seq(Src &g, const Geo &G, uint8_t *perm, int ps, Mask &mask, int &ar,
                                                 int &ac, int &ad, int &gr, int &gc) {
    const uint32_t nw = g.below((uint32_t)G.budget + 1u);
    for (int i = 0; i < G.ni; i++) perm[i * ps] = (uint8_t)i;
    for (int i = G.ni - 1; i >= 1; i--) {
        const uint32_t j = g.interval((uint32_t)i);
        const uint8_t a = perm[i * ps], b = perm[j * ps];
        perm[i * ps] = b;
        perm[j * ps] = a;
    }
    mask.w[0] = mask.w[1] = mask.w[2] = mask.w[3] = 0u;
    for (uint32_t k = 0; k < nw; k++) mask_set(mask, perm[k * ps], 1u);
    const uint32_t nfree = (uint32_t)G.ni - nw;
    const uint32_t gk = g.below(nfree);
    const int goal = perm[(nw + gk) * ps];
    const uint32_t ak = g.below(nfree - 1u);
    const int agent = perm[(nw + (ak < gk ? ak : ak + 1u)) * ps];
    ad = (int)g.below(4u);
    gr = goal / G.iw + 1;
    gc = goal % G.iw + 1;
    ar = agent / G.iw + 1;
    ac = agent % G.iw + 1;
}

// All 32 lanes of the warp call this (uniform `need`); lanes with their bit set get a
// level for their own key (k0, k1).  skey: [LPW] x 2 u64 scratch.
template <int LPW>
__device__ __forceinline__ void warp_sample_batch(unsigned need, uint64_t k0, uint64_t k1, const Geo &G,
                                                  uint32_t *sw, uint8_t *perm, uint64_t *skey, Mask &mask, int &ar,
                                                  int &ac, int &ad, int &gr, int &gc) {
    const int lane = threadIdx.x & 31;
    const bool mine = (need >> lane) & 1u;
    if (mine) {
        skey[2 * lane] = k0;
        skey[2 * lane + 1] = k1;
    }
    __syncwarp();
    const int cnt = __popc(need);
    for (int x = lane; x < cnt * kSNB; x += 32) {
        const int idx = x / kSNB, b = x - idx * kSNB;
        const int L = (int)__fns(need, 0, idx + 1);
        uint64_t o0, o1, o2, o3;
        philox_block((uint64_t)b + 1ull, skey[2 * L], skey[2 * L + 1], o0, o1, o2, o3);
        uint32_t *d = sw + (8 * b) * LPW + L;
        d[0 * LPW] = (uint32_t)o0;
        d[1 * LPW] = (uint32_t)(o0 >> 32);
        d[2 * LPW] = (uint32_t)o1;
        d[3 * LPW] = (uint32_t)(o1 >> 32);
        d[4 * LPW] = (uint32_t)o2;
        d[5 * LPW] = (uint32_t)(o2 >> 32);
        d[6 * LPW] = (uint32_t)o3;
        d[7 * LPW] = (uint32_t)(o3 >> 32);
    }
    __syncwarp();
    if (mine) {
        LaneStream s{sw + lane, LPW, 0u, k0, k1, 0ull, 0ull, 0ull, 0ull, 0ull};
        sample_level_seq(s, G, perm + lane, LPW, mask, ar, ac, ad, gr, gc);
    }
    __syncwarp();
}

}  // namespace amz
