// amz_sampler.cuh -- warp-cooperative sample_random_level (amaze/generator.py:36-52).
//
// One level per warp, bit-identical to numpy's stream consumption:
//   * the level's Philox4x64-10 blocks are counter-indexed, so lane b computes block
//     b+1 and the warp stages the first kWNB blocks (kWNB*8 u32 words) in shared memory;
//     words past that are computed on demand (numpy's next_uint32 order: lo, hi of each
//     u64, u64s in block order);
//   * integers(0, n) (Lemire) draws run as uniform scalar code;
//   * the Fisher-Yates of permutation(ni) (masked rejection per step) is resolved 32
//     stream words at a time, and the permuted array is read off the transpositions
//     without replaying them (see warp_sample_level).
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

// Per-warp shared scratch of warp_sample_level.
struct WarpSampler {
    uint32_t sw[kWNW];   // staged stream words
    uint32_t L[128][4];  // L[q]: bit set of the steps i with j_i == q (128-bit)
    __align__(16) uint8_t J[128];  // j_i of Fisher-Yates step i (J[0] = 0)
    uint8_t T[128];      // terminal of the succ chain from i (pointer jumping)
};

// Phase 2 of warp_sample_level: kTrack = false reads the permutation off the swap lists
// (fewest instructions: throughput kernels that sample many levels); kTrack = true
// follows each lane's 4 elements through the 120 transpositions (4 independent select
// chains: lowest latency for one level on the dynamics' critical path).

// smallest element > after of the 128-bit set L[q], or -1
__device__ __forceinline__ int set_next(const WarpSampler &X, int q, int after) {
    const int s = after + 1;
    for (int w = s >> 5; w < 4; w++) {
        uint32_t bits = X.L[q][w];
        if (w == (s >> 5)) bits &= ~0u << (s & 31);
        if (bits) return w * 32 + __ffs(bits) - 1;
    }
    return -1;
}

// All 32 lanes call with the same key; every lane returns the same level.
//   1. j_i for every step i (numpy's masked rejection, i = ni-1 .. 1) in windows of 32
//      stream words.  Word k of a window serves step i - c_k, c_k = accepted words
//      before it, and is accepted iff (w_k & mask(i - c_k)) <= i - c_k: a triangular
//      system solved by Jacobi sweeps (ballot + popc) from "all accepted"; it reaches
//      the unique fixed point in ~4 sweeps, so a window settles ~25 steps at once.
//   2. the permuted array without replaying the swaps: reading the transpositions
//      backwards, position k holds the element reached by jumping first to the next
//      step after k that drew the same j as k (or to j_k itself if there is none), then
//      along succ(q) = first step after q that drew q.  The succ chains are collapsed by
//      pointer jumping.
#ifdef AMZ_SAMP_PROF
__device__ long long g_samp_prof[8];
#define SAMP_T(k_) \
    do { if ((threadIdx.x & 31) == 0) g_samp_prof[k_] += clock64(); } while (0)
#else
#define SAMP_T(k_) \
    do {           \
    } while (0)
#endif
template <bool kTrack = false>
__device__ __forceinline__ void warp_sample_level(uint64_t k0, uint64_t k1, const Geo &G, WarpSampler &X, Mask &mask,
                                                  int &ar, int &ac, int &ad, int &gr, int &gc) {
    const int lane = threadIdx.x & 31;
    const int ni = G.ni;
    if (!kTrack)
        for (int x = lane; x < 128; x += 32) reinterpret_cast<uint4 *>(&X.L[0][0])[x] = make_uint4(0u, 0u, 0u, 0u);
    SAMP_T(0);
    warp_stage_stream(k0, k1, X.sw);
    SAMP_T(1);
    const WarpStream S{X.sw, k0, k1};
    uint32_t p = 0;
    const uint32_t nw = S.below(p, (uint32_t)G.budget + 1u);
    SAMP_T(2);
    // ---- 1. j_i ----
    const unsigned lt = (1u << lane) - 1u;
    int i = ni - 1;
    while (i >= 1) {
        const uint32_t w = S.word(p + lane);
        // c = accepted words before this lane; the step this word serves is i - c.
        // Jacobi sweep from "all accepted" to the (unique) fixed point.
        int c = lane, ik;
        bool acc;
        uint32_t v;
        unsigned A;
        while (true) {
            ik = i - c;
            v = ik >= 1 ? (w & (0xFFFFFFFFu >> __clz(ik))) : 0xFFFFFFFFu;
            acc = ik >= 1 && v <= (uint32_t)ik;
            A = __ballot_sync(0xFFFFFFFFu, acc);
            const int c2 = __popc(A & lt);
            if (__all_sync(0xFFFFFFFFu, c2 == c)) break;
            c = c2;
        }
        if (acc) X.J[ik] = (uint8_t)v;
        const int na = __popc(A);
        p += (i - na >= 1) ? 32u : (uint32_t)(32 - __clz(A));  // through the last accepted word
        i -= na;
    }
    if (lane == 0) X.J[0] = 0;
    __syncwarp();
    SAMP_T(3);
    if (kTrack) {
        // ---- 2. final positions of this lane's elements ----
        int q0 = lane, q1 = lane + 32, q2 = lane + 64, q3 = lane + 96;
#pragma unroll 4
        for (int i = ni - 1; i >= 1; i--) {
            const int j = X.J[i];
            q0 = q0 == i ? j : (q0 == j ? i : q0);
            q1 = q1 == i ? j : (q1 == j ? i : q1);
            q2 = q2 == i ? j : (q2 == j ? i : q2);
            q3 = q3 == i ? j : (q3 == j ? i : q3);
        }
        SAMP_T(4);
        mask.w[0] = __ballot_sync(0xFFFFFFFFu, lane < ni && q0 < (int)nw);
        mask.w[1] = __ballot_sync(0xFFFFFFFFu, lane + 32 < ni && q1 < (int)nw);
        mask.w[2] = __ballot_sync(0xFFFFFFFFu, lane + 64 < ni && q2 < (int)nw);
        mask.w[3] = __ballot_sync(0xFFFFFFFFu, lane + 96 < ni && q3 < (int)nw);
        auto element = [&](int target) {  // the element whose final position is target
            const int e = (lane < ni && q0 == target)        ? lane
                          : (lane + 32 < ni && q1 == target) ? lane + 32
                          : (lane + 64 < ni && q2 == target) ? lane + 64
                          : (lane + 96 < ni && q3 == target) ? lane + 96
                                                             : -1;
            const unsigned b = __ballot_sync(0xFFFFFFFFu, e >= 0);
            return __shfl_sync(0xFFFFFFFFu, e, __ffs(b) - 1);
        };
        // goal = free[gk], agent = (free without goal)[ak]; free = final positions nw..ni-1
        const uint32_t nfree = (uint32_t)ni - nw;
        const uint32_t gk = S.below(p, nfree);
        const uint32_t ak = S.below(p, nfree - 1u);
        ad = (int)S.below(p, 4u);
        const int goal = element((int)(nw + gk)), agent = element((int)(nw + (ak < gk ? ak : ak + 1u)));
        gr = goal / G.iw + 1;
        gc = goal % G.iw + 1;
        ar = agent / G.iw + 1;
        ac = agent % G.iw + 1;
        SAMP_T(5);
    } else {
        // ---- 2. final positions ----
        for (int k = lane; k < ni; k += 32) atomicOr(&X.L[X.J[k]][k >> 5], 1u << (k & 31));
        __syncwarp();
        for (int k = lane; k < ni; k += 32) {
            const int sn = set_next(X, k, k);
            X.T[k] = (uint8_t)(sn >= 0 ? sn : k);
        }
        __syncwarp();
        while (true) {  // T[k] <- T[T[k]] until every chain is collapsed
            bool moved = false;
            for (int k = lane; k < ni; k += 32) {
                const int t = X.T[k], tt = X.T[t];
                if (tt != t) {
                    X.T[k] = (uint8_t)tt;
                    moved = true;
                }
            }
            __syncwarp();
            if (!__any_sync(0xFFFFFFFFu, moved)) break;
        }
        auto element = [&](int k) {
            const int q = X.J[k];
            const int sn = set_next(X, q, k);
            return sn >= 0 ? (int)X.T[sn] : q;
        };
        uint32_t m0 = 0u, m1 = 0u, m2 = 0u, m3 = 0u;
        for (int k = lane; k < (int)nw; k += 32) {
            const int e = element(k);
            const uint32_t b = 1u << (e & 31);
            const int q = e >> 5;
            m0 |= q == 0 ? b : 0u;
            m1 |= q == 1 ? b : 0u;
            m2 |= q == 2 ? b : 0u;
            m3 |= q == 3 ? b : 0u;
        }
        mask.w[0] = __reduce_or_sync(0xFFFFFFFFu, m0);
        mask.w[1] = __reduce_or_sync(0xFFFFFFFFu, m1);
        mask.w[2] = __reduce_or_sync(0xFFFFFFFFu, m2);
        mask.w[3] = __reduce_or_sync(0xFFFFFFFFu, m3);
        // goal = free[gk], agent = (free without goal)[ak]; free = final positions nw..ni-1
        const uint32_t nfree = (uint32_t)ni - nw;
        const uint32_t gk = S.below(p, nfree);
        const uint32_t ak = S.below(p, nfree - 1u);
        ad = (int)S.below(p, 4u);
        const int goal = element((int)(nw + gk)), agent = element((int)(nw + (ak < gk ? ak : ak + 1u)));
        gr = goal / G.iw + 1;
        gc = goal % G.iw + 1;
        ar = agent / G.iw + 1;
        ac = agent % G.iw + 1;
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------------
// Thread sampler: one level per thread, for throughput kernels (DR resets, batched level
// generation).  The same stream consumption as warp_sample_level, as a word-driven state
// machine: in each round every thread of the warp computes the next Philox block of its
// own key (uniform control flow: block r for everyone in round r) and feeds its 8 words,
// in numpy's order, through its draw state -- Lemire for the wall count, the masked
// rejection of each Fisher-Yates step (the swap in the thread's slice of shared
// memory), Lemire for goal / agent / heading.  A warp samples 32 levels with about the
// instructions warp_sample_level spends on one.
// ---------------------------------------------------------------------------------
constexpr int kTSlice = 132;  // bytes of shared memory per thread (33 words: conflict-free same-index access)

template <int kPhases>
__device__ __forceinline__ void ts_settle(int &phase, int &i, uint32_t &n, uint32_t &thr, uint32_t (&res)[5], int ni,
                                          uint32_t bound0) {
    // advance past phases that draw nothing (Lemire with n <= 1: numpy returns low; a
    // Fisher-Yates with no step left)
#pragma unroll 1
    while (phase < kPhases) {
        if (phase == 1) {
            if (i >= 1) return;
            phase = 2;
            continue;
        }
        n = phase == 0 ? bound0 : phase == 2 ? (uint32_t)ni - res[0] : phase == 3 ? (uint32_t)ni - res[0] - 1u : 4u;
        if (n > 1u) {
            thr = (0u - n) % n;
            return;
        }
        res[phase] = 0u;
        phase++;
        if (phase == 1) i = ni - 1;
    }
}

// arr: this thread's kTSlice-byte slice (4-byte aligned).  Threads with active = false
// run the rounds idle and return nothing.
__device__ __forceinline__ void thread_sample_level(uint64_t k0, uint64_t k1, const Geo &G, uint8_t *arr, bool active,
                                                    Mask &mask, int &ar, int &ac, int &ad, int &gr, int &gc) {
    const int ni = G.ni;
    uint32_t *aw = reinterpret_cast<uint32_t *>(arr);
#pragma unroll 8
    for (int w = 0; w < 32; w++) aw[w] = 0x03020100u + 0x04040404u * (uint32_t)w;  // arange(ni) (+ padding)
    int phase = active ? 0 : 5, i = 0;
    uint32_t n = 0, thr = 0, res[5] = {0u, 0u, 0u, 0u, 0u};
    ts_settle<5>(phase, i, n, thr, res, ni, (uint32_t)G.budget + 1u);
    const unsigned am = __activemask();
    // block r+1 is computed while block r's words are consumed (two independent chains)
    uint64_t o[4];
    philox_block(1, k0, k1, o[0], o[1], o[2], o[3]);
    for (uint64_t blk = 1; __any_sync(am, phase < 5); blk++) {
        uint64_t nx[4];
        philox_block(blk + 1, k0, k1, nx[0], nx[1], nx[2], nx[3]);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const uint32_t w = (q & 1) ? (uint32_t)(o[q >> 1] >> 32) : (uint32_t)o[q >> 1];
            if (phase == 1) {
                const uint32_t v = w & (0xFFFFFFFFu >> __clz(i));
                if (v <= (uint32_t)i) {
                    const uint8_t a = arr[i], b = arr[v];
                    arr[i] = b;
                    arr[v] = a;
                    if (--i < 1) ts_settle<5>(phase, i, n, thr, res, ni, 0u);
                }
            } else if (phase < 5) {
                const uint64_t m = (uint64_t)w * n;
                if ((uint32_t)m >= thr) {
                    res[phase] = (uint32_t)(m >> 32);
                    phase++;
                    if (phase == 1) i = ni - 1;
                    ts_settle<5>(phase, i, n, thr, res, ni, 0u);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 4; q++) o[q] = nx[q];
    }
    if (!active) return;
    // walls: the interior cells at positions [0, nw) of the permuted array
    const uint32_t nw = res[0];
    uint32_t m0 = 0u, m1 = 0u, m2 = 0u, m3 = 0u;
    for (uint32_t k = 0; k < nw; k++) {
        const uint32_t e = arr[k];
        const uint32_t b = 1u << (e & 31u), qw = e >> 5;
        m0 |= qw == 0u ? b : 0u;
        m1 |= qw == 1u ? b : 0u;
        m2 |= qw == 2u ? b : 0u;
        m3 |= qw == 3u ? b : 0u;
    }
    mask.w[0] = m0;
    mask.w[1] = m1;
    mask.w[2] = m2;
    mask.w[3] = m3;
    // goal = free[gk], agent = (free without goal)[ak]; free = positions nw..ni-1
    const uint32_t gk = res[2], ak = res[3];
    const int goal = arr[nw + gk], agent = arr[nw + (ak < gk ? ak : ak + 1u)];
    ad = (int)res[4];
    gr = goal / G.iw + 1;
    gc = goal % G.iw + 1;
    ar = agent / G.iw + 1;
    ac = agent % G.iw + 1;
}

// Every lane whose bit is set in `need` gets the level of its own key (k0, k1), one
// warp-cooperative sample per requesting lane.
template <bool kTrack = false>
__device__ __forceinline__ void warp_sample_each(unsigned need, uint64_t k0, uint64_t k1, const Geo &G,
                                                 WarpSampler &X, Mask &mask, int &ar, int &ac, int &ad, int &gr,
                                                 int &gc) {
    const int lane = threadIdx.x & 31;
    while (need) {
        const int tl = __ffs(need) - 1;
        need &= need - 1;
        const uint64_t a = __shfl_sync(0xFFFFFFFFu, k0, tl), b = __shfl_sync(0xFFFFFFFFu, k1, tl);
        Mask m;
        int r0, c0, d0, g0, h0;
        warp_sample_level<kTrack>(a, b, G, X, m, r0, c0, d0, g0, h0);
        if (lane == tl) {
            mask = m;
            ar = r0;
            ac = c0;
            ad = d0;
            gr = g0;
            gc = h0;
        }
    }
}

}  // namespace amz
