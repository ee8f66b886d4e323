// amz_level.cuh -- level geometry, DR generator, ACCEL mutator, wall boards.
//
// Level bit layout: interior cell (r, c) -> bit (r-1)*(W-2) + (c-1) of a 128-bit
// mask (amz_level_t.walls).  Border cells are implicit walls.
//
// A "board" is the per-lane rendering form of a level: 16 u32 words, word k holding
// the wall bits of grid row k in its low half (bit c = column c, borders included) and
// of grid column k in its high half (bit r = row r).  Observations are cut from it as
// V-bit slices (amz_env.cu), one board word per view row.
#pragma once
#include <stdint.h>

#include "amz_rng.cuh"

namespace amz {

struct Geo {
    int H, W, V, iw, ni, tep, budget;
    bool see;
};

inline Geo make_geo(const amz_params_t &p) {
    Geo g;
    g.H = p.height;
    g.W = p.width;
    g.V = p.agent_view_size;
    g.iw = p.width - 2;
    g.ni = (p.height - 2) * (p.width - 2);
    g.tep = p.max_episode_steps;
    g.budget = p.wall_budget;
    g.see = p.see_through_walls != 0;
    return g;
}

struct Mask {
    uint32_t w[4];
};

__device__ __forceinline__ uint32_t mask_word(const Mask &m, int i) {
    return i == 0 ? m.w[0] : i == 1 ? m.w[1] : i == 2 ? m.w[2] : m.w[3];
}

__device__ __forceinline__ bool mask_bit(const Mask &m, int i) { return (mask_word(m, i >> 5) >> (i & 31)) & 1u; }

__device__ __forceinline__ void mask_set(Mask &m, int i, uint32_t v) {
    uint32_t b = v << (i & 31);
    int k = i >> 5;
    m.w[0] |= k == 0 ? b : 0u;
    m.w[1] |= k == 1 ? b : 0u;
    m.w[2] |= k == 2 ? b : 0u;
    m.w[3] |= k == 3 ? b : 0u;
}

__device__ __forceinline__ void mask_flip(Mask &m, int i) {
    uint32_t b = 1u << (i & 31);
    int k = i >> 5;
    m.w[0] ^= k == 0 ? b : 0u;
    m.w[1] ^= k == 1 ? b : 0u;
    m.w[2] ^= k == 2 ? b : 0u;
    m.w[3] ^= k == 3 ? b : 0u;
}

// `len` (<= 16) bits starting at bit `off`
__device__ __forceinline__ uint32_t mask_bits(const Mask &m, int off, int len) {
    int k = off >> 5;
    uint32_t lo = mask_word(m, k), hi = k < 3 ? mask_word(m, k + 1) : 0u;
    return __funnelshift_r(lo, hi, off & 31) & ((1u << len) - 1u);
}

// index of the k-th (0-based) set bit of a 128-bit mask (k < popcount)
__device__ __forceinline__ int mask_select(const Mask &m, uint32_t k) {
    int base = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        uint32_t w = m.w[i];
        uint32_t c = __popc(w);
        if (k < c) return base + (int)__fns(w, 0, (int)k + 1);
        k -= c;
        base += 32;
    }
    return -1;
}

// mutate_level (amaze/generator.py:55-84): goal relocation w.p. 0.05 to the k-th
// row-major non-wall non-agent interior cell, else toggle the k-th row-major interior
// cell other than agent and goal.
__device__ __forceinline__ void mutate_level_dev(Stream &g, const Geo &G, int n_edits, Mask &mask, int ar,
                                                 int ac, int &gr, int &gc) {
    const int agent = (ar - 1) * G.iw + (ac - 1);
    int goal = (gr - 1) * G.iw + (gc - 1);
    Mask full;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        int lo = i * 32;
        full.w[i] = G.ni >= lo + 32 ? 0xFFFFFFFFu : (G.ni > lo ? (1u << (G.ni - lo)) - 1u : 0u);
    }
    for (int e = 0; e < n_edits; e++) {
        if (g.random() < 0.05) {
            Mask fr;
#pragma unroll
            for (int i = 0; i < 4; i++) fr.w[i] = full.w[i] & ~mask.w[i];
            if (!mask_bit(mask, agent)) mask_flip(fr, agent);
            uint32_t nf = __popc(fr.w[0]) + __popc(fr.w[1]) + __popc(fr.w[2]) + __popc(fr.w[3]);
            goal = mask_select(fr, g.below(nf));
        } else {
            const int s1 = agent < goal ? agent : goal, s2 = agent < goal ? goal : agent;
            const uint32_t ncand = (uint32_t)G.ni - 1u - (agent != goal ? 1u : 0u);
            int k = (int)g.below(ncand);
            int idx = k + (k >= s1 ? 1 : 0);
            if (agent != goal) idx += (idx >= s2 ? 1 : 0);
            mask_flip(mask, idx);
        }
    }
    gr = goal / G.iw + 1;
    gc = goal % G.iw + 1;
}

// Board words (see header comment): rows in the low 16 bits, columns in the high 16.
// Bit-matrix transpose by recursive block swaps (4 stages).
__device__ __forceinline__ void build_board(const Mask &m, const Geo &G, uint32_t *board, int stride) {
    uint32_t a[16];
    const uint32_t rowfull = (1u << G.W) - 1u;
#pragma unroll
    for (int r = 0; r < 16; r++) {
        uint32_t v;
        if (r == 0 || r == G.H - 1)
            v = rowfull;
        else if (r < G.H - 1)
            v = 1u | (mask_bits(m, (r - 1) * G.iw, G.iw) << 1) | (1u << (G.W - 1));
        else
            v = 0u;
        a[r] = v;
    }
    uint32_t t[16];
#pragma unroll
    for (int r = 0; r < 16; r++) t[r] = a[r];
#pragma unroll
    for (int k = 3; k >= 0; k--) {  // s = 8, 4, 2, 1 (a linear counter, so it fully unrolls)
        const int s = 1 << k;
        const uint32_t msk = s == 8 ? 0x00FFu : s == 4 ? 0x0F0Fu : s == 2 ? 0x3333u : 0x5555u;
#pragma unroll
        for (int i = 0; i < 16; i++) {
            if ((i & s) == 0) {
                uint32_t x = ((t[i] >> s) ^ t[i + s]) & msk;
                t[i + s] ^= x;
                t[i] ^= x << s;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 16; k++) board[k * stride] = a[k] | (t[k] << 16);
}

// build_board by a whole warp for one level (m warp-uniform): lane r < 16 forms row word
// r, and the 16 column words are 16 ballots of one bit of every row (the transpose).
__device__ __forceinline__ uint32_t warp_board_word(const Mask &m, const Geo &G) {
    const int lane = threadIdx.x & 31;
    uint32_t v = 0u;
    if (lane == 0 || lane == G.H - 1)
        v = (1u << G.W) - 1u;
    else if (lane < G.H - 1)
        v = 1u | (mask_bits(m, (lane - 1) * G.iw, G.iw) << 1) | (1u << (G.W - 1));
    uint32_t col = 0u;
#pragma unroll
    for (int c = 0; c < 16; c++) {
        const uint32_t b = __ballot_sync(0xFFFFFFFFu, (v >> c) & 1u) & 0xFFFFu;
        col = lane == c ? b : col;
    }
    return v | (col << 16);  // board word `lane` (meaningful for lanes < 16)
}

// amz_level_t <-> registers
__device__ __forceinline__ void load_level(const amz_level_t *lv, Mask &m, int &ar, int &ac, int &ad, int &gr,
                                           int &gc) {
    const uint4 w = *reinterpret_cast<const uint4 *>(lv->walls);
    const uint2 p = *reinterpret_cast<const uint2 *>(&lv->agent_r);
    m.w[0] = w.x;
    m.w[1] = w.y;
    m.w[2] = w.z;
    m.w[3] = w.w;
    ar = p.x & 0xFF;
    ac = (p.x >> 8) & 0xFF;
    ad = (p.x >> 16) & 0xFF;
    gr = p.x >> 24;
    gc = p.y & 0xFF;
}

__device__ __forceinline__ void store_level(amz_level_t *lv, const Mask &m, int ar, int ac, int ad, int gr, int gc) {
    uint4 w = make_uint4(m.w[0], m.w[1], m.w[2], m.w[3]);
    uint4 p = make_uint4((uint32_t)ar | ((uint32_t)ac << 8) | ((uint32_t)ad << 16) | ((uint32_t)gr << 24),
                         (uint32_t)gc, 0u, 0u);
    reinterpret_cast<uint4 *>(lv)[0] = w;
    reinterpret_cast<uint4 *>(lv)[1] = p;
}

}  // namespace amz
