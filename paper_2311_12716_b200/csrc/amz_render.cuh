// amz_render.cuh -- dynamics and egocentric observation of one lane.
//
// transition/compute_reward/step_batch: amaze/env.py:64-84, 320-349.
// observe_batch/view_offsets/apply_occlusion: amaze/env.py:87-137, 352-364.
//
// View row vr looks `ahead = V-1-vr` cells forward; its V cells run along the agent's
// right vector.  For headings N/S that is a slice of grid row r -/+ ahead, for E/W a
// slice of grid column c +/- ahead, reversed for S and W.  So every view row is one
// board word, one shift and (for S/W) one bit reversal; out-of-grid cells come from the
// same shift applied to an "inside" mask.  The goal (burned over walls, as
// MazeStateBatch.tile_codes does, amaze/env.py:254-258) is placed by inverting the
// view transform once per observation.
#pragma once
#include <stdint.h>

#include "amz_level.cuh"

namespace amz {

// dr, dc per heading, clockwise from north (amaze/level.py:19-27)
__device__ __forceinline__ int dir_dr(int d) { return d == 0 ? -1 : (d == 2 ? 1 : 0); }
__device__ __forceinline__ int dir_dc(int d) { return d == 1 ? 1 : (d == 3 ? -1 : 0); }

struct LaneDyn {
    int r, c, d, time;
};

// One transition; returns reached.  Unknown action codes are no-ops with time + 1,
// exactly as step_batch treats them.  `board` gives the wall bits of grid row k at
// board[k * stride] (low 16 bits).  Branch-free: lanes of a warp taking different
// actions do not serialise.  Turn deltas and heading vectors come from nibble tables:
// turn (a=0: +3, a=1: +1, else 0) = 0x13 >> 4a; dr+1 per heading = 0x1210 >> 4d,
// dc+1 per heading = 0x0121 >> 4d (N, E, S, W as amaze/level.py:19-27).
__device__ __forceinline__ bool lane_transition(LaneDyn &s, int a, int gr, int gc, const uint32_t *board,
                                                int stride) {
    const uint32_t ua = (uint32_t)a < 3u ? (uint32_t)a : 3u;
    const int d = (s.d + (int)((0x13u >> (4u * ua)) & 0xFu)) & 3;
    const bool fwd = ua == 2u;
    const int dr = (int)((0x1210u >> (4 * d)) & 0xFu) - 1;
    const int dc = (int)((0x0121u >> (4 * d)) & 0xFu) - 1;
    const int tr = fwd ? s.r + dr : s.r, tc = fwd ? s.c + dc : s.c;
    const bool blocked = (board[tr * stride] >> tc) & 1u;
    s.r = blocked ? s.r : tr;
    s.c = blocked ? s.c : tc;
    s.d = d;
    s.time += 1;
    return s.r == gr && s.c == gc;
}

// 1.0 - 0.9 * time / max_episode_steps with numpy's float64 operation order
__device__ __forceinline__ double goal_reward(int time, int tep) {
    return __dsub_rn(1.0, __ddiv_rn(__dmul_rn(0.9, (double)time), (double)tep));
}

// Observation of one lane: V*V tile codes written to out[vr*V + vc] (out may be shared).
template <int V>
__device__ __forceinline__ void lane_render(int r, int c, int d, int gr, int gc, int H, int W, bool see,
                                            const uint32_t *board, int stride, uint8_t *out) {
    constexpr int h = V / 2;
    constexpr uint32_t vm = (1u << V) - 1u;
    const bool ns = (d & 1) == 0;
    const bool rev = d >= 2;
    const int fr = dir_dr(d), fc = dir_dc(d);
    const int center = ns ? c : r;
    const int nlines = ns ? H : W;
    const int llen = ns ? W : H;
    const int sh = center - h + 8;
    const uint32_t inside = ((((1u << llen) - 1u) << 8) >> sh) & vm;
    // goal position in view coordinates
    const int dr = gr - r, dcol = gc - c;
    const int g_ahead = dr * fr + dcol * fc;
    const int g_side = dr * fc - dcol * fr;  // right = (fc, -fr)
    const bool g_vis = g_ahead >= 0 && g_ahead < V && g_side >= -h && g_side <= h;
    const int g_vr = V - 1 - g_ahead, g_vc = g_side + h;

    uint32_t wall[V], inb[V];
#pragma unroll
    for (int vr = 0; vr < V; vr++) {
        const int ahead = V - 1 - vr;
        const int line = ns ? r + fr * ahead : c + fc * ahead;
        uint32_t wb = 0u, ib = 0u;
        if (line >= 0 && line < nlines) {
            uint32_t word = board[line * stride];
            word = ns ? (word & 0xFFFFu) : (word >> 16);
            wb = ((word << 8) >> sh) & vm;
            ib = inside;
        }
        if (rev) {
            wb = __brev(wb) >> (32 - V);
            ib = __brev(ib) >> (32 - V);
        }
        wall[vr] = wb;
        inb[vr] = ib;
    }
    uint32_t vis[V];
    if (see) {
#pragma unroll
        for (int vr = 0; vr < V; vr++) vis[vr] = vm;
    } else {
        // apply_occlusion (amaze/env.py:111-137): goal cells are transparent
        uint32_t tr[V];
#pragma unroll
        for (int vr = 0; vr < V; vr++) {
            uint32_t gbit = (g_vis && g_vr == vr) ? (1u << g_vc) : 0u;
            tr[vr] = inb[vr] & (~wall[vr] | gbit) & vm;
        }
#pragma unroll
        for (int vr = V - 1; vr >= 0; vr--) {
            uint32_t v;
            if (vr == V - 1) {
                v = 1u << h;
            } else {
                uint32_t through = vis[vr + 1] & tr[vr + 1];
                v = (through | (through >> 1) | (through << 1)) & vm;
            }
#pragma unroll
            for (int k = h + 1; k < V; k++) v |= ((v >> (k - 1)) & (tr[vr] >> (k - 1)) & 1u) << k;
#pragma unroll
            for (int k = h - 1; k >= 0; k--) v |= ((v >> (k + 1)) & (tr[vr] >> (k + 1)) & 1u) << k;
            vis[vr] = v;
        }
    }
#pragma unroll
    for (int vr = 0; vr < V; vr++) {
        const uint32_t shown = vis[vr] & inb[vr];
#pragma unroll
        for (int vc = 0; vc < V; vc++) {
            uint32_t code;
            if (!((shown >> vc) & 1u))
                code = 3u;
            else if (g_vis && g_vr == vr && g_vc == vc)
                code = 2u;
            else
                code = (wall[vr] >> vc) & 1u;
            out[vr * V + vc] = (uint8_t)code;
        }
    }
}

struct LaneRec {
    LaneDyn s;
    int gr, gc, hr, hc, hd;
    bool term;
};

__device__ __forceinline__ LaneRec unpack_st(uint4 v) {
    LaneRec L;
    L.s.r = v.x & 0xFF;
    L.s.c = (v.x >> 8) & 0xFF;
    L.s.d = (v.x >> 16) & 0xFF;
    L.term = (v.x >> 24) != 0;
    L.gr = v.y & 0xFF;
    L.gc = (v.y >> 8) & 0xFF;
    L.hr = (v.y >> 16) & 0xFF;
    L.hc = v.y >> 24;
    L.hd = v.z & 0xFF;
    L.s.time = (int)(v.z >> 8);
    return L;
}

__device__ __forceinline__ uint4 pack_st(const LaneRec &L) {
    return make_uint4((uint32_t)L.s.r | ((uint32_t)L.s.c << 8) | ((uint32_t)L.s.d << 16) |
                          ((uint32_t)L.term << 24),
                      (uint32_t)L.gr | ((uint32_t)L.gc << 8) | ((uint32_t)L.hr << 16) | ((uint32_t)L.hc << 24),
                      (uint32_t)L.hd | ((uint32_t)L.s.time << 8), 0u);
}

}  // namespace amz
