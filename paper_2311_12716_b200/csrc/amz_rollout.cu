// amz_rollout.cu -- T fused env steps of every lane (the env side of
// agents/rollout.py:120-179 with an action stream), split into two kernels.
//
// k_dyn (dynamics, sequential per lane).  One thread per lane, LPW lanes per warp,
// every warp independent.  Per step: transition + reward/done (amaze/env.py:320-349),
// one 32-bit pose record (row, col, heading, level epoch) and the fused auto-reset
// (env/wrappers.py:59-78).  The lanes of a warp that finish on the same step get their
// RESAMPLE levels from one staged SIMT sampler pass (amz_sampler.cuh): the warp
// computes all their Philox blocks round-robin, then each runs its Fisher-Yates.  Each
// level a lane plays ("epoch") is published as a 20-word record (wall board + goal) at
// slot lane + epoch * B.  The action stream is prefetched 32 steps ahead with cp.async.
//
// k_render (observations, fully parallel over (t, lane)).  Each thread renders the
// observation before step t of one lane from its pose record and epoch board
// (observe_batch + apply_occlusion, amaze/env.py:111-137, 352-364) into shared memory;
// the CTA's 128 consecutive (t, lane) records are one contiguous 128*V*V-byte run of the
// time-major view tensor and leave with cp.async.bulk (TMA bulk copy, SASS UBLKCP).
//
// The split takes the 25-byte render and its stores off the per-lane sequential chain:
// the dynamics loop is ~20 instructions per step, the render is embarrassingly
// parallel and HBM-bound.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "amz_internal.h"
#include "amz_render.cuh"
#include "amz_sampler.cuh"

#ifndef AMZ_DYN8_MINB
#define AMZ_DYN8_MINB 4
#endif
#ifndef AMZ_DYN8_TRACK
#define AMZ_DYN8_TRACK false
#endif
#ifndef AMZ_DYN2_MINB
#define AMZ_DYN2_MINB 1
#endif

namespace amz {

namespace {

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(smem_addr(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// The action stream is read ACH steps ahead of use: a warp's next ACH x NL action
// bytes are copied into a shared ring with cp.async while it simulates the current
// ACH steps (a per-lane dependent loop cannot hide HBM latency otherwise).
constexpr int ACH = 32;
template <int NL>
__device__ __forceinline__ void fetch_actions(uint8_t (*ring)[NL], const uint8_t *actions, int64_t B, int64_t lane0,
                                             int nv, int t0, int T, int lane, bool vec) {
    if (vec) {
        // NL/4 threads per step, 4 bytes each
        constexpr int TPS = NL / 4;
        for (int x = lane; x < ACH * TPS; x += 32) {
            const int j = x / TPS, q = x % TPS;
            const int t = t0 + j;
            if (t < T) cp_async4(&ring[j][q * 4], actions + (int64_t)t * B + lane0 + q * 4);
        }
    } else {
        for (int x = lane; x < ACH * NL; x += 32) {
            const int j = x / NL, q = x % NL;
            const int t = t0 + j;
            if (t < T && q < nv) ring[j][q] = actions[(int64_t)t * B + lane0 + q];
        }
    }
    cp_commit();
}

// wall / in-grid bits of view row vr (bit k = view column k)
template <int V, int BS = 32>
__device__ __forceinline__ void row_bits(int r, int c, int d, int H, int W, const uint32_t *board, int vr,
                                         uint32_t &wall, uint32_t &inb) {
    constexpr int h = V / 2;
    constexpr uint32_t vm = (1u << V) - 1u;
    const bool ns = (d & 1) == 0;
    const int ahead = V - 1 - vr;
    const int line = ns ? r + dir_dr(d) * ahead : c + dir_dc(d) * ahead;
    const int nlines = ns ? H : W;
    const int llen = ns ? W : H;
    const int sh = (ns ? c : r) - h + 8;
    uint32_t wb = 0u, ib = 0u;
    if (line >= 0 && line < nlines) {
        uint32_t word = board[line * BS];
        word = ns ? (word & 0xFFFFu) : (word >> 16);
        wb = ((word << 8) >> sh) & vm;
        ib = ((((1u << llen) - 1u) << 8) >> sh) & vm;
    }
    if (d >= 2) {
        wb = __brev(wb) >> (32 - V);
        ib = __brev(ib) >> (32 - V);
    }
    wall = wb;
    inb = ib;
}

// bytes of one view row (codes: hidden/OOB 3, wall 1, goal 2, empty 0) -> out[0..V).
// V <= 5 spreads the wall and hidden bit masks to bytes through a 32-entry table.
template <int V>
__device__ __forceinline__ void emit_row(uint32_t wall, uint32_t inb, bool goal_here, int g_vc,
                                         const uint64_t *spread, uint8_t *o) {
    constexpr uint32_t vm = (1u << V) - 1u;
    if (V <= 5) {
        // bit j -> byte j by one multiply (partial products at bits 7j never overlap)
        auto spr = [](uint32_t x) { return ((uint64_t)x * 0x10204081ull) & 0x0101010101ull; };
        uint64_t bytes = spr(wall & inb) | (spr(~inb & vm) * 3ull);
        if (goal_here) bytes = (bytes & ~(0xFFull << (8 * g_vc))) | (2ull << (8 * g_vc));
        const uint32_t lo = (uint32_t)bytes, hi = (uint32_t)(bytes >> 32);
        o[0] = (uint8_t)lo;
        if (V > 1) o[1] = (uint8_t)(lo >> 8);
        if (V > 2) o[2] = (uint8_t)(lo >> 16);
        if (V > 3) o[3] = (uint8_t)(lo >> 24);
        if (V > 4) o[4] = (uint8_t)hi;
    } else {
#pragma unroll
        for (int j = 0; j < V; j++) {
            uint32_t code = ((inb >> j) & 1u) ? ((wall >> j) & 1u) : 3u;
            if (goal_here && g_vc == j) code = 2u;
            o[j] = (uint8_t)code;
        }
    }
}

// 5-bit mask -> 5 bytes of 0/1 (built once per CTA)
__device__ __forceinline__ void init_spread(uint64_t *spread) {
    for (int e = threadIdx.x; e < 32; e += blockDim.x) {
        uint64_t v = 0;
#pragma unroll
        for (int j = 0; j < 5; j++) v |= (uint64_t)((e >> j) & 1) << (8 * j);
        spread[e] = v;
    }
}

// observe_batch + apply_occlusion (amaze/env.py:111-137, 352-364) for one lane
template <int V, bool SEE, int BS = 32>
__device__ __forceinline__ void render_lane(int r, int c, int d, int gr, int gc, int H, int W, const uint32_t *board,
                                            const uint64_t *spread, uint8_t *out, int only_k = -1, int G = 1) {
    constexpr int h = V / 2;
    constexpr uint32_t vm = (1u << V) - 1u;
    const int fr = dir_dr(d), fc = dir_dc(d);
    const int dr = gr - r, dcol = gc - c;
    const int g_ahead = dr * fr + dcol * fc;
    const int g_side = dr * fc - dcol * fr;
    const bool g_vis = g_ahead >= 0 && g_ahead < V && g_side >= -h && g_side <= h;
    const int g_vr = V - 1 - g_ahead, g_vc = g_side + h;
    uint32_t wall[V], inb[V];
#pragma unroll
    for (int vr = 0; vr < V; vr++) row_bits<V, BS>(r, c, d, H, W, board, vr, wall[vr], inb[vr]);
    if (!SEE) {
        uint32_t tr[V], vis[V];
#pragma unroll
        for (int vr = 0; vr < V; vr++) {
            const uint32_t gbit = (g_vis && g_vr == vr) ? (1u << g_vc) : 0u;
            tr[vr] = inb[vr] & (~wall[vr] | gbit) & vm;
        }
#pragma unroll
        for (int vr = V - 1; vr >= 0; vr--) {
            uint32_t v;
            if (vr == V - 1) {
                v = 1u << h;
            } else {
                const uint32_t through = vis[vr + 1] & tr[vr + 1];
                v = (through | (through >> 1) | (through << 1)) & vm;
            }
#pragma unroll
            for (int kk = h + 1; kk < V; kk++) v |= ((v >> (kk - 1)) & (tr[vr] >> (kk - 1)) & 1u) << kk;
#pragma unroll
            for (int kk = h - 1; kk >= 0; kk--) v |= ((v >> (kk + 1)) & (tr[vr] >> (kk + 1)) & 1u) << kk;
            vis[vr] = v;
        }
#pragma unroll
        for (int vr = 0; vr < V; vr++) inb[vr] &= vis[vr];
    }
#pragma unroll
    for (int vr = 0; vr < V; vr++) {
        if (only_k >= 0 && vr % G != only_k) continue;
        const bool goal_here = g_vis && g_vr == vr && ((inb[vr] >> g_vc) & 1u);
        emit_row<V>(wall[vr], inb[vr], goal_here, g_vc, spread, out + vr * V);
    }
}


// See-through 5x5 observation (the default view) with word-level arithmetic, from a
// staged board (16 line words; any index is readable, so rows off the grid read line
// L & 15 and are overwritten by the off-grid code).  A view row is one board word (grid
// row for N/S headings, grid column for E/W); its 5-cell window becomes code bytes
// (3 off-grid, 1 wall, 0 empty) by one multiply-spread, the S/W mirror is a byte
// permute.  The off-grid codes of the observation's two row kinds (in-grid line:
// the columns outside the grid; off-grid line: all five) are built once, a row is
// (window bits * spread) | off-grid codes -- 3 | wall = 3, so neither the window nor the
// line needs masking -- and the goal byte is NOT patched: the caller stores it at byte
// offset *gpos (-1: not visible) after the row words.
__device__ __forceinline__ void render5_see_rows(int r, int c, int d, int gr, int gc, int H, int W,
                                                 const uint32_t *board, uint32_t (&w)[7], int &gpos) {
    const bool ns = (d & 1) == 0;
    const int sgn = (d == 0 || d == 3) ? -1 : 1;
    const int base = ns ? r : c, center = ns ? c : r;
    const uint32_t nlines = (uint32_t)(ns ? H : W);
    const int llen = ns ? W : H;
    const int up = ns ? 16 : 0;
    const int sx = 14 + center;
    const uint32_t obm = ~(((((1u << llen) - 1u) << 16) >> sx)) & 31u;  // off-grid cells of an in-grid line
    const uint32_t obl = ((obm * 0x00204081u) & 0x01010101u) * 3u, obh = (obm >> 4) * 3u;
    const bool rev = d >= 2;
    const uint32_t sel0 = rev ? 0x1234u : 0x3210u, sel1 = rev ? 0x5550u : 0x5554u;
    const int fr = dir_dr(d), fc = dir_dc(d);
    const int dr = gr - r, dcol = gc - c;
    const int g_ahead = dr * fr + dcol * fc, g_side = dr * fc - dcol * fr;
    gpos = (g_ahead >= 0 && g_ahead < 5 && g_side >= -2 && g_side <= 2) ? (4 - g_ahead) * 5 + g_side + 2 : -1;
    const int L0 = base + 4 * sgn;
    uint32_t lo[5], hi[5];
#pragma unroll
    for (int vr = 0; vr < 5; vr++) {
        const int L = L0 - sgn * vr;
        const bool in = (uint32_t)L < nlines;
        const uint32_t bw = board[L & 15];
        const uint32_t x = ((bw << up) >> sx) & 31u;
        const uint32_t l4 = ((x * 0x00204081u) & 0x01010101u) | (in ? obl : 0x03030303u);
        const uint32_t h1 = (x >> 4) | (in ? obh : 3u);
        lo[vr] = __byte_perm(l4, h1, sel0);
        hi[vr] = __byte_perm(l4, h1, sel1);
    }
    w[0] = lo[0];
    w[1] = hi[0] | (lo[1] << 8);
    w[2] = (lo[1] >> 24) | (hi[1] << 8) | (lo[2] << 16);
    w[3] = (lo[2] >> 16) | (hi[2] << 16) | (lo[3] << 24);
    w[4] = (lo[3] >> 8) | (hi[3] << 24);
    w[5] = lo[4];
    w[6] = hi[4];
}
// Warp-collective store of each lane's 25 bytes (7 words from render5_see_rows) at byte
// offset 25 * idx of a 16-byte-aligned staging row, idx = lane index in the row (the
// warp's lanes hold consecutive idx, idx % 32 == lane): 6-7 aligned 32-bit stores per
// lane instead of 25 byte stores; the word a lane shares with its successor is merged
// by a shuffle.  Every lane of the warp must call it (live = false: nothing stored).
__device__ __forceinline__ void store_obs25(uint8_t *stage, int idx, bool live, const uint32_t (&w)[7]) {
    const int o = idx & 3;  // (25 * idx) mod 4
    const int sh = 8 * o;
    uint32_t a[7];
    a[0] = w[0] << sh;
#pragma unroll
    for (int k = 1; k < 7; k++) a[k] = __funnelshift_l(w[k - 1], w[k], sh);
    const uint32_t nxt = __shfl_down_sync(0xFFFFFFFFu, live ? a[0] : 0u, 1);
    if (o != 3) a[6] |= nxt;  // this lane's last word is the successor's first
    if (!live) return;
    uint32_t *dst = reinterpret_cast<uint32_t *>(stage) + ((25 * idx) >> 2);
    if (o == 0) dst[0] = a[0];
#pragma unroll
    for (int k = 1; k < 7; k++) dst[k] = a[k];
}

constexpr int kRec = 20;  // u32 words per epoch record: board[16], goal, pad

}  // namespace

// ---------------------------------------------------------------------------------
// phase 1: dynamics
// ---------------------------------------------------------------------------------
#ifdef AMZ_DYN_PROF
__device__ unsigned long long g_dyn_prof[65536][8];
__device__ unsigned long long g_dyn_prof2[65536][8];
#define DYN_ACC2(k_, v_)                                                                                        \
    do {                                                                                                        \
        const int64_t wi_ = (int64_t)blockIdx.x * WPC + (threadIdx.x >> 5);                                     \
        if ((threadIdx.x & 31) == 0 && wi_ < 65536) g_dyn_prof2[wi_][k_] += (unsigned long long)(clock64() - v_); \
    } while (0)
__device__ __forceinline__ unsigned smid_() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
#define DYN_MARK(k_)                                                                         \
    do {                                                                                     \
        const int64_t wi_ = (int64_t)blockIdx.x * WPC + (threadIdx.x >> 5);                  \
        if ((threadIdx.x & 31) == 0 && wi_ < 65536) g_dyn_prof[wi_][k_] = clock64() | ((unsigned long long)smid_() << 56); \
    } while (0)
#define DYN_T0(v_) const long long v_ = clock64()
#define DYN_ACC(k_, v_)                                                                                        \
    do {                                                                                                        \
        const int64_t wi_ = (int64_t)blockIdx.x * WPC + (threadIdx.x >> 5);                                     \
        if ((threadIdx.x & 31) == 0 && wi_ < 65536) g_dyn_prof[wi_][k_] += (unsigned long long)(clock64() - v_); \
    } while (0)
#else
#define DYN_T0(v_) \
    do {           \
    } while (0)
#define DYN_ACC(k_, v_) \
    do {                \
    } while (0)
#define DYN_MARK(k_) \
    do {             \
    } while (0)
#define DYN_ACC2(k_, v_) \
    do {                 \
    } while (0)
#endif

// move-table rows per lane: 5 (the 4 headings + an identity row, so a turn is the same
// byte load as a move: the shortest chain, for the latency-bound small batches) or 4
// (LPW >= 8: a turn selects the old position instead -- 8 KB less shared memory per
// CTA, which with <= 128 registers gives the many-wave large batch a 4th resident CTA)
template <int LPW>
constexpr int kMtRows = LPW >= 8 ? 4 : 5;
template <int LPW>
struct DynSmem {
    uint32_t board[16][LPW];
    uint8_t mt[LPW][kMtRows<LPW>][256];  // move table: position after a step, [heading (or 4 = no move)][pos]
    uint8_t act[2][ACH][LPW];
    uint32_t aw[LPW][ACH / 4 + 2];  // this chunk's actions per lane, 4 steps per word (+2 zero pad)
    uint32_t rec[LPW][ACH + 8];     // this chunk's step records per lane (+8: a batch stores all 8)
    WarpSampler samp;
    __align__(16) amz_level_t spec[LPW];  // the lanes' prepared timeout levels
};

// Move table of lane L (whole warp): mt[e][pos], pos = r | c << 4, is the position after
// a forward move in heading e (unchanged when the target cell is a wall, as
// lane_transition), and mt[4][pos] = pos (turns / no-ops).  A step of the position
// chain is then one shared byte load.  A table word holds rows r0..r0+3 of column c:
// the four wall flags of their targets are one shift of a column's wall bits (board
// word high halves; off-grid targets count as walls), and the bytes are
// pos + off * (not blocked), byte-parallel.
template <int LPW>
__device__ __forceinline__ void build_move_table(const uint32_t *board, int L, uint8_t *mt) {
    const int lane = threadIdx.x & 31;
    // table word w = lane + 32 k (k = 0..9): heading e = k >> 1, column c = lane / 4 +
    // 8 (k & 1), rows r0..r0+3 with r0 = 4 (lane & 3).  A lane only ever needs columns
    // c0 - 1 .. c0 + 1 and c0 + 7 .. c0 + 9 (c0 = lane / 4): six loads up front, then
    // ten independent words.
    auto col = [&](int x) -> uint32_t { return (x >= 0 && x < 16) ? (board[x * LPW + L] >> 16) : 0xFFFFu; };
    const int c0 = lane >> 2, r0 = (lane & 3) << 2;
    uint32_t cm[2], cc[2], cp[2];
#pragma unroll
    for (int h = 0; h < 2; h++) {
        cm[h] = col(c0 + 8 * h - 1);
        cc[h] = col(c0 + 8 * h);
        cp[h] = col(c0 + 8 * h + 1);
    }
#pragma unroll
    for (int k = 0; k < 2 * kMtRows<LPW>; k++) {
        const int e = k >> 1, h = k & 1, c = c0 + 8 * h;
        const uint32_t base4 = (uint32_t)(r0 | (c << 4)) * 0x01010101u + 0x03020100u;
        uint32_t out = base4;
        if (e < 4) {
            uint32_t m;
            int off;
            if (e == 0) {  // N
                m = ((cc[h] << 1) | 1u) >> r0;
                off = -1;
            } else if (e == 2) {  // S
                m = (cc[h] | 0x10000u) >> (r0 + 1);
                off = 1;
            } else if (e == 1) {  // E
                m = cp[h] >> r0;
                off = 16;
            } else {  // W
                m = cm[h] >> r0;
                off = -16;
            }
            const uint32_t open = ~m & 0xFu;
            const uint32_t spread = (open * 0x00204081u) & 0x01010101u;
            out = base4 + spread * (uint32_t)off;
        }
        reinterpret_cast<uint32_t *>(mt)[lane + 32 * k] = out;
    }
    __syncwarp();
}

// resident CTAs per SM the register budget is sized for: the large-batch instantiation
// (LPW 8) runs many waves, so it trades registers for a 4th resident CTA (128 registers,
// no spills; with the 4-row move table its CTA fits 4 per SM in shared memory too)
template <int LPW>
struct DynOcc {
    static constexpr int kMinBlocks = LPW >= 8 ? AMZ_DYN8_MINB : (LPW <= 2 ? AMZ_DYN2_MINB : 1);
    // sampler variant: element tracking (lowest latency) where the per-warp chain bounds
    // the rollout; swap-list read-off (fewest instructions) in the many-wave large batch
    static constexpr bool kTrack = LPW >= 8 ? AMZ_DYN8_TRACK : true;
    // persistent warps over a lane-group queue (the many-wave large batch; E.work, zero
    // between launches): a warp takes
    // the next group as soon as it finishes one, instead of a CTA holding its slot until
    // its slowest warp is done (achieved occupancy 18% of the 25% resident at 65536 lanes)
    static constexpr bool kPersist = LPW >= 8;
};
template <int LPW, int WPC>
__global__ void __launch_bounds__(32 * WPC, DynOcc<LPW>::kMinBlocks) k_dyn(Geo G, EnvDev E, int T, const uint8_t *__restrict__ actions, int mode,
                                                  amz_seed_t wrap, uint32_t step0, double *__restrict__ reward,
                                                  uint8_t *__restrict__ done, uint32_t *__restrict__ poses,
                                                  uint32_t *__restrict__ epochs, uint32_t *__restrict__ final_pose,
                                                  const amz_level_t *__restrict__ spec,
                                                  const uint32_t *__restrict__ spec_step, int avec, int use_lut) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    static_assert((LPW % 4 == 0 || LPW == 2) && LPW <= 32, "lane-major action gather: LPW 2 or a multiple of 4");

    DynSmem<LPW> &S = reinterpret_cast<DynSmem<LPW> *>(smem)[warp];
    // goal rewards R[time] = 1 - 0.9*time/T_ep (numpy's op order), tabulated per CTA
    double *s_rew = reinterpret_cast<double *>(smem + WPC * sizeof(DynSmem<LPW>));
    if (use_lut)
        for (int tt = threadIdx.x; tt <= G.tep; tt += blockDim.x) s_rew[tt] = goal_reward(tt, G.tep);
    __syncthreads();
    pdl_wait();  // lane state from the reset
    if (E.iter && mode == AMZ_RESET_RESAMPLE) {  // graph replay: root.fold_in(*iter).fold_in(1)
        seed_absorb(wrap, *E.iter);
        seed_absorb(wrap, 1u);
    }
    // the render may launch now: everything before this grid is complete (pdl_wait), every
    // CTA of it is resident, and the render waits per lane group (E.gdone)
    if (E.gdone) pdl_trigger();
    const int64_t B = E.B;
    const int64_t ngroups = (B + LPW - 1) / LPW;
    int64_t grp = (int64_t)blockIdx.x * WPC + warp;  // first group static, then the queue
    for (; grp < ngroups;) {
    DYN_MARK(0);
    const int64_t lane0 = grp * LPW;
    const int64_t l = lane0 + lane;
    const bool live = lane < LPW && l < B;
    const int nv = (int)((B - lane0) < LPW ? (B - lane0) : LPW);
    uint32_t *bd = &S.board[0][lane < LPW ? lane : 0];
    const uint8_t *mtl = &S.mt[lane < LPW ? lane : 0][0][0];

    LaneRec L{};
    L.s.r = L.s.c = 1;  // idle lanes step harmlessly inside the grid
    Mask m;
    bool lvl_changed = false;
    uint32_t epoch = 0, my_spec = 0xFFFFFFFFu;
    if (live) {
        L = unpack_st(E.st[l]);
        uint32_t *rec = epochs + (size_t)l * kRec;
        // all loads before any store: epochs may alias E.board as far as the compiler
        // knows, and interleaving would serialise 16 global round trips
        uint32_t v[16];
#pragma unroll
        for (int w = 0; w < 16; w++) v[w] = E.board[w * B + l];
#pragma unroll
        for (int w = 0; w < 16; w++) {
            bd[w * LPW] = v[w];
            rec[w] = v[w];
        }
        rec[16] = (uint32_t)L.gr | ((uint32_t)L.gc << 8);
        if (mode == AMZ_RESET_RESAMPLE) {
            my_spec = spec_step[l];
            if (my_spec != 0xFFFFFFFFu) {  // in flight with the first action chunk
                cp_async16(&S.spec[lane], spec + l);
                cp_async16(reinterpret_cast<uint8_t *>(&S.spec[lane]) + 16, reinterpret_cast<const uint8_t *>(spec + l) + 16);
            }
        }
    }
    __syncwarp();
    for (int q = 0; q < nv; q++) build_move_table<LPW>(&S.board[0][0], q, &S.mt[q][0][0]);
    const bool vec = avec && nv == LPW && LPW % 4 == 0;
    fetch_actions<LPW>(S.act[0], actions, B, lane0, nv, 0, T, lane, vec);
    __syncwarp();
    const uint8_t *ap = &S.act[0][0][lane < LPW ? lane : 0];
    // Packed lane state ps = r | c << 4 | heading << 8 | epoch << 12 (the pose record
    // layout).  A forward move adds a signed nibble offset to ps; a turn rewrites bits
    // 8-9.  Idle lanes never finish (goal 0xFF is unreachable from (1, 1), tep = inf).
    uint32_t ps = (uint32_t)L.s.r | ((uint32_t)L.s.c << 4) | ((uint32_t)L.s.d << 8);
    uint32_t g = live ? ((uint32_t)L.gr | ((uint32_t)L.gc << 4)) : 0xFFu;
    int time = L.s.time;
    const int tep = live ? G.tep : 0x7FFFFFFF;
    uint4 *pq = reinterpret_cast<uint4 *>(poses) + l;  // steps 4q..4q+3 of lane l at pq[q * B]

    // Episode ends at step t of the lanes with dn: RESAMPLE levels (prepared timeout level
    // or the warp-cooperative sampler), board + move table, epoch record, reset.
    auto episode_end = [&](int t, bool dn) {
        const unsigned fin = __ballot_sync(0xFFFFFFFFu, dn);
        if (fin) {
            DYN_T0(c_evt);
            if (mode == AMZ_RESET_RESAMPLE) {
                const uint32_t gstep = step0 + (uint32_t)t;
                const bool hit = dn && my_spec == gstep;
                const unsigned need = __ballot_sync(0xFFFFFFFFu, dn && !hit);
                int ar = 0, acol = 0, ad = 0, gr = 0, gc = 0;
                DYN_ACC2(0, c_evt);
                if (need) {
                    DYN_T0(c_key);
                    uint64_t k0 = 0, k1 = 0;
                    if (dn && !hit) {
                        amz_seed_t sd = wrap;
                        seed_absorb(sd, gstep);
                        seed_absorb(sd, E.lane_offset + (uint32_t)l);
                        seed_key(sd, k0, k1);
                    }
                    DYN_ACC2(1, c_key);
                    DYN_T0(c_smp);
                    warp_sample_each<DynOcc<LPW>::kTrack>(need, k0, k1, G, S.samp, m, ar, acol, ad, gr, gc);
                    DYN_ACC(5, c_smp);
#ifdef AMZ_DYN_PROF
                    if (lane == 0) g_dyn_prof[(int64_t)blockIdx.x * WPC + warp][7] += __popc(need);
#endif
                }
                DYN_T0(c_bb);
                if (hit) load_level(&S.spec[lane], m, ar, acol, ad, gr, gc);
                if (dn) {
                    L.hr = ar;
                    L.hc = acol;
                    L.hd = ad;
                    L.gr = gr;
                    L.gc = gc;
                    lvl_changed = true;
                    epoch++;
                }
                DYN_ACC2(2, c_bb);
            }
            if (mode == AMZ_RESET_RESAMPLE) {
                // per finishing lane q, the whole warp: board words (ballot transpose), the
                // epoch record, the move table
                __syncwarp();
                DYN_T0(c_tbl);
                unsigned chg = fin & ((LPW >= 32) ? 0xFFFFFFFFu : ((1u << LPW) - 1u));
                while (chg) {
                    const int q = __ffs(chg) - 1;
                    chg &= chg - 1;
                    Mask mq;
#pragma unroll
                    for (int i = 0; i < 4; i++) mq.w[i] = __shfl_sync(0xFFFFFFFFu, m.w[i], q);
                    const uint32_t eq = __shfl_sync(0xFFFFFFFFu, epoch, q);
                    const uint32_t gq = __shfl_sync(0xFFFFFFFFu, (uint32_t)L.gr | ((uint32_t)L.gc << 8), q);
                    const uint32_t bw = warp_board_word(mq, G);
                    uint32_t *rec = epochs + ((size_t)eq * B + lane0 + q) * kRec;
                    if (lane < 16) {
                        S.board[lane][q] = bw;
                        rec[lane] = bw;
                    } else if (lane == 16) {
                        rec[16] = gq;
                    }
                    __syncwarp();
                    build_move_table<LPW>(&S.board[0][0], q, &S.mt[q][0][0]);
                }
                DYN_ACC(6, c_tbl);
            }
            if (dn) {
                ps = (uint32_t)L.hr | ((uint32_t)L.hc << 4) | ((uint32_t)L.hd << 8) | (epoch << 12);
                g = (uint32_t)L.gr | ((uint32_t)L.gc << 4);
                time = 0;
            }
            DYN_ACC(4, c_evt);
#ifdef AMZ_DYN_PROF
            if (lane == 0) g_dyn_prof[(int64_t)blockIdx.x * WPC + warp][7] += (1ull << 32) + ((unsigned long long)__popc(fin) << 48);
#endif
        }
    };

    DYN_MARK(1);
    for (int t0 = 0; t0 < T; t0 += ACH) {
        fetch_actions<LPW>(S.act[((t0 / ACH) + 1) & 1], actions, B, lane0, nv, t0 + ACH, T, lane, vec);
        cp_wait<1>();
        __syncwarp();
        const int tn = (T - t0) < ACH ? (T - t0) : ACH;
        {
            // lane-major copy of the chunk's actions (4 steps per word)
            const int me = lane < LPW ? lane : 0;
            const uint32_t *row = reinterpret_cast<const uint32_t *>(&S.act[(t0 / ACH) & 1][0][0]) + (me >> 2);
            const uint32_t sel = (uint32_t)(me & 3) | ((uint32_t)(4 + (me & 3)) << 4);
            if (lane < LPW) {
                if (LPW % 4 == 0) {
#pragma unroll
                    for (int q = 0; q < ACH / 4; q++) {
                        const uint32_t lo = __byte_perm(row[(4 * q) * (LPW / 4)], row[(4 * q + 1) * (LPW / 4)], sel);
                        const uint32_t hi = __byte_perm(row[(4 * q + 2) * (LPW / 4)], row[(4 * q + 3) * (LPW / 4)], sel);
                        S.aw[me][q] = __byte_perm(lo, hi, 0x5410);
                    }
                } else {
                    const uint8_t *ab = &S.act[(t0 / ACH) & 1][0][me];
#pragma unroll
                    for (int q = 0; q < ACH / 4; q++)
                        S.aw[me][q] = (uint32_t)ab[(4 * q) * LPW] | ((uint32_t)ab[(4 * q + 1) * LPW] << 8) |
                                      ((uint32_t)ab[(4 * q + 2) * LPW] << 16) | ((uint32_t)ab[(4 * q + 3) * LPW] << 24);
                }
                S.aw[me][ACH / 4] = S.aw[me][ACH / 4 + 1] = 0u;
            }
            __syncwarp();
        }
        // Speculative batches of up to 8 steps: the position chain alone (heading by byte
        // prefix sums of the SWAR-decoded actions, a move = one move-table byte load).  The
        // warp keeps the steps up to the first episode end of any of its lanes (exact for
        // every lane), handles that end, and continues from the next step -- nothing is
        // recomputed.
        int j = 0;
        while (j < tn) {
            const int n = (tn - j) < 8 ? (tn - j) : 8;
            const int me = lane < LPW ? lane : 0;
            const uint32_t *awl = &S.aw[me][j >> 2];
            const int sh = 8 * (j & 3);
            const uint32_t a0 = __funnelshift_r(awl[0], awl[1], sh), a1 = __funnelshift_r(awl[1], awl[2], sh);
            uint32_t pos = ps & 0xFFu, d = (ps >> 8) & 3u;
            const uint32_t hi = ps & 0xFFFFF000u;
            uint32_t ew[2], dw[2];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint32_t a = h ? a1 : a0;
                const uint32_t left = __vcmpeq4(a, 0u), right = __vcmpeq4(a, 0x01010101u);
                const uint32_t fwd = __vcmpeq4(a, 0x02020202u);
                const uint32_t turn = (left & 0x03030303u) | (right & 0x01010101u);
                const uint32_t da = (turn * 0x01010101u + d * 0x01010101u) & 0x03030303u;  // after
                dw[h] = (da << 8) | d;                                                     // before
                ew[h] = (da & fwd) | (0x04040404u & ~fwd);
                d = da >> 24;
            }
            uint32_t rec[8], pkw[2] = {0u, 0u};  // positions after each step, one byte each
            unsigned ev = (time + n >= tep) ? (1u << (tep - time - 1)) : 0u;  // timeout step, if inside
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const uint32_t e = (ew[k >> 2] >> (8 * (k & 3))) & 0xFFu;
                const uint32_t db = (dw[k >> 2] >> (8 * (k & 3))) & 0x3u;
                rec[k] = pos | (db << 8) | hi;
                if constexpr (kMtRows<LPW> == 5) {
                    pos = mtl[e * 256u + pos];
                } else {
                    const uint32_t np = mtl[(e & 3u) * 256u + pos];
                    pos = e < 4u ? np : pos;
                }
                pkw[k >> 2] |= pos << (8 * (k & 3));
                ev |= (unsigned)(pos == g) << k;
            }
            ev &= (1u << n) - 1u;
            const unsigned kl = ev ? (unsigned)(__ffs(ev) - 1) : 8u;
            const unsigned km = __reduce_min_sync(0xFFFFFFFFu, kl);
            const int cnt = km < (unsigned)n ? (int)km + 1 : n;
            const bool dn = kl == km && km < (unsigned)n;
            // position after step cnt - 1 (byte-packed: an array indexed at run time would
            // live in local memory)
            const uint32_t pe = ((((cnt - 1) >> 2) ? pkw[1] : pkw[0]) >> (8 * ((cnt - 1) & 3))) & 0xFFu;
            const bool reached = dn && pe == g;  // km = cnt - 1 whenever dn
            if (lane < LPW) {
                // all 8 records unconditionally (those past cnt are rewritten by the next
                // batch, which starts at j + cnt), then the episode-end flags
#pragma unroll
                for (int k = 0; k < 8; k++) S.rec[me][j + k] = rec[k];
                if (dn) S.rec[me][j + km] |= ((uint32_t)reached << 10) | (1u << 11);
            }
            const uint32_t de = cnt == 8 ? d : ((((cnt >> 2) ? dw[1] : dw[0]) >> (8 * (cnt & 3))) & 3u);
            ps = pe | (de << 8) | hi;
            time += cnt;
            j += cnt;
            if (km < (unsigned)n) {
                const int t = t0 + j - 1;
                if (reached && live) reward[(int64_t)t * B + l] = use_lut ? s_rew[time] : goal_reward(time, G.tep);
                episode_end(t, dn);
            }
        }
        // the chunk's records: quads of lane L at pq[(t0 / 4 + q) * B]
        __syncwarp();
        for (int x = lane; x < nv * (ACH / 4); x += 32) {
            const int qq = x / (ACH / 4), cq = x - qq * (ACH / 4);
            if (4 * cq < tn)
                reinterpret_cast<uint4 *>(poses)[(size_t)((t0 >> 2) + cq) * B + lane0 + qq] =
                    *reinterpret_cast<const uint4 *>(&S.rec[qq][4 * cq]);
        }
        __syncwarp();
    }
    DYN_MARK(2);
    L.s.r = (int)(ps & 15u);
    L.s.c = (int)((ps >> 4) & 15u);
    L.s.d = (int)((ps >> 8) & 3u);
    L.s.time = time;
    L.term = false;
    if (live) {
        final_pose[l] = ps;
        E.st[l] = pack_st(L);
        if (lvl_changed) {
            E.mask[l] = make_uint4(m.w[0], m.w[1], m.w[2], m.w[3]);
#pragma unroll
            for (int w = 0; w < 16; w++) E.board[w * B + l] = bd[w * LPW];
        }
    }
    DYN_MARK(3);
    if (E.gdone) {  // publish: this warp's poses, epoch records, final poses and lane state
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(E.gdone + (lane0 >> 7), 1u);
    }
    if (!DynOcc<LPW>::kPersist) break;
    __syncwarp();  // every lane is done with the group's shared state
    unsigned nxt = 0;
    if (lane == 0) {
        nxt = atomicAdd(E.work, 1u);
        // every warp's last fetch fails, so a launch makes exactly ngroups fetches: the
        // one that returns ngroups - 1 is the last and re-zeroes the queue for the next
        if ((int64_t)nxt == ngroups - 1) *E.work = 0u;
    }
    grp = (int64_t)gridDim.x * WPC + __shfl_sync(0xFFFFFFFFu, nxt, 0);
    }
}

#ifdef AMZ_DYN_PROF
extern "C" int amz_debug_dyn_prof2(void *host) {
    return (int)cudaMemcpyFromSymbol(host, g_dyn_prof2, sizeof(g_dyn_prof2));
}
extern "C" int amz_debug_dyn_prof(void *out) {
    return (int)cudaMemcpyFromSymbol(out, g_dyn_prof, sizeof(g_dyn_prof));
}
extern "C" int amz_debug_dyn_prof_reset(const void *zero) {
    cudaMemcpyToSymbol(g_dyn_prof2, zero, sizeof(g_dyn_prof2));
    return (int)cudaMemcpyToSymbol(g_dyn_prof, zero, sizeof(g_dyn_prof));
}
#endif

// Speculative timeout levels: a lane that never reaches the goal times out at the step
// where its time hits max_episode_steps; that level's key is known now, so it is
// sampled up front with everyone else's (kSpecLPW lanes per warp, warp-cooperative).
constexpr int kSpecLPW = 1;
__global__ void __launch_bounds__(128) k_spec_levels(Geo G, EnvDev E, int T, amz_seed_t wrap, uint32_t step0,
                                                     amz_level_t *__restrict__ spec, uint32_t *__restrict__ spec_step) {
    constexpr int LPW = kSpecLPW;
    __shared__ __align__(16) WarpSampler X[4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t l0 = ((int64_t)blockIdx.x * 4 + warp) * LPW;
    if (l0 >= E.B) return;
    if (E.iter) {
        seed_absorb(wrap, *E.iter);
        seed_absorb(wrap, 1u);
    }
    const int64_t l = l0 + lane;
    bool mine = false;
    uint64_t k0 = 0, k1 = 0;
    int s_to = -1;
    if (lane < LPW && l < E.B) {
        const LaneRec L = unpack_st(E.st[l]);
        s_to = G.tep - L.s.time - 1;
        mine = s_to >= 0 && s_to < T;
        if (mine) {
            amz_seed_t sd = wrap;
            seed_absorb(sd, step0 + (uint32_t)s_to);
            seed_absorb(sd, E.lane_offset + (uint32_t)l);
            seed_key(sd, k0, k1);
        } else {
            spec_step[l] = 0xFFFFFFFFu;
        }
    }
    const unsigned need = __ballot_sync(0xFFFFFFFFu, mine);
    if (!need) return;
    Mask m;
    int ar, ac, ad, gr, gc;
    warp_sample_each(need, k0, k1, G, X[warp], m, ar, ac, ad, gr, gc);
    if (mine) {
        store_level(spec + l, m, ar, ac, ad, gr, gc);
        spec_step[l] = step0 + (uint32_t)s_to;
    }
}

// ---------------------------------------------------------------------------------
// phase 2: observations
// ---------------------------------------------------------------------------------
// One persistent launch renders the T*B step observations (tiles [0, g1)) and the B
// final observations (tiles [g1, g1 + ceil(B/128))), 128 observations per tile.  A CTA
// loops over tiles with two staging buffers: the bulk store of one tile drains while the
// next tile renders, and the spread table is built once per CTA.
template <int V, bool SEE>
__global__ void __launch_bounds__(128) k_render(Geo G, int64_t B, int64_t n, const uint32_t *__restrict__ poses,
                                                const uint32_t *__restrict__ final_pose,
                                                const uint32_t *__restrict__ epochs, uint8_t *__restrict__ view,
                                                uint8_t *__restrict__ dirs, double *__restrict__ reward,
                                                uint8_t *__restrict__ done, uint8_t *__restrict__ fview,
                                                uint8_t *__restrict__ fdir, int bulk_ok, int64_t g1, int64_t ntiles) {
    constexpr int VV = V * V;
    __shared__ __align__(128) uint8_t s_view[2][128 * VV];
    __shared__ __align__(16) uint8_t s_dir[2][128];
    __shared__ __align__(16) uint8_t s_done[2][128];
    __shared__ uint64_t s_spread[32];
    __shared__ int64_t s_t0;
    init_spread(s_spread);
    pdl_wait();  // poses / epochs from k_dyn
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
        const int buf = it & 1;
        const bool fin = tile >= g1;
        const int64_t base = (fin ? tile - g1 : tile) * 128;
        const int64_t cnt = fin ? B : n;
        if (threadIdx.x == 0) {
            s_t0 = fin ? 0 : base / B;  // one 64-bit division per tile
            if (bulk_ok) bulk_wait_read<1>();  // this buffer's previous bulk store has been read
        }
        __syncthreads();
        uint8_t *vout = fin ? fview : view;
        uint8_t *dout = fin ? fdir : dirs;
        uint8_t *nout = fin ? nullptr : done;
        const int64_t i = base + threadIdx.x;
        if (i < cnt) {
            uint32_t pr;
            int64_t l;
            if (fin) {
                l = i;
                pr = final_pose[l];
            } else {
                int64_t t = s_t0;
                l = i - t * B;
                while (l >= B) {
                    l -= B;
                    t++;
                }
                // quad layout: steps 4q..4q+3 of lane l are the uint4 at (q * B + l)
                pr = poses[((t >> 2) * B + l) * 4 + (t & 3)];
            }
            const uint32_t *rec = epochs + ((size_t)(pr >> 12) * B + l) * kRec;
            const uint32_t gw = rec[16];
            const int r = pr & 15, c = (pr >> 4) & 15, d = (pr >> 8) & 3;
            render_lane<V, SEE, 1>(r, c, d, gw & 0xFF, (gw >> 8) & 0xFF, G.H, G.W, rec, s_spread,
                                   s_view[buf] + threadIdx.x * VV);
            s_dir[buf][threadIdx.x] = (uint8_t)d;
            s_done[buf][threadIdx.x] = (uint8_t)((pr >> 11) & 1u);
            if (!fin && reward && !((pr >> 10) & 1u)) reward[i] = 0.0;
        }
        const int nvalid = (int)((cnt - base) < 128 ? (cnt - base) : 128);
        if (bulk_ok && nvalid == 128) {
            fence_proxy_async();
            __syncthreads();
            if (threadIdx.x == 0) {
                bulk_store(vout + base * VV, s_view[buf], 128 * VV);
                if (dout) bulk_store(dout + base, s_dir[buf], 128);
                if (nout) bulk_store(nout + base, s_done[buf], 128);
                bulk_commit();
            }
        } else {
            __syncthreads();
            for (int x = threadIdx.x; x < nvalid * VV; x += 128) vout[base * VV + x] = s_view[buf][x];
            if (threadIdx.x < nvalid) {
                if (dout) dout[base + threadIdx.x] = s_dir[buf][threadIdx.x];
                if (nout) nout[base + threadIdx.x] = s_done[buf][threadIdx.x];
            }
        }
    }
    if (threadIdx.x == 0 && bulk_ok) bulk_wait_all();
}

template <int LPW, int WPC>
static void launch_dyn(const Geo &G, const EnvDev &E, int T, const uint8_t *actions, int mode, const amz_seed_t &wrap,
                       uint32_t step0, double *reward, uint8_t *done, uint32_t *poses, uint32_t *epochs,
                       uint32_t *final_pose, amz_level_t *spec, uint32_t *spec_step, int spec_ready, cudaStream_t s) {
    // the goal-reward table: small batches only (LPW >= 8 spends the shared memory on a
    // 4th resident CTA; a goal reach is rare, its one division is off the step chain)
    const int use_lut = G.tep <= 4096 && LPW < 8;
    const size_t sm = (size_t)WPC * sizeof(DynSmem<LPW>) + (use_lut ? ((size_t)G.tep + 1) * 8 : 0);
    ensure_dyn_smem((const void *)k_dyn<LPW, WPC>, (int)sm);
    const int avec = (E.B % 4 == 0) && ((((uintptr_t)actions) & 3u) == 0);
    if (mode == AMZ_RESET_RESAMPLE && !spec_ready)
        k_spec_levels<<<(unsigned)((E.B + 4 * kSpecLPW - 1) / (4 * kSpecLPW)), 128, 0, s>>>(G, E, T, wrap, step0, spec,
                                                                                           spec_step);
    const int64_t warps = (E.B + LPW - 1) / LPW;
    int64_t ctas = (warps + WPC - 1) / WPC;
    if (DynOcc<LPW>::kPersist) {  // one resident wave, the rest from the queue
        static int nsm[64] = {0};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev >= 0 && dev < 64 && !nsm[dev]) cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev);
        // all 4 CTAs per SM the registers allow (3, leaving room for render CTAs beside
        // the dynamics, measured 0.429 -> 0.488 ms at 65536 lanes)
        const int64_t wave = (int64_t)(dev >= 0 && dev < 64 && nsm[dev] ? nsm[dev] : 148) * DynOcc<LPW>::kMinBlocks;
        if (ctas > wave) ctas = wave;
    }

    launch_pdl(k_dyn<LPW, WPC>, dim3((unsigned)ctas), dim3(32 * WPC), sm, s, G, E, T, actions,
               mode, wrap, step0, reward, done, poses, epochs, final_pose, (const amz_level_t *)spec,
               (const uint32_t *)spec_step, avec, use_lut);
}

// Quad tiles: a CTA renders 128 consecutive lanes x 4 consecutive steps, one lane per
// thread.  The lane's 4 step records are one 16-byte load (the uint4 quad k_dyn stores),
// the epoch record address and goal word are fetched once per epoch (a lane rarely
// changes level inside 4 steps), and the CTA's 4 output rows -- 128 consecutive
// observations of one step each -- leave as 4 bulk copies (plus dir / done rows).
// Tiles [0, nq * ng) are (quad, lane group) pairs, quad-major; tiles past that render
// the final observations.
template <int V, bool SEE>
__device__ __forceinline__ void render_obs(int r, int c, int d, uint32_t gw, const Geo &G, const uint32_t *rec,
                                           const uint64_t *spread, uint8_t *out) {
    render_lane<V, SEE, 1>(r, c, d, gw & 0xFF, (gw >> 8) & 0xFF, G.H, G.W, rec, spread, out);
}

template <int V, bool SEE>
__global__ void __launch_bounds__(128) k_render_q(Geo G, int64_t B, int T, const uint32_t *__restrict__ poses,
                                                  const uint32_t *__restrict__ final_pose,
                                                  const uint32_t *__restrict__ epochs, uint8_t *__restrict__ view,
                                                  uint8_t *__restrict__ dirs, double *__restrict__ reward,
                                                  uint8_t *__restrict__ done, uint8_t *__restrict__ fview,
                                                  uint8_t *__restrict__ fdir, int bulk_ok, int64_t ng, int64_t nq,
                                                  uint32_t *gdone, uint32_t *gpass, int lpw, int gmajor) {
    constexpr int VV = V * V;
    __shared__ __align__(128) uint8_t s_view[4][128 * VV];
    __shared__ __align__(16) uint8_t s_dir[4][128];
    __shared__ __align__(16) uint8_t s_done[4][128];
    __shared__ uint64_t s_spread[32];
    // see-through 5x5: each thread's current epoch board (16 line words) staged at a
    // 17-word stride (conflict-free), so a view row is one LDS instead of an LDG whose 32
    // lanes hit ~20 L1 lines (records are 80 B apart)
    constexpr int kBS = (V == 5 && SEE) ? 17 : 1;
    __shared__ uint32_t s_brd[128 * kBS];
    if (!(V == 5 && SEE)) init_spread(s_spread);
    const int tid = threadIdx.x;
    const int64_t tile = blockIdx.x;
    bool fin;
    int64_t q, g;
    if (gmajor) {  // a group's tiles together, in the order the dynamics' queue finishes
                   // groups (persistent k_dyn; 65536 lanes 0.433 -> 0.429 ms)
        const int64_t tpg = nq + (fview ? 1 : 0);
        g = tile / tpg;
        q = tile - g * tpg;
        fin = q == nq;
        if (fin) q = 0;
    } else {  // quad-major
        fin = tile >= nq * ng;
        q = fin ? 0 : tile / ng;
        g = fin ? tile - nq * ng : tile - (tile / ng) * ng;
    }
    const int64_t l = g * 128 + tid;
    const bool live = l < B;
    const int nvalid = (int)((B - g * 128) < 128 ? (B - g * 128) : 128);
    const int nsteps = fin ? 1 : ((T - 4 * (int)q) < 4 ? (T - 4 * (int)q) : 4);
    if (gdone) {
        // this tile's lane group: all of its k_dyn warps have published (launched early by
        // k_dyn's trigger, so the wait overlaps the dynamics' tail).  Bounded: a lost
        // count leaves wrong outputs after ~4 s instead of a hung GPU
        if (tid == 0) {
            const uint32_t want = (uint32_t)((nvalid + lpw - 1) / lpw);
            uint64_t t0 = 0, now = 0;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            for (;;) {
                uint32_t got;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(got) : "l"(gdone + g) : "memory");
                if (got >= want) break;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                if (now - t0 > 4000000000ull) break;
                __nanosleep(200);
            }
            // the group's last tile past its wait zeroes the counters for the next rollout
            // (every tile of this launch has read gdone[g] by then; the next k_dyn runs
            // after this grid completes)
            const uint32_t tiles = (uint32_t)(nq + (fview ? 1 : 0));
            if (atomicAdd(gpass + g, 1u) == tiles - 1u) {
                gdone[g] = 0u;
                gpass[g] = 0u;
            }
        }
        __syncthreads();
    } else {
        __syncthreads();
        pdl_wait();  // poses / epochs from k_dyn
    }
    uint4 pq = make_uint4(0u, 0u, 0u, 0u);
    if (live) pq = fin ? make_uint4(final_pose[l], 0u, 0u, 0u) : reinterpret_cast<const uint4 *>(poses)[q * B + l];
    uint32_t ep = 0xFFFFFFFFu, gw = 0u;
    const uint32_t *rec = nullptr;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        if (k < nsteps) {  // uniform across the CTA
            const uint32_t pr = k == 0 ? pq.x : k == 1 ? pq.y : k == 2 ? pq.z : pq.w;
            if (live) {
                if ((pr >> 12) != ep) {
                    ep = pr >> 12;
                    rec = epochs + ((size_t)ep * B + l) * kRec;
                    gw = rec[16];
                    if constexpr (V == 5 && SEE) {
                        const uint4 *r4 = reinterpret_cast<const uint4 *>(rec);
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const uint4 x = __ldg(r4 + j);
                            s_brd[tid * kBS + 4 * j] = x.x;
                            s_brd[tid * kBS + 4 * j + 1] = x.y;
                            s_brd[tid * kBS + 4 * j + 2] = x.z;
                            s_brd[tid * kBS + 4 * j + 3] = x.w;
                        }
                    }
                }
                s_dir[k][tid] = (uint8_t)((pr >> 8) & 3);
                s_done[k][tid] = (uint8_t)((pr >> 11) & 1u);
                if (!fin && reward && !((pr >> 10) & 1u)) reward[(4 * q + k) * B + l] = 0.0;
            }
            if constexpr (V == 5 && SEE) {
                uint32_t w[7] = {0u, 0u, 0u, 0u, 0u, 0u, 0u};
                int gpos = -1;
                if (live)
                    render5_see_rows(pr & 15, (pr >> 4) & 15, (pr >> 8) & 3, gw & 0xFF, (gw >> 8) & 0xFF, G.H, G.W,
                                     s_brd + tid * kBS, w, gpos);
                store_obs25(s_view[k], tid, live, w);  // warp-collective
                __syncwarp();  // the lane's first word may have been stored by its predecessor
                if (gpos >= 0) s_view[k][tid * VV + gpos] = 2;  // the goal (never off-grid or a wall)
            } else {
                if (live)
                    render_obs<V, SEE>(pr & 15, (pr >> 4) & 15, (pr >> 8) & 3, gw, G, rec, s_spread,
                                       s_view[k] + tid * VV);
            }
        }
    }
    uint8_t *vout = fin ? fview : view;
    uint8_t *dout = fin ? fdir : dirs;
    uint8_t *nout = fin ? nullptr : done;
    if (bulk_ok && nvalid == 128) {
        fence_proxy_async();
        __syncthreads();
        if (tid < nsteps) {
            const int64_t row = (fin ? 0 : (4 * q + tid) * B) + g * 128;
            bulk_store(vout + row * VV, s_view[tid], 128 * VV);
            if (dout) bulk_store(dout + row, s_dir[tid], 128);
            if (nout) bulk_store(nout + row, s_done[tid], 128);
            bulk_commit();
            bulk_wait_all();
        }
    } else {
        __syncthreads();
        for (int k = 0; k < nsteps; k++) {
            const int64_t row = (fin ? 0 : (4 * q + k) * B) + g * 128;
            for (int x = tid; x < nvalid * VV; x += 128) vout[row * VV + x] = s_view[k][x];
            if (tid < nvalid) {
                if (dout) dout[row + tid] = s_dir[k][tid];
                if (nout) nout[row + tid] = s_done[k][tid];
            }
        }
    }
}

template <int V, bool SEE>
static void launch_render(const Geo &G, int64_t B, int64_t n, const uint32_t *poses, const uint32_t *final_pose,
                          const uint32_t *epochs, uint8_t *view, uint8_t *dirs, double *reward, uint8_t *done,
                          uint8_t *fview, uint8_t *fdir, uint32_t *gdone, uint32_t *gpass, int lpw, cudaStream_t s) {
    auto al16 = [](const void *p) { return p == nullptr || (((uintptr_t)p) & 15u) == 0; };
    static const int legacy = getenv("AMZ_RENDER_LEGACY") ? atoi(getenv("AMZ_RENDER_LEGACY")) : 0;
    if (!legacy) {
        const int bulk = al16(view) && al16(dirs) && al16(done) && al16(fview) && al16(fdir) && B % 16 == 0;
        const int T = (int)(n / B);
        const int64_t ng = (B + 127) / 128, nq = (T + 3) / 4;
        const int64_t nt = nq * ng + (fview ? ng : 0);
        launch_pdl(k_render_q<V, SEE>, dim3((unsigned)nt), dim3(128), 0, s, G, B, T, poses, final_pose, epochs, view,
                   dirs, reward, done, fview, fdir, bulk, ng, nq, gdone, gpass, lpw, gdone && lpw >= 8 ? 1 : 0);
        return;
    }
    const int bulk = al16(view) && al16(dirs) && al16(done) && al16(fview) && al16(fdir);
    const int64_t g1 = (n + 127) / 128, g2 = fview ? (B + 127) / 128 : 0, nt = g1 + g2;
    const int64_t grid = nt < 148 * 12 ? nt : 148 * 12;
    launch_pdl(k_render<V, SEE>, dim3((unsigned)grid), dim3(128), 0, s, G, B, n, poses, final_pose, epochs, view, dirs,
               reward, done, fview, fdir, bulk, g1, nt);
}

int launch_env_rollout(const Geo &G, const EnvDev &E, int T, const uint8_t *actions, int mode,
                       const amz_seed_t &wrap, uint32_t step0, uint8_t *view, uint8_t *dirs, double *reward,
                       uint8_t *done, uint8_t *fview, uint8_t *fdir, uint32_t *poses, uint32_t *epochs,
                       uint32_t *final_pose, amz_level_t *spec, uint32_t *spec_step, int spec_ready,
                       cudaStream_t s) {
    if (E.B <= 0) return 0;
    // few lanes per warp: the per-lane chain is latency-bound, and a warp stalls for
    // every resample of any of its lanes, so small warps finish sooner.  AMZ_DYN_LPW
    // (4, 8, 16) overrides the choice for tuning runs (tools/dyn_lpw.sh).
    static const int forced = getenv("AMZ_DYN_LPW") ? atoi(getenv("AMZ_DYN_LPW")) : 0;
    const int lpw = (forced == 2 || forced == 8 || forced == 16) ? forced : (E.B <= 148 * 8 * 16 ? 4 : 8);
    if (forced == 2)
        launch_dyn<2, 4>(G, E, T, actions, mode, wrap, step0, reward, done, poses, epochs, final_pose, spec, spec_step, spec_ready, s);
    else if (forced == 8)
        launch_dyn<8, 4>(G, E, T, actions, mode, wrap, step0, reward, done, poses, epochs, final_pose, spec, spec_step, spec_ready, s);
    else if (forced == 16)
        launch_dyn<16, 4>(G, E, T, actions, mode, wrap, step0, reward, done, poses, epochs, final_pose, spec, spec_step, spec_ready, s);
    else if (E.B <= 148 * 8 * 16)
        launch_dyn<4, 4>(G, E, T, actions, mode, wrap, step0, reward, done, poses, epochs, final_pose, spec, spec_step, spec_ready,
                         s);
    else
        launch_dyn<8, 4>(G, E, T, actions, mode, wrap, step0, reward, done, poses, epochs, final_pose, spec,
                         spec_step, spec_ready, s);
    const int64_t n = (int64_t)T * E.B;
#define AMZ_RR(VV_)                                                                                         \
    case VV_:                                                                                               \
        if (G.see)                                                                                          \
            launch_render<VV_, true>(G, E.B, n, poses, final_pose, epochs, view, dirs, reward, done, fview, \
                                     fdir, E.gdone, E.gpass, lpw, s);                                                \
        else                                                                                                \
            launch_render<VV_, false>(G, E.B, n, poses, final_pose, epochs, view, dirs, reward, done, fview, \
                                      fdir, E.gdone, E.gpass, lpw, s);                                               \
        return 0;
    switch (G.V) {
        AMZ_RR(3)
        AMZ_RR(5)
        AMZ_RR(7)
        AMZ_RR(9)
        default:
            return AMZ_ECONFIG;
    }
#undef AMZ_RR
}

// ---------------------------------------------------------------------------------
// DR level generation: kGenLPW levels per warp, warp-cooperative sampler
// ---------------------------------------------------------------------------------
constexpr int kGenLPW = 1;
__global__ void __launch_bounds__(128) k_sample_levels_w(Geo G, amz_seed_t prefix, uint32_t lane0,
                                                         const uint32_t *__restrict__ lane_ids, int64_t n,
                                                         amz_level_t *__restrict__ out) {
    pdl_wait();  // PDL: the predecessor kernel has completed (its launch overlapped)
    constexpr int LPW = kGenLPW;
    __shared__ __align__(16) WarpSampler X[4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i0 = ((int64_t)blockIdx.x * 4 + warp) * LPW;
    if (i0 >= n) return;
    const int64_t i = i0 + lane;
    const bool mine = lane < LPW && i < n;
    uint64_t k0 = 0, k1 = 0;
    if (mine) {
        amz_seed_t s = prefix;
        seed_absorb(s, lane_ids ? lane_ids[i] : lane0 + (uint32_t)i);
        seed_key(s, k0, k1);
    }
    const unsigned need = __ballot_sync(0xFFFFFFFFu, mine);
    Mask m;
    int ar, ac, ad, gr, gc;
    warp_sample_each(need, k0, k1, G, X[warp], m, ar, ac, ad, gr, gc);
    if (mine) store_level(out + i, m, ar, ac, ad, gr, gc);
}

// One thread per level (thread_sample_level) for large batches.
__global__ void __launch_bounds__(64) k_sample_levels_t(Geo G, amz_seed_t prefix, uint32_t lane0,
                                                        const uint32_t *__restrict__ lane_ids, int64_t n,
                                                        amz_level_t *__restrict__ out) {
    pdl_wait();  // PDL: the predecessor kernel has completed (its launch overlapped)
    __shared__ __align__(16) uint8_t arr[64 * kTSlice];
    const int64_t i = (int64_t)blockIdx.x * 64 + threadIdx.x;
    if ((int64_t)blockIdx.x * 64 + (threadIdx.x & ~31) >= n) return;  // whole warps only
    const bool mine = i < n;
    uint64_t k0 = 0, k1 = 0;
    if (mine) {
        amz_seed_t sd = prefix;
        seed_absorb(sd, lane_ids ? lane_ids[i] : lane0 + (uint32_t)i);
        seed_key(sd, k0, k1);
    }
    Mask m;
    int ar = 0, ac = 0, ad = 0, gr = 0, gc = 0;
    thread_sample_level(k0, k1, G, arr + threadIdx.x * kTSlice, mine, m, ar, ac, ad, gr, gc);
    if (mine) store_level(out + i, m, ar, ac, ad, gr, gc);
}

int launch_sample_levels(const Geo &G, const amz_seed_t &prefix, uint32_t lane0, const uint32_t *ids, int64_t n,
                         amz_level_t *out, cudaStream_t s) {
    if (n <= 0) return 0;
    // one warp per level while the batch is small (latency), one thread per level from
    // 16384 levels on (throughput; the same levels)
    if (n >= 16384)
        launch_pdl(k_sample_levels_t, dim3((unsigned)((n + 63) / 64)), dim3(64), 0, s, G, prefix, lane0, ids, n, out);
    else
        launch_pdl(k_sample_levels_w, dim3((unsigned)((n + 4 * kGenLPW - 1) / (4 * kGenLPW))), dim3(128), 0, s, G,
                   prefix, lane0, ids, n, out);
    return 0;
}

}  // namespace amz
