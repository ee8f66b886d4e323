// amz_rollout.cu -- fused T-step rollout of every lane (the env side of
// agents/rollout.py:120-179 with an action stream), B200 layout.
//
// One warp owns 32 consecutive lanes (one lane per thread) and is independent of every
// other warp: no CTA-wide barrier anywhere in the step loop.  Per step a lane renders
// its observation (V row slices of its wall board in shared memory, expanded to bytes
// through a 32-entry spread table), applies its action and writes reward/done into a
// shared-memory staging ring.  Every NS steps lane 0 ships the warp's staged chunk with
// cp.async.bulk (TMA bulk-copy engine, SASS UBLKCP): for each step one contiguous run
// per output array (view 32*V*V bytes, dir 32, reward 256, done 32).  Chunks are
// double-buffered, so the copies of chunk c drain while chunk c+1 is computed.
//
// Auto-reset levels.  A RESAMPLE reset draws the level of key wrap ++ [step, lane].
// Under random or weak policies almost every reset is a timeout, and a lane's timeout
// step is known before the rollout starts, so k_spec_levels samples those levels up
// front, fully parallel (one warp per lane, amz_sampler.cuh).  A reset at exactly that
// step loads the precomputed level (it is the same key, hence the same level); any
// other reset (a solved episode) is sampled inline by the whole warp cooperatively.
#include <cuda_runtime.h>
#include <stdint.h>

#include "amz_internal.h"
#include "amz_render.cuh"
#include "amz_sampler.cuh"

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
        uint64_t bytes = spread[wall & inb] | (spread[~inb & vm] * 3ull);
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

// rows vr = k, k+G, ... of one lane's observation (G threads per lane); see-through only
template <int V, int G, int BS>
__device__ __forceinline__ void render_rows_see(int r, int c, int d, int gr, int gc, int H, int W,
                                                const uint32_t *board, const uint64_t *spread, int k, uint8_t *out) {
    constexpr int h = V / 2;
    const int fr = dir_dr(d), fc = dir_dc(d);
    const int dr = gr - r, dcol = gc - c;
    const int g_ahead = dr * fr + dcol * fc;
    const int g_side = dr * fc - dcol * fr;
    const bool g_vis = g_ahead >= 0 && g_ahead < V && g_side >= -h && g_side <= h;
    const int g_vr = V - 1 - g_ahead, g_vc = g_side + h;
    for (int vr = k; vr < V; vr += G) {
        uint32_t wall, inb;
        row_bits<V, BS>(r, c, d, H, W, board, vr, wall, inb);
        emit_row<V>(wall, inb, g_vis && g_vr == vr, g_vc, spread, out + vr * V);
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

template <int V, int NS>
struct WarpSmem {
    uint8_t act[2][ACH][32];
    uint8_t view[2 * NS][32 * V * V];
    double rew[2 * NS][32];
    uint8_t dir[2 * NS][32];
    uint8_t done[2 * NS][32];
    uint32_t board[16][32];
    uint32_t stream[kWNW];
};

}  // namespace

// ---------------------------------------------------------------------------------
// speculative timeout levels: lane l times out (if it never reaches the goal) at the
// step where its time reaches max_episode_steps; sample that level now.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_spec_levels(Geo G, EnvDev E, int T, amz_seed_t wrap, uint32_t step0,
                                                     amz_level_t *__restrict__ spec, uint32_t *__restrict__ spec_step) {
    __shared__ __align__(16) uint32_t sw[4][kWNW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t l = (int64_t)blockIdx.x * 4 + warp;
    if (l >= E.B) return;
    const LaneRec L = unpack_st(E.st[l]);
    const int s_to = G.tep - L.s.time - 1;
    if (s_to < 0 || s_to >= T) {
        if (lane == 0) spec_step[l] = 0xFFFFFFFFu;
        return;
    }
    amz_seed_t sd = wrap;
    seed_absorb(sd, step0 + (uint32_t)s_to);
    seed_absorb(sd, E.lane_offset + (uint32_t)l);
    uint64_t k0, k1;
    seed_key(sd, k0, k1);
    Mask m;
    int ar, ac, ad, gr, gc;
    warp_sample_level(k0, k1, G, sw[warp], m, ar, ac, ad, gr, gc);
    if (lane == 0) {
        store_level(spec + l, m, ar, ac, ad, gr, gc);
        spec_step[l] = step0 + (uint32_t)s_to;
    }
}

template <int V, bool SEE, int NS, int WPC>
__global__ void __launch_bounds__(32 * WPC) k_rollout(Geo G, EnvDev E, int T, const uint8_t *__restrict__ actions,
                                                      int mode, amz_seed_t wrap, uint32_t step0,
                                                      uint8_t *__restrict__ view, uint8_t *__restrict__ dirs,
                                                      double *__restrict__ reward, uint8_t *__restrict__ done,
                                                      uint8_t *__restrict__ fview, uint8_t *__restrict__ fdir,
                                                      const amz_level_t *__restrict__ spec,
                                                      const uint32_t *__restrict__ spec_step, int bulk_ok) {
    constexpr int VV = V * V;
    constexpr int VIEWB = 32 * VV;
    using WS = WarpSmem<V, NS>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *s_spread = reinterpret_cast<uint64_t *>(smem);  // [32] spread table
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WS &S = reinterpret_cast<WS *>(smem + 256)[warp];
    init_spread(s_spread);
    __syncthreads();

    const int64_t B = E.B;
    const int64_t lane0 = ((int64_t)blockIdx.x * WPC + warp) * 32;
    if (lane0 >= B) return;
    const int64_t l = lane0 + lane;
    const bool live = l < B;
    const int nv = (int)((B - lane0) < 32 ? (B - lane0) : 32);
    uint32_t *bd = &S.board[0][lane];

    LaneRec L;
    Mask m;
    bool lvl_changed = false;
    uint32_t my_spec = 0xFFFFFFFFu;
    if (live) {
        L = unpack_st(E.st[l]);
#pragma unroll
        for (int w = 0; w < 16; w++) bd[w * 32] = E.board[w * B + l];
        if (mode == AMZ_RESET_RESAMPLE) my_spec = spec_step[l];
    } else {
        L = LaneRec{};
    }
    const bool avec = bulk_ok && nv == 32;
    fetch_actions<32>(S.act[0], actions, B, lane0, nv, 0, T, lane, avec);
    __syncwarp();

    static_assert(ACH % NS == 0, "action chunk must hold whole staging chunks");
    const int nchunks = (T + NS - 1) / NS;
    for (int c = 0; c < nchunks; c++) {
        const int hb = (c & 1) * NS;
        const int t0 = c * NS;
        const int ns = (T - t0) < NS ? (T - t0) : NS;
        if ((t0 % ACH) == 0) {
            fetch_actions<32>(S.act[((t0 / ACH) + 1) & 1], actions, B, lane0, nv, t0 + ACH, T, lane, avec);
            cp_wait<1>();
            __syncwarp();
        }
#pragma unroll
        for (int j = 0; j < NS; j++) {
            if (j >= ns) break;
            const int s = hb + j;
            const int ta = t0 + j;
            const uint8_t aj = S.act[(ta / ACH) & 1][ta % ACH][lane];
            bool dn = false;
            if (live) {
                render_lane<V, SEE>(L.s.r, L.s.c, L.s.d, L.gr, L.gc, G.H, G.W, bd, s_spread, &S.view[s][lane * VV]);
                S.dir[s][lane] = (uint8_t)L.s.d;
                const bool reached = lane_transition(L.s, aj, L.gr, L.gc, bd, 32);
                dn = reached || L.s.time >= G.tep;
                S.rew[s][lane] = reached ? goal_reward(L.s.time, G.tep) : 0.0;
                S.done[s][lane] = dn;
            }
            const unsigned any = __ballot_sync(0xFFFFFFFFu, dn);
            if (any) {
                const uint32_t gstep = step0 + (uint32_t)(t0 + j);
                if (mode == AMZ_RESET_RESAMPLE) {
                    const bool hit = dn && my_spec == gstep;
                    if (hit) {
                        int ar, ac, ad, gr, gc;
                        load_level(spec + l, m, ar, ac, ad, gr, gc);
                        build_board(m, G, bd, 32);
                        L.hr = ar;
                        L.hc = ac;
                        L.hd = ad;
                        L.gr = gr;
                        L.gc = gc;
                        lvl_changed = true;
                    }
                    unsigned todo = __ballot_sync(0xFFFFFFFFu, dn && !hit);
                    while (todo) {
                        const int tl = __ffs(todo) - 1;
                        todo &= todo - 1;
                        amz_seed_t sd = wrap;
                        seed_absorb(sd, gstep);
                        seed_absorb(sd, E.lane_offset + (uint32_t)(lane0 + tl));
                        uint64_t k0, k1;
                        seed_key(sd, k0, k1);
                        Mask nm;
                        int ar, ac, ad, gr, gc;
                        warp_sample_level(k0, k1, G, S.stream, nm, ar, ac, ad, gr, gc);
                        if (lane == tl) {
                            m = nm;
                            build_board(m, G, bd, 32);
                            L.hr = ar;
                            L.hc = ac;
                            L.hd = ad;
                            L.gr = gr;
                            L.gc = gc;
                            lvl_changed = true;
                        }
                        __syncwarp();
                    }
                }
                if (dn) {
                    L.s.r = L.hr;
                    L.s.c = L.hc;
                    L.s.d = L.hd;
                    L.s.time = 0;
                    L.term = false;
                }
                __syncwarp();
            }
        }
        // ---- chunk end: ship the warp's NS staged steps ----
        __syncwarp();
        if (bulk_ok) {
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                for (int j = 0; j < ns; j++) {
                    const int s = hb + j;
                    const int64_t row = (int64_t)(t0 + j) * B + lane0;
                    bulk_store(view + row * VV, S.view[s], VIEWB);
                    bulk_store(dirs + row, S.dir[s], 32);
                    bulk_store(reward + row, S.rew[s], 256);
                    bulk_store(done + row, S.done[s], 32);
                }
                bulk_commit();
                bulk_wait_read<1>();  // chunk c-1 finished reading the other half
            }
        } else {
            for (int j = 0; j < ns; j++) {
                const int s = hb + j;
                const int64_t row = (int64_t)(t0 + j) * B + lane0;
                for (int x = lane; x < nv * VV; x += 32) view[row * VV + x] = S.view[s][x];
                if (lane < nv) {
                    dirs[row + lane] = S.dir[s][lane];
                    reward[row + lane] = S.rew[s][lane];
                    done[row + lane] = S.done[s][lane];
                }
            }
        }
        __syncwarp();
    }
    // ---- cursor observation + state write-back ----
    if (bulk_ok && lane == 0) bulk_wait_read<0>();
    __syncwarp();
    if (live) {
        render_lane<V, SEE>(L.s.r, L.s.c, L.s.d, L.gr, L.gc, G.H, G.W, bd, s_spread, &S.view[0][lane * VV]);
        S.dir[0][lane] = (uint8_t)L.s.d;
        E.st[l] = pack_st(L);
        if (lvl_changed) {
            E.mask[l] = make_uint4(m.w[0], m.w[1], m.w[2], m.w[3]);
#pragma unroll
            for (int w = 0; w < 16; w++) E.board[w * B + l] = bd[w * 32];
        }
    }
    __syncwarp();
    if (bulk_ok) {
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            if (fview) bulk_store(fview + lane0 * VV, S.view[0], VIEWB);
            if (fdir) bulk_store(fdir + lane0, S.dir[0], 32);
            bulk_commit();
            bulk_wait_all();
        }
    } else {
        if (fview)
            for (int x = lane; x < nv * VV; x += 32) fview[lane0 * VV + x] = S.view[0][x];
        if (fdir && lane < nv) fdir[lane0 + lane] = S.dir[0][lane];
    }
}


// ---------------------------------------------------------------------------------
// small batches: 4 threads per lane, 8 lanes per warp, every warp independent.
// The group computes its lane's transition redundantly, renders rows k, k+4 of the
// observation, and the warp writes each step's 8-lane output runs with 8-byte stores.
// ---------------------------------------------------------------------------------
template <int V, bool SEE>
__global__ void __launch_bounds__(128) k_rollout_g4(Geo G, EnvDev E, int T, const uint8_t *__restrict__ actions,
                                                   int mode, amz_seed_t wrap, uint32_t step0,
                                                   uint8_t *__restrict__ view, uint8_t *__restrict__ dirs,
                                                   double *__restrict__ reward, uint8_t *__restrict__ done,
                                                   uint8_t *__restrict__ fview, uint8_t *__restrict__ fdir,
                                                   const amz_level_t *__restrict__ spec,
                                                   const uint32_t *__restrict__ spec_step, int vec_ok) {
    constexpr int VV = V * V;
    constexpr int VB = 8 * VV;  // view bytes per warp-step
    constexpr int VBP = (VB + 15) & ~15;
    struct alignas(16) WS {
        uint8_t act[2][ACH][8];
        uint8_t view[VBP];
        double rew[8];
        uint8_t dir[8];
        uint8_t done[8];
        uint32_t board[16][8];
        uint32_t stream[kWNW];
    };
    __shared__ uint64_t s_spread[32];
    __shared__ WS wsm[4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane >> 2, k = lane & 3;
    WS &S = wsm[warp];
    init_spread(s_spread);
    __syncthreads();
    const int64_t B = E.B;
    const int64_t lane0 = ((int64_t)blockIdx.x * 4 + warp) * 8;
    if (lane0 >= B) return;
    const int64_t l = lane0 + grp;
    const bool live = l < B;
    const int nv = (int)((B - lane0) < 8 ? (B - lane0) : 8);
    const bool vec = vec_ok && nv == 8;
    uint32_t *bd = &S.board[0][grp];
    LaneRec L{};
    Mask m;
    bool lvl_changed = false;
    uint32_t my_spec = 0xFFFFFFFFu;
    if (live) {
        L = unpack_st(E.st[l]);
        for (int w = k; w < 16; w += 4) bd[w * 8] = E.board[w * B + l];
        if (mode == AMZ_RESET_RESAMPLE) my_spec = spec_step[l];
    }
    const bool avec = vec_ok && nv == 8;
    fetch_actions<8>(S.act[0], actions, B, lane0, nv, 0, T, lane, avec);
    __syncwarp();
    for (int t = 0; t < T; t++) {
        if ((t % ACH) == 0) {
            // chunk t/ACH is in flight since one chunk ago; start the next one
            fetch_actions<8>(S.act[((t / ACH) + 1) & 1], actions, B, lane0, nv, t + ACH, T, lane, avec);
            cp_wait<1>();
            __syncwarp();
        }
        const uint8_t a = S.act[(t / ACH) & 1][t % ACH][grp];
        bool dn = false;
        if (live) {
            if (SEE)
                render_rows_see<V, 4, 8>(L.s.r, L.s.c, L.s.d, L.gr, L.gc, G.H, G.W, bd, s_spread, k,
                                         S.view + grp * VV);
            else
                render_lane<V, false, 8>(L.s.r, L.s.c, L.s.d, L.gr, L.gc, G.H, G.W, bd, s_spread,
                                         S.view + grp * VV, k, 4);
            if (k == 0) S.dir[grp] = (uint8_t)L.s.d;
            const bool reached = lane_transition(L.s, a, L.gr, L.gc, bd, 8);
            dn = reached || L.s.time >= G.tep;
            if (k == 1) {
                S.rew[grp] = reached ? goal_reward(L.s.time, G.tep) : 0.0;
                S.done[grp] = dn;
            }
        }
        __syncwarp();
        // ship this step's 8-lane runs
        const int64_t row = (int64_t)t * B + lane0;
        if (vec) {
            for (int x = lane; x < VB / 8; x += 32)
                reinterpret_cast<uint64_t *>(view + row * VV)[x] = reinterpret_cast<const uint64_t *>(S.view)[x];
            if (lane < 8) reward[row + lane] = S.rew[lane];
            if (lane == 8) *reinterpret_cast<uint64_t *>(dirs + row) = *reinterpret_cast<const uint64_t *>(S.dir);
            if (lane == 9) *reinterpret_cast<uint64_t *>(done + row) = *reinterpret_cast<const uint64_t *>(S.done);
        } else {
            for (int x = lane; x < nv * VV; x += 32) view[row * VV + x] = S.view[x];
            if (lane < nv) {
                reward[row + lane] = S.rew[lane];
                dirs[row + lane] = S.dir[lane];
                done[row + lane] = S.done[lane];
            }
        }
        const unsigned any = __ballot_sync(0xFFFFFFFFu, dn && k == 0);
        if (any) {
            const uint32_t gstep = step0 + (uint32_t)t;
            if (mode == AMZ_RESET_RESAMPLE) {
                const bool hit = dn && my_spec == gstep;
                if (hit) {
                    int ar, ac, ad, gr, gc;
                    load_level(spec + l, m, ar, ac, ad, gr, gc);
                    if (k == 0) build_board(m, G, bd, 8);
                    L.hr = ar;
                    L.hc = ac;
                    L.hd = ad;
                    L.gr = gr;
                    L.gc = gc;
                    lvl_changed = true;
                }
                unsigned todo = __ballot_sync(0xFFFFFFFFu, dn && !hit && k == 0);
                while (todo) {
                    const int tl = __ffs(todo) - 1;  // lane index of the group leader
                    todo &= todo - 1;
                    amz_seed_t sd = wrap;
                    seed_absorb(sd, gstep);
                    seed_absorb(sd, E.lane_offset + (uint32_t)(lane0 + (tl >> 2)));
                    uint64_t k0, k1;
                    seed_key(sd, k0, k1);
                    Mask nm;
                    int ar, ac, ad, gr, gc;
                    warp_sample_level(k0, k1, G, S.stream, nm, ar, ac, ad, gr, gc);
                    if (grp == (tl >> 2)) {
                        m = nm;
                        if (k == 0) build_board(m, G, bd, 8);
                        L.hr = ar;
                        L.hc = ac;
                        L.hd = ad;
                        L.gr = gr;
                        L.gc = gc;
                        lvl_changed = true;
                    }
                    __syncwarp();
                }
            }
            if (dn) {
                L.s.r = L.hr;
                L.s.c = L.hc;
                L.s.d = L.hd;
                L.s.time = 0;
                L.term = false;
            }
        }
        __syncwarp();
    }
    // cursor observation + state write-back
    if (live) {
        if (SEE)
            render_rows_see<V, 4, 8>(L.s.r, L.s.c, L.s.d, L.gr, L.gc, G.H, G.W, bd, s_spread, k, S.view + grp * VV);
        else
            render_lane<V, false, 8>(L.s.r, L.s.c, L.s.d, L.gr, L.gc, G.H, G.W, bd, s_spread, S.view + grp * VV, k,
                                     4);
        if (k == 0) {
            S.dir[grp] = (uint8_t)L.s.d;
            E.st[l] = pack_st(L);
            if (lvl_changed) E.mask[l] = make_uint4(m.w[0], m.w[1], m.w[2], m.w[3]);
        }
        if (lvl_changed)
            for (int w = k; w < 16; w += 4) E.board[w * B + l] = bd[w * 8];
    }
    __syncwarp();
    if (fview)
        for (int x = lane; x < nv * VV; x += 32) fview[lane0 * VV + x] = S.view[x];
    if (fdir && lane < nv) fdir[lane0 + lane] = S.dir[lane];
}

template <int V, bool SEE>
static int launch_rollout_g4(const Geo &G, const EnvDev &E, int T, const uint8_t *actions, int mode,
                             const amz_seed_t &wrap, uint32_t step0, uint8_t *view, uint8_t *dirs, double *reward,
                             uint8_t *done, uint8_t *fview, uint8_t *fdir, cudaStream_t s) {
    auto al8 = [](const void *p) { return (((uintptr_t)p) & 7u) == 0; };
    const int vec = (E.B % 8 == 0) && al8(view) && al8(dirs) && al8(reward) && al8(done) &&
                    ((((uintptr_t)actions) & 3u) == 0);
    if (mode == AMZ_RESET_RESAMPLE)
        k_spec_levels<<<(unsigned)((E.B + 3) / 4), 128, 0, s>>>(G, E, T, wrap, step0, E.spec, E.spec_step);
    const unsigned grid = (unsigned)((E.B + 31) / 32);
    k_rollout_g4<V, SEE><<<grid, 128, 0, s>>>(G, E, T, actions, mode, wrap, step0, view, dirs, reward, done, fview,
                                              fdir, E.spec, E.spec_step, vec);
    return 0;
}

template <int V, bool SEE, int NS, int WPC>
static int launch_rollout_t(const Geo &G, const EnvDev &E, int T, const uint8_t *actions, int mode,
                            const amz_seed_t &wrap, uint32_t step0, uint8_t *view, uint8_t *dirs, double *reward,
                            uint8_t *done, uint8_t *fview, uint8_t *fdir, cudaStream_t s) {
    const size_t sm = 256 + (size_t)WPC * sizeof(WarpSmem<V, NS>);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_rollout<V, SEE, NS, WPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        attr = true;
    }
    auto al16 = [](const void *p) { return p == nullptr || (((uintptr_t)p) & 15u) == 0; };
    const int bulk = (E.B % 32 == 0) && al16(view) && al16(dirs) && al16(reward) && al16(done) && al16(fview) &&
                     al16(fdir) && ((((uintptr_t)actions) & 3u) == 0);
    if (mode == AMZ_RESET_RESAMPLE)
        k_spec_levels<<<(unsigned)((E.B + 3) / 4), 128, 0, s>>>(G, E, T, wrap, step0, E.spec, E.spec_step);
    const int64_t warps = (E.B + 31) / 32;
    const unsigned grid = (unsigned)((warps + WPC - 1) / WPC);
    k_rollout<V, SEE, NS, WPC><<<grid, 32 * WPC, sm, s>>>(G, E, T, actions, mode, wrap, step0, view, dirs, reward,
                                                          done, fview, fdir, E.spec, E.spec_step, bulk);
    return 0;
}

template <int V, bool SEE>
static int launch_rollout_v(const Geo &G, const EnvDev &E, int T, const uint8_t *actions, int mode,
                            const amz_seed_t &wrap, uint32_t step0, uint8_t *view, uint8_t *dirs, double *reward,
                            uint8_t *done, uint8_t *fview, uint8_t *fdir, cudaStream_t s) {
    // small batches: 4 threads per lane (keeps ~3.5+ warps per SM at 4096 lanes);
    // large batches: one lane per thread, TMA bulk stores
    if (E.B <= 148 * 32 * 4)
        return launch_rollout_g4<V, SEE>(G, E, T, actions, mode, wrap, step0, view, dirs, reward, done, fview, fdir,
                                         s);
    return launch_rollout_t<V, SEE, 4, 4>(G, E, T, actions, mode, wrap, step0, view, dirs, reward, done, fview, fdir,
                                          s);
}

int launch_env_rollout(const Geo &G, const EnvDev &E, int T, const uint8_t *actions, int mode,
                       const amz_seed_t &wrap, uint32_t step0, uint8_t *view, uint8_t *dirs, double *reward,
                       uint8_t *done, uint8_t *fview, uint8_t *fdir, cudaStream_t s) {
    if (E.B <= 0) return 0;
#define AMZ_RV(VV_)                                                                                              \
    case VV_:                                                                                                    \
        return G.see ? launch_rollout_v<VV_, true>(G, E, T, actions, mode, wrap, step0, view, dirs, reward, done, \
                                                   fview, fdir, s)                                               \
                     : launch_rollout_v<VV_, false>(G, E, T, actions, mode, wrap, step0, view, dirs, reward, done, \
                                                    fview, fdir, s);
    switch (G.V) {
        AMZ_RV(3)
        AMZ_RV(5)
        AMZ_RV(7)
        AMZ_RV(9)
        default:
            return AMZ_ECONFIG;
    }
#undef AMZ_RV
}

// DR level generation: one warp per level (amz_sampler.cuh)
__global__ void __launch_bounds__(128) k_sample_levels_w(Geo G, amz_seed_t prefix, uint32_t lane0,
                                                         const uint32_t *__restrict__ lane_ids, int64_t n,
                                                         amz_level_t *__restrict__ out) {
    __shared__ __align__(16) uint32_t sw[4][kWNW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * 4 + warp;
    if (i >= n) return;
    amz_seed_t s = prefix;
    seed_absorb(s, lane_ids ? lane_ids[i] : lane0 + (uint32_t)i);
    uint64_t k0, k1;
    seed_key(s, k0, k1);
    Mask m;
    int ar, ac, ad, gr, gc;
    warp_sample_level(k0, k1, G, sw[warp], m, ar, ac, ad, gr, gc);
    if (lane == 0) store_level(out + i, m, ar, ac, ad, gr, gc);
}

int launch_sample_levels(const Geo &G, const amz_seed_t &prefix, uint32_t lane0, const uint32_t *ids, int64_t n,
                         amz_level_t *out, cudaStream_t s) {
    if (n <= 0) return 0;
    k_sample_levels_w<<<(unsigned)((n + 3) / 4), 128, 0, s>>>(G, prefix, lane0, ids, n, out);
    return 0;
}

}  // namespace amz
