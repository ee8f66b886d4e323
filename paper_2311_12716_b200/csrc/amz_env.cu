// amz_env.cu -- level generation / mutation kernels and the batched AMaze environment.
//
// Lane state (SoA, resident in HBM, owned by amz_env_t):
//   st[B]    uint4   x = r | c<<8 | d<<16 | terminal<<24
//                    y = goal_r | goal_c<<8 | home_r<<16 | home_c<<24
//                    z = home_dir | time<<8
//   mask[B]  uint4   the lane's level (interior wall bits)
//   board    u32 [16][B]  rendering form of the level (amz_level.cuh)
// The per-step kernel reads st/board from HBM; the fused rollout kernel keeps st in
// registers and the boards in shared memory for all T steps.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "amz_internal.h"
#include "amz_render.cuh"
#include "amz_sampler.cuh"

namespace amz {

// ---------------------------------------------------------------------------------
// level generation / mutation / validation
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_mutate_levels(Geo G, amz_seed_t prefix, uint32_t lane0, int64_t n,
                                                       const amz_level_t *__restrict__ parents,
                                                       const int32_t *__restrict__ pidx, int n_edits,
                                                       amz_level_t *__restrict__ out) {
    pdl_wait();  // PDL: the predecessor kernel has completed (its launch overlapped)
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    amz_seed_t s = prefix;
    seed_absorb(s, lane0 + (uint32_t)i);
    Stream g;
    g.init(s);
    Mask m;
    int ar, ac, ad, gr, gc;
    load_level(parents + (pidx ? pidx[i] : i), m, ar, ac, ad, gr, gc);
    mutate_level_dev(g, G, n_edits, m, ar, ac, gr, gc);
    store_level(out + i, m, ar, ac, ad, gr, gc);
}

// MazeLevel.validate (amaze/level.py:50-66) on packed levels
__device__ __forceinline__ bool level_ok(const Geo &G, const amz_level_t *lv) {
    Mask m;
    int ar, ac, ad, gr, gc;
    load_level(lv, m, ar, ac, ad, gr, gc);
    if (ar < 1 || ar > G.H - 2 || ac < 1 || ac > G.W - 2) return false;
    if (gr < 1 || gr > G.H - 2 || gc < 1 || gc > G.W - 2) return false;
    if (ad > 3) return false;
    if (ar == gr && ac == gc) return false;
    if (mask_bit(m, (ar - 1) * G.iw + ac - 1) || mask_bit(m, (gr - 1) * G.iw + gc - 1)) return false;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        int lo = k * 32;
        uint32_t valid = G.ni >= lo + 32 ? 0xFFFFFFFFu : (G.ni > lo ? (1u << (G.ni - lo)) - 1u : 0u);
        if (m.w[k] & ~valid) return false;
    }
    return true;
}

__global__ void k_check_levels(Geo G, const amz_level_t *__restrict__ lv, int64_t n,
                               unsigned long long *__restrict__ first_bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && !level_ok(G, lv + i)) atomicMin(first_bad, (unsigned long long)i);
}

// ---------------------------------------------------------------------------------
// lane state helpers
// ---------------------------------------------------------------------------------
// Copy a warp's staged V*V-byte records (stage = 32*VV bytes) to dst[0 .. nvalid*VV).
__device__ __forceinline__ void warp_flush(const uint8_t *stage, uint8_t *dst, int nbytes, int lane) {
    if ((((uintptr_t)dst) & 15u) == 0 && (nbytes & 15) == 0) {
        const uint4 *s4 = reinterpret_cast<const uint4 *>(stage);
        uint4 *d4 = reinterpret_cast<uint4 *>(dst);
        for (int k = lane; k < (nbytes >> 4); k += 32) d4[k] = s4[k];
    } else {
        for (int k = lane; k < nbytes; k += 32) dst[k] = stage[k];
    }
}

// ---------------------------------------------------------------------------------
// reset_to_levels / observe / accessors
// ---------------------------------------------------------------------------------
template <int V>
__global__ void __launch_bounds__(128) k_env_reset(Geo G, EnvDev E, const amz_level_t *__restrict__ levels,
                                                   const int64_t *__restrict__ lanes, int64_t n,
                                                   uint8_t *__restrict__ view, int64_t *__restrict__ dirs) {
    pdl_wait();  // PDL: the predecessor kernel has completed (its launch overlapped)
    __shared__ uint8_t stage[128 * V * V];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t wbase = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    uint8_t *my = stage + threadIdx.x * V * V;
    bool ok = i < n;
    int64_t l = i;
    if (ok && lanes) {
        l = lanes[i];
        if (l < 0 || l >= E.B) {  // never write outside the lane arrays: flag it instead
            atomicOr(E.err, 2);
            ok = false;
        }
    }
    if (ok) {
        Mask m;
        LaneRec L;
        load_level(levels + i, m, L.s.r, L.s.c, L.s.d, L.gr, L.gc);
        L.hr = L.s.r;
        L.hc = L.s.c;
        L.hd = L.s.d;
        L.s.time = 0;
        L.term = false;
        E.st[l] = pack_st(L);
        E.mask[l] = make_uint4(m.w[0], m.w[1], m.w[2], m.w[3]);
        build_board(m, G, E.board + l, (int)E.B);
        if (dirs) dirs[i] = L.s.d;
        if (view) lane_render<V>(L.s.r, L.s.c, L.s.d, L.gr, L.gc, G.H, G.W, G.see, E.board + l, (int)E.B, my);
    }
    if (view) {
        __syncwarp();
        if (wbase < n) {
            int nv = (int)(((n - wbase) < 32) ? (n - wbase) : 32);
            warp_flush(stage + (threadIdx.x & ~31) * V * V, view + wbase * V * V, nv * V * V, lane);
        }
    }
}

// Domain-randomised reset fused with level generation (VectorBatchEnv.reset,
// env/batch.py:86-95 over amaze/generator.py:36-52): one warp per lane samples the
// level of key prefix ++ [global lane] (warp-cooperative sampler), then writes the lane
// state, board and observation.  With a wrapper key it also prepares the lane's timeout
// level for the first RESAMPLE rollout (key wrap ++ [tep - 1, global lane]: a fresh
// episode times out at step tep - 1), so that rollout needs no k_spec_levels pass.
// 7 resident CTAs per SM (<= 73 registers): a 4096-lane reset is 1024 CTAs, one wave on
// 148 SMs; at 78 registers (6 per SM) the last 136 CTAs ran as a second wave (27 -> 38 us)
template <int V>
__global__ void __launch_bounds__(128, 7) k_env_reset_dr(Geo G, EnvDev E, amz_seed_t prefix, int prep,
                                                      amz_seed_t wrap, amz_level_t *__restrict__ spec,
                                                      uint32_t *__restrict__ spec_step, uint8_t *__restrict__ view,
                                                      int64_t *__restrict__ dirs) {
    __shared__ __align__(16) WarpSampler X[4];
    __shared__ uint8_t stage[4][V * V];
    __shared__ uint32_t sboard[4][16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t l = (int64_t)blockIdx.x * 4 + warp;
    if (l >= E.B) return;
    const uint32_t gl = E.lane_offset + (uint32_t)l;
    uint64_t k0, k1;
    {
        amz_seed_t sd = prefix;
        if (E.iter) {  // graph replay: this iteration's lane-level stream root.fold_in(it).fold_in(0)
            seed_absorb(sd, *E.iter);
            seed_absorb(sd, 0u);
        }
        seed_absorb(sd, gl);
        seed_key(sd, k0, k1);
    }
    Mask m;
    LaneRec L;
    warp_sample_level(k0, k1, G, X[warp], m, L.s.r, L.s.c, L.s.d, L.gr, L.gc);
    if (lane == 0) {
        L.hr = L.s.r;
        L.hc = L.s.c;
        L.hd = L.s.d;
        L.s.time = 0;
        L.term = false;
        E.st[l] = pack_st(L);
        E.mask[l] = make_uint4(m.w[0], m.w[1], m.w[2], m.w[3]);
        if (dirs) dirs[l] = L.s.d;
    }
    {
        const uint32_t bw = warp_board_word(m, G);  // the sampler's mask is warp-uniform
        if (lane < 16) {
            E.board[lane * E.B + l] = bw;
            sboard[warp][lane] = bw;
        }
    }
    __syncwarp();
    if (view && G.see && V * V <= 32) {
        // see-through: every cell is independent -- one lane per cell (the level is
        // warp-uniform), instead of lane 0 rendering all V*V
        if (lane < V * V) {
            const int vr = lane / V, side = lane % V - V / 2, ahead = V - 1 - vr;
            const int fr = dir_dr(L.s.d), fc = dir_dc(L.s.d);
            const int cr = L.s.r + fr * ahead + fc * side, cc = L.s.c + fc * ahead - fr * side;
            uint32_t code = 3u;  // off-grid
            if (cr >= 0 && cr < G.H && cc >= 0 && cc < G.W)
                code = (cr == L.gr && cc == L.gc) ? 2u : ((sboard[warp][cr] >> cc) & 1u);
            view[l * V * V + lane] = (uint8_t)code;
        }
    } else {
        if (lane == 0 && view)
            lane_render<V>(L.s.r, L.s.c, L.s.d, L.gr, L.gc, G.H, G.W, G.see, sboard[warp], 1, stage[warp]);
        __syncwarp();
        if (view)
            for (int j = lane; j < V * V; j += 32) view[l * V * V + j] = stage[warp][j];
    }
    if (prep) {
        amz_seed_t sd = wrap;
        if (E.iter) {  // root.fold_in(it).fold_in(1): the iteration's auto-reset stream
            seed_absorb(sd, *E.iter);
            seed_absorb(sd, 1u);
        }
        seed_absorb(sd, (uint32_t)(G.tep - 1));
        seed_absorb(sd, gl);
        seed_key(sd, k0, k1);
        Mask ms;
        int ar, ac, ad, gr, gc;
        warp_sample_level(k0, k1, G, X[warp], ms, ar, ac, ad, gr, gc);
        if (lane == 0) {
            store_level(spec + l, ms, ar, ac, ad, gr, gc);
            spec_step[l] = (uint32_t)(G.tep - 1);
        }
    }
}

constexpr int64_t kThreadSamplerMin = 16384;  // levels per launch from which one thread per level wins

// Thread-per-level DR reset (the throughput sampler, thread_sample_level): a CTA owns 32
// lanes; warp 0 samples their levels (key prefix ++ [global lane]) and writes lane state,
// board and observation per thread, warp 1 (with a wrapper key) their timeout levels
// (key wrap ++ [tep - 1, global lane]).  Same levels as k_env_reset_dr (one warp per
// level), at ~1/10 of its instructions per level.
template <int V>
__global__ void __launch_bounds__(64) k_env_reset_dr_t(Geo G, EnvDev E, amz_seed_t prefix, int prep, amz_seed_t wrap,
                                                       amz_level_t *__restrict__ spec,
                                                       uint32_t *__restrict__ spec_step, uint8_t *__restrict__ view,
                                                       int64_t *__restrict__ dirs) {
    __shared__ __align__(16) uint8_t arr[64 * kTSlice];
    __shared__ __align__(16) uint8_t stage[32 * V * V];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 1 && !prep) return;
    const int64_t l0 = (int64_t)blockIdx.x * 32, l = l0 + lane;
    const bool live = l < E.B;
    const uint32_t gl = E.lane_offset + (uint32_t)l;
    uint64_t k0, k1;
    {
        amz_seed_t sd = warp == 0 ? prefix : wrap;
        if (E.iter) {  // graph replay: root.fold_in(it).fold_in(0) (lanes) / .fold_in(1) (auto-reset stream)
            seed_absorb(sd, *E.iter);
            seed_absorb(sd, (uint32_t)warp);
        }
        if (warp == 1) seed_absorb(sd, (uint32_t)(G.tep - 1));
        seed_absorb(sd, gl);
        seed_key(sd, k0, k1);
    }
    Mask m;
    int ar = 0, ac = 0, ad = 0, gr = 0, gc = 0;
    thread_sample_level(k0, k1, G, arr + threadIdx.x * kTSlice, live, m, ar, ac, ad, gr, gc);
    if (warp == 1) {
        if (live) {
            store_level(spec + l, m, ar, ac, ad, gr, gc);
            spec_step[l] = (uint32_t)(G.tep - 1);
        }
        return;
    }
    if (live) {
        LaneRec L;
        L.s.r = L.hr = ar;
        L.s.c = L.hc = ac;
        L.s.d = L.hd = ad;
        L.gr = gr;
        L.gc = gc;
        L.s.time = 0;
        L.term = false;
        E.st[l] = pack_st(L);
        E.mask[l] = make_uint4(m.w[0], m.w[1], m.w[2], m.w[3]);
        build_board(m, G, E.board + l, (int)E.B);
        if (dirs) dirs[l] = ad;
        if (view) lane_render<V>(ar, ac, ad, gr, gc, G.H, G.W, G.see, E.board + l, (int)E.B, stage + lane * V * V);
    }
    if (view) {
        __syncwarp();
        const int nv = (int)((E.B - l0) < 32 ? (E.B - l0) : 32);
        warp_flush(stage, view + l0 * V * V, nv * V * V, lane);
    }
}

template <int V>
__global__ void __launch_bounds__(128) k_env_observe(Geo G, EnvDev E, uint8_t *__restrict__ view,
                                                     int64_t *__restrict__ dirs) {
    __shared__ uint8_t stage[128 * V * V];
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t wbase = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    if (l < E.B) {
        LaneRec L = unpack_st(E.st[l]);
        if (dirs) dirs[l] = L.s.d;
        lane_render<V>(L.s.r, L.s.c, L.s.d, L.gr, L.gc, G.H, G.W, G.see, E.board + l, (int)E.B,
                       stage + threadIdx.x * V * V);
    }
    __syncwarp();
    if (wbase < E.B && view) {
        int nv = (int)(((E.B - wbase) < 32) ? (E.B - wbase) : 32);
        warp_flush(stage + (threadIdx.x & ~31) * V * V, view + wbase * V * V, nv * V * V, lane);
    }
}

__global__ void k_env_levels(EnvDev E, amz_level_t *__restrict__ out) {
    pdl_wait();  // PDL: the predecessor kernel has completed (its launch overlapped)
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= E.B) return;
    LaneRec L = unpack_st(E.st[l]);
    uint4 w = E.mask[l];
    Mask m;
    m.w[0] = w.x;
    m.w[1] = w.y;
    m.w[2] = w.z;
    m.w[3] = w.w;
    store_level(out + l, m, L.hr, L.hc, L.hd, L.gr, L.gc);
}

__global__ void k_env_state(EnvDev E, int32_t *__restrict__ out) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= E.B) return;
    LaneRec L = unpack_st(E.st[l]);
    out[l * 5 + 0] = L.s.r;
    out[l * 5 + 1] = L.s.c;
    out[l * 5 + 2] = L.s.d;
    out[l * 5 + 3] = L.s.time;
    out[l * 5 + 4] = L.term;
}

__global__ void k_env_set_state(EnvDev E, const int32_t *__restrict__ in) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= E.B) return;
    LaneRec L = unpack_st(E.st[l]);
    L.s.r = in[l * 5 + 0];
    L.s.c = in[l * 5 + 1];
    L.s.d = in[l * 5 + 2];
    L.s.time = in[l * 5 + 3];
    L.term = in[l * 5 + 4] != 0;
    E.st[l] = pack_st(L);
}

// ---------------------------------------------------------------------------------
// one step of every lane (+ fused auto-reset)
// ---------------------------------------------------------------------------------
__device__ __forceinline__ int load_action(const void *a, int dtype, int64_t i) {
    if (dtype == 0) return reinterpret_cast<const uint8_t *>(a)[i];
    if (dtype == 1) {
        int v = reinterpret_cast<const int32_t *>(a)[i];
        return (v < 0 || v > 2) ? 3 : v;
    }
    long long v = reinterpret_cast<const int64_t *>(a)[i];
    return (v < 0 || v > 2) ? 3 : (int)v;
}

template <int V>
__global__ void __launch_bounds__(128) k_env_step(Geo G, EnvDev E, const void *__restrict__ actions, int adtype,
                                                  int mode, amz_seed_t wrap, uint32_t step_base,
                                                  const uint32_t *__restrict__ step_dev,
                                                  const amz_seed_t *__restrict__ wrap_dev,
                                                  uint8_t *__restrict__ view, int64_t *__restrict__ dirs,
                                                  double *__restrict__ reward, uint8_t *__restrict__ done,
                                                  double *__restrict__ solved, int64_t *__restrict__ times,
                                                  const int *__restrict__ term_in, int *__restrict__ term_out) {
    // graph replay: key and step come from device memory the captured graph updates
    const uint32_t step_idx = step_dev ? *step_dev : step_base;
    if (wrap_dev) wrap = *wrap_dev;
    __shared__ __align__(16) uint8_t stage[128 * V * V];
    __shared__ __align__(16) WarpSampler sw[4];
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t wbase = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    if (mode == AMZ_RESET_NONE && *term_in > 0) {
        // step_batch raises on terminal lanes before touching anything (amaze/env.py:325-326)
        if (l == 0) {
            *term_out = *term_in;
            atomicOr(E.err, 1);
        }
        return;
    }
    const bool live = l < E.B;
    bool dn = false;
    LaneRec L{};
    uint32_t *bd = E.board + l;
    if (live) {
        L = unpack_st(E.st[l]);
        const int a = load_action(actions, adtype, l);
        const bool reached = lane_transition(L.s, a, L.gr, L.gc, bd, (int)E.B);
        dn = reached || L.s.time >= G.tep;
        if (reward) reward[l] = reached ? goal_reward(L.s.time, G.tep) : 0.0;
        if (done) done[l] = dn;
        if (solved) solved[l] = reached ? 1.0 : 0.0;
        if (times) times[l] = L.s.time;
    }
    if (mode == AMZ_RESET_RESAMPLE) {
        // the warp samples each finished lane's level cooperatively (amz_sampler.cuh)
        unsigned todo = __ballot_sync(0xFFFFFFFFu, dn);
        while (todo) {
            const int tl = __ffs(todo) - 1;
            todo &= todo - 1;
            amz_seed_t sd = wrap;
            seed_absorb(sd, step_idx);  // step_base + the device step counter, if any
            seed_absorb(sd, E.lane_offset + (uint32_t)(wbase + tl));
            uint64_t k0, k1;
            seed_key(sd, k0, k1);
            Mask m;
            int ar, ac, ad, gr, gc;
            warp_sample_level(k0, k1, G, sw[warp], m, ar, ac, ad, gr, gc);
            if (lane == tl) {
                build_board(m, G, bd, (int)E.B);
                E.mask[l] = make_uint4(m.w[0], m.w[1], m.w[2], m.w[3]);
                L.hr = ar;
                L.hc = ac;
                L.hd = ad;
                L.gr = gr;
                L.gc = gc;
            }
            __syncwarp();
        }
    }
    if (live) {
        if (dn) {
            if (mode == AMZ_RESET_NONE) {
                L.term = true;
            } else {
                L.s.r = L.hr;
                L.s.c = L.hc;
                L.s.d = L.hd;
                L.s.time = 0;
                L.term = false;
            }
        }
        E.st[l] = pack_st(L);
        if (dirs) dirs[l] = L.s.d;
        if (view) lane_render<V>(L.s.r, L.s.c, L.s.d, L.gr, L.gc, G.H, G.W, G.see, bd, (int)E.B,
                                 stage + threadIdx.x * V * V);
    }
    if (mode == AMZ_RESET_NONE) {
        unsigned b = __ballot_sync(0xFFFFFFFFu, dn);
        if (lane == 0 && b) atomicAdd(term_out, __popc(b));
    }
    if (view) {
        __syncwarp();
        if (wbase < E.B) {
            int nv = (int)(((E.B - wbase) < 32) ? (E.B - wbase) : 32);
            warp_flush(stage + (threadIdx.x & ~31) * V * V, view + wbase * V * V, nv * V * V, lane);
        }
    }
}

// ---------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------
static inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// Threads per block for one-lane-per-thread kernels: spread small batches over all
// 148 SMs (one warp per SM for B <= 4736) instead of packing them into a few CTAs.
static inline int lanes_per_cta(int64_t n) {
    const int64_t per_sm = (n + 147) / 148;
    int t = (int)(((per_sm + 31) / 32) * 32);
    return t < 32 ? 32 : (t > 128 ? 128 : t);
}

int launch_mutate_levels(const Geo &G, const amz_seed_t &prefix, uint32_t lane0, int64_t n, const amz_level_t *par,
                         const int32_t *pidx, int n_edits, amz_level_t *out, cudaStream_t s) {
    if (n <= 0) return 0;
    const int nt = lanes_per_cta(n);
    launch_pdl(k_mutate_levels, dim3((unsigned)blocks_for(n, nt)), dim3(nt), 0, s, G, prefix, lane0, n, par, pidx, n_edits,
               out);
    return 0;
}

int launch_check_levels(const Geo &G, const amz_level_t *lv, int64_t n, unsigned long long *first_bad,
                        cudaStream_t s) {
    if (n <= 0) return 0;
    k_check_levels<<<blocks_for(n, 256), 256, 0, s>>>(G, lv, n, first_bad);
    return 0;
}

#define AMZ_DISPATCH_V(V_, ...)                                            \
    switch (V_) {                                                         \
        case 3: { constexpr int VT = 3; __VA_ARGS__; } break;             \
        case 5: { constexpr int VT = 5; __VA_ARGS__; } break;             \
        case 7: { constexpr int VT = 7; __VA_ARGS__; } break;             \
        case 9: { constexpr int VT = 9; __VA_ARGS__; } break;             \
        default: return AMZ_ECONFIG;                                      \
    }

int launch_env_reset(const Geo &G, const EnvDev &E, const amz_level_t *lv, const int64_t *lanes, int64_t n,
                     uint8_t *view, int64_t *dirs, cudaStream_t s) {
    if (n <= 0) return 0;
    AMZ_DISPATCH_V(G.V, (launch_pdl(k_env_reset<VT>, dim3((unsigned)blocks_for(n, 128)), dim3(128), 0, s, G, E, lv,
                                    lanes, n, view, dirs)));
    return 0;
}

__global__ void k_iter_advance(uint32_t *iter, uint32_t by) { *iter += by; }

// Host -> device copy of pinned host memory by a kernel reading it through its unified
// address (16-byte loads across PCIe, many in flight).  Used for the per-step input feed
// of a captured graph: a memcpy node whose source is host memory made the driver read
// that buffer at ~23 GB/s (eager and graph alike, once captured), this kernel moves it at
// the link rate, concurrently with the step's kernels.
__global__ void __launch_bounds__(256) k_copy_h2d(uint4 *__restrict__ dst, const uint4 *__restrict__ src, int64_t n16,
                                                 uint8_t *__restrict__ dst_tail, const uint8_t *__restrict__ src_tail,
                                                 int tail) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {  // four 16-byte loads in flight per thread
        const uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
        dst[i] = a;
        dst[i + stride] = b;
        dst[i + 2 * stride] = c;
        dst[i + 3 * stride] = d;
    }
    for (; i < n16; i += stride) dst[i] = src[i];
    if (blockIdx.x == 0 && threadIdx.x < tail) dst_tail[threadIdx.x] = src_tail[threadIdx.x];
}

int launch_copy_h2d(void *dst, const void *src, size_t bytes, int ctas, cudaStream_t s) {
    const int64_t n16 = (int64_t)(bytes / 16);
    const int tail = (int)(bytes - (size_t)n16 * 16);
    k_copy_h2d<<<ctas, 256, 0, s>>>(reinterpret_cast<uint4 *>(dst), reinterpret_cast<const uint4 *>(src), n16,
                                    reinterpret_cast<uint8_t *>(dst) + n16 * 16,
                                    reinterpret_cast<const uint8_t *>(src) + n16 * 16, tail);
    return 0;
}

int launch_iter_advance(uint32_t *iter, uint32_t by, cudaStream_t s) {
    k_iter_advance<<<1, 1, 0, s>>>(iter, by);
    return 0;
}

int launch_env_reset_dr(const Geo &G, const EnvDev &E, const amz_seed_t &prefix, const amz_seed_t *wrap,
                        amz_level_t *spec, uint32_t *spec_step, uint8_t *view, int64_t *dirs, cudaStream_t s) {
    if (E.B <= 0) return 0;
    const amz_seed_t w = wrap ? *wrap : amz_seed_t{};
    const int prep = wrap != nullptr;
    // one warp per level while the batch is small (latency: 4096 lanes 32 us vs 53 us for
    // the thread sampler, which then has < 2 warps per SM), one thread per level beyond
    // (throughput: 65536 lanes 113 us vs 369 us); AMZ_RESET_WARP=0/1 forces one
    static const int forced = getenv("AMZ_RESET_WARP") ? atoi(getenv("AMZ_RESET_WARP")) : -1;
    const bool warp_sampler = forced >= 0 ? forced != 0 : E.B < kThreadSamplerMin;
    if (warp_sampler) {
        AMZ_DISPATCH_V(G.V, (k_env_reset_dr<VT><<<(unsigned)((E.B + 3) / 4), 128, 0, s>>>(G, E, prefix, prep, w, spec,
                                                                                             spec_step, view, dirs)));
    } else {
        AMZ_DISPATCH_V(G.V, (k_env_reset_dr_t<VT><<<(unsigned)((E.B + 31) / 32), 64, 0, s>>>(G, E, prefix, prep, w,
                                                                                                spec, spec_step, view,
                                                                                                dirs)));
    }
    return 0;
}

int launch_env_observe(const Geo &G, const EnvDev &E, uint8_t *view, int64_t *dirs, cudaStream_t s) {
    if (E.B <= 0) return 0;
    AMZ_DISPATCH_V(G.V, (k_env_observe<VT><<<blocks_for(E.B, 128), 128, 0, s>>>(G, E, view, dirs)));
    return 0;
}

int launch_env_levels(const EnvDev &E, amz_level_t *out, cudaStream_t s) {
    if (E.B > 0) launch_pdl(k_env_levels, dim3((unsigned)blocks_for(E.B, 256)), dim3(256), 0, s, E, out);
    return 0;
}

int launch_env_state(const EnvDev &E, int32_t *out, cudaStream_t s) {
    if (E.B > 0) k_env_state<<<blocks_for(E.B, 256), 256, 0, s>>>(E, out);
    return 0;
}

int launch_env_set_state(const EnvDev &E, const int32_t *in, cudaStream_t s) {
    if (E.B > 0) k_env_set_state<<<blocks_for(E.B, 256), 256, 0, s>>>(E, in);
    return 0;
}

int launch_env_step(const Geo &G, const EnvDev &E, const void *actions, int adtype, int mode,
                    const amz_seed_t &wrap, uint32_t step_idx, const uint32_t *step_dev,
                    const amz_seed_t *wrap_dev, uint8_t *view,
                    int64_t *dirs, double *reward,
                    uint8_t *done, double *solved, int64_t *times, const int *term_in, int *term_out,
                    cudaStream_t s) {
    if (E.B <= 0) return 0;
    const int V = G.V;
    AMZ_DISPATCH_V(V, (k_env_step<VT><<<blocks_for(E.B, 128), 128, 0, s>>>(G, E, actions, adtype, mode, wrap,
                                                                          step_idx, step_dev, wrap_dev, view, dirs,
                                                                          reward,
                                                                          done,
                                                                          solved, times, term_in, term_out)));
    return 0;
}

}  // namespace amz
