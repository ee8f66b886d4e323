// amz_plr.cu -- device-resident PLR level buffer: rank-prioritised replay sampling and
// the sequential buffer_update of SPEC.md:373-377, made fast without changing its
// result.  Semantics (and the open choices SPEC leaves, pinned the same way) follow
// oracle/plr_np.py.
//
// Buffer arrays live in HBM (slots 0..size-1 are valid; slots fill in order and are
// only ever overwritten by eviction).  Both kernels run as ONE CTA: K <= 4096 fits
// its shared memory, and the sampler's cumsum and the update's candidate loop are
// inherently ordered.
//
// Sampling (k_plr_sample):
//   1. rank: CUB block radix sort, (seq asc) then stable (score desc)
//   2. w = LUT[rank]  (host LUT (1/r)^(1/beta), computed by numpy -> bit-exact)
//   3. sum(w) in numpy's pairwise order (parallel leaves, ordered combine)
//   4. P = (1-rho) w/sum(w) + rho st/sum(st); cdf = sequential cumsum / cdf[-1]
//      (numpy Generator.choice), u_i = i-th random() of the key's stream
//      (counter-based: block i/4 of Philox), slot_i = searchsorted(cdf, u_i, 'right')
// Update (k_plr_update): see the comment above the kernel.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/block/block_radix_sort.cuh>

#include "amz_internal.h"

namespace amz {

constexpr int kPlrThreads = 1024;
constexpr int kPlrMaxK = 4096;
constexpr int kHash = 8192;  // smem hash table entries (>= 2 * K)

__device__ __forceinline__ uint32_t level_hash(const uint4 &w, uint32_t pose) {
    uint32_t h = 0x9E3779B9u;
    h = (h ^ w.x) * 0x85EBCA6Bu;
    h = (h ^ w.y) * 0xC2B2AE35u;
    h = (h ^ w.z) * 0x85EBCA6Bu;
    h = (h ^ w.w) * 0xC2B2AE35u;
    h = (h ^ pose) * 0x27D4EB2Fu;
    return h ^ (h >> 15);
}

// pose word = agent_r | agent_c<<8 | agent_dir<<16 | goal_r<<24, second word goal_c
__device__ __forceinline__ void level_key(const amz_level_t *lv, uint4 &w, uint32_t &p0, uint32_t &p1) {
    w = *reinterpret_cast<const uint4 *>(lv->walls);
    const uint2 p = *reinterpret_cast<const uint2 *>(&lv->agent_r);
    p0 = p.x;
    p1 = p.y & 0xFFu;
}

__device__ __forceinline__ bool key_eq(const amz_level_t *a, const uint4 &w, uint32_t p0, uint32_t p1) {
    uint4 x;
    uint32_t q0, q1;
    level_key(a, x, q0, q1);
    return x.x == w.x && x.y == w.y && x.z == w.z && x.w == w.w && q0 == p0 && q1 == p1;
}

// numpy float64 maximum/ordering helpers
__device__ __forceinline__ bool entry_less(double sa, int64_t la, int64_t qa, double sb, int64_t lb, int64_t qb) {
    if (sa != sb) return sa < sb;
    if (la != lb) return la < lb;
    return qa < qb;
}

// ---------------------------------------------------------------------------------
// numpy pairwise sum of x[0..n) evaluated by a whole CTA (leaves in parallel).
// Returns the sum in thread 0 (valid after the call in all threads via smem).
// ---------------------------------------------------------------------------------
__device__ double block_pairwise_sum(const double *x, int n, double *leafbuf /* >= 64 */, int *leafinfo /* >= 3*64+1 */) {
    // thread 0 walks numpy's recursion (pw(s, n) = n <= 128 ? leaf : pw(left) + pw(right),
    // left length n/2 rounded down to a multiple of 8) and records, per leaf, its range
    // and how many pending sums close after it.
    if (threadIdx.x == 0) {
        int fs[24], fn[24], st[24];
        int fp = 1, nl = 0;
        fs[0] = 0;
        fn[0] = n;
        st[0] = 0;
        while (fp > 0) {
            const int i = fp - 1;
            if (st[i] == 0 && fn[i] <= 128) {
                leafinfo[1 + 3 * nl] = fs[i];
                leafinfo[2 + 3 * nl] = fn[i];
                leafinfo[3 + 3 * nl] = 0;
                nl++;
                fp--;
            } else if (st[i] < 2) {
                int n2 = fn[i] / 2;
                n2 -= n2 % 8;
                const int cs = st[i] == 0 ? fs[i] : fs[i] + n2;
                const int cn = st[i] == 0 ? n2 : fn[i] - n2;
                st[i]++;
                fs[fp] = cs;
                fn[fp] = cn;
                st[fp] = 0;
                fp++;
            } else {
                leafinfo[3 + 3 * (nl - 1)]++;
                fp--;
            }
        }
        leafinfo[0] = nl;
    }
    __syncthreads();
    const int nl = leafinfo[0];
    for (int li = threadIdx.x; li < nl; li += blockDim.x) {
        const int s = leafinfo[1 + 3 * li], len = leafinfo[2 + 3 * li];
        double res;
        if (len < 8) {
            res = 0.0;
            for (int k = 0; k < len; k++) res = res + x[s + k];
        } else {
            double r[8];
#pragma unroll
            for (int k = 0; k < 8; k++) r[k] = x[s + k];
            int k = 8;
            const int l8 = len - len % 8;
            for (; k < l8; k += 8) {
#pragma unroll
                for (int j = 0; j < 8; j++) r[j] = r[j] + x[s + k + j];
            }
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
            for (; k < len; k++) res = res + x[s + k];
        }
        leafbuf[li] = res;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double stk[40];
        int sp = 0;
        for (int li = 0; li < nl; li++) {
            stk[sp++] = leafbuf[li];
            for (int a = 0; a < leafinfo[3 + 3 * li]; a++) {
                double b = stk[--sp];
                double c = stk[--sp];
                stk[sp++] = c + b;
            }
        }
        leafbuf[0] = stk[0];
    }
    __syncthreads();
    return leafbuf[0];
}

// ---------------------------------------------------------------------------------
// sampling
// ---------------------------------------------------------------------------------
#ifndef AMZ_SORT_BITS
#define AMZ_SORT_BITS 4
#endif
using SampleSort = cub::BlockRadixSort<unsigned long long, kPlrThreads, 4, int, AMZ_SORT_BITS>;
struct SampleSmem {
    typename SampleSort::TempStorage sort;
    double p[kPlrMaxK];
    double leaf[64];
    int leafinfo[3 * 64 + 4];
    unsigned long long st_total;
    unsigned long long seq_min, seq_max;
    int rank_slot[kPlrMaxK];
};

__global__ void __launch_bounds__(kPlrThreads, 1)
    k_plr_sample(PlrDev D, amz_seed_t key, int64_t n, double one_minus_rho, double rho,
                 const double *__restrict__ lut, int64_t iter, int32_t *__restrict__ slots_out,
                 amz_level_t *__restrict__ levels_out, double *__restrict__ maxret_out,
                 double *__restrict__ score_out, int *__restrict__ err) {
    extern __shared__ __align__(16) uint8_t smraw[];
    SampleSmem &S = *reinterpret_cast<SampleSmem *>(smraw);
    const int tid = threadIdx.x;
    const int size = (int)D.meta[0];
    if (size <= 0) {
        if (tid == 0) atomicOr(err, 2);
        return;
    }
    // ---- 1. ranks: sort by seq asc, then stable by score desc ----
    // seq values are distinct and span a narrow range: the first sort only runs over the
    // bits of (seq - min seq), with the padding keys (all ones) above every valid key
    using Sort = SampleSort;
    unsigned long long keys[4];
    int vals[4];
    if (tid == 0) {
        S.seq_min = ~0ull;
        S.seq_max = 0ull;
    }
    __syncthreads();
    {
        unsigned long long mn = ~0ull, mx = 0ull;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int i = tid * 4 + k;
            keys[k] = i < size ? (unsigned long long)D.seq[i] : 0ull;
            if (i < size) {
                mn = keys[k] < mn ? keys[k] : mn;
                mx = keys[k] > mx ? keys[k] : mx;
            }
        }
        atomicMin(&S.seq_min, mn);
        atomicMax(&S.seq_max, mx);
    }
    __syncthreads();
    const unsigned long long smin = S.seq_min;
    const int seq_bits = 64 - __clzll((long long)(S.seq_max - smin + 1ull));
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int i = tid * 4 + k;
        keys[k] = i < size ? keys[k] - smin : ~0ull;
        vals[k] = i;
    }
    Sort(S.sort).Sort(keys, vals, 0, seq_bits < 1 ? 1 : seq_bits);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int i = vals[k];
        // descending score = ascending bitwise-inverted key; non-negative doubles order like their bits
        unsigned long long b = 0ull;
        if (i < size) {
            double s = D.score[i];
            s = s == 0.0 ? 0.0 : s;  // -0.0 ties with 0.0, as in numpy's sort
            unsigned long long u = (unsigned long long)__double_as_longlong(s);
            // total order for all doubles: flip negatives entirely, positives' sign bit
            u = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
            b = ~u;
        } else {
            b = ~0ull;
        }
        keys[k] = b;
    }
    Sort(S.sort).Sort(keys, vals);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int pos = tid * 4 + k;
        if (vals[k] < size) S.rank_slot[vals[k]] = pos;  // rank - 1
    }
    if (tid == 0) S.st_total = 0ull;
    __syncthreads();
    // ---- 2./3. weights and their pairwise sum (slot order) ----
    unsigned long long my_st = 0ull;
    for (int i = tid; i < size; i += blockDim.x) {
        S.p[i] = lut[S.rank_slot[i]];
        my_st += (unsigned long long)(iter - D.last[i]);
    }
    // staleness total (exact integer sum)
    for (int o = 16; o > 0; o >>= 1) my_st += __shfl_down_sync(0xFFFFFFFFu, my_st, o);
    if ((tid & 31) == 0) atomicAdd(&S.st_total, my_st);
    const double wsum = block_pairwise_sum(S.p, size, S.leaf, S.leafinfo);
    const long long tot = (long long)S.st_total;
    // ---- 4. P, cdf ----
    for (int i = tid; i < size; i += blockDim.x) {
        const double ps = S.p[i] / wsum;
        if (tot == 0) {
            S.p[i] = ps;
        } else {
            const double pc = (double)(iter - D.last[i]) / (double)tot;
            S.p[i] = one_minus_rho * ps + rho * pc;
        }
    }
    __syncthreads();
    if (tid == 0) {
        // numpy's sequential cumsum; the next 16 loads are issued ahead of this block's
        // stores so only the add chain is serial
        constexpr int CB = 16;
        double acc = 0.0, cur[CB], nxt[CB];
#pragma unroll
        for (int j = 0; j < CB; j++) cur[j] = j < size ? S.p[j] : 0.0;
        for (int b = 0; b < size; b += CB) {
#pragma unroll
            for (int j = 0; j < CB; j++) nxt[j] = b + CB + j < size ? S.p[b + CB + j] : 0.0;
#pragma unroll
            for (int j = 0; j < CB; j++) {
                acc = acc + cur[j];
                cur[j] = acc;
            }
#pragma unroll
            for (int j = 0; j < CB; j++)
                if (b + j < size) S.p[b + j] = cur[j];
#pragma unroll
            for (int j = 0; j < CB; j++) cur[j] = nxt[j];
        }
    }
    __syncthreads();
    const double last_cdf = S.p[size - 1];
    __syncthreads();
    for (int i = tid; i < size; i += blockDim.x) S.p[i] = S.p[i] / last_cdf;
    __syncthreads();
    // ---- draws ----
    uint64_t k0, k1;
    seed_key(key, k0, k1);
    for (int64_t d = tid; d < n; d += blockDim.x) {
        uint64_t o[4];
        philox_block((uint64_t)(d >> 2) + 1ull, k0, k1, o[0], o[1], o[2], o[3]);
        const uint64_t r = o[d & 3];
        const double u = (double)(r >> 11) * (1.0 / 9007199254740992.0);
        // searchsorted(cdf, u, side='right'): first index with cdf[idx] > u
        int lo = 0, hi = size;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (S.p[mid] <= u)
                lo = mid + 1;
            else
                hi = mid;
        }
        const int slot = lo < size ? lo : size - 1;
        slots_out[d] = slot;
        if (levels_out) levels_out[d] = D.levels[slot];
        if (maxret_out) maxret_out[d] = D.maxret[slot];
        if (score_out) score_out[d] = D.score[slot];
    }
    __syncthreads();
    // sampled entries: last_sampled = iter (after every probability used the old values)
    for (int64_t d = tid; d < n; d += blockDim.x) D.last[slots_out[d]] = iter;
}

// ---------------------------------------------------------------------------------
// update
//
// Exact sequential semantics, cheap in practice:
//   A  (all threads)  smem hash of the current buffer keys; each candidate looks up
//                     its initial slot (init_match) and its first in-batch twin
//                     (twin_first, via a global hash with atomicMin)
//   B  (all threads)  m_low = min(current min score, scores of candidates that can
//                     update in place).  If the buffer starts full, a candidate with
//                     no key match and score <= m_low can never enter (the minimum never
//                     drops below m_low), so it is skipped; everything else is
//                     "relevant" and compacted in order.
//   C  (one warp)     replays the relevant candidates in order against an indexed
//                     64-ary min-heap of (score, tb) in shared memory, tb = last_sampled
//                     << 32 | seq (the stale-first eviction order): an in-place update is
//                     one sift, an eviction is replace-top + sift-down, candidate data are
//                     prefetched into shared memory by the whole CTA chunk by chunk, and
//                     level / max_return copies are deferred to a parallel epilogue.
// ---------------------------------------------------------------------------------
constexpr int kChunk = 1024;  // relevant candidates staged per round (reuses the hash table's space)
struct CandChunk {
    double sc[kChunk];
    int32_t cid[kChunk];
    int32_t tf[kChunk];
    int32_t im[kChunk];
};
struct UpdSmem {
    uint64_t hk[kPlrMaxK];  // heap: order-preserving score key (score_key)
    uint64_t ht[kPlrMaxK];  // heap: tie-break key (last_sampled << 32) | seq
    int hslot[kPlrMaxK];    // heap entry -> buffer slot
    int pos[kPlrMaxK];      // buffer slot -> heap entry
    union {
        uint32_t hash[kHash];
        CandChunk chunk;
    } u;
    int owner[kPlrMaxK];   // first-candidate index of the key now in the slot, -1 = initial entry
    int src[kPlrMaxK];     // candidate whose level the slot now holds (-1 = unchanged)
    int mr_src[kPlrMaxK];  // candidate whose score / max_return the slot now holds (-1 = unchanged)
    uint32_t replaced[kPlrMaxK / 32];
    double mlow;
    int64_t next_seq;
    int n_rel;
    int full;
    int size;
    int rcur;     // next chunk position for warp 0
    int bulk_hi;  // end of the in-place run to apply in bulk (-1 = none)
};
static_assert(sizeof(CandChunk) <= sizeof(uint32_t) * kHash, "chunk must fit in the hash table space");

// Scores enter the heap as order-preserving unsigned keys (-0.0 folded onto +0.0, as the
// float compare of the reference sees them), so every comparison is integer and a warp
// arg-min is a redux.sync on the high word (ties fall through to the lower words).
__device__ __forceinline__ uint64_t score_key(double s) {
    s = s == 0.0 ? 0.0 : s;
    const uint64_t u = (uint64_t)__double_as_longlong(s);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ bool ukey_lt(uint64_t ka, uint64_t ta, uint64_t kb, uint64_t tb) {
    return ka < kb || (ka == kb && ta < tb);
}
__device__ __forceinline__ void heap_put(UpdSmem &S, int h, uint64_t k, uint64_t t, int slot) {
    S.hk[h] = k;
    S.ht[h] = t;
    S.hslot[h] = slot;
    S.pos[slot] = h;
}
// lanes whose bit is set in `eq` compete; narrows `eq` to the lanes holding the minimum of v
__device__ __forceinline__ unsigned warp_argmin_word(unsigned eq, uint32_t v, int lane) {
    const bool in = (eq >> lane) & 1u;
    const uint32_t m = __reduce_min_sync(0xFFFFFFFFu, in ? v : 0xFFFFFFFFu);
    return __ballot_sync(0xFFFFFFFFu, in && v == m);
}
// 64-ary min-heap (children of h are 64h+1 .. 64h+64; up to 4160 entries -> 2 levels below
// the root).  The entry x = (xk, xt, xs) is sifted from the hole h: at each level lane l
// loads children 64h+1+2l and 64h+2+2l and keeps the smaller, then a ballot of "child < x"
// and a redux arg-min over the lanes; the winning lane moves its child into the hole.
// Whole warp, uniform control flow.
__device__ __forceinline__ void sift_down_w(UpdSmem &S, int h, int n, uint64_t xk, uint64_t xt, int xs, int lane) {
    while (true) {
        const int c0 = 64 * h + 1 + 2 * lane;
        uint64_t ck = ~0ull, ct = ~0ull;
        int cs = 0, cc = c0;
        const bool valid = c0 < n;
        if (valid) {
            ck = S.hk[c0];
            ct = S.ht[c0];
            cs = S.hslot[c0];
            if (c0 + 1 < n) {
                const uint64_t k1 = S.hk[c0 + 1], t1 = S.ht[c0 + 1];
                if (ukey_lt(k1, t1, ck, ct)) {
                    ck = k1;
                    ct = t1;
                    cs = S.hslot[c0 + 1];
                    cc = c0 + 1;
                }
            }
        }
        unsigned eq = __ballot_sync(0xFFFFFFFFu, valid && ukey_lt(ck, ct, xk, xt));
        if (eq == 0u) break;
        eq = warp_argmin_word(eq, (uint32_t)(ck >> 32), lane);
        if (__popc(eq) > 1) eq = warp_argmin_word(eq, (uint32_t)ck, lane);
        if (__popc(eq) > 1) eq = warp_argmin_word(eq, (uint32_t)(ct >> 32), lane);
        if (__popc(eq) > 1) eq = warp_argmin_word(eq, (uint32_t)ct, lane);
        const int win = __ffs(eq) - 1;
        if (lane == win) heap_put(S, h, ck, ct, cs);
        h = __shfl_sync(0xFFFFFFFFu, cc, win);
    }
    if (lane == 0) heap_put(S, h, xk, xt, xs);
    __syncwarp();
}
__device__ __forceinline__ void sift_up_w(UpdSmem &S, int h, uint64_t xk, uint64_t xt, int xs, int lane) {
    while (h > 0) {
        const int p = (h - 1) >> 6;
        const uint64_t pk = S.hk[p], pt = S.ht[p];
        if (!ukey_lt(xk, xt, pk, pt)) break;
        const int ps = S.hslot[p];
        if (lane == 0) heap_put(S, h, pk, pt, ps);
        h = p;
    }
    if (lane == 0) heap_put(S, h, xk, xt, xs);
    __syncwarp();
}
// one thread (heapify: disjoint subtrees per level)
__device__ __forceinline__ void heap_down_t(UpdSmem &S, int h, int n) {
    const uint64_t xk = S.hk[h], xt = S.ht[h];
    const int xs = S.hslot[h];
    while (true) {
        const int c0 = 64 * h + 1;
        if (c0 >= n) break;
        const int ce = c0 + 64 < n ? c0 + 64 : n;
        int m = c0;
        uint64_t mk = S.hk[c0], mt = S.ht[c0];
        for (int c = c0 + 1; c < ce; c++) {
            const uint64_t k = S.hk[c], t = S.ht[c];
            if (ukey_lt(k, t, mk, mt)) {
                m = c;
                mk = k;
                mt = t;
            }
        }
        if (!ukey_lt(mk, mt, xk, xt)) break;
        heap_put(S, h, mk, mt, S.hslot[m]);
        h = m;
    }
    heap_put(S, h, xk, xt, xs);
}

// the buffer slot candidate r of the staged chunk updates in place, or -1
__device__ __forceinline__ int cand_present(const UpdSmem &S, const UpdScratch &W, int r) {
    const int im = S.u.chunk.im[r];
    if (im >= 0 && !((S.replaced[im >> 5] >> (im & 31)) & 1u)) return im;
    const int f = S.u.chunk.tf[r];
    return f != S.u.chunk.cid[r] ? W.keyslot[f] : -1;
}
// length of the run of consecutive in-place candidates starting at r (whole warp)
__device__ __forceinline__ int inplace_run(const UpdSmem &S, const UpdScratch &W, int r, int cn, int lane) {
    int L = 0;
    while (true) {
        const int i = r + L + lane;
        const bool pr = i < cn && cand_present(S, W, i) >= 0;
        const unsigned fail = ~__ballot_sync(0xFFFFFFFFu, pr);
        if (fail) return L + __ffs(fail) - 1;
        L += 32;
    }
}
constexpr int kBulkRun = 64;  // shorter in-place runs stay on the sequential warp path

__global__ void k_plr_cand_prep(PlrDev D, const amz_level_t *__restrict__ cand, int64_t n, UpdScratch W,
                                int64_t hsize) {
    // twin detection over candidates: global open-addressing table keeps min index
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        uint4 w;
        uint32_t p0, p1;
        level_key(cand + c, w, p0, p1);
        uint32_t h = level_hash(w, p0 ^ (p1 << 24)) & (uint32_t)(hsize - 1);
        while (true) {
            uint32_t cur = W.chash[h];
            if (cur == 0u) {
                uint32_t prev = atomicCAS(&W.chash[h], 0u, (uint32_t)(c + 1));
                if (prev == 0u) break;
                cur = prev;
            }
            if (key_eq(cand + (cur - 1), w, p0, p1)) {
                atomicMin(&W.chash[h], (uint32_t)(c + 1));
                break;
            }
            h = (h + 1) & (uint32_t)(hsize - 1);
        }
        W.keyslot[c] = -1;
    }
}

__global__ void k_plr_cand_twin(const amz_level_t *__restrict__ cand, int64_t n, UpdScratch W, int64_t hsize) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        uint4 w;
        uint32_t p0, p1;
        level_key(cand + c, w, p0, p1);
        uint32_t h = level_hash(w, p0 ^ (p1 << 24)) & (uint32_t)(hsize - 1);
        while (true) {
            uint32_t cur = W.chash[h];
            if (cur != 0u && key_eq(cand + (cur - 1), w, p0, p1)) {
                W.twin_first[c] = (int32_t)(cur - 1);
                break;
            }
            h = (h + 1) & (uint32_t)(hsize - 1);
        }
    }
}

__global__ void __launch_bounds__(kPlrThreads, 1)
    k_plr_update(PlrDev D, const amz_level_t *__restrict__ cand, const double *__restrict__ cscore,
                 const double *__restrict__ cmax, int64_t n, int64_t iter, UpdScratch W) {
    extern __shared__ __align__(16) uint8_t smraw[];
    UpdSmem &S = *reinterpret_cast<UpdSmem *>(smraw);
    const int tid = threadIdx.x, lane = tid & 31;
    const int K = (int)D.K;
    const int size0 = (int)D.meta[0];
    // ---- A: load the buffer into the heap arrays + key hash ----
    for (int i = tid; i < kHash; i += blockDim.x) S.u.hash[i] = 0u;
    for (int i = tid; i < kPlrMaxK / 32; i += blockDim.x) S.replaced[i] = 0u;
    if (tid == 0) {
        S.n_rel = 0;
        S.full = size0 >= K;
    }
    __syncthreads();
    double my_min = __longlong_as_double(0x7FF0000000000000ll);  // +inf
    for (int i = tid; i < size0; i += blockDim.x) {
        const double sc = D.score[i];
        S.hk[i] = score_key(sc);
        S.ht[i] = ((uint64_t)D.last[i] << 32) | (uint32_t)D.seq[i];
        S.hslot[i] = i;
        S.pos[i] = i;
        S.owner[i] = -1;
        S.src[i] = -1;
        S.mr_src[i] = -1;
        my_min = fmin(my_min, sc);
        uint4 w;
        uint32_t p0, p1;
        level_key(D.levels + i, w, p0, p1);
        uint32_t h = level_hash(w, p0 ^ (p1 << 24)) & (kHash - 1);
        while (atomicCAS(&S.u.hash[h], 0u, (uint32_t)(i + 1)) != 0u) h = (h + 1) & (kHash - 1);
    }
    __syncthreads();
    for (int64_t c = tid; c < n; c += blockDim.x) {
        uint4 w;
        uint32_t p0, p1;
        level_key(cand + c, w, p0, p1);
        uint32_t h = level_hash(w, p0 ^ (p1 << 24)) & (kHash - 1);
        int m = -1;
        while (true) {
            uint32_t cur = S.u.hash[h];
            if (cur == 0u) break;
            if (key_eq(D.levels + (cur - 1), w, p0, p1)) {
                m = (int)(cur - 1);
                break;
            }
            h = (h + 1) & (kHash - 1);
        }
        W.init_match[c] = m;
        // candidates that can update an entry in place bound the running minimum from below
        if (m >= 0 || W.twin_first[c] != (int32_t)c) my_min = fmin(my_min, cscore[c]);
    }
    // block min
    for (int o = 16; o > 0; o >>= 1) my_min = fmin(my_min, __shfl_xor_sync(0xFFFFFFFFu, my_min, o));
    __shared__ double wmin[32];
    if (lane == 0) wmin[tid >> 5] = my_min;
    __syncthreads();
    if (tid == 0) {
        double m = wmin[0];
        for (int k = 1; k < (int)(blockDim.x >> 5); k++) m = fmin(m, wmin[k]);
        S.mlow = m;
    }
    // ---- heapify, level-parallel (all sift-downs of one level touch disjoint subtrees) ----
    // level starts of the 64-ary heap: 0, 1, 65, 4161
    {
        const int starts[4] = {0, 1, 65, 4161};
        for (int lv = 2; lv >= 0; lv--) {
            __syncthreads();
            const int lo = starts[lv], hi = min(starts[lv + 1], size0);
            for (int h = lo + tid; h < hi; h += blockDim.x) heap_down_t(S, h, size0);
        }
    }
    __syncthreads();
    // ---- B: relevant candidates, compacted in order (block-wide, chunk by chunk) ----
    __shared__ int wcount[32];
    for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t c = base + tid;
        bool rel = false;
        if (c < n) {
            const bool later_twin = W.twin_first[c] != (int32_t)c;
            rel = !S.full || W.init_match[c] >= 0 || later_twin || !(cscore[c] <= S.mlow);
        }
        unsigned b = __ballot_sync(0xFFFFFFFFu, rel);
        if (lane == 0) wcount[tid >> 5] = __popc(b);
        __syncthreads();
        if (tid == 0) {
            int acc = S.n_rel;
            for (int k = 0; k < (int)(blockDim.x >> 5); k++) {
                int v = wcount[k];
                wcount[k] = acc;
                acc += v;
            }
            S.n_rel = acc;
        }
        __syncthreads();
        if (rel) W.rel[wcount[tid >> 5] + __popc(b & ((1u << lane) - 1u))] = (int32_t)c;
        __syncthreads();
    }
    // A skipped first occurrence is never inserted (score <= mlow), so its later twins,
    // which are always relevant, correctly find no entry for the key (keyslot = -1).

    // ---- C: ordered replay (warp 0); long in-place runs applied by the whole CTA ----
    // In-place updates never change which later candidates find their key (only fills and
    // evictions do), so warp 0 scans ahead for the run of consecutive in-place candidates
    // starting at r.  A run of >= kBulkRun is applied in bulk: the last candidate per slot
    // wins (atomicMax on the candidate index, which is increasing along the order), and the
    // heap is rebuilt level-parallel.  (score, last_sampled, seq) is a total order (seq is
    // unique), so the heap's shape never affects which entry is the minimum.
    const int nrel = S.n_rel;
    if (tid == 0) {
        S.size = size0;
        S.next_seq = D.meta[1];
    }
    for (int base = 0; base < nrel; base += kChunk) {
        const int cn = (nrel - base) < kChunk ? (nrel - base) : kChunk;
        __syncthreads();
        for (int i = tid; i < cn; i += blockDim.x) {
            const int c = W.rel[base + i];
            S.u.chunk.cid[i] = c;
            S.u.chunk.sc[i] = cscore[c];
            S.u.chunk.tf[i] = W.twin_first[c];
            S.u.chunk.im[i] = W.init_match[c];
        }
        if (tid == 0) S.rcur = 0;
        __syncthreads();
        while (true) {
            if (tid < 32) {
                int size = S.size;
                int64_t next_seq = S.next_seq;
                int r = S.rcur, scan_end = r, bulk_hi = -1;
                // candidate fields are prefetched one ahead (the replaced bit and the twin's
                // keyslot are read after the previous candidate is applied)
                int c_n = 0, f_n = 0, im_n = -1;
                double sc_n = 0.0;
                if (r < cn) {
                    c_n = S.u.chunk.cid[r];
                    sc_n = S.u.chunk.sc[r];
                    f_n = S.u.chunk.tf[r];
                    im_n = S.u.chunk.im[r];
                }
                for (; r < cn; r++) {
                    const int c = c_n, f = f_n, im = im_n;
                    const double sc = sc_n;
                    if (r + 1 < cn) {
                        c_n = S.u.chunk.cid[r + 1];
                        sc_n = S.u.chunk.sc[r + 1];
                        f_n = S.u.chunk.tf[r + 1];
                        im_n = S.u.chunk.im[r + 1];
                    }
                    int present = -1;
                    if (im >= 0 && !((S.replaced[im >> 5] >> (im & 31)) & 1u)) present = im;
                    if (present < 0 && f != c) present = W.keyslot[f];
                    // only an in-place candidate can open a run worth applying in bulk
                    if (present >= 0 && r >= scan_end) {
                        const int L = inplace_run(S, W, r, cn, lane);
                        if (L >= kBulkRun) {
                            bulk_hi = r + L;
                            break;
                        }
                        scan_end = r + L;
                    }
                    const uint64_t sk = score_key(sc);
                    if (present >= 0) {  // identical level: score / max_return in place (tb unchanged)
                        const int h = S.pos[present];
                        const uint64_t ok = S.hk[h], ot = S.ht[h];
                        __syncwarp();
                        if (lane == 0) S.mr_src[present] = c;
                        if (sk < ok)
                            sift_up_w(S, h, sk, ot, present, lane);
                        else if (sk > ok)
                            sift_down_w(S, h, size, sk, ot, present, lane);
                        __syncwarp();
                        continue;
                    }
                    const uint64_t tbn = ((uint64_t)iter << 32) | (uint32_t)next_seq;
                    int slot;
                    if (size < K) {  // fill
                        slot = size;
                        const int h = size++;
                        __syncwarp();
                        sift_up_w(S, h, sk, tbn, slot, lane);
                    } else {  // evict the (score, last_sampled, seq) minimum iff strictly better
                        if (!(sk > S.hk[0])) continue;
                        slot = S.hslot[0];
                        const int ow = S.owner[slot];
                        __syncwarp();
                        if (lane == 0 && ow >= 0) W.keyslot[ow] = -1;
                        sift_down_w(S, 0, size, sk, tbn, slot, lane);
                    }
                    if (lane == 0) {
                        S.owner[slot] = f;
                        S.replaced[slot >> 5] |= 1u << (slot & 31);
                        S.src[slot] = c;
                        S.mr_src[slot] = c;
                        W.keyslot[f] = slot;
                    }
                    __syncwarp();
                    next_seq++;
                }
                __syncwarp();
                if (lane == 0) {
                    S.size = size;
                    S.next_seq = next_seq;
                    S.rcur = r;
                    S.bulk_hi = bulk_hi;
                }
            }
            __syncthreads();
            const int lo = S.rcur, hi = S.bulk_hi;
            if (hi < 0) break;
            for (int i = lo + tid; i < hi; i += blockDim.x) atomicMax(&S.mr_src[cand_present(S, W, i)], S.u.chunk.cid[i]);
            __syncthreads();
            for (int i = lo + tid; i < hi; i += blockDim.x) {
                const int p = cand_present(S, W, i);
                if (S.mr_src[p] == S.u.chunk.cid[i]) S.hk[S.pos[p]] = score_key(S.u.chunk.sc[i]);
            }
            const int hs = S.size;
            const int starts[4] = {0, 1, 65, 4161};
            for (int lv = 2; lv >= 0; lv--) {
                __syncthreads();
                const int l0 = starts[lv], l1 = min(starts[lv + 1], hs);
                for (int h = l0 + tid; h < l1; h += blockDim.x) heap_down_t(S, h, hs);
            }
            __syncthreads();
            if (tid == 0) S.rcur = hi;
            __syncthreads();
        }
    }
    __syncthreads();
    // ---- epilogue: scatter the heap back to slots, deferred level / max_return copies ----
    const int fsize = S.size;
    for (int h = tid; h < fsize; h += blockDim.x) {
        const int slot = S.hslot[h];
        const uint64_t tb = S.ht[h];
        D.last[slot] = (int64_t)(tb >> 32);
        D.seq[slot] = (int64_t)(uint32_t)tb;
        if (S.src[slot] >= 0) D.levels[slot] = cand[S.src[slot]];
        const int mr = S.mr_src[slot];
        if (mr >= 0) {
            D.score[slot] = cscore[mr];
            D.maxret[slot] = cmax[mr];
        }
    }
    if (tid == 0) {
        D.meta[0] = fsize;
        D.meta[1] = S.next_seq;
    }
}

// top-q replay lanes by score (ties -> lower lane index), single CTA
__global__ void k_top_q(const double *__restrict__ scores, int64_t n, int q, int32_t *__restrict__ out) {
    __shared__ double bs[32];
    __shared__ int bi[32];
    __shared__ int chosen[64];
    for (int k = 0; k < q; k++) {
        double best = 0.0;
        int besti = -1;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            bool skip = false;
            for (int j = 0; j < k; j++) skip |= chosen[j] == (int)i;
            if (skip) continue;
            const double s = scores[i];
            if (besti < 0 || s > best || (s == best && (int)i < besti)) {
                best = s;
                besti = (int)i;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double s2 = __shfl_xor_sync(0xFFFFFFFFu, best, o);
            const int i2 = __shfl_xor_sync(0xFFFFFFFFu, besti, o);
            if (i2 >= 0 && (besti < 0 || s2 > best || (s2 == best && i2 < besti))) {
                best = s2;
                besti = i2;
            }
        }
        if ((threadIdx.x & 31) == 0) {
            bs[threadIdx.x >> 5] = best;
            bi[threadIdx.x >> 5] = besti;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double b = 0.0;
            int ix = -1;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
                if (bi[w] >= 0 && (ix < 0 || bs[w] > b || (bs[w] == b && bi[w] < ix))) {
                    b = bs[w];
                    ix = bi[w];
                }
            }
            chosen[k] = ix;
            out[k] = ix;
        }
        __syncthreads();
    }
}

size_t plr_sample_smem() { return sizeof(SampleSmem); }
size_t plr_update_smem() { return sizeof(UpdSmem); }

int launch_plr_sample(const PlrDev &D, const amz_seed_t &key, int64_t n, double omr, double rho, const double *lut,
                      int64_t iter, int32_t *slots, amz_level_t *levels, double *maxret, double *score, int *err,
                      cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_plr_sample, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SampleSmem));
        attr = true;
    }
    k_plr_sample<<<1, kPlrThreads, sizeof(SampleSmem), s>>>(D, key, n, omr, rho, lut, iter, slots, levels, maxret,
                                                             score, err);
    return 0;
}

int launch_plr_update(const PlrDev &D, const amz_level_t *cand, const double *cs, const double *cm, int64_t n,
                      int64_t iter, const UpdScratch &W, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_plr_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(UpdSmem));
        attr = true;
    }
    if (n <= 0) return 0;
    int64_t hsize = 1;
    while (hsize < 2 * n) hsize <<= 1;
    cudaMemsetAsync(W.chash, 0, hsize * sizeof(uint32_t), s);
    const int g = (int)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184);
    k_plr_cand_prep<<<g, 256, 0, s>>>(D, cand, n, W, hsize);
    k_plr_cand_twin<<<g, 256, 0, s>>>(cand, n, W, hsize);
    k_plr_update<<<1, kPlrThreads, sizeof(UpdSmem), s>>>(D, cand, cs, cm, n, iter, W);
    return 0;
}

int launch_top_q(const double *scores, int64_t n, int q, int32_t *out, cudaStream_t s) {
    k_top_q<<<1, 256, 0, s>>>(scores, n, q, out);
    return 0;
}

}  // namespace amz
