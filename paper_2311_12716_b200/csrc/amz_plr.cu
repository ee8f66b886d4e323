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
constexpr int kMaxDevices = 64;
#ifdef AMZ_PLR_STATS
__device__ long long g_samp_clk[16];
#define SAMP_CLK(k_)                                       \
    do {                                                   \
        __syncthreads();                                   \
        if (threadIdx.x == 0) g_samp_clk[k_] = clock64();  \
    } while (0)
extern "C" int amz_debug_samp_clk(void *host) {
    return (int)cudaMemcpyFromSymbol(host, g_samp_clk, sizeof(g_samp_clk));
}
#else
#define SAMP_CLK(k_) \
    do {             \
    } while (0)
#endif

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
// numpy pairwise sum of x[0..n) (numpy/_core/src/umath/loops_utils.h.src pairwise_sum):
// n < 8 sequential; n <= 128 eight accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
// then the n % 8 tail; beyond, left half n2 = n/2 rounded down to a multiple of 8, and
// the result is pw(left) + pw(right).  The recursion tree (<= 127 nodes for n <= 4096)
// is built level by level by warp 0, the leaves are summed in parallel and the internal
// nodes evaluated bottom-up -- every node is the same single addition of the same two
// operands as numpy's recursion, so the result is bit-identical.
// ---------------------------------------------------------------------------------
constexpr int kPwNodes = 128;
struct PwTree {
    int start[kPwNodes], len[kPwNodes], left[kPwNodes], depth[kPwNodes];
    double val[kPwNodes];
    int n_nodes, max_depth;
};
__device__ __forceinline__ double pw_leaf(const double *x, int s, int len) {
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
    return res;
}
// whole CTA; returns the sum in every thread
__device__ double block_pairwise_sum(const double *x, int n, PwTree &P) {
    const int tid = threadIdx.x;
    if (tid < 32) {
        // level-by-level expansion: nodes of one level are contiguous, children appended
        if (tid == 0) {
            P.start[0] = 0;
            P.len[0] = n;
            P.depth[0] = 0;
            P.left[0] = -1;
            P.n_nodes = 1;
            P.max_depth = 0;
        }
        __syncwarp();
        int lo = 0, hi = 1, d = 0;
        while (lo < hi) {
            // count splits of this level (in order) and append their children
            const int cnt = hi - lo;
            int base = hi;
            for (int c0 = 0; c0 < cnt; c0 += 32) {
                const int i = lo + c0 + tid;
                const bool split = c0 + tid < cnt && P.len[i] > 128;
                const unsigned b = __ballot_sync(0xFFFFFFFFu, split);
                if (split) {
                    const int k = base + 2 * __popc(b & ((1u << tid) - 1u));
                    int n2 = P.len[i] / 2;
                    n2 -= n2 % 8;
                    P.start[k] = P.start[i];
                    P.len[k] = n2;
                    P.start[k + 1] = P.start[i] + n2;
                    P.len[k + 1] = P.len[i] - n2;
                    P.depth[k] = P.depth[k + 1] = d + 1;
                    P.left[k] = P.left[k + 1] = -1;
                    P.left[i] = k;
                }
                base += 2 * __popc(b);
            }
            __syncwarp();
            lo = hi;
            hi = base;
            if (hi > lo) d++;
        }
        if (tid == 0) {
            P.n_nodes = hi;
            P.max_depth = d;
        }
    }
    __syncthreads();
    const int nn = P.n_nodes;
    for (int i = tid; i < nn; i += blockDim.x)
        if (P.left[i] < 0) P.val[i] = pw_leaf(x, P.start[i], P.len[i]);
    __syncthreads();
    for (int d = P.max_depth - 1; d >= 0; d--) {
        for (int i = tid; i < nn; i += blockDim.x)
            if (P.depth[i] == d && P.left[i] >= 0) P.val[i] = P.val[P.left[i]] + P.val[P.left[i] + 1];
        __syncthreads();
    }
    return P.val[0];
}

// ---------------------------------------------------------------------------------
// sampling
//   1. ranks: one bitonic sort (1024 threads, 78 compare-exchange stages over the next
//      power of two >= size) by (score desc, seq asc) -- the order numpy's lexsort of
//      (seq, -score) gives (rank ties -> older insertion first)
//   2. w = LUT[rank - 1] ((1/rank)^(1/beta), numpy's host LUT); proportional:
//      w = score^(1/beta)
//   3. sum(w) in numpy's pairwise order
//   4. P = (1-rho) w/sum(w) + rho st/sum(st); cdf = sequential cumsum (one thread: it is
//      numpy's order) while the other warps draw the uniforms u_i = i-th random() of the
//      key's stream (counter-based: block i/4 of Philox); then cdf /= cdf[-1] and
//      slot_i = searchsorted(cdf, u_i, 'right')
// ---------------------------------------------------------------------------------
constexpr int kSampU = 4096;  // uniforms precomputed during the cumsum
struct SampleSmem {
    double u[kSampU];  // uniforms of the first kSampU draws
    double p[kPlrMaxK];
    PwTree pw;
    unsigned long long st_total;
};

// rank - 1 of every entry under (score desc, seq asc) -- numpy's lexsort((seq, -score)),
// rank ties -> older insertion first -- by direct counting over a 2-D grid: CTA (bi, bj)
// stages entries [bj*RJ, (bj+1)*RJ) in shared memory and thread i adds the number of them
// before entry i to rank[i] (zeroed first).  4000^2 comparisons over ~128 CTAs take a few
// microseconds; a single-CTA sort of the same keys (CUB block radix, 64-bit score keys)
// was ~45 us and a bitonic network ~80 us.
constexpr int kRankThreads = 256;
constexpr int kRankJ = 256;
__device__ __forceinline__ void rank_keys(const PlrDev &D, int j, uint64_t &k, uint64_t &q) {
    double sc = D.score[j];
    sc = sc == 0.0 ? 0.0 : sc;  // -0.0 ties with 0.0, as in numpy's sort
    const uint64_t u = (uint64_t)__double_as_longlong(sc);
    k = (u >> 63) ? ~u : (u | 0x8000000000000000ull);  // ascending = score asc
    q = (uint64_t)D.seq[j] ^ 0x8000000000000000ull;     // signed -> unsigned order
}
__global__ void __launch_bounds__(kRankThreads) k_plr_rank(PlrDev D, int32_t *__restrict__ rank) {
    pdl_wait();  // PDL: the predecessor kernel has completed (its launch overlapped)
    __shared__ uint64_t sk[kRankJ];
    __shared__ uint64_t sq[kRankJ];
    const int size = (int)D.meta[0];
    const int j0 = blockIdx.y * kRankJ;
    const int nj = min(kRankJ, size - j0);
    if (nj <= 0) return;
    for (int j = threadIdx.x; j < nj; j += blockDim.x) rank_keys(D, j0 + j, sk[j], sq[j]);
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= size) return;
    uint64_t ki, qi;
    rank_keys(D, i, ki, qi);
    int r = 0;
#pragma unroll 8
    for (int j = 0; j < nj; j++) r += (sk[j] > ki) | ((sk[j] == ki) & (sq[j] < qi));
    if (r) atomicAdd(&rank[i], r);
}

__global__ void __launch_bounds__(kPlrThreads, 1)
    k_plr_sample(PlrDev D, const int32_t *__restrict__ rank, amz_seed_t key, int64_t n, double one_minus_rho,
                 double rho, const double *__restrict__ lut, int prop, double inv_beta, int64_t iter,
                 int32_t *__restrict__ slots_out, amz_level_t *__restrict__ levels_out, double *__restrict__ maxret_out,
                 double *__restrict__ score_out, int *__restrict__ err) {
    pdl_wait();  // PDL: the predecessor kernel has completed (its launch overlapped)
    extern __shared__ __align__(16) uint8_t smraw[];
    SampleSmem &S = *reinterpret_cast<SampleSmem *>(smraw);
    const int tid = threadIdx.x;
    const int size = (int)D.meta[0];
    if (size <= 0) {
        if (tid == 0) atomicOr(err, 2);
        return;
    }
    SAMP_CLK(0);
    if (tid == 0) S.st_total = 0ull;
    __syncthreads();
    // ---- 2./3. weights and their pairwise sum (slot order) ----
    unsigned long long my_st = 0ull;
    bool bad = false;
    for (int i = tid; i < size; i += blockDim.x) {
        if (prop) {  // proportional: score^(1/beta) (numpy's np.power; CUDA pow is within 2 ulp of it)
            const double w = pow(D.score[i], inv_beta);
            bad |= !(w >= 0.0);  // a negative score: numpy's choice rejects NaN probabilities
            S.p[i] = w;
        } else {
            S.p[i] = lut[rank[i]];
        }
        my_st += (unsigned long long)(iter - D.last[i]);
    }
    if (bad) atomicOr(err, 8);
    for (int o = 16; o > 0; o >>= 1) my_st += __shfl_down_sync(0xFFFFFFFFu, my_st, o);
    if ((tid & 31) == 0) atomicAdd(&S.st_total, my_st);
    __syncthreads();
    SAMP_CLK(4);
    const double wsum = block_pairwise_sum(S.p, size, S.pw);
    if (prop && tid == 0 && !(wsum > 0.0)) atomicOr(err, 8);  // every score 0: 0/0 probabilities
    const long long tot = (long long)S.st_total;
    SAMP_CLK(5);
    // ---- 4. P ----
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
    SAMP_CLK(6);
    uint64_t k0, k1;
    seed_key(key, k0, k1);
    const int nu = n < kSampU ? (int)n : kSampU;
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
    } else if ((tid >> 5) & 3) {
        // meanwhile: the first nu uniforms, one Philox block per 4 draws, on the warps of
        // the other three schedulers (warp 0's scheduler stays free for the add chain)
        const int w = tid >> 5, q0 = (w - 1 - (w >> 2)) * 32 + (tid & 31), nw = 24 * 32;
        for (int q = q0; q < (nu + 3) / 4; q += nw) {
            uint64_t o[4];
            philox_block((uint64_t)q + 1ull, k0, k1, o[0], o[1], o[2], o[3]);
#pragma unroll
            for (int j = 0; j < 4; j++)
                if (4 * q + j < nu) S.u[4 * q + j] = (double)(o[j] >> 11) * (1.0 / 9007199254740992.0);
        }
    }
    __syncthreads();
    SAMP_CLK(7);
    const double last_cdf = S.p[size - 1];
    __syncthreads();
    for (int i = tid; i < size; i += blockDim.x) S.p[i] = S.p[i] / last_cdf;
    __syncthreads();
    SAMP_CLK(8);
    // ---- draws ----
    for (int64_t d = tid; d < n; d += blockDim.x) {
        double u;
        if (d < nu) {
            u = S.u[d];
        } else {
            uint64_t o0, o1, o2, o3;
            philox_block((uint64_t)(d >> 2) + 1ull, k0, k1, o0, o1, o2, o3);
            const int j = (int)(d & 3);
            const uint64_t r = j == 0 ? o0 : j == 1 ? o1 : j == 2 ? o2 : o3;
            u = (double)(r >> 11) * (1.0 / 9007199254740992.0);
        }
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
    SAMP_CLK(9);
    // sampled entries: last_sampled = iter (after every probability used the old values)
    for (int64_t d = tid; d < n; d += blockDim.x) D.last[slots_out[d]] = iter;
    SAMP_CLK(10);
}

// ---------------------------------------------------------------------------------
// update
//
// Exact sequential semantics of SPEC.md:373-377 (oracle/plr_np.py LevelBuffer.update),
// parallel wherever the order provably cannot matter:
//   A  (all threads)  smem hash of the current buffer keys; each candidate looks up
//                     its initial slot (init_match) and its first in-batch twin
//                     (twin_first, via a global hash with atomicMin).  Tie keys are
//                     made relative: tb = (last - lmin) << bq | (seq - qmin), exact
//                     for any int64 last_sampled / seq whose spans fit 64 bits together
//                     (else the update is refused: error bit 4, ContractViolation)
//   B  (all threads)  m_low = min(current min score, scores of candidates that can
//                     update in place).  If the buffer starts full, a candidate with
//                     no key match and score <= m_low can never enter (the minimum never
//                     drops below m_low), so it is skipped; everything else is
//                     "relevant" and compacted in order.
//   C  (one warp)     replays the relevant candidates in order.  The buffer's
//                     (score key, tb) live in flat shared arrays; the eviction order
//                     needs only the bottom: a BOTTOM CACHE of the 64 smallest entries
//                     sits in warp 0's registers (2 per lane) with its minimum and
//                     maximum kept as warp-uniform values, and every entry outside it
//                     is larger than its maximum.  An eviction takes the cached minimum
//                     (one warp reduction refreshes it), an in-place update edits the
//                     cache only if the entry is in it or drops below its maximum; an
//                     emptied cache is rebuilt by the CTA (128-bit MSD radix select).
//                     Warp-batched stretches: the leading run of candidates that change
//                     neither presence nor the cache (in place outside the cache and
//                     above its maximum; absent and not above the minimum of a full
//                     buffer) is applied 32 at a time, the last writer per slot found
//                     by match.any.  Presence of a candidate's key: its initial slot
//                     while not replaced, else (a level present at kernel start that
//                     was evicted and inserted again by a twin) the shared reslot map,
//                     else (a later twin of a new level) the global keyslot.  Level /
//                     max_return copies are deferred to a parallel epilogue.  Two kinds
//                     of stretch leave warp 0 for the whole CTA:
//     bulk in-place run (>= kBulkRun consecutive candidates whose level is present):
//                     last writer per slot by atomicMax;
//     insert run (>= kRunMin consecutive candidates that are certainly new: no key
//                     match at kernel start, first of their key in the batch):
//                     a streaming top-K in parallel (k_plr_update comment below,
//                     tools/plr_insert_runs_proto.py is the host prototype).
// ---------------------------------------------------------------------------------
constexpr int kChunk = 1024;  // relevant candidates staged per round (reuses the hash table's space)
#ifdef AMZ_PLR_STATS
// [0] sequential candidates (warp 0), [1] of them in place, [2] bulk runs, [3] bulk
// candidates, [4] insert_runs calls, [5] insert passes, [6] candidates consumed by runs,
// [7] relevant candidates, [8] calls, [9] bottom-cache rebuilds, [10] warp-batched candidates,
// [11] cycles of phase B, [12] cycles of phase C, [13] batch steps, [14] cycles in batch steps
__device__ unsigned long long g_plr_stats[40];
#define PLR_STAT(k_, v_) atomicAdd(&g_plr_stats[k_], (unsigned long long)(v_))
#define PLR_CLK(v_) const long long v_ = clock64()
extern "C" int amz_debug_plr_stats(void *host, int reset) {
    int rc = (int)cudaMemcpyFromSymbol(host, g_plr_stats, sizeof(g_plr_stats));
    if (reset) {
        unsigned long long z[40] = {};
        cudaMemcpyToSymbol(g_plr_stats, z, sizeof(z));
    }
    return rc;
}
#else
#define PLR_STAT(k_, v_) \
    do {                 \
    } while (0)
#define PLR_CLK(v_) \
    do {            \
    } while (0)
#endif
constexpr int kRunMin = 96;   // shorter insert runs stay on the sequential warp path
constexpr int kBulkRun = 64;  // shorter in-place runs stay on the sequential warp path
struct CandChunk {
    uint64_t sk[kChunk];  // score keys (score_key of the candidates' scores)
    int32_t cid[kChunk];
    int32_t tf[kChunk];
    int32_t im[kChunk];
};

// Insert runs (whole CTA): relevant candidates from r0 on that are certainly new (no key
// match at kernel start, first of their key in the batch), until the first one that is
// not.  With free slots as virtual entries of score -inf (evicted in slot order) the
// sequential rule is a streaming top-K of the buffer under the order
//   x < y  <=>  score_x < score_y, or equal scores and x entered first
// (every stored entry entered before every run candidate: tb(stored) < tb(new), checked
// by run_ok).  For the live candidates of a pass, in arrival order,
//   accept_i <=> #{live j < i : s_j > s_i} < #{buffer x : s_x <= s_i}
//   the p acceptances evict the p smallest of (buffer U accepted), in order; the k-th
//   acceptance takes the slot of the k-th eviction (chained through re-evicted ones);
//   the minimum present when candidate i arrives is merged element q_i (q_i =
//   acceptances before i): later acceptances all exceed it.
// The order differs from the rule only when s_i equals that minimum's score (the rule
// rejects; the order would accept): the first such candidate f is found exactly, the
// prefix before it is committed (a prefix of the streaming process is the same
// process), f and every later candidate with score <= s_f are rejected (the minimum
// never drops), and the next pass runs over the rest.  The sorted buffer is sorted once
// per call and then kept sorted by merging each pass's commits into it.
constexpr int kRunM = 256;  // live candidates per pass (4 threads per candidate)
struct RunArr {
    uint64_t lk[kRunM];        // live candidates' score keys, arrival order
    uint64_t ask[kRunM];       // this pass's acceptances sorted by (score, arrival)
    uint64_t apk[kRunM];       // the committed acceptances, sorted
    uint64_t mkey[kRunM + 1];  // score keys of the first p+1 elements of the merged order
    int32_t lc[kRunM];         // live candidates' ids
    int32_t lq[kRunM];         // acceptances before each live candidate
    int32_t acand[kRunM];      // acceptance index -> live index
    int32_t arank[kRunM];      // acceptance index -> position in ask
    int32_t abelow[kRunM];     // acceptance index -> #buffer entries <= its score
    int32_t apos2[kRunM];      // ask position -> position in apk (committed only)
    int32_t aslot[kRunM];      // acceptance index -> slot
    int32_t mref[kRunM + 1];   // merged order: >= 0 sorted buffer position, < 0 -(acceptance + 1)
};
using RunSort = cub::BlockRadixSort<unsigned long long, kPlrThreads, 4, int, 4>;
struct SortedEntries {
    uint64_t ekey[kPlrMaxK];  // score keys of the buffer (virtual free slots = 0), eviction order
    int32_t eslot[kPlrMaxK];
};
constexpr int kCache = 64;  // bottom cache entries (two per lane of warp 0)
struct UpdSmem {
    uint64_t key[kPlrMaxK];  // slot -> order-preserving score key (score_key)
    uint64_t tie[kPlrMaxK];  // slot -> relative tie key (last - lmin) << bq | (seq - qmin)
    union {
        uint32_t hash[kHash];
        CandChunk chunk;
        RunArr run;
    } u;
    int owner[kPlrMaxK];   // first-candidate index of the key now in the slot, -1 = initial entry
    int src[kPlrMaxK];     // candidate whose level the slot now holds (-1 = unchanged)
    int mr_src[kPlrMaxK];  // candidate whose score / max_return the slot now holds (-1 = unchanged)
    uint32_t replaced[kPlrMaxK / 32];
    // keys present at kernel start whose slot was taken, then inserted again by a later
    // twin: reslot[initial slot] = the slot holding the key now (-1 = absent), and
    // origin[slot] = the initial slot of the key a slot holds (-1 = initial entry or a
    // key new to the buffer) -- the replay twins' presence without the global keyslot
    int16_t reslot[kPlrMaxK];
    int16_t origin[kPlrMaxK];
    union {
        typename RunSort::TempStorage sort;
        SortedEntries e;
    } r1;
    uint32_t evicted[kRunM / 32];  // insert run: acceptances evicted again inside the pass
    // bottom cache: the kCache smallest (key, tie) entries of the buffer (warp 0 keeps it
    // in registers while it replays candidates; rebuilt by the CTA when invalid)
    int cslot[kCache];
    uint64_t ckey[kCache];
    uint64_t ctie[kCache];
    uint8_t sel[kPlrMaxK];  // cache rebuild: selected slots
    uint8_t incache[kPlrMaxK];  // slot is in the bottom cache (meaningful while cvalid)
    int hist[256];
    int sel_b, sel_below, sel_cnt;
    int cvalid;
    uint64_t bmk, bmt;  // bulk run: the bottom cache's maximum
    int bulk_bad;       // bulk run: updated entries that touch the cache ...
    int bulk_list[kCache];  // ... and their slots
    double mlow;
    int64_t next_seq;
    int64_t lmin, qmin, lmax, qmax, last_max0;
    unsigned long long tie_max;
    int bq;
    int n_rel;
    int full;
    int size;
    int rcur;      // next chunk position for warp 0
    int action;    // 0 = chunk done, 1 = bulk in-place run [rcur, arg), 2 = insert run, 3 = rebuild the cache
    int arg;
    int run_ok;
    int flag_first;
    int n_virtual;
};
static_assert(sizeof(CandChunk) <= sizeof(uint32_t) * kHash, "chunk must fit in the hash table space");
static_assert(sizeof(RunArr) <= sizeof(uint32_t) * kHash, "run scratch must fit in the hash table space");
static_assert(sizeof(UpdSmem) + 1024 <= 227 * 1024, "update shared memory over the 227 KB opt-in limit");

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
__device__ __forceinline__ uint64_t tie_pack(const UpdSmem &S, int64_t last, int64_t seq) {
    const uint64_t q = (uint64_t)seq - (uint64_t)S.qmin;
    return S.bq >= 64 ? q : ((((uint64_t)last - (uint64_t)S.lmin) << S.bq) | q);
}
__device__ __forceinline__ bool ukey_le(uint64_t ka, uint64_t ta, uint64_t kb, uint64_t tb) {
    return ka < kb || (ka == kb && ta <= tb);
}
// lanes whose bit is set in `eq` compete; narrows `eq` to the lanes holding the minimum of v
__device__ __forceinline__ unsigned warp_argmin_word(unsigned eq, uint32_t v, int lane) {
    const bool in = (eq >> lane) & 1u;
    const uint32_t m = __reduce_min_sync(0xFFFFFFFFu, in ? v : 0xFFFFFFFFu);
    return __ballot_sync(0xFFFFFFFFu, in && v == m);
}
// The lane holding the lexicographic minimum (or, with mx, maximum) of (k, t) among the
// lanes with `has`, or -1.  (key, tie) pairs are unique, so the winner is unique.
__device__ __forceinline__ int warp_lex_pick(bool has, uint64_t k, uint64_t t, bool mx, int lane) {
    unsigned eq = __ballot_sync(0xFFFFFFFFu, has);
    if (!eq) return -1;
    const uint64_t kk = mx ? ~k : k, tt = mx ? ~t : t;
    eq = warp_argmin_word(eq, (uint32_t)(kk >> 32), lane);
    if (__popc(eq) > 1) eq = warp_argmin_word(eq, (uint32_t)kk, lane);
    if (__popc(eq) > 1) eq = warp_argmin_word(eq, (uint32_t)(tt >> 32), lane);
    if (__popc(eq) > 1) eq = warp_argmin_word(eq, (uint32_t)tt, lane);
    return __ffs(eq) - 1;
}

// The bottom cache in warp 0's registers: lane l holds entries l (.0) and l + 32 (.1);
// slot < 0 = free.  Invariant while valid: every buffer entry outside the cache is
// larger than the cache maximum, and the cache is not empty.  The maximum and the
// minimum (value and position) are kept as warp-uniform state, so an eviction reads
// its victim without a warp reduction and only the operations that remove an extreme
// pay one (warp_lex_pick).
struct BottomCache {
    int s0, s1;
    uint64_t k0, k1, t0, t1;
    uint64_t mk, mt;  // maximum (uniform) ...
    int xl, xw;       // ... at lane xl, entry xw
    uint64_t nk, nt;  // minimum (uniform) ...
    int nl, nw, ns;   // ... at lane nl, entry nw, buffer slot ns
    int n;            // entries (uniform)
    bool valid;       // uniform
    uint8_t *flag;    // UpdSmem::incache

    __device__ __forceinline__ void load(UpdSmem &S, int lane) {
        flag = S.incache;
        s0 = S.cslot[lane];
        s1 = S.cslot[lane + 32];
        k0 = S.ckey[lane];
        k1 = S.ckey[lane + 32];
        t0 = S.ctie[lane];
        t1 = S.ctie[lane + 32];
        valid = S.cvalid != 0;
        mk = mt = nk = nt = 0;
        xl = xw = nl = nw = 0;
        ns = -1;
        n = __popc(__ballot_sync(0xFFFFFFFFu, s0 >= 0)) + __popc(__ballot_sync(0xFFFFFFFFu, s1 >= 0));
        if (valid) {
            refresh_max(lane);
            refresh_min(lane);
        }
    }
    __device__ __forceinline__ void store(UpdSmem &S, int lane) const {
        S.cslot[lane] = s0;
        S.cslot[lane + 32] = s1;
        S.ckey[lane] = k0;
        S.ckey[lane + 32] = k1;
        S.ctie[lane] = t0;
        S.ctie[lane + 32] = t1;
        if (lane == 0) S.cvalid = valid ? 1 : 0;
    }
    // this lane's extreme of its two entries (mx: maximum); which = 0 / 1
    __device__ __forceinline__ bool local(bool mx, uint64_t &k, uint64_t &t, int &which) const {
        const bool a = s0 >= 0, b = s1 >= 0;
        if (a && (!b || (mx ? !ukey_le(k0, t0, k1, t1) : ukey_le(k0, t0, k1, t1)))) {
            k = k0;
            t = t0;
            which = 0;
        } else {
            k = k1;
            t = t1;
            which = 1;
        }
        return a || b;
    }
    // recompute the maximum / minimum of a non-empty cache
    __device__ __forceinline__ void refresh_max(int lane) {
        uint64_t k, t;
        int w;
        const bool has = local(true, k, t, w);
        xl = warp_lex_pick(has, k, t, true, lane);
        mk = __shfl_sync(0xFFFFFFFFu, k, xl);
        mt = __shfl_sync(0xFFFFFFFFu, t, xl);
        xw = __shfl_sync(0xFFFFFFFFu, w, xl);
    }
    __device__ __forceinline__ void refresh_min(int lane) {
        uint64_t k, t;
        int w;
        const bool has = local(false, k, t, w);
        nl = warp_lex_pick(has, k, t, false, lane);
        nk = __shfl_sync(0xFFFFFFFFu, k, nl);
        nt = __shfl_sync(0xFFFFFFFFu, t, nl);
        nw = __shfl_sync(0xFFFFFFFFu, w, nl);
        ns = __shfl_sync(0xFFFFFFFFu, w ? s1 : s0, nl);
    }
    __device__ __forceinline__ void remove_at(int wl, int ww, int lane) {
        if (lane == wl) {
            flag[ww ? s1 : s0] = 0;
            if (ww)
                s1 = -1;
            else
                s0 = -1;
        }
        n--;
    }
    // drop the minimum (its slot is being evicted); an emptied cache becomes invalid
    __device__ __forceinline__ void pop_min(int lane) {
        remove_at(nl, nw, lane);
        if (n == 0)
            valid = false;
        else
            refresh_min(lane);  // the maximum is another entry: unchanged
    }
    // the entry holding slot s: (lane, which), or lane -1
    __device__ __forceinline__ void find(int s, int &wl, int &ww) const {
        const unsigned f0 = __ballot_sync(0xFFFFFFFFu, s0 == s), f1 = __ballot_sync(0xFFFFFFFFu, s1 == s);
        if (f0) {
            wl = __ffs(f0) - 1;
            ww = 0;
        } else if (f1) {
            wl = __ffs(f1) - 1;
            ww = 1;
        } else {
            wl = -1;
            ww = 0;
        }
    }
    // insert (s, k, t) below the maximum; a full cache first drops its maximum (which
    // then lies outside, above the new maximum)
    __device__ __forceinline__ void insert(int s, uint64_t k, uint64_t t, int lane) {
        const bool drop = n == 2 * 32;
        if (drop) remove_at(xl, xw, lane);
        const unsigned f0 = __ballot_sync(0xFFFFFFFFu, s0 < 0), f1 = __ballot_sync(0xFFFFFFFFu, s1 < 0);
        const int wl = f0 ? __ffs(f0) - 1 : __ffs(f1) - 1;
        const int ww = f0 ? 0 : 1;
        if (lane == wl) {
            flag[s] = 1;
            if (ww) {
                s1 = s;
                k1 = k;
                t1 = t;
            } else {
                s0 = s;
                k0 = k;
                t0 = t;
            }
        }
        n++;
        if (drop) refresh_max(lane);
        if (ukey_le(k, t, nk, nt)) {  // the new minimum
            nk = k;
            nt = t;
            nl = wl;
            nw = ww;
            ns = s;
        }
    }
    // the cached entry (wl, ww) of slot s takes key k (its tie t unchanged): it stays if
    // still below the maximum, else it leaves the cache
    __device__ __forceinline__ void rekey(int s, int wl, int ww, uint64_t k, uint64_t t, int lane) {
        const bool was_max = wl == xl && ww == xw, was_min = wl == nl && ww == nw;
        if (ukey_le(k, t, mk, mt)) {
            if (lane == wl) {
                if (ww)
                    k1 = k;
                else
                    k0 = k;
            }
            if (was_max) refresh_max(lane);
            if (was_min) {
                refresh_min(lane);
            } else if (ukey_le(k, t, nk, nt)) {
                nk = k;
                nt = t;
                nl = wl;
                nw = ww;
                ns = s;
            }
        } else {  // rose above the maximum: outside now
            remove_at(wl, ww, lane);
            if (n == 0) {
                valid = false;
                return;
            }
            if (was_max) refresh_max(lane);
            if (was_min) refresh_min(lane);
        }
    }
};

// the slot holding the key of candidate c (initial match im, twin-first f), or -1
__device__ __forceinline__ int present_slot(const UpdSmem &S, const UpdScratch &W, int im, int f, int c) {
    if (im >= 0) return ((S.replaced[im >> 5] >> (im & 31)) & 1u) ? (int)S.reslot[im] : im;
    return f != c ? W.keyslot[f] : -1;  // a later twin of a level new to the buffer
}
// the buffer slot candidate r of the staged chunk updates in place, or -1
__device__ __forceinline__ int cand_present(const UpdSmem &S, const UpdScratch &W, int r) {
    return present_slot(S, W, S.u.chunk.im[r], S.u.chunk.tf[r], S.u.chunk.cid[r]);
}
// certainly new at any point of the batch: no key match at kernel start, first of its key
__device__ __forceinline__ bool cand_pure(const UpdSmem &S, int r) {
    return S.u.chunk.im[r] < 0 && S.u.chunk.tf[r] == S.u.chunk.cid[r];
}
// length of the run of consecutive in-place candidates starting at r (whole warp)
__device__ __forceinline__ int inplace_run(const UpdSmem &S, const UpdScratch &W, int r, int cn, int lane,
                                           unsigned ok0) {
    const unsigned fail0 = ~ok0;
    if (fail0) return __ffs(fail0) - 1;
    int L = 32;
    while (true) {
        const int i = r + L + lane;
        const bool pr = i < cn && cand_present(S, W, i) >= 0;
        const unsigned fail = ~__ballot_sync(0xFFFFFFFFu, pr);
        if (fail) return L + __ffs(fail) - 1;
        L += 32;
    }
}
// length of the run of consecutive certainly-new candidates starting at r (whole warp)
// ok0: the first window's ballot (lanes r..r+31), when the caller already has it
__device__ __forceinline__ int pure_run(const UpdSmem &S, int r, int cn, int lane, unsigned ok0) {
    const unsigned fail0 = ~ok0;
    if (fail0) return __ffs(fail0) - 1;
    int L = 32;
    while (L < kRunMin) {
        const int i = r + L + lane;
        const bool pr = i < cn && cand_pure(S, i);
        const unsigned fail = ~__ballot_sync(0xFFFFFFFFu, pr);
        if (fail) return L + __ffs(fail) - 1;
        L += 32;
    }
    return L;
}

__device__ __forceinline__ int upper_bound_u64(const uint64_t *a, int n, uint64_t x) {  // # a[i] <= x
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int lower_bound_u64(const uint64_t *a, int n, uint64_t x) {  // # a[i] < x
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// block-wide exclusive prefix count of `flag` (kPlrThreads threads); returns the total
__device__ __forceinline__ int block_excl_count(bool flag, int &excl, int *wscan) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned b = __ballot_sync(0xFFFFFFFFu, flag);
    if (lane == 0) wscan[w] = __popc(b);
    __syncthreads();
    if (w == 0) {
        const int v = lane < (int)(blockDim.x >> 5) ? wscan[lane] : 0;
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += y;
        }
        wscan[lane] = x - v;  // exclusive
        if (lane == 31) wscan[32] = x;
    }
    __syncthreads();
    excl = wscan[w] + __popc(b & ((1u << lane) - 1u));
    const int tot = wscan[32];
    __syncthreads();
    return tot;
}

// Whole CTA: the kCache smallest (key, tie) among slots [0, n) into the cache arrays, by
// a most-significant-digit radix select over the 128-bit values (8-bit digits; stops as
// soon as the remaining bucket fits exactly).
__device__ void cache_rebuild(UpdSmem &S, int n, int *wscan) {
    const int tid = threadIdx.x;
    const int c = n < kCache ? n : kCache;
    uint64_t pk = 0, pt = 0, mk = 0, mt = 0;  // prefix value / mask of the bytes fixed so far
    int need = c;
    for (int i = tid; i < kPlrMaxK; i += blockDim.x) {
        S.sel[i] = 0;
        S.incache[i] = 0;
    }
    __syncthreads();
    for (int d = 15; d >= 0 && need > 0; d--) {
        for (int i = tid; i < 256; i += blockDim.x) S.hist[i] = 0;
        __syncthreads();
        const int sh = 8 * (d & 7);
        for (int i = tid; i < n; i += blockDim.x) {
            if (S.sel[i]) continue;
            const uint64_t k = S.key[i], t = S.tie[i];
            if ((k & mk) != pk || (t & mt) != pt) continue;
            atomicAdd(&S.hist[(int)(((d >= 8 ? k : t) >> sh) & 0xFFu)], 1);
        }
        __syncthreads();
        if (tid < 32) {  // bucket b holding the need-th value
            int v[8], tot = 0;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                v[j] = S.hist[tid * 8 + j];
                tot += v[j];
            }
            int inc = tot;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
                if (tid >= o) inc += y;
            }
            int before = inc - tot;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                if (before < need && before + v[j] >= need) {
                    S.sel_b = tid * 8 + j;
                    S.sel_below = before;
                    S.sel_cnt = v[j];
                }
                before += v[j];
            }
        }
        __syncthreads();
        const int b = S.sel_b, below = S.sel_below, cnt = S.sel_cnt;
        const uint64_t byte = (uint64_t)b << sh;
        for (int i = tid; i < n; i += blockDim.x) {  // buckets below b are in
            if (S.sel[i]) continue;
            const uint64_t k = S.key[i], t = S.tie[i];
            if ((k & mk) != pk || (t & mt) != pt) continue;
            const int bb = (int)(((d >= 8 ? k : t) >> sh) & 0xFFu);
            if (bb < b || (bb == b && cnt == need - below)) S.sel[i] = 1;
        }
        if (d >= 8) {
            pk |= byte;
            mk |= 0xFFull << sh;
        } else {
            pt |= byte;
            mt |= 0xFFull << sh;
        }
        need = cnt == need - below ? 0 : need - below;
        __syncthreads();
    }
    // compact the selected slots into the cache
    for (int i = tid; i < kCache; i += blockDim.x) S.cslot[i] = -1;
    __syncthreads();
    int off = 0;
    for (int base = 0; base < n; base += blockDim.x) {
        const int i = base + tid;
        const bool in = i < n && S.sel[i];
        int e = 0;
        const int tot = block_excl_count(in, e, wscan);
        if (in) {
            S.cslot[off + e] = i;
            S.ckey[off + e] = S.key[i];
            S.ctie[off + e] = S.tie[i];
            S.incache[i] = 1;
        }
        off += tot;
    }
    __syncthreads();
    if (tid == 0) S.cvalid = c > 0 ? 1 : 0;
    __syncthreads();
}

__device__ int insert_runs(UpdSmem &S, const UpdScratch &W, const double *__restrict__ cscore, int64_t iter,
                           int r0, int rend, int E, int *wscan) {
    // E = buffer capacity K: sort items [0, E) are the buffer (stored + virtual free
    // slots), items [E, kPlrMaxK) padding that sorts last
    const int tid = threadIdx.x, ci = tid >> 2, part = tid & 3;
    RunArr &R = S.u.run;
    // ---- the buffer sorted by (score, tie): tie order (stable), then score order ----
    {
        const int size0 = S.size;
        unsigned long long keys[4];
        int vals[4];
        unsigned long long tmax = 0ull;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int i = tid * 4 + k;  // slot (stored for i < size0, free otherwise)
            keys[k] = i < size0 ? S.tie[i] : (unsigned long long)i;  // virtual: slot order
            vals[k] = i;
            tmax = keys[k] > tmax ? keys[k] : tmax;
        }
        if (tid == 0) S.tie_max = 0ull;
        __syncthreads();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xFFFFFFFFu, tmax, o);
            tmax = y > tmax ? y : tmax;
        }
        if ((tid & 31) == 0) atomicMax(&S.tie_max, tmax);  // one per warp (not 1024 on one word)
        __syncthreads();
        const int tbits = 64 - __clzll((long long)(S.tie_max | 1ull));
        RunSort(S.r1.sort).Sort(keys, vals, 0, tbits);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int slot = vals[k];
            keys[k] = slot < size0 ? S.key[slot] : (slot < E ? 0ull : ~0ull);
        }
        RunSort(S.r1.sort).Sort(keys, vals);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 4; k++) {
            S.r1.e.ekey[tid * 4 + k] = keys[k];
            S.r1.e.eslot[tid * 4 + k] = vals[k];
        }
    }
    const uint64_t *ekey = S.r1.e.ekey;
    int pos = r0;
    bool more = true;
    while (more && pos < rend) {
        // ---- next chunk of certainly-new candidates ----
        if (tid == 0) S.flag_first = kRunM;
        __syncthreads();
        int c = -1;
        if (tid < kRunM) {
            const int idx = pos + tid;
            bool ok = idx < rend;
            if (ok) {
                c = W.rel[idx];
                ok = W.init_match[c] < 0 && W.twin_first[c] == c;
            }
            if (!ok) atomicMin(&S.flag_first, tid);
        }
        __syncthreads();
        int m = S.flag_first;
        if (m < kRunM) more = false;
        if (m == 0) break;
        if (tid < m) {
            R.lc[tid] = c;
            R.lk[tid] = score_key(cscore[c]);
        }
        pos += m;
        // ---- passes over the live candidates ----
        while (m > 0) {
            if (tid == 0) PLR_STAT(5, 1);
            __syncthreads();
            if (tid == 0) {
                S.flag_first = m;
                S.n_virtual = 0;
            }
            const int size_cur = S.size;
            const int64_t seq0 = S.next_seq;
            const bool live = ci < m;
            const uint64_t si = live ? R.lk[ci] : 0ull;
            int below = 0, g = 0;
            if (live) {
                below = upper_bound_u64(ekey, E, si);
                for (int j = part; j < ci; j += 4) g += R.lk[j] > si;
            }
            g += __shfl_xor_sync(0xFFFFFFFFu, g, 1);
            g += __shfl_xor_sync(0xFFFFFFFFu, g, 2);
            const bool acc = live && g < below;
            int q = 0;
            const int p = block_excl_count(part == 0 && acc, q, wscan);
            q = __shfl_sync(0xFFFFFFFFu, q, (threadIdx.x & 31) & ~3);  // the group's part-0 count
            if (part == 0 && live) R.lq[ci] = q;
            if (part == 0 && acc) {
                R.acand[q] = ci;
                R.abelow[q] = below;
            }
            __syncthreads();
            // rank among this pass's acceptances (score, then arrival)
            int rk = 0;
            if (acc)
                for (int k = part; k < p; k += 4) {
                    const int j = R.acand[k];
                    const uint64_t sj = R.lk[j];
                    rk += sj < si || (sj == si && j < ci);
                }
            rk += __shfl_xor_sync(0xFFFFFFFFu, rk, 1);
            rk += __shfl_xor_sync(0xFFFFFFFFu, rk, 2);
            if (part == 0 && acc) {
                R.ask[rk] = si;
                R.arank[q] = rk;
            }
            __syncthreads();
            // the first p+1 elements of the merged order (buffer before acceptance at equal score)
            for (int k = tid; k <= p && k < E; k += blockDim.x) {
                const int mi = k + lower_bound_u64(R.ask, p, ekey[k]);
                if (mi <= p) {
                    R.mkey[mi] = ekey[k];
                    R.mref[mi] = k;
                }
            }
            if (part == 0 && acc) {
                const int mi = rk + below;
                if (mi <= p) {
                    R.mkey[mi] = si;
                    R.mref[mi] = -(q + 1);
                }
            }
            __syncthreads();
            // exact ties: the minimum present at arrival is merged element q_i
            if (part == 0 && live && R.mkey[R.lq[ci]] == si) atomicMin(&S.flag_first, ci);
            for (int k = tid; k < kRunM / 32; k += blockDim.x) S.evicted[k] = 0u;
            __syncthreads();
            const int f = S.flag_first;
            const int pc = f < m ? R.lq[f] : p;  // acceptances committed (arrival < f)
            // ---- slots: the j-th acceptance takes the slot of the j-th eviction ----
            for (int j = tid; j < pc; j += blockDim.x) {
                const int v = R.mref[j];
                if (v >= 0) {
                    const int slot = S.r1.e.eslot[v];
                    R.aslot[j] = slot;
                    if (slot >= size_cur) {
                        atomicAdd(&S.n_virtual, 1);
                    } else if (S.owner[slot] >= 0) {
                        W.keyslot[S.owner[slot]] = -1;  // inserted earlier in this update: evicted
                        const int og = S.origin[slot];
                        if (og >= 0) S.reslot[og] = -1;
                    }
                } else {
                    R.aslot[j] = -1;
                    const int qq = -v - 1;
                    atomicOr(&S.evicted[qq >> 5], 1u << (qq & 31));
                }
            }
            __syncthreads();
            while (true) {  // pointer jumping along chains of re-evicted acceptances
                int ns = -1, nv = 0;
                bool pend = false;
                if (tid < pc && R.aslot[tid] < 0) {
                    const int par = -R.mref[tid] - 1;
                    const int ps = R.aslot[par];
                    pend = true;
                    if (ps >= 0)
                        ns = ps;
                    else
                        nv = R.mref[par];
                }
                __syncthreads();
                if (pend) {
                    if (ns >= 0)
                        R.aslot[tid] = ns;
                    else
                        R.mref[tid] = nv;
                }
                if (!__syncthreads_or(pend)) break;
            }
            // ---- apply: final occupants ----
            for (int j = tid; j < pc; j += blockDim.x) {
                const int li = R.acand[j];
                const int cj = R.lc[li];
                if ((S.evicted[j >> 5] >> (j & 31)) & 1u) {
                    W.keyslot[cj] = -1;  // inserted and evicted again inside the pass
                    continue;
                }
                const int slot = R.aslot[j];
                S.key[slot] = R.lk[li];
                S.tie[slot] = tie_pack(S, iter, seq0 + j);
                S.owner[slot] = cj;
                S.origin[slot] = -1;  // run candidates are new to the buffer
                S.src[slot] = cj;
                S.mr_src[slot] = cj;
                atomicOr(&S.replaced[slot >> 5], 1u << (slot & 31));
                W.keyslot[cj] = slot;
            }
            // the committed acceptances sorted (apk): ask positions whose acceptance index is
            // < pc, compacted in order; apos2[ask position] = its position in apk
            __syncthreads();
            if (tid < p) R.apos2[R.arank[tid]] = tid;  // ask position -> acceptance index
            __syncthreads();
            const bool cm = tid < p && R.apos2[tid] < pc;
            int e2 = 0;
            block_excl_count(cm, e2, wscan);
            if (cm) {
                R.apk[e2] = R.ask[tid];
                R.apos2[tid] = e2;
            }
            __syncthreads();
            uint64_t nk[4];
            int ns[4], np[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int e = tid * 4 + k;
                np[k] = -1;
                if (e < E && pc > 0) {
                    nk[k] = ekey[e];
                    ns[k] = S.r1.e.eslot[e];
                    np[k] = e + lower_bound_u64(R.apk, pc, nk[k]) - pc;
                }
            }
            uint64_t ak = 0ull;
            int as = 0, ap = -1;
            if (tid < pc && !((S.evicted[tid >> 5] >> (tid & 31)) & 1u)) {
                const int r = R.arank[tid];
                ak = R.ask[r];
                as = R.aslot[tid];
                ap = R.apos2[r] + R.abelow[tid] - pc;
            }
            __syncthreads();
            if (pc > 0) {
#pragma unroll
                for (int k = 0; k < 4; k++)
                    if (np[k] >= 0) {
                        S.r1.e.ekey[np[k]] = nk[k];
                        S.r1.e.eslot[np[k]] = ns[k];
                    }
                if (ap >= 0) {
                    S.r1.e.ekey[ap] = ak;
                    S.r1.e.eslot[ap] = as;
                }
            }
            if (tid == 0) {
                S.size = size_cur + S.n_virtual;
                S.next_seq = seq0 + pc;
            }
            // ---- next pass: drop f and every later candidate with score <= s_f ----
            int nm = 0;
            if (f < m) {
                const uint64_t mu = R.lk[f];
                const bool keepc = part == 0 && live && ci > f && si > mu;
                const int cc = live ? R.lc[ci] : 0;
                int e3 = 0;
                nm = block_excl_count(keepc, e3, wscan);
                if (keepc) {
                    R.lk[e3] = si;
                    R.lc[e3] = cc;
                }
            }
            m = nm;
        }
    }
    __syncthreads();
    // the bottom cache straight from the sorted buffer (no radix-select rebuild): the
    // remaining virtual free slots (key 0) sort first, then the real entries in (score,
    // tie) order -- the first kCache of those
    {
        const int sz = S.size, first = E - sz, c = sz < kCache ? sz : kCache;
        for (int i = tid; i < kPlrMaxK; i += blockDim.x) S.incache[i] = 0;
        __syncthreads();
        if (tid < kCache) {
            int slot = -1;
            if (tid < c) {
                slot = S.r1.e.eslot[first + tid];
                S.ckey[tid] = S.key[slot];
                S.ctie[tid] = S.tie[slot];
                S.incache[slot] = 1;
            }
            S.cslot[tid] = slot;
        }
        if (tid == 0) S.cvalid = c > 0 ? 1 : 0;
    }
    __syncthreads();
    return pos - r0;
}

__global__ void k_plr_cand_prep(PlrDev D, const amz_level_t *__restrict__ cand, int64_t n, UpdScratch W,
                                int64_t hsize) {
    pdl_wait();  // PDL: the predecessor kernel has completed (its launch overlapped)
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
    pdl_wait();  // PDL: the predecessor kernel has completed (its launch overlapped)
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

__device__ __forceinline__ int bits_for(uint64_t span) { return span ? 64 - __clzll((long long)span) : 0; }

__global__ void __launch_bounds__(kPlrThreads, 1)
    k_plr_update(PlrDev D, const amz_level_t *__restrict__ cand, const double *__restrict__ cscore,
                 const double *__restrict__ cmax, int64_t n, int64_t iter, UpdScratch W, int *err) {
    pdl_wait();  // PDL: the predecessor kernel has completed (its launch overlapped)
    extern __shared__ __align__(16) uint8_t smraw[];
    UpdSmem &S = *reinterpret_cast<UpdSmem *>(smraw);
    __shared__ int wscan[33];
    const int tid = threadIdx.x, lane = tid & 31;
    const int K = (int)D.K;
    const int size0 = (int)D.meta[0];
    PLR_CLK(clk_a);
    // ---- A: tie-key frame, buffer into the heap arrays + key hash ----
    for (int i = tid; i < kHash; i += blockDim.x) S.u.hash[i] = 0u;
    for (int i = tid; i < kPlrMaxK / 32; i += blockDim.x) S.replaced[i] = 0u;
    for (int i = tid; i < kPlrMaxK; i += blockDim.x) {
        S.owner[i] = -1;
        S.src[i] = -1;
        S.mr_src[i] = -1;
        S.reslot[i] = -1;
        S.origin[i] = -1;
    }
    if (tid == 0) {
        S.n_rel = 0;
        S.full = size0 >= K;
        S.next_seq = D.meta[1];
        S.lmin = iter;
        S.lmax = iter;
        S.last_max0 = INT64_MIN;
        S.qmin = D.meta[1];
        S.qmax = D.meta[1] + n;
    }
    __syncthreads();
#ifdef AMZ_PLR_STATS
    if (tid == 0) PLR_STAT(36, clock64() - clk_a);
#endif
    {
        long long lmn = iter, lmx = iter, qmn = S.qmin, lm0 = INT64_MIN;
#pragma unroll 4
        for (int i = tid; i < size0; i += blockDim.x) {
            const long long l = D.last[i], q = D.seq[i];
            lmn = l < lmn ? l : lmn;
            lmx = l > lmx ? l : lmx;
            lm0 = l > lm0 ? l : lm0;
            qmn = q < qmn ? q : qmn;
        }
        // warp reductions first: 1024 threads' 64-bit shared atomics on four words serialise
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long a = __shfl_xor_sync(0xFFFFFFFFu, lmn, o), b = __shfl_xor_sync(0xFFFFFFFFu, lmx, o);
            const long long c = __shfl_xor_sync(0xFFFFFFFFu, lm0, o), d = __shfl_xor_sync(0xFFFFFFFFu, qmn, o);
            lmn = a < lmn ? a : lmn;
            lmx = b > lmx ? b : lmx;
            lm0 = c > lm0 ? c : lm0;
            qmn = d < qmn ? d : qmn;
        }
        if (lane == 0) {
            atomicMin((long long *)&S.lmin, lmn);
            atomicMax((long long *)&S.lmax, lmx);
            atomicMax((long long *)&S.last_max0, lm0);
            atomicMin((long long *)&S.qmin, qmn);
        }
    }
    __syncthreads();
    if (tid == 0) {
        const int bl = bits_for((uint64_t)S.lmax - (uint64_t)S.lmin);
        const int bq = bits_for((uint64_t)S.qmax - (uint64_t)S.qmin);
        S.bq = bq;
        S.run_ok = (bl + bq <= 64) ? 1 : -1;
        if (S.run_ok > 0) S.run_ok = S.last_max0 <= iter ? 1 : 0;  // stored ties below every new one
    }
    __syncthreads();
    if (S.run_ok < 0) {  // (last, seq) spans do not fit one 64-bit tie key: refuse, unchanged
        if (tid == 0) atomicOr(err, 4);
        return;
    }
#ifdef AMZ_PLR_STATS
    if (tid == 0) PLR_STAT(37, clock64() - clk_a);
#endif
    double my_min = __longlong_as_double(0x7FF0000000000000ll);  // +inf
    // keys, tie keys and the key hash.  The hash is built in two steps: every entry stores
    // itself into its home slot (plain stores, one wins per slot), then only the losers
    // insert by atomicCAS from the next slot on -- four times fewer shared atomics than a
    // CAS per entry, which serialised (~12k cycles for K = 4000).  Linear probing stays
    // valid: a loser's run from its home slot to its place is occupied when it lands.
    static_assert(kPlrMaxK <= 4 * kPlrThreads, "four buffer entries per thread");
    uint32_t hh[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int i = tid + k * kPlrThreads;
        hh[k] = 0u;
        if (i < size0) {
            const double sc = D.score[i];
            const long long la = D.last[i], sq = D.seq[i];
            uint4 w;
            uint32_t p0, p1;
            level_key(D.levels + i, w, p0, p1);
            S.key[i] = score_key(sc);
            S.tie[i] = tie_pack(S, la, sq);
            my_min = fmin(my_min, sc);
            hh[k] = level_hash(w, p0 ^ (p1 << 24)) & (kHash - 1);
            S.u.hash[hh[k]] = (uint32_t)(i + 1);
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int i = tid + k * kPlrThreads;
        if (i < size0 && S.u.hash[hh[k]] != (uint32_t)(i + 1)) {
            uint32_t h = (hh[k] + 1u) & (kHash - 1);
            while (atomicCAS(&S.u.hash[h], 0u, (uint32_t)(i + 1)) != 0u) h = (h + 1) & (kHash - 1);
        }
    }
    __syncthreads();
#ifdef AMZ_PLR_STATS
    if (tid == 0) PLR_STAT(38, clock64() - clk_a);
#endif
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
    if (tid == 0) S.cvalid = 0;
    __syncthreads();
    PLR_CLK(clk_b);
    if (tid == 0) PLR_STAT(34, clk_b - clk_a);
    // ---- B: relevant candidates, compacted in order (block-wide, chunk by chunk) ----
    for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t c = base + tid;
        bool rel = false;
        if (c < n) {
            const bool later_twin = W.twin_first[c] != (int32_t)c;
            rel = !S.full || W.init_match[c] >= 0 || later_twin || !(cscore[c] <= S.mlow);
        }
        int excl = 0;
        const int tot = block_excl_count(rel, excl, wscan);
        if (rel) W.rel[S.n_rel + excl] = (int32_t)c;
        __syncthreads();
        if (tid == 0) S.n_rel += tot;
        __syncthreads();
    }
    // A skipped first occurrence is never inserted (score <= mlow), so its later twins,
    // which are always relevant, correctly find no entry for the key (keyslot = -1).

    PLR_CLK(clk_c);
    if (tid == 0) PLR_STAT(11, clk_c - clk_b);
    // ---- C: ordered replay (warp 0); bulk in-place runs and insert runs by the CTA ----
    // In-place updates never change which later candidates find their key (only fills and
    // evictions do), so warp 0 scans ahead for the run of consecutive in-place candidates
    // starting at r.  A run of >= kBulkRun is applied in bulk: the last candidate per slot
    // wins (atomicMax on the candidate index, which is increasing along the order), and the
    // heap is rebuilt level-parallel.  (score, tb) is a total order (seq is unique), so the
    // heap's shape never affects which entry is the minimum.
    const int nrel = S.n_rel;
    if (tid == 0) {
        S.size = size0;
        PLR_STAT(7, nrel);
        PLR_STAT(8, 1);
    }
    int base = 0;
    while (base < nrel) {
        const int cn = (nrel - base) < kChunk ? (nrel - base) : kChunk;
        __syncthreads();
        for (int i = tid; i < cn; i += blockDim.x) {
            const int c = W.rel[base + i];
            S.u.chunk.cid[i] = c;
            S.u.chunk.sk[i] = score_key(cscore[c]);
            S.u.chunk.tf[i] = W.twin_first[c];
            S.u.chunk.im[i] = W.init_match[c];
        }
        __syncthreads();
        PLR_CLK(clk_w0);
        if (tid < 32) {
            int size = S.size;
            int64_t next_seq = S.next_seq;
            const bool run_ok = S.run_ok > 0;
            int r = 0, scan_end = 0, pscan_end = 0, action = 0, arg = 0;
            BottomCache bc;
            bc.load(S, lane);
            // candidate fields are prefetched one ahead (the replaced bit and the twin's
            // keyslot are read after the previous candidate is applied)
            int c_n = 0, f_n = 0, im_n = -1;
            uint64_t sk_n = 0ull;
            if (r < cn) {
                c_n = S.u.chunk.cid[r];
                sk_n = S.u.chunk.sk[r];
                f_n = S.u.chunk.tf[r];
                im_n = S.u.chunk.im[r];
            }
#ifdef AMZ_PLR_STATS
            long long clk_sc = 0;
#endif
            for (; r < cn; r++) {
#ifdef AMZ_PLR_STATS
                if (clk_sc && lane == 0) {
                    PLR_STAT(20, clock64() - clk_sc);
                    PLR_STAT(21, 1);
                }
                clk_sc = 0;
#endif
                int present;  // candidate r's in-place slot or -1 (lane 0 of the batch probe)
                unsigned pres_b, pure_b;  // the probe's lanes r..r+31: present / certainly new
                // Warp-batched fast path: the leading stretch of "simple" candidates -- in
                // place (key present), slot outside the bottom cache and new key above the
                // cache maximum -- changes neither presence nor the cache, so the stretch
                // is applied at once (the last candidate per slot wins)
                {
                    PLR_CLK(clk_bt);
                    const int i = r + lane;
                    bool simple = false, prs = false;
                    int ps = -1, ci = 0;
                    uint64_t ski = 0;
                    // an absent key is certainly rejected (a no-op) when the buffer is full and
                    // its score does not beat the cache minimum, which no simple op changes
                    const bool rej_ok = bc.valid && size >= K;
                    const uint64_t mink = bc.nk;
#ifdef AMZ_PLR_STATS
                    bool gread = false;
#endif
                    if (i < cn) {
                        // branch-free where the lanes disagree (initial match or not, present
                        // or not): every load issues, clamped, and selects pick the result
                        ci = S.u.chunk.cid[i];
                        const int imi = S.u.chunk.im[i], fi = S.u.chunk.tf[i];
                        const int imc = imi < 0 ? 0 : imi;
                        prs = imi < 0 && fi == ci;  // certainly new
                        const uint32_t rw = S.replaced[imc >> 5];
                        const int rs = S.reslot[imc];
                        ski = S.u.chunk.sk[i];
                        ps = ((rw >> (imc & 31)) & 1u) ? rs : imi;
                        if (imi < 0) {
                            ps = -1;
                            if (fi != ci) ps = W.keyslot[fi];  // a later twin of a new level (rare)
                        }
#ifdef AMZ_PLR_STATS
                        gread = imi < 0 && fi != ci;
#endif
                        const int pc = ps < 0 ? 0 : ps;
                        const bool inc = S.incache[pc] != 0;
                        const uint64_t tp = S.tie[pc];
                        const bool sin = !bc.valid || (!inc && !ukey_le(ski, tp, bc.mk, bc.mt));
                        const bool sab = rej_ok && !(ski > mink);
                        simple = ps >= 0 ? sin : sab;
                    }
#ifdef AMZ_PLR_STATS
                    {
                        const bool sv = __ballot_sync(0xFFFFFFFFu, simple) != 0;  // the chain settles here
                        if (lane == 0) {
                            PLR_STAT(32, clock64() - clk_bt + (sv ? 0 : 0));
                            PLR_STAT(33, 1);
                        }
                    }
#endif
                    present = __shfl_sync(0xFFFFFFFFu, ps, 0);
                    pres_b = __ballot_sync(0xFFFFFFFFu, i < cn && ps >= 0);
                    pure_b = __ballot_sync(0xFFFFFFFFu, prs);
#ifdef AMZ_PLR_STATS
                    {
                        const unsigned gr = __ballot_sync(0xFFFFFFFFu, gread);
                        if (lane == 0) {
                            PLR_STAT(30, gr != 0);
                            PLR_STAT(31, 1);
                        }
                    }
#endif
                    const unsigned bad = ~__ballot_sync(0xFFFFFFFFu, simple);
                    const int k = bad ? __ffs(bad) - 1 : 32;
                    if (k > 0) {
                        const bool act = lane < k && ps >= 0;  // rejected absent keys change nothing
                        // last writer per slot: candidate ids grow along the order, so the
                        // slot's atomicMax is the last writer (match.any was slower here)
                        if (act) atomicMax(&S.mr_src[ps], ci);
                        __syncwarp();
                        if (act && S.mr_src[ps] == ci) S.key[ps] = ski;
                        if (lane == 0) {
                            PLR_STAT(10, k);
                            PLR_STAT(13, 1);
                            PLR_STAT(14, clock64() - clk_bt);
                        }
                        __syncwarp();
                        r += k - 1;  // the loop's r++ moves past the stretch
                        if (r + 1 < cn) {
                            c_n = S.u.chunk.cid[r + 1];
                            sk_n = S.u.chunk.sk[r + 1];
                            f_n = S.u.chunk.tf[r + 1];
                            im_n = S.u.chunk.im[r + 1];
                        }
                        continue;
                    }
                }
#ifdef AMZ_PLR_STATS
                clk_sc = clock64();
#endif
                const int c = c_n, f = f_n, im = im_n;
                const uint64_t sk = sk_n;
                if (r + 1 < cn) {
                    c_n = S.u.chunk.cid[r + 1];
                    sk_n = S.u.chunk.sk[r + 1];
                    f_n = S.u.chunk.tf[r + 1];
                    im_n = S.u.chunk.im[r + 1];
                }
                // a stretch of certainly-new candidates worth a parallel insert run
                if (run_ok && im < 0 && f == c && r >= pscan_end) {
                    const int L = pure_run(S, r, cn, lane, pure_b);
                    if (L >= kRunMin) {
                        action = 2;
                        arg = L;
                        break;
                    }
                    pscan_end = r + L;
                }
                // only an in-place candidate can open a run worth applying in bulk
                if (present >= 0 && r >= scan_end) {
                    PLR_CLK(clk_ir);
                    const int L = inplace_run(S, W, r, cn, lane, pres_b);
                    if (lane == 0) PLR_STAT(15, clock64() - clk_ir);
                    if (L >= kBulkRun) {
                        action = 1;
                        arg = r + L;
                        break;
                    }
                    scan_end = r + L;
                }
                if (lane == 0) PLR_STAT(0, 1);
#ifdef AMZ_PLR_STATS
                if (lane == 0) PLR_STAT(22, clock64() - clk_sc);
#endif
#ifdef AMZ_PLR_STATS
                const long long clk_body = clock64();
#endif
                if (present >= 0) {
                    if (lane == 0) PLR_STAT(1, 1);  // identical level: score / max_return in place (tb unchanged)
                    const int s2 = present;
                    const uint64_t st = S.tie[s2];
                    __syncwarp();
                    if (lane == 0) {
                        S.key[s2] = sk;
                        S.mr_src[s2] = c;
                    }
                    if (bc.valid) {  // keep the bottom cache exact
                        int wl, ww;
                        bc.find(s2, wl, ww);
                        if (wl >= 0)
                            bc.rekey(s2, wl, ww, sk, st, lane);
                        else if (ukey_le(sk, st, bc.mk, bc.mt))
                            bc.insert(s2, sk, st, lane);
                    }
                    __syncwarp();
#ifdef AMZ_PLR_STATS
                    if (lane == 0) PLR_STAT(23, clock64() - clk_body);
#endif
                    continue;
                }
                const uint64_t tbn = tie_pack(S, iter, next_seq);
                int slot;
                if (size < K) {  // fill
                    slot = size++;
                    __syncwarp();
                    if (lane == 0) {
                        S.key[slot] = sk;
                        S.tie[slot] = tbn;
                    }
                    if (bc.valid && ukey_le(sk, tbn, bc.mk, bc.mt)) bc.insert(slot, sk, tbn, lane);
#ifdef AMZ_PLR_STATS
                    if (lane == 0) { PLR_STAT(24, clock64() - clk_body); PLR_STAT(25, 1); }
#endif
                } else {  // evict the (score, last_sampled, seq) minimum iff strictly better
                    if (!bc.valid) {  // the CTA rebuilds the cache, then this candidate again
                        action = 3;
                        break;
                    }
                    const uint64_t mink = bc.nk;
                    const int ms = bc.ns;
#ifdef AMZ_PLR_STATS
                    if (lane == 0) { PLR_STAT(26, clock64() - clk_body); PLR_STAT(27, 1); }
#endif
                    if (!(sk > mink)) continue;
                    slot = ms;
                    const int ow = S.owner[slot], og = S.origin[slot];
                    __syncwarp();
                    if (lane == 0) {
                        if (ow >= 0) W.keyslot[ow] = -1;
                        if (og >= 0) S.reslot[og] = -1;
                        S.key[slot] = sk;
                        S.tie[slot] = tbn;
                    }
                    bc.pop_min(lane);  // empty -> invalid (rebuilt before the next eviction)
                    if (bc.valid && ukey_le(sk, tbn, bc.mk, bc.mt)) bc.insert(slot, sk, tbn, lane);
#ifdef AMZ_PLR_STATS
                    if (lane == 0) { PLR_STAT(28, clock64() - clk_body); PLR_STAT(29, 1); }
#endif
                }
                if (lane == 0) {
                    S.owner[slot] = f;
                    S.origin[slot] = (int16_t)im;
                    if (im >= 0) S.reslot[im] = (int16_t)slot;
                    S.replaced[slot >> 5] |= 1u << (slot & 31);
                    S.src[slot] = c;
                    S.mr_src[slot] = c;
                    W.keyslot[f] = slot;
                }
                __syncwarp();
                next_seq++;
            }
            __syncwarp();
            bc.store(S, lane);
            if (lane == 0) {
                S.size = size;
                S.next_seq = next_seq;
                S.rcur = r;
                S.action = action;
                S.arg = arg;
            }
        }
        __syncthreads();
        if (tid == 0) {
            PLR_STAT(16, clock64() - clk_w0);
            PLR_STAT(17, 1);
        }
        const int lo = S.rcur, action = S.action, arg = S.arg;
        if (action == 0) {
            base += cn;
            continue;
        }
        if (action == 3) {  // the bottom cache: the kCache smallest entries, by radix select
            if (tid == 0) PLR_STAT(9, 1);
            PLR_CLK(clk_rb);
            cache_rebuild(S, S.size, wscan);
            if (tid == 0) PLR_STAT(18, clock64() - clk_rb);
            base += lo;
            continue;
        }
        if (action == 1) {  // bulk in-place run [lo, arg)
            if (tid == 0) {
                PLR_STAT(2, 1);
                PLR_STAT(3, arg - lo);
            }
            const int hi = arg;
            // the bottom cache survives the run if no updated entry is in it or lands at or
            // below its maximum (every entry outside then still lies above the maximum)
            const bool cv = S.cvalid != 0;
            if (tid < 32 && cv) {
                uint64_t k = 0, t = 0;
                bool has = false;
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int j = tid + 32 * h;
                    if (S.cslot[j] >= 0) {
                        const uint64_t kj = S.ckey[j], tj = S.ctie[j];
                        if (!has || !ukey_le(kj, tj, k, t)) {
                            k = kj;
                            t = tj;
                        }
                        has = true;
                    }
                }
                const int win = warp_lex_pick(has, k, t, true, tid);
                if (tid == win) {
                    S.bmk = k;
                    S.bmt = t;
                }
            }
            if (tid == 0) S.bulk_bad = 0;
            for (int i = lo + tid; i < hi; i += blockDim.x)
                atomicMax(&S.mr_src[cand_present(S, W, i)], S.u.chunk.cid[i]);
            __syncthreads();
            for (int i = lo + tid; i < hi; i += blockDim.x) {
                const int p = cand_present(S, W, i);
                if (S.mr_src[p] == S.u.chunk.cid[i]) {
                    const uint64_t nk = S.u.chunk.sk[i];
                    S.key[p] = nk;
                    if (cv && (S.incache[p] || ukey_le(nk, S.tie[p], S.bmk, S.bmt))) {
                        const int j = atomicAdd(&S.bulk_bad, 1);  // entries the cache must absorb
                        if (j < kCache) S.bulk_list[j] = p;
                    }
                }
            }
            __syncthreads();
            const int nb = S.bulk_bad;
            if (nb > kCache) {
                if (tid == 0) S.cvalid = 0;  // too many: rebuilt when next needed
            } else if (nb > 0 && tid < 32) {
                // warp 0 replays them into the cache (a changed member: rekey; an outside
                // entry now at or below the maximum: insert) -- a few warp operations each
                // instead of the CTA-wide rebuild
                BottomCache bc;
                bc.load(S, tid);
                for (int j = 0; j < nb && bc.valid; j++) {
                    const int p = S.bulk_list[j];
                    const uint64_t k = S.key[p], t = S.tie[p];
                    int wl, ww;
                    bc.find(p, wl, ww);
                    if (wl >= 0)
                        bc.rekey(p, wl, ww, k, t, tid);
                    else if (ukey_le(k, t, bc.mk, bc.mt))
                        bc.insert(p, k, t, tid);
                }
                __syncwarp();
                bc.store(S, tid);
            }
            __syncthreads();
            if (tid == 0 && nb > kCache) PLR_STAT(39, 1);
            base += hi;
            continue;
        }
        // insert run [base + lo, base + lo + arg)
        {
            PLR_CLK(clk_in);
            const int used = insert_runs(S, W, cscore, iter, base + lo, nrel, K, wscan);
            if (tid == 0) PLR_STAT(19, clock64() - clk_in);
            if (tid == 0) {
                PLR_STAT(4, 1);
                PLR_STAT(6, used);
            }
            base += lo + used;
        }
    }
    __syncthreads();
    PLR_CLK(clk_e);
    if (tid == 0) PLR_STAT(12, clk_e - clk_c);
    // ---- epilogue: tie keys back to last_sampled / seq, deferred level / max_return copies ----
    const int fsize = S.size;
    const uint64_t qmask = S.bq >= 64 ? ~0ull : ((1ull << S.bq) - 1ull);
    for (int slot = tid; slot < fsize; slot += blockDim.x) {
        const uint64_t tb = S.tie[slot];
        D.last[slot] = (int64_t)((S.bq >= 64 ? 0ull : (tb >> S.bq)) + (uint64_t)S.lmin);
        D.seq[slot] = (int64_t)((tb & qmask) + (uint64_t)S.qmin);
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
#ifdef AMZ_PLR_STATS
    __syncthreads();
    if (tid == 0) PLR_STAT(35, clock64() - clk_e);
#endif
}

// top-q replay lanes by score (ties -> lower lane index), single CTA
__global__ void k_top_q(const double *__restrict__ scores, int64_t n, int q, int32_t *__restrict__ out) {
    pdl_wait();  // PDL: the predecessor kernel has completed (its launch overlapped)
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

// 64-bit digest of the buffer state (valid slots + meta) for the replica drift check:
// a wrapping sum of per-slot mixes (slot index, level words, score / max_return bits,
// last_sampled, seq), so it is order-free across threads and equal iff (up to hash
// collisions) the replicas hold the same entries in the same slots.
__device__ __forceinline__ uint64_t mix64(uint64_t h, uint64_t v) {
    h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    h ^= h >> 31;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 29;
    return h;
}
__global__ void __launch_bounds__(256) k_plr_digest(PlrDev D, int64_t *__restrict__ out) {
    __shared__ unsigned long long acc;
    if (threadIdx.x == 0) acc = 0ull;
    __syncthreads();
    const int64_t size = D.meta[0];
    unsigned long long mine = 0ull;
    for (int64_t i = threadIdx.x; i < size && i < D.K; i += blockDim.x) {
        const uint4 *lw = reinterpret_cast<const uint4 *>(D.levels + i);
        const uint4 a = lw[0], b = lw[1];
        uint64_t h = mix64(0x243F6A8885A308D3ull, (uint64_t)i);
        h = mix64(h, ((uint64_t)a.y << 32) | a.x);
        h = mix64(h, ((uint64_t)a.w << 32) | a.z);
        h = mix64(h, ((uint64_t)b.y << 32) | b.x);
        h = mix64(h, ((uint64_t)b.w << 32) | b.z);
        h = mix64(h, (uint64_t)__double_as_longlong(D.score[i]));
        h = mix64(h, (uint64_t)__double_as_longlong(D.maxret[i]));
        h = mix64(h, (uint64_t)D.last[i]);
        h = mix64(h, (uint64_t)D.seq[i]);
        mine += h;
    }
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xFFFFFFFFu, mine, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&acc, mine);
    __syncthreads();
    if (threadIdx.x == 0) out[0] = (int64_t)mix64(mix64(acc, (uint64_t)size), (uint64_t)D.meta[1]);
}

int launch_plr_digest(const PlrDev &D, int64_t *out, cudaStream_t s) {
    k_plr_digest<<<1, 256, 0, s>>>(D, out);
    return 0;
}

size_t plr_sample_smem() { return sizeof(SampleSmem); }
size_t plr_update_smem() { return sizeof(UpdSmem); }

int launch_plr_sample(const PlrDev &D, int32_t *rank, const amz_seed_t &key, int64_t n, double omr, double rho,
                      const double *lut, int prop, double inv_beta, int64_t iter, int32_t *slots, amz_level_t *levels,
                      double *maxret, double *score, int *err, cudaStream_t s) {
    static bool attr[kMaxDevices] = {};  // the attribute is per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= kMaxDevices || !attr[dev]) {
        cudaFuncSetAttribute(k_plr_sample, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SampleSmem));
        if (dev < kMaxDevices) attr[dev] = true;
    }
    if (!prop) {  // ranks only for rank prioritisation
        cudaMemsetAsync(rank, 0, (size_t)D.K * sizeof(int32_t), s);
        launch_pdl(k_plr_rank, dim3((unsigned)((D.K + kRankThreads - 1) / kRankThreads),
                                   (unsigned)((D.K + kRankJ - 1) / kRankJ)),
                   dim3(kRankThreads), 0, s, D, rank);
    }
    launch_pdl(k_plr_sample, dim3(1), dim3(kPlrThreads), sizeof(SampleSmem), s, D, (const int32_t *)rank, key, n,
               omr, rho, lut, prop, inv_beta, iter, slots, levels, maxret, score, err);
    return 0;
}

// the candidates' twin table (k_plr_cand_prep / _twin): depends on the candidate levels
// only, so it can run ahead of the update (amz_plr_prepare)
int launch_plr_prepare(const PlrDev &D, const amz_level_t *cand, int64_t n, const UpdScratch &W, cudaStream_t s) {
    if (n <= 0) return 0;
    int64_t hsize = 1;
    while (hsize < 2 * n) hsize <<= 1;
    cudaMemsetAsync(W.chash, 0, hsize * sizeof(uint32_t), s);
    const int g = (int)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184);
    launch_pdl(k_plr_cand_prep, g, dim3(256), 0, s, D, cand, n, W, hsize);
    launch_pdl(k_plr_cand_twin, g, dim3(256), 0, s, cand, n, W, hsize);
    return 0;
}

int launch_plr_update(const PlrDev &D, const amz_level_t *cand, const double *cs, const double *cm, int64_t n,
                      int64_t iter, const UpdScratch &W, int *err, cudaStream_t s, int prepared) {
    static bool attr[kMaxDevices] = {};  // the attribute is per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= kMaxDevices || !attr[dev]) {
        cudaFuncSetAttribute(k_plr_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(UpdSmem));
        if (dev < kMaxDevices) attr[dev] = true;
    }
    if (n <= 0) return 0;
    if (!prepared) launch_plr_prepare(D, cand, n, W, s);
    launch_pdl(k_plr_update, dim3(1), dim3(kPlrThreads), sizeof(UpdSmem), s, D, cand, cs, cm, n, iter, W, err);
    return 0;
}

int launch_top_q(const double *scores, int64_t n, int q, int32_t *out, cudaStream_t s) {
    launch_pdl(k_top_q, dim3(1), dim3(256), 0, s, scores, n, q, out);
    return 0;
}

}  // namespace amz
