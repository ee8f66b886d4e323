// amz_score.cu -- fused GAE + episode statistics + MaxMC / PVL regret scores.
//
// One thread per lane over time-major [T][B] arrays (every warp access is a
// contiguous 256-B row segment).  Three passes per lane, all in the reference's
// float64 operation order so results are bit-identical to numpy:
//   1. forward   agents/rollout.py:155-189  per_lane_episode_stats -> running max return
//   2. reverse   agents/gae.py:32-36        delta = (r + (g*nd)*V') - V ; A = delta + ((g*l)*nd)*A'
//   3. forward   runners/scoring.py:18-31   mean over t, summed in numpy's pairwise order
// Build flags include --fmad=false so no multiply-add is contracted.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "amz_internal.h"

namespace amz {

// numpy pairwise_sum recursion: n <= 128 is a leaf; otherwise split at n/2 rounded
// down to a multiple of 8 (numpy/_core/src/umath/loops_utils.h.src).
static int plan_rec(int start, int n, PairwisePlan &p) {
    if (n <= 128) {
        if (p.n_leaves >= kMaxLeaves) return -1;
        p.leaf_end[p.n_leaves] = start + n;
        p.adds[p.n_leaves] = 0;
        p.n_leaves++;
        return 0;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    if (plan_rec(start, n2, p) || plan_rec(start + n2, n - n2, p)) return -1;
    p.adds[p.n_leaves - 1]++;
    return 0;
}

int make_pairwise_plan(int n, PairwisePlan &p) {
    p.n_leaves = 0;
    return plan_rec(0, n, p);
}

// numpy maximum for float64: NaN in the first operand propagates
__device__ __forceinline__ double np_max(double a, double b) { return (a >= b || isnan(a)) ? a : b; }

// Streaming evaluation of numpy's pairwise sum in index order.  Leaf starts are
// multiples of 8, so the accumulator of element t is t & 7.
struct PairwiseSum {
    double r[8];
    double res;
    double stk[8];
    int sp, li, lstart, lend, llen, l8;

    __device__ __forceinline__ void begin(const PairwisePlan &P) {
        sp = 0;
        li = 0;
        lstart = 0;
        lend = P.leaf_end[0];
        llen = lend;
        l8 = llen - llen % 8;
        res = 0.0;
    }
    __device__ __forceinline__ double combine() const {
        return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    }
    __device__ __forceinline__ void add(double x, int t, int j, const PairwisePlan &P) {
        const int p = t - lstart;
        if (llen < 8) {
            res = res + x;
        } else if (p < 8) {
            r[j] = x;
        } else if (p < l8) {
            r[j] = r[j] + x;
        } else {
            if (p == l8) res = combine();
            res = res + x;
        }
        if (t == lend - 1) {
            if (llen >= 8 && l8 == llen) res = combine();
            stk[sp++] = res;
            for (int k = 0; k < P.adds[li]; k++) {
                double b = stk[--sp];
                double a = stk[--sp];
                stk[sp++] = a + b;
            }
            li++;
            if (li < P.n_leaves) {
                lstart = lend;
                lend = P.leaf_end[li];
                llen = lend - lstart;
                l8 = llen - llen % 8;
                res = 0.0;
            }
        }
    }
    __device__ __forceinline__ double total() const { return stk[0]; }
};

__global__ void __launch_bounds__(64) k_gae_score(int T, int64_t B, const double *__restrict__ rw,
                                                  const double *__restrict__ val, const uint8_t *__restrict__ dn,
                                                  const double *__restrict__ last, double gamma, double gl,
                                                  const double *__restrict__ prior, int score_fn, int disc,
                                                  double *__restrict__ adv, double *__restrict__ ret,
                                                  double *__restrict__ scores, double *__restrict__ maxret,
                                                  int64_t *__restrict__ st_eps, double *__restrict__ st_mean,
                                                  double *__restrict__ st_max, double *__restrict__ st_solved,
                                                  const int do_gae, const PairwisePlan P) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= B) return;
    const bool noclamp = (score_fn & AMZ_SCORE_NOCLAMP) != 0;
    const bool prior_final = (score_fn & AMZ_SCORE_PRIOR_FINAL) != 0;
    score_fn &= 0xFF;
    // ---- pass 1: completed-episode statistics (forward) ----
    const double g1 = disc ? gamma : 1.0;
    double acc = 0.0, dsc = 1.0, tot = 0.0, best = 0.0;
    int64_t cnt = 0, hits = 0;
    for (int t0 = 0; t0 < (prior_final ? 0 : T); t0 += 8) {
        double xr[8];
        uint8_t xd[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int t = t0 + j;
            xr[j] = t < T ? rw[(int64_t)t * B + l] : 0.0;
            xd[j] = t < T ? dn[(int64_t)t * B + l] : 0;
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
            if (t0 + j < T) {
                acc = acc + dsc * xr[j];
                dsc = dsc * g1;
                if (xd[j]) {
                    cnt++;
                    tot = tot + acc;
                    best = np_max(best, acc);
                    hits += acc > 0.0;
                    acc = 0.0;
                }
            }
        }
    }
    const double mx = prior_final ? prior[l] : np_max(prior ? prior[l] : 0.0, best);
    if (maxret) maxret[l] = mx;
    if (st_eps) st_eps[l] = cnt;
    if (st_mean) st_mean[l] = cnt > 0 ? tot / (double)cnt : 0.0;
    if (st_max) st_max[l] = best;
    if (st_solved) st_solved[l] = cnt > 0 ? (double)hits / (double)cnt : 0.0;

    // ---- pass 2: GAE (reverse) ----
    double nxt = do_gae ? last[l] : 0.0, run = 0.0;
    for (int t1 = do_gae ? T : 0; t1 > 0; t1 -= 8) {
        double xr[8], xv[8];
        uint8_t xd[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int t = t1 - 1 - j;
            xr[j] = t >= 0 ? rw[(int64_t)t * B + l] : 0.0;
            xv[j] = t >= 0 ? val[(int64_t)t * B + l] : 0.0;
            xd[j] = t >= 0 ? dn[(int64_t)t * B + l] : 0;
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int t = t1 - 1 - j;
            if (t >= 0) {
                const double keep = 1.0 - (xd[j] ? 1.0 : 0.0);
                const double delta = (xr[j] + (gamma * keep) * nxt) - xv[j];
                run = delta + (gl * keep) * run;
                adv[(int64_t)t * B + l] = run;
                ret[(int64_t)t * B + l] = run + xv[j];
                nxt = xv[j];
            }
        }
    }

    // ---- pass 3: mean over the lane's slice in pairwise order (forward) ----
    if (scores) {
        PairwiseSum S;
        S.begin(P);
        const double *src = score_fn == AMZ_SCORE_PVL ? adv : val;
        for (int t0 = 0; t0 < T; t0 += 8) {
            double x[8];
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int t = t0 + j;
                x[j] = t < T ? src[(int64_t)t * B + l] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int t = t0 + j;
                if (t < T) {
                    const double e = score_fn == AMZ_SCORE_PVL ? np_max(x[j], 0.0) : mx - x[j];
                    S.add(e, t, j, P);
                }
            }
        }
        const double sc = S.total() / (double)T;
        scores[l] = noclamp ? sc : np_max(sc, 0.0);
    }
}

// Two warps per 32 lanes: warp 0 runs pass 1 (forward statistics) while warp 1 runs
// pass 2 (reverse GAE) -- the passes are independent -- then the pairwise leaves of
// pass 3 are split between the two warps and warp 0 combines them in numpy's order.
// This halves the per-lane sequential chain, which is what bounds small batches.
__device__ __forceinline__ double leaf_sum(const double *__restrict__ src, int64_t B, int64_t l, int s, int len,
                                           int fn, double mx) {
    auto elem = [&](int t) {
        const double x = src[(int64_t)t * B + l];
        return fn == AMZ_SCORE_PVL ? np_max(x, 0.0) : mx - x;
    };
    if (len < 8) {
        double res = 0.0;
        for (int k = 0; k < len; k++) res = res + elem(s + k);
        return res;
    }
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; k++) r[k] = elem(s + k);
    const int l8 = len - len % 8;
    for (int k = 8; k < l8; k += 8) {
        double x[8];
#pragma unroll
        for (int j = 0; j < 8; j++) x[j] = elem(s + k + j);
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = r[j] + x[j];
    }
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (int k = l8; k < len; k++) res = res + elem(s + k);
    return res;
}

__global__ void __launch_bounds__(64) k_gae_score2(int T, int64_t B, const double *__restrict__ rw,
                                                   const double *__restrict__ val, const uint8_t *__restrict__ dn,
                                                   const double *__restrict__ last, double gamma, double gl,
                                                   const double *__restrict__ prior, int score_fn, int disc,
                                                   double *adv, double *__restrict__ ret,
                                                   double *__restrict__ scores, double *__restrict__ maxret,
                                                   int64_t *__restrict__ st_eps, double *__restrict__ st_mean,
                                                   double *__restrict__ st_max, double *__restrict__ st_solved,
                                                   const int do_gae, const PairwisePlan P) {
    __shared__ double s_mx[32];
    __shared__ double s_leaf[kMaxLeaves][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t l = (int64_t)blockIdx.x * 32 + lane;
    const bool live = l < B;
    const bool noclamp = (score_fn & AMZ_SCORE_NOCLAMP) != 0;
    const bool prior_final = (score_fn & AMZ_SCORE_PRIOR_FINAL) != 0;
    const int fn = score_fn & 0xFF;
    if (warp == 0 && live) {
        // ---- pass 1: completed-episode statistics (forward) ----
        const double g1 = disc ? gamma : 1.0;
        double acc = 0.0, dsc = 1.0, tot = 0.0, best = 0.0;
        int64_t cnt = 0, hits = 0;
        for (int t0 = 0; t0 < (prior_final ? 0 : T); t0 += 8) {
            double xr[8];
            uint8_t xd[8];
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int t = t0 + j;
                xr[j] = t < T ? rw[(int64_t)t * B + l] : 0.0;
                xd[j] = t < T ? dn[(int64_t)t * B + l] : 0;
            }
#pragma unroll
            for (int j = 0; j < 8; j++) {
                if (t0 + j < T) {
                    acc = acc + dsc * xr[j];
                    dsc = dsc * g1;
                    if (xd[j]) {
                        cnt++;
                        tot = tot + acc;
                        best = np_max(best, acc);
                        hits += acc > 0.0;
                        acc = 0.0;
                    }
                }
            }
        }
        const double mx = prior_final ? prior[l] : np_max(prior ? prior[l] : 0.0, best);
        s_mx[lane] = mx;
        if (maxret) maxret[l] = mx;
        if (st_eps) st_eps[l] = cnt;
        if (st_mean) st_mean[l] = cnt > 0 ? tot / (double)cnt : 0.0;
        if (st_max) st_max[l] = best;
        if (st_solved) st_solved[l] = cnt > 0 ? (double)hits / (double)cnt : 0.0;
    }
    if (warp == 1 && live && do_gae) {
        // ---- pass 2: GAE (reverse) ----
        double nxt = last[l], run = 0.0;
        for (int t1 = T; t1 > 0; t1 -= 8) {
            double xr[8], xv[8];
            uint8_t xd[8];
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int t = t1 - 1 - j;
                xr[j] = t >= 0 ? rw[(int64_t)t * B + l] : 0.0;
                xv[j] = t >= 0 ? val[(int64_t)t * B + l] : 0.0;
                xd[j] = t >= 0 ? dn[(int64_t)t * B + l] : 0;
            }
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int t = t1 - 1 - j;
                if (t >= 0) {
                    const double keep = 1.0 - (xd[j] ? 1.0 : 0.0);
                    const double delta = (xr[j] + (gamma * keep) * nxt) - xv[j];
                    run = delta + (gl * keep) * run;
                    adv[(int64_t)t * B + l] = run;
                    ret[(int64_t)t * B + l] = run + xv[j];
                    nxt = xv[j];
                }
            }
        }
        __threadfence_block();  // PVL's pass 3 reads these advantages in the other warp
    }
    if (!scores) return;
    __syncthreads();
    // ---- pass 3: pairwise leaves split across the two warps ----
    const double *src = fn == AMZ_SCORE_PVL ? adv : val;
    const double mx = s_mx[lane];
    if (live) {
        int start = 0;
        for (int li = 0; li < P.n_leaves; li++) {
            const int end = P.leaf_end[li];
            if ((li & 1) == warp) s_leaf[li][lane] = leaf_sum(src, B, l, start, end - start, fn, mx);
            start = end;
        }
    }
    __syncthreads();
    if (warp == 0 && live) {
        double stk[16];
        int sp = 0;
        for (int li = 0; li < P.n_leaves; li++) {
            stk[sp++] = s_leaf[li][lane];
            for (int k = 0; k < P.adds[li]; k++) {
                const double b = stk[--sp];
                const double a = stk[--sp];
                stk[sp++] = a + b;
            }
        }
        const double sc = stk[0] / (double)T;
        scores[l] = noclamp ? sc : np_max(sc, 0.0);
    }
}

int launch_gae_score(int T, int64_t B, const double *r, const double *v, const uint8_t *d, const double *last,
                     double gamma, double lam, const double *prior, int score_fn, int disc, double *adv,
                     double *ret, double *scores, double *maxret, const amz_episode_stats_t *stats,
                     cudaStream_t s, int do_gae) {
    if (B <= 0 || T <= 0) return 0;
    PairwisePlan P;
    if (make_pairwise_plan(T, P)) return AMZ_ECONFIG;
    const double gl = gamma * lam;  // Python evaluates gamma * lam first (agents/gae.py:35)
    if (B <= 148 * 32 * 8) {
        k_gae_score2<<<(unsigned)((B + 31) / 32), 64, 0, s>>>(
            T, B, r, v, d, last, gamma, gl, prior, score_fn, disc, adv, ret, scores, maxret,
            stats ? stats->episodes : nullptr, stats ? stats->mean_return : nullptr,
            stats ? stats->max_return : nullptr, stats ? stats->solved_rate : nullptr, do_gae, P);
        return 0;
    }
    const int threads = B >= 148 * 64 ? 64 : 32;
    k_gae_score<<<(unsigned)((B + threads - 1) / threads), threads, 0, s>>>(
        T, B, r, v, d, last, gamma, gl, prior, score_fn, disc, adv, ret, scores, maxret,
        stats ? stats->episodes : nullptr, stats ? stats->mean_return : nullptr,
        stats ? stats->max_return : nullptr, stats ? stats->solved_rate : nullptr, do_gae, P);
    return 0;
}

}  // namespace amz
