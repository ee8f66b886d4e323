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

// ---------------------------------------------------------------------------------
// k_gae_score3: the same three passes for 16 lanes per CTA, with the [T][16] columns
// streamed through an 8-stage cp.async ring (8 steps per stage) so that every warp has
// ~64 steps of loads in flight instead of one dependent DRAM round trip per 8 steps.
// Pass 2 keeps the pass-3 source column (advantages for PVL, values for MaxMC) in
// shared memory, so pass 3 reads no global memory.  Needs B % 16 == 0 (16-B aligned
// rows of the done bytes) and T <= kG3MaxT; launch_gae_score falls back otherwise.
// ---------------------------------------------------------------------------------
constexpr int kG3LW = 16;     // lanes per CTA
constexpr int kG3GS = 8;      // steps per stage
constexpr int kG3NS = 8;      // stages in flight
constexpr int kG3MaxT = 256;  // pass-3 column kept in shared memory
struct G3Stage {
    double r[kG3GS][kG3LW];
    double v[kG3GS][kG3LW];
    uint8_t d[kG3GS][kG3LW];
};
struct G3Smem {
    G3Stage ring[2][kG3NS];
    double src[kG3MaxT][kG3LW];
    double leaf[kMaxLeaves][kG3LW];
    double mx[kG3LW];
};

__device__ __forceinline__ void g3_cp16(void *sdst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(sdst)),
                 "l"(gsrc)
                 : "memory");
}

__global__ void __launch_bounds__(64) k_gae_score3(int T, int64_t B, const double *__restrict__ rw,
                                                   const double *__restrict__ val, const uint8_t *__restrict__ dn,
                                                   const double *__restrict__ last, double gamma, double gl,
                                                   const double *__restrict__ prior, int score_fn, int disc,
                                                   double *__restrict__ adv, double *__restrict__ ret,
                                                   double *__restrict__ scores, double *__restrict__ maxret,
                                                   int64_t *__restrict__ st_eps, double *__restrict__ st_mean,
                                                   double *__restrict__ st_max, double *__restrict__ st_solved,
                                                   const PairwisePlan P) {
    extern __shared__ __align__(16) uint8_t g3raw[];
    G3Smem &S = *reinterpret_cast<G3Smem *>(g3raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t l0 = (int64_t)blockIdx.x * kG3LW;
    const int64_t l = l0 + lane;
    const bool noclamp = (score_fn & AMZ_SCORE_NOCLAMP) != 0;
    const bool prior_final = (score_fn & AMZ_SCORE_PRIOR_FINAL) != 0;
    const int fn = score_fn & 0xFF;
    const bool pvl = fn == AMZ_SCORE_PVL;
    // warp 0: forward (rewards, dones); warp 1: reverse (rewards, values, dones)
    const bool rev = warp == 1;
    const int nst = (warp == 0 && prior_final) ? 0 : (T + kG3GS - 1) / kG3GS;
    G3Stage *ring = S.ring[warp];
    // stage copy plan (fixed per thread): rewards and values rows j = lane>>3 and
    // j+4, 16-B chunk q = lane&7; done rows j = lane (lanes 0..7)
    const int cq = lane & 7, cj = lane >> 3;
    auto issue = [&](int st) {
        if (st < nst) {
            G3Stage &G = ring[st % kG3NS];
            const int k0 = st * kG3GS;
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int j = cj + 4 * h, k = k0 + j;
                if (k < T) {
                    const int64_t row = (int64_t)(rev ? T - 1 - k : k) * B + l0;
                    g3_cp16(&G.r[j][2 * cq], rw + row + 2 * cq);
                    if (rev) g3_cp16(&G.v[j][2 * cq], val + row + 2 * cq);
                }
            }
            if (lane < kG3GS && k0 + lane < T)
                g3_cp16(&G.d[lane][0], dn + (int64_t)(rev ? T - 1 - (k0 + lane) : k0 + lane) * B + l0);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
#pragma unroll 1
    for (int st = 0; st < kG3NS - 1; st++) issue(st);

    const bool act = lane < kG3LW;
    const bool keep_src = pvl;  // MaxMC's source (values) is staged by this warp too
    // pass 1 state
    const double g1 = disc ? gamma : 1.0;
    double acc = 0.0, dsc = 1.0, tot = 0.0, best = 0.0;
    int cnt = 0, hits = 0;
    // pass 2 state
    double nxt = (rev && act) ? last[l] : 0.0, run = 0.0;
    const double g0 = gamma * 0.0, gl0 = gl * 0.0;  // x * keep for keep = 0.0, sign included
    int64_t off = (int64_t)(T - 1) * B + l;         // reverse walk over [t][B]
    // per_lane_episode_stats step: the episode bookkeeping only runs on a done
    auto fwd_step = [&](double r, bool dd) {
        acc = acc + dsc * r;
        dsc = dsc * g1;
        if (dd) {
            cnt++;
            tot = tot + acc;
            best = np_max(best, acc);
            hits += acc > 0.0;
            acc = 0.0;
        }
    };
    auto rev_step = [&](double r, double xv, bool dd, int t) {
        // gamma * keep and (gamma * lam) * keep with keep in {0.0, 1.0}
        const double gk = dd ? g0 : gamma, glk = dd ? gl0 : gl;
        const double delta = (r + gk * nxt) - xv;
        run = delta + glk * run;
        adv[off] = run;
        ret[off] = run + xv;
        off -= B;
        nxt = xv;
        S.src[t][lane] = keep_src ? run : xv;
    };
#pragma unroll 1
    for (int st = 0; st < nst; st++) {
        issue(st + kG3NS - 1);
        asm volatile("cp.async.wait_group %0;\n" ::"n"(kG3NS - 1) : "memory");
        __syncwarp();
        const G3Stage &G = ring[st % kG3NS];
        const int jn = (T - st * kG3GS) < kG3GS ? (T - st * kG3GS) : kG3GS;
        if (act) {
            if (!rev) {
                if (jn == kG3GS) {
#pragma unroll
                    for (int j = 0; j < kG3GS; j++) fwd_step(G.r[j][lane], G.d[j][lane] != 0);
                } else {
                    for (int j = 0; j < jn; j++) fwd_step(G.r[j][lane], G.d[j][lane] != 0);
                }
            } else {
                const int tb = T - 1 - st * kG3GS;
                if (jn == kG3GS) {
#pragma unroll
                    for (int j = 0; j < kG3GS; j++) rev_step(G.r[j][lane], G.v[j][lane], G.d[j][lane] != 0, tb - j);
                } else {
                    for (int j = 0; j < jn; j++) rev_step(G.r[j][lane], G.v[j][lane], G.d[j][lane] != 0, tb - j);
                }
            }
        }
        __syncwarp();
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    if (!rev && act) {
        const double mx = prior_final ? prior[l] : np_max(prior ? prior[l] : 0.0, best);
        S.mx[lane] = mx;
        if (maxret) maxret[l] = mx;
        if (st_eps) st_eps[l] = (int64_t)cnt;
        if (st_mean) st_mean[l] = cnt > 0 ? tot / (double)cnt : 0.0;
        if (st_max) st_max[l] = best;
        if (st_solved) st_solved[l] = cnt > 0 ? (double)hits / (double)cnt : 0.0;
    }
    if (!scores) return;
    __syncthreads();
    // ---- pass 3 from shared memory: leaves split between the warps ----
    if (act) {
        const double mx = S.mx[lane];
        auto elem = [&](int t) {
            const double x = S.src[t][lane];
            return pvl ? np_max(x, 0.0) : mx - x;
        };
        int start = 0;
        for (int li = 0; li < P.n_leaves; li++) {
            const int end = P.leaf_end[li];
            if ((li & 1) == warp) {
                const int len = end - start;
                double res = 0.0;
                if (len < 8) {
                    for (int k = 0; k < len; k++) res = res + elem(start + k);
                } else {
                    double r[8];
#pragma unroll
                    for (int k = 0; k < 8; k++) r[k] = elem(start + k);
                    const int l8 = len - len % 8;
                    for (int k = 8; k < l8; k += 8) {
#pragma unroll
                        for (int j = 0; j < 8; j++) r[j] = r[j] + elem(start + k + j);
                    }
                    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
                    for (int k = l8; k < len; k++) res = res + elem(start + k);
                }
                S.leaf[li][lane] = res;
            }
            start = end;
        }
    }
    __syncthreads();
    if (warp == 0 && act) {
        double stk[16];
        int sp = 0;
        for (int li = 0; li < P.n_leaves; li++) {
            stk[sp++] = S.leaf[li][lane];
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
    const bool g3 = do_gae && T <= kG3MaxT && B % kG3LW == 0 && B % 16 == 0 && ((uintptr_t)r & 15u) == 0 &&
                    ((uintptr_t)v & 15u) == 0 && ((uintptr_t)d & 15u) == 0;
    if (g3) {
        const size_t sm = sizeof(G3Smem);
        cudaFuncSetAttribute(k_gae_score3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_gae_score3<<<(unsigned)(B / kG3LW), 64, sm, s>>>(
            T, B, r, v, d, last, gamma, gl, prior, score_fn, disc, adv, ret, scores, maxret,
            stats ? stats->episodes : nullptr, stats ? stats->mean_return : nullptr,
            stats ? stats->max_return : nullptr, stats ? stats->solved_rate : nullptr, P);
        return 0;
    }
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
