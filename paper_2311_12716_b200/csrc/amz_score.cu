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
#include <stdlib.h>

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

template <typename VT>
__global__ void __launch_bounds__(64) k_gae_score(int T, int64_t B, const double *__restrict__ rw,
                                                  const VT *__restrict__ val, const uint8_t *__restrict__ dn,
                                                  const VT *__restrict__ last, double gamma, double gl,
                                                  const double *__restrict__ prior, int score_fn, int disc,
                                                  double *__restrict__ adv, double *__restrict__ ret,
                                                  double *__restrict__ scores, double *__restrict__ maxret,
                                                  int64_t *__restrict__ st_eps, double *__restrict__ st_mean,
                                                  double *__restrict__ st_max, double *__restrict__ st_solved,
                                                  const int do_gae, const PairwisePlan P) {
    pdl_wait();  // rewards / dones from the rollout (launch_pdl)
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
    double nxt = do_gae ? (double)last[l] : 0.0, run = 0.0;
    for (int t1 = do_gae ? T : 0; t1 > 0; t1 -= 8) {
        double xr[8], xv[8];
        uint8_t xd[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int t = t1 - 1 - j;
            xr[j] = t >= 0 ? rw[(int64_t)t * B + l] : 0.0;
            xv[j] = t >= 0 ? (double)val[(int64_t)t * B + l] : 0.0;
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
        const bool pv = score_fn == AMZ_SCORE_PVL;
        for (int t0 = 0; t0 < T; t0 += 8) {
            double x[8];
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int t = t0 + j;
                x[j] = t < T ? (pv ? adv[(int64_t)t * B + l] : (double)val[(int64_t)t * B + l]) : 0.0;
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
template <typename ST>
__device__ __forceinline__ double leaf_sum(const ST *__restrict__ src, int64_t B, int64_t l, int s, int len,
                                           int fn, double mx) {
    auto elem = [&](int t) {
        const double x = (double)src[(int64_t)t * B + l];
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

template <typename VT>
__global__ void __launch_bounds__(64) k_gae_score2(int T, int64_t B, const double *__restrict__ rw,
                                                   const VT *__restrict__ val, const uint8_t *__restrict__ dn,
                                                   const VT *__restrict__ last, double gamma, double gl,
                                                   const double *__restrict__ prior, int score_fn, int disc,
                                                   double *adv, double *__restrict__ ret,
                                                   double *__restrict__ scores, double *__restrict__ maxret,
                                                   int64_t *__restrict__ st_eps, double *__restrict__ st_mean,
                                                   double *__restrict__ st_max, double *__restrict__ st_solved,
                                                   const int do_gae, const PairwisePlan P) {
    __shared__ double s_mx[32];
    __shared__ double s_leaf[kMaxLeaves][32];
    pdl_wait();
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
        double nxt = (double)last[l], run = 0.0;
        for (int t1 = T; t1 > 0; t1 -= 8) {
            double xr[8], xv[8];
            uint8_t xd[8];
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int t = t1 - 1 - j;
                xr[j] = t >= 0 ? rw[(int64_t)t * B + l] : 0.0;
                xv[j] = t >= 0 ? (double)val[(int64_t)t * B + l] : 0.0;
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
    const double mx = s_mx[lane];
    if (live) {
        int start = 0;
        for (int li = 0; li < P.n_leaves; li++) {
            const int end = P.leaf_end[li];
            if ((li & 1) == warp)
                s_leaf[li][lane] = fn == AMZ_SCORE_PVL ? leaf_sum(adv, B, l, start, end - start, fn, mx)
                                                       : leaf_sum(val, B, l, start, end - start, fn, mx);
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

__device__ __forceinline__ void g3_cp16(void *sdst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(sdst)),
                 "l"(gsrc)
                 : "memory");
}

// ---------------------------------------------------------------------------------
// k_gae_score4: 16 lanes per CTA, 4 warps, whole columns in shared memory (T <= 256).
//   load   all 128 threads stream the CTA's [T][16] rewards / values / dones into shared
//          memory with cp.async (bandwidth-bound: every warp keeps ~35 16-B copies in
//          flight);
//   prep   warps 1-3 compute the data-parallel part of the GAE recurrence,
//          delta_t = (r_t + (gamma*keep_t) * V_{t+1}) - V_t, while warp 0 runs
//          per_lane_episode_stats forward over (r, done);
//   scan   warp 1 runs the reverse recurrence A_t = delta_t + ((gamma*lam)*keep_t) * A_{t+1}
//          alone: two dependent float64 ops per step;
//   out    all threads store A and R = A + V and sum the pass-3 leaves from shared memory.
// Same float64 operations in the same order as the reference (bit-exact).
// ---------------------------------------------------------------------------------
constexpr int kG4MaxT = 256;
template <int kG4LW, typename VT>
struct G4Smem {
    double r[kG4MaxT][kG4LW];    // rewards
    VT v[kG4MaxT][kG4LW];        // values (f64, or the policy's f32)
    double a[kG4MaxT][kG4LW];    // delta, then advantages (in place)
    uint8_t d[kG4MaxT][kG4LW];   // dones
    double leaf[kMaxLeaves][kG4LW];
    double mx[kG4LW];
};

__device__ __forceinline__ void g4_cp8(void *sdst, const void *gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((uint32_t)__cvta_generic_to_shared(sdst)),
                 "l"(gsrc)
                 : "memory");
}

template <int kG4LW, typename VT>
__global__ void __launch_bounds__(128) k_gae_score4(int T, int64_t B, const double *__restrict__ rw,
                                                    const VT *__restrict__ val, const uint8_t *__restrict__ dn,
                                                    const VT *__restrict__ last, double gamma, double gl,
                                                    const double *__restrict__ prior, int score_fn, int disc,
                                                    double *__restrict__ adv, double *__restrict__ ret,
                                                    double *__restrict__ scores, double *__restrict__ maxret,
                                                    int64_t *__restrict__ st_eps, double *__restrict__ st_mean,
                                                    double *__restrict__ st_max, double *__restrict__ st_solved,
                                                    const PairwisePlan P) {
    extern __shared__ __align__(16) uint8_t g4raw[];
    G4Smem<kG4LW, VT> &S = *reinterpret_cast<G4Smem<kG4LW, VT> *>(g4raw);
    pdl_wait();
    constexpr int CR = kG4LW / 2;                            // 16-B chunks per row of r
    constexpr int CV = kG4LW * (int)sizeof(VT) / 16;         // ... and of v
    constexpr int EV = 16 / (int)sizeof(VT);                 // values per chunk
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t l0 = (int64_t)blockIdx.x * kG4LW;
    const bool noclamp = (score_fn & AMZ_SCORE_NOCLAMP) != 0;
    const bool prior_final = (score_fn & AMZ_SCORE_PRIOR_FINAL) != 0;
    const int fn = score_fn & 0xFF;
    const bool pvl = fn == AMZ_SCORE_PVL;
    // ---- load: CR + CV 16-B chunks of r and v per row, one chunk of dones ----
    for (int x = tid; x < T * (CR + CV + 1); x += 128) {
        const int t = x / (CR + CV + 1), q = x - t * (CR + CV + 1);
        const int64_t row = (int64_t)t * B + l0;
        if (q < CR)
            g3_cp16(&S.r[t][2 * q], rw + row + 2 * q);
        else if (q < CR + CV)
            g3_cp16(&S.v[t][EV * (q - CR)], val + row + EV * (q - CR));
        else if (kG4LW == 16)
            g3_cp16(&S.d[t][0], dn + row);
        else
            g4_cp8(&S.d[t][0], dn + row);
    }
    asm volatile("cp.async.commit_group;\n" "cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    // ---- pass 1 (warp 0): per_lane_episode_stats forward, beside prep and the scan ----
    if (warp == 0 && lane < kG4LW) {
        const int64_t l = l0 + lane;
        const double g1 = disc ? gamma : 1.0;
        double acc = 0.0, dsc = 1.0, tot = 0.0, best = 0.0;
        int cnt = 0, hits = 0;
        for (int t = 0; t < (prior_final ? 0 : T); t++) {
            acc = acc + dsc * S.r[t][lane];
            dsc = dsc * g1;
            if (S.d[t][lane]) {
                cnt++;
                tot = tot + acc;
                best = np_max(best, acc);
                hits += acc > 0.0;
                acc = 0.0;
            }
        }
        const double mx = prior_final ? prior[l] : np_max(prior ? prior[l] : 0.0, best);
        S.mx[lane] = mx;
        if (maxret) maxret[l] = mx;
        if (st_eps) st_eps[l] = (int64_t)cnt;
        if (st_mean) st_mean[l] = cnt > 0 ? tot / (double)cnt : 0.0;
        if (st_max) st_max[l] = best;
        if (st_solved) st_solved[l] = cnt > 0 ? (double)hits / (double)cnt : 0.0;
    } else if (warp >= 1) {
        // ---- prep (warps 1-3): delta_t ----
        const double g0 = gamma * 0.0;
        for (int x = tid - 32; x < T * kG4LW; x += 96) {
            const int t = x / kG4LW, c = x - t * kG4LW;
            const double nxt = t + 1 < T ? (double)S.v[t + 1][c] : (double)last[l0 + c];
            const double gk = S.d[t][c] ? g0 : gamma;
            S.a[t][c] = (S.r[t][c] + gk * nxt) - (double)S.v[t][c];
        }
        // warps 1-3 only: pass 1 keeps running in warp 0 meanwhile
        asm volatile("bar.sync 1, 96;\n" ::: "memory");
        // ---- pass 2 (warp 1): the reverse scan, A_t over delta_t in shared memory.  The
        // operands of step t - 2 are loaded before step t's store (volatile asm keeps that
        // order; plain code would wait for each load behind the previous store) ----
        if (warp == 1 && lane < kG4LW) {
            const double gl0 = gl * 0.0;
            double run = 0.0;
            auto ld = [&](int t, double &x, uint32_t &dd) {
                asm volatile("ld.shared.f64 %0, [%1];"
                             : "=d"(x)
                             : "r"((uint32_t)__cvta_generic_to_shared(&S.a[t][lane])));
                asm volatile("ld.shared.u8 %0, [%1];"
                             : "=r"(dd)
                             : "r"((uint32_t)__cvta_generic_to_shared(&S.d[t][lane])));
            };
            double x0 = 0.0, x1 = 0.0;
            uint32_t d0 = 0u, d1 = 0u;
            ld(T - 1, x0, d0);
            if (T >= 2) ld(T - 2, x1, d1);
            for (int t = T - 1; t >= 0; t--) {
                double x2 = 0.0;
                uint32_t d2 = 0u;
                if (t >= 2) ld(t - 2, x2, d2);
                run = x0 + (d0 ? gl0 : gl) * run;  // A_t = delta_t + glk * A_{t+1}
                asm volatile("st.shared.f64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&S.a[t][lane])),
                             "d"(run)
                             : "memory");
                x0 = x1;
                d0 = d1;
                x1 = x2;
                d1 = d2;
            }
        }
    }
    __syncthreads();
    // A and R = A + V written out by the whole CTA (row segments of kG4LW doubles)
    for (int x = tid; x < T * kG4LW; x += 128) {
        const int t = x / kG4LW, c = x - t * kG4LW;
        const double a = S.a[t][c];
        const int64_t o = (int64_t)t * B + l0 + c;
        adv[o] = a;
        ret[o] = a + (double)S.v[t][c];
    }
    if (!scores) return;
    // ---- pass 3: pairwise leaves from shared memory, 8 lanes x leaves over the warps ----
    for (int x = tid; x < P.n_leaves * kG4LW; x += 128) {
        const int li = x / kG4LW, c = x - li * kG4LW;
        const int start = li == 0 ? 0 : P.leaf_end[li - 1], end = P.leaf_end[li];
        const double mx = S.mx[c];
        auto elem = [&](int t) { return pvl ? np_max(S.a[t][c], 0.0) : mx - (double)S.v[t][c]; };
        const int len = end - start;
        double res = 0.0;
        if (len < 8) {
            for (int k = 0; k < len; k++) res = res + elem(start + k);
        } else {
            double rr[8];
#pragma unroll
            for (int k = 0; k < 8; k++) rr[k] = elem(start + k);
            const int l8 = len - len % 8;
            for (int k = 8; k < l8; k += 8) {
#pragma unroll
                for (int j = 0; j < 8; j++) rr[j] = rr[j] + elem(start + k + j);
            }
            res = ((rr[0] + rr[1]) + (rr[2] + rr[3])) + ((rr[4] + rr[5]) + (rr[6] + rr[7]));
            for (int k = l8; k < len; k++) res = res + elem(start + k);
        }
        S.leaf[li][c] = res;
    }
    __syncthreads();
    if (tid < kG4LW) {
        double stk[16];
        int sp = 0;
        for (int li = 0; li < P.n_leaves; li++) {
            stk[sp++] = S.leaf[li][tid];
            for (int k = 0; k < P.adds[li]; k++) {
                const double b = stk[--sp];
                const double a = stk[--sp];
                stk[sp++] = a + b;
            }
        }
        const double sc = stk[0] / (double)T;
        scores[l0 + tid] = noclamp ? sc : np_max(sc, 0.0);
    }
}

// ---------------------------------------------------------------------------------
// k_gae_score7: whole 16-lane columns in shared memory (r, V f64, done u8: 68 KB, so 3
// CTAs per SM), persistent over the 16-lane groups.  Per group:
//   load   all 128 threads cp.async the [T][16] columns (16-B copies, 17 per row);
//   warp 0 pass 1 forward over (r, done) in shared memory;
//   warp 1 pass 2 reverse, delta_t computed inline (its shared loads do not depend on
//          the chain, so they issue ahead of it), A_t and R_t = A_t + V_t stored
//          straight to global (128-B row segments); for PVL, A_{t+1} replaces V_{t+1}
//          in shared memory once step t has consumed it;
//   all    pass 3 leaves from shared memory.
// The three CTAs of an SM overlap one another's load, chain and store phases.
// ---------------------------------------------------------------------------------
constexpr int kG7MaxT = 256, kG7LW = 16;
// kA: PVL's advantages get their own column (f32 values cannot hold them); with f64
// values they replace V in place
template <typename VT, bool kA>
struct G7Smem {
    double r[kG7MaxT][kG7LW];
    VT v[kG7MaxT][kG7LW];
    double a[kA ? kG7MaxT : 1][kG7LW];
    uint8_t d[kG7MaxT][kG7LW];
    double leaf[4][kG7LW];
    double mx[kG7LW];
};

template <typename VT, bool kA>
__global__ void __launch_bounds__(128) k_gae_score7(int T, int64_t B, const double *__restrict__ rw,
                                                    const VT *__restrict__ val, const uint8_t *__restrict__ dn,
                                                    const VT *__restrict__ last, double gamma, double gl,
                                                    const double *__restrict__ prior, int score_fn, int disc,
                                                    double *__restrict__ adv, double *__restrict__ ret,
                                                    double *__restrict__ scores, double *__restrict__ maxret,
                                                    int64_t *__restrict__ st_eps, double *__restrict__ st_mean,
                                                    double *__restrict__ st_max, double *__restrict__ st_solved,
                                                    const PairwisePlan P) {
    extern __shared__ __align__(16) uint8_t g7raw[];
    G7Smem<VT, kA> &S = *reinterpret_cast<G7Smem<VT, kA> *>(g7raw);
    pdl_wait();
    constexpr int CR = kG7LW / 2;                     // 16-B chunks per row of r
    constexpr int CV = kG7LW * (int)sizeof(VT) / 16;  // ... and of v
    constexpr int EV = 16 / (int)sizeof(VT);          // values per chunk
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool noclamp = (score_fn & AMZ_SCORE_NOCLAMP) != 0;
    const bool prior_final = (score_fn & AMZ_SCORE_PRIOR_FINAL) != 0;
    const int fn = score_fn & 0xFF;
    const bool pvl = fn == AMZ_SCORE_PVL;
    const int64_t ngroups = B / kG7LW;
    for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const int64_t l0 = g * kG7LW;
        for (int x = tid; x < T * (CR + CV + 1); x += 128) {
            const int t = x / (CR + CV + 1), q = x - t * (CR + CV + 1);
            const int64_t row = (int64_t)t * B + l0;
            if (q < CR)
                g3_cp16(&S.r[t][2 * q], rw + row + 2 * q);
            else if (q < CR + CV)
                g3_cp16(&S.v[t][EV * (q - CR)], val + row + EV * (q - CR));
            else
                g3_cp16(&S.d[t][0], dn + row);
        }
        asm volatile("cp.async.commit_group;\n" "cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        if (warp == 0 && lane < kG7LW) {
            // ---- pass 1: per_lane_episode_stats (forward) ----
            const int64_t l = l0 + lane;
            const double g1 = disc ? gamma : 1.0;
            double acc = 0.0, dsc = 1.0, tot = 0.0, best = 0.0;
            int cnt = 0, hits = 0;
            const int T1 = prior_final ? 0 : T;
            for (int t = 0; t < T1; t++) {
                acc = acc + dsc * S.r[t][lane];
                dsc = dsc * g1;
                if (S.d[t][lane]) {
                    cnt++;
                    tot = tot + acc;
                    best = np_max(best, acc);
                    hits += acc > 0.0;
                    acc = 0.0;
                }
            }
            const double mx = prior_final ? prior[l] : np_max(prior ? prior[l] : 0.0, best);
            S.mx[lane] = mx;
            if (maxret) maxret[l] = mx;
            if (st_eps) st_eps[l] = (int64_t)cnt;
            if (st_mean) st_mean[l] = cnt > 0 ? tot / (double)cnt : 0.0;
            if (st_max) st_max[l] = best;
            if (st_solved) st_solved[l] = cnt > 0 ? (double)hits / (double)cnt : 0.0;
        } else if (warp == 1 && lane < kG7LW) {
            // ---- pass 2: GAE (reverse), delta inline ----
            const int64_t l = l0 + lane;
            const double g0 = gamma * 0.0, gl0 = gl * 0.0;
            double nxt = (double)last[l], run = 0.0;
            double *pa = adv + (int64_t)(T - 1) * B + l, *pr = ret + (int64_t)(T - 1) * B + l;
            int t = T - 1;
            for (; t >= 7; t -= 8) {
                double xr[8], xv[8];
                uint32_t xd[8];
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    xr[j] = S.r[t - j][lane];
                    xv[j] = (double)S.v[t - j][lane];
                    xd[j] = S.d[t - j][lane];
                }
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const double delta = (xr[j] + (xd[j] ? g0 : gamma) * nxt) - xv[j];
                    run = delta + (xd[j] ? gl0 : gl) * run;
                    *pa = run;
                    *pr = run + xv[j];
                    pa -= B;
                    pr -= B;
                    if (kA)
                        S.a[t - j][lane] = run;
                    else if (pvl)
                        S.v[t - j][lane] = (VT)run;  // (f64 values) V_t is dead once delta_t is formed
                    nxt = xv[j];
                }
            }
            for (; t >= 0; t--) {
                const double xr = S.r[t][lane], xv = (double)S.v[t][lane];
                const uint32_t xd = S.d[t][lane];
                const double delta = (xr + (xd ? g0 : gamma) * nxt) - xv;
                run = delta + (xd ? gl0 : gl) * run;
                *pa = run;
                *pr = run + xv;
                pa -= B;
                pr -= B;
                if (kA)
                    S.a[t][lane] = run;
                else if (pvl)
                    S.v[t][lane] = (VT)run;
                nxt = xv;
            }
        }
        __syncthreads();
        if (scores) {
            // ---- pass 3: one (leaf, lane) per thread from shared memory ----
            for (int x = tid; x < P.n_leaves * kG7LW; x += 128) {
                const int li = x / kG7LW, c = x - li * kG7LW;
                const int start = li == 0 ? 0 : P.leaf_end[li - 1], end = P.leaf_end[li];
                const double mx = S.mx[c];
                auto elem = [&](int t) {
                    return pvl ? np_max(kA ? S.a[t][c] : (double)S.v[t][c], 0.0) : mx - (double)S.v[t][c];
                };
                const int len = end - start;
                double res = 0.0;
                if (len < 8) {
                    for (int k = 0; k < len; k++) res = res + elem(start + k);
                } else {
                    double rr[8];
#pragma unroll
                    for (int k = 0; k < 8; k++) rr[k] = elem(start + k);
                    const int l8 = len - len % 8;
                    for (int k = 8; k < l8; k += 8) {
#pragma unroll
                        for (int j = 0; j < 8; j++) rr[j] = rr[j] + elem(start + k + j);
                    }
                    res = ((rr[0] + rr[1]) + (rr[2] + rr[3])) + ((rr[4] + rr[5]) + (rr[6] + rr[7]));
                    for (int k = l8; k < len; k++) res = res + elem(start + k);
                }
                S.leaf[li][c] = res;
            }
            __syncthreads();
            if (tid < kG7LW) {
                double stk[4];
                int sp = 0;
                for (int li = 0; li < P.n_leaves; li++) {
                    stk[sp++] = S.leaf[li][tid];
                    for (int k = 0; k < P.adds[li]; k++) {
                        const double b = stk[--sp];
                        const double a = stk[--sp];
                        stk[sp++] = a + b;
                    }
                }
                const double sc = stk[0] / (double)T;
                scores[l0 + tid] = noclamp ? sc : np_max(sc, 0.0);
            }
        }
        __syncthreads();  // the columns are reloaded for the next group
    }
}

template <typename VT>
static int launch_gae_score_t(int T, int64_t B, const double *r, const VT *v, const uint8_t *d, const VT *last,
                              double gamma, double lam, const double *prior, int score_fn, int disc, double *adv,
                              double *ret, double *scores, double *maxret, const amz_episode_stats_t *stats,
                              cudaStream_t s, int do_gae) {
    if (B <= 0 || T <= 0) return 0;
    PairwisePlan P;
    if (make_pairwise_plan(T, P)) return AMZ_ECONFIG;
    const double gl = gamma * lam;  // Python evaluates gamma * lam first (agents/gae.py:35)
    // measured on B200 (T = 256, tools/gae_large.py): the whole-column kernel k_gae_score4
    // wins up to ~12k lanes (latency), the persistent 16-lane-column kernel k_gae_score7
    // beyond (bit-identical outputs; 65536 lanes 0.213 -> 0.163 ms, 262144 0.638 -> 0.600);
    // the streaming kernels cover layouts those two cannot take (unaligned, B % 16 != 0,
    // T > 256, statistics-only calls)
    const bool aligned = ((uintptr_t)r & 15u) == 0 && ((uintptr_t)v & 15u) == 0 && ((uintptr_t)d & 15u) == 0;
    const bool g3 = do_gae && T <= kG4MaxT && B <= 12288 && B % 16 == 0 && aligned;
    const bool g7 = do_gae && T <= kG7MaxT && B % kG7LW == 0 && aligned;
    static const int lw = getenv("AMZ_GAE_LW") ? atoi(getenv("AMZ_GAE_LW")) : 8;
    static const int gsel = getenv("AMZ_GAE_KERNEL") ? atoi(getenv("AMZ_GAE_KERNEL")) : 0;  // tuning runs
    auto st = [&](int k) -> void * {
        if (!stats) return nullptr;
        return k == 0 ? (void *)stats->episodes
                      : k == 1 ? (void *)stats->mean_return : k == 2 ? (void *)stats->max_return : (void *)stats->solved_rate;
    };
    int64_t *s_eps = (int64_t *)st(0);
    double *s_mean = (double *)st(1), *s_max = (double *)st(2), *s_sol = (double *)st(3);
    if (gsel == 2) goto k2;
    if (gsel == 1) goto k1;
    if ((gsel == 4 || (gsel == 0 && g3)) && do_gae && T <= kG4MaxT && B % 16 == 0 && aligned) {
        if (lw == 16 || gsel == 4) {
            const size_t sm = sizeof(G4Smem<16, VT>);
            ensure_dyn_smem((const void *)k_gae_score4<16, VT>, (int)sm);
            launch_pdl(k_gae_score4<16, VT>, dim3((unsigned)(B / 16)), dim3(128), sm, s, T, B, r, v, d, last, gamma, gl,
                       prior, score_fn, disc, adv, ret, scores, maxret, s_eps, s_mean, s_max, s_sol, P);
            return 0;
        }
        const size_t sm = sizeof(G4Smem<8, VT>);
        ensure_dyn_smem((const void *)k_gae_score4<8, VT>, (int)sm);
        launch_pdl(k_gae_score4<8, VT>, dim3((unsigned)(B / 8)), dim3(128), sm, s, T, B, r, v, d, last, gamma, gl, prior,
                   score_fn, disc, adv, ret, scores, maxret, s_eps, s_mean, s_max, s_sol, P);
        return 0;
    }
    if (g7 && (gsel == 0 || gsel == 7)) {
        static const int m7 = getenv("AMZ_GAE_M") ? atoi(getenv("AMZ_GAE_M")) : 0;  // CTAs per SM (tuning)
        auto go = [&](auto kern, size_t sm) {
            ensure_dyn_smem((const void *)kern, (int)sm);
            int dev = 0, nsm = 148, occ = 1;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, sm);
            if (occ < 1) occ = 1;
            const int m = m7 > 0 && m7 < occ ? m7 : occ;
            const int64_t ng = B / kG7LW;
            const unsigned grid = (unsigned)(ng < (int64_t)nsm * m ? ng : (int64_t)nsm * m);
            launch_pdl(kern, dim3(grid), dim3(128), sm, s, T, B, r, v, d, last, gamma, gl, prior, score_fn, disc, adv, ret,
                       scores, maxret, s_eps, s_mean, s_max, s_sol, P);
        };
        // f64 values: PVL's advantages overwrite V in place; f32 values: a separate column
        if (sizeof(VT) == 8 || (score_fn & 0xFF) != AMZ_SCORE_PVL)
            go(k_gae_score7<VT, false>, sizeof(G7Smem<VT, false>));
        else
            go(k_gae_score7<VT, true>, sizeof(G7Smem<VT, true>));
        return 0;
    }
k2:
    if (gsel == 2 || B <= 131072) {
        launch_pdl(k_gae_score2<VT>, dim3((unsigned)((B + 31) / 32)), dim3(64), 0, s, T, B, r, v, d, last, gamma, gl,
                   prior, score_fn, disc, adv, ret, scores, maxret, s_eps, s_mean, s_max, s_sol, do_gae, P);
        return 0;
    }
k1:
    const int threads = B >= 148 * 64 ? 64 : 32;
    launch_pdl(k_gae_score<VT>, dim3((unsigned)((B + threads - 1) / threads)), dim3(threads), 0, s, T, B, r, v, d, last,
               gamma, gl, prior, score_fn, disc, adv, ret, scores, maxret, s_eps, s_mean, s_max, s_sol, do_gae, P);
    return 0;
}

int launch_gae_score(int T, int64_t B, const double *r, const double *v, const uint8_t *d, const double *last,
                     double gamma, double lam, const double *prior, int score_fn, int disc, double *adv,
                     double *ret, double *scores, double *maxret, const amz_episode_stats_t *stats,
                     cudaStream_t s, int do_gae) {
    return launch_gae_score_t<double>(T, B, r, v, d, last, gamma, lam, prior, score_fn, disc, adv, ret, scores,
                                      maxret, stats, s, do_gae);
}

int launch_gae_score_v32(int T, int64_t B, const double *r, const float *v, const uint8_t *d, const float *last,
                         double gamma, double lam, const double *prior, int score_fn, int disc, double *adv,
                         double *ret, double *scores, double *maxret, const amz_episode_stats_t *stats,
                         cudaStream_t s) {
    return launch_gae_score_t<float>(T, B, r, v, d, last, gamma, lam, prior, score_fn, disc, adv, ret, scores,
                                     maxret, stats, s, 1);
}

}  // namespace amz
