// amz_policy.cu -- the policy hand-off of the rollout loop:
// logits -> sampled action + its log-probability, numpy-exact.
//
//   sample_actions   agents/rollout.py:145-152  z = x - max; p = exp(z) / sum(exp(z));
//                                               u = g.random(B)[lane]; a = min(#(u > cumsum(p)), A-1)
//   log_softmax_np   agents/ppo.py:136-138      z - log(sum(exp(z)))
//   PPOAgent.act     agents/ppo.py:82-96        greedy = argmax(logits), log_probs gathered at a
//
// One thread per lane.  Row sums follow numpy's reduction for a contiguous last axis
// (sequential below 8 elements, 8-accumulator pairwise blocks from 8 on); the uniform is
// the lane-th double of the step's Philox stream (numpy hands the u64s of block b,
// counter b+1, out in order).  exp/log are CUDA's (<= 1 ulp); numpy's may differ in the
// last bit, which moves an action only when u lies within an ulp of a CDF boundary.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "amz_internal.h"
#include "amz_rng.cuh"

namespace amz {

constexpr int kMaxActions = 16;

// numpy pairwise_sum for n <= 16 (numpy/_core/src/umath/loops_utils.h.src)
__device__ __forceinline__ double np_row_sum(const double *e, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; i++) res = __dadd_rn(res, e[i]);
        return res;
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(e[0], e[1]), __dadd_rn(e[2], e[3])),
                           __dadd_rn(__dadd_rn(e[4], e[5]), __dadd_rn(e[6], e[7])));
    for (int i = 8; i < n; i++) res = __dadd_rn(res, e[i]);
    return res;
}

// KA > 0: the action count fixed at compile time (AMaze's 3), so x/z/e live in registers;
// KA = 0: any A <= kMaxActions (the arrays then sit in local memory)
template <typename TL, int KA>
__global__ void __launch_bounds__(128) k_policy_head(const TL *__restrict__ logits, int64_t B, int A_, uint64_t k0,
                                                     uint64_t k1, const amz_seed_t *__restrict__ prefix_dev,
                                                     const uint32_t *__restrict__ step_dev, int greedy,
                                                     int64_t lane0, int64_t *__restrict__ act64,
                                                     uint8_t *__restrict__ act8, double *__restrict__ logp) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B) return;
    const int A = KA > 0 ? KA : A_;
    constexpr int NA = KA > 0 ? KA : kMaxActions;
    double x[NA], z[NA], e[NA];
    const TL *row = logits + i * A;
    double mx = (double)row[0];
#pragma unroll
    for (int a = 0; a < A; a++) {
        x[a] = (double)row[a];
        if (!isnan(mx) && (isnan(x[a]) || x[a] > mx)) mx = x[a];
    }
#pragma unroll
    for (int a = 0; a < A; a++) {
        z[a] = __dsub_rn(x[a], mx);
        e[a] = exp(z[a]);
    }
    const double s = np_row_sum(e, A);
    int act;
    if (greedy) {
        // np.argmax: first maximum, a NaN wins at its first occurrence
        act = 0;
        double xa = x[0];
#pragma unroll
        for (int a = 1; a < A; a++) {
            if (!isnan(xa) && (isnan(x[a]) || x[a] > xa)) {
                act = a;
                xa = x[a];
            }
        }
    } else {
        if (prefix_dev) {  // graph replay: the key prefix and the step word come from device memory
            amz_seed_t pre = *prefix_dev;
            seed_absorb(pre, *step_dev);
            seed_key(pre, k0, k1);
        }
        const uint64_t q = (uint64_t)(lane0 + i);
        uint64_t o0, o1, o2, o3;
        philox_block((q >> 2) + 1ull, k0, k1, o0, o1, o2, o3);
        const uint32_t w = (uint32_t)(q & 3u);
        const uint64_t r = w == 0 ? o0 : w == 1 ? o1 : w == 2 ? o2 : o3;
        const double u = (double)(r >> 11) * (1.0 / 9007199254740992.0);
        int cnt = 0;
        double cum = 0.0;
#pragma unroll
        for (int a = 0; a < A; a++) {
            const double p = __ddiv_rn(e[a], s);
            cum = a == 0 ? p : __dadd_rn(cum, p);
            cnt += u > cum;
        }
        act = cnt < A - 1 ? cnt : A - 1;
    }
    if (act64) act64[i] = act;
    if (act8) act8[i] = (uint8_t)act;
    if (logp) {
        double za = z[0];
#pragma unroll
        for (int a = 1; a < A; a++)
            if (a == act) za = z[a];
        logp[i] = __dsub_rn(za, log(s));
    }
}

int launch_policy_head(const void *logits, int dtype, int64_t B, int A, uint64_t k0, uint64_t k1,
                       const amz_seed_t *prefix_dev, const uint32_t *step_dev, int greedy, int64_t lane0, int64_t *act64,
                       uint8_t *act8, double *logp, cudaStream_t s) {
    if (B <= 0) return 0;
    if (A < 1 || A > kMaxActions) return AMZ_ESHAPE;
    const unsigned g = (unsigned)((B + 127) / 128);
    if (dtype == 0 && A == 3)
        k_policy_head<float, 3><<<g, 128, 0, s>>>((const float *)logits, B, A, k0, k1, prefix_dev, step_dev, greedy,
                                                  lane0, act64, act8, logp);
    else if (dtype == 0)
        k_policy_head<float, 0><<<g, 128, 0, s>>>((const float *)logits, B, A, k0, k1, prefix_dev, step_dev, greedy,
                                                  lane0, act64, act8, logp);
    else if (A == 3)
        k_policy_head<double, 3><<<g, 128, 0, s>>>((const double *)logits, B, A, k0, k1, prefix_dev, step_dev, greedy,
                                                   lane0, act64, act8, logp);
    else
        k_policy_head<double, 0><<<g, 128, 0, s>>>((const double *)logits, B, A, k0, k1, prefix_dev, step_dev, greedy,
                                                   lane0, act64, act8, logp);
    return 0;
}

}  // namespace amz
