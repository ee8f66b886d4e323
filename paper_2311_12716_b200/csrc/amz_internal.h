// amz_internal.h -- declarations shared by the .cu translation units (not part of the ABI).
#pragma once
#include <mutex>
#include <unordered_map>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/amaze_b200.h"
#include "amz_level.cuh"

namespace amz {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, size): made on
// every launch it cost the rollout call ~0.4 ms of host time
inline void ensure_dyn_smem(const void *kern, int bytes) {
    static std::mutex mu;
    static std::unordered_map<uint64_t, int> done;  // (kernel, device) -> bytes already allowed
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t key = (uint64_t)(uintptr_t)kern ^ ((uint64_t)(uint32_t)dev << 52);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = done.find(key);
        if (it != done.end() && it->second >= bytes) return;
    }
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    std::lock_guard<std::mutex> lk(mu);
    int &b = done[key];
    if (bytes > b) b = bytes;
}

// Programmatic dependent launch along the rollout chain (k_env_reset_dr -> k_dyn ->
// k_render -> GAE): a dependent kernel is launched with launch_pdl, runs its
// shared-memory-only prologue, then pdl_wait() -- which returns once the preceding grid
// has completed and its writes are visible -- before touching global memory the
// preceding kernels write.  No kernel triggers early (pdl_trigger): measured on B200,
// dependents launched at the start of k_dyn parked their CTAs on the SMs and slowed it
// (step 0.152 -> 0.156 ms), while the implicit trigger at completion gains ~1-3%
// (launch processing and the dependents' prologues overlap the tail).  Both are no-ops
// for ordinary launches; AMZ_NO_PDL=1 launches without the attribute (A/B runs).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    static const bool off = getenv("AMZ_NO_PDL") != nullptr;  // A/B runs
    cfg.attrs = at;
    cfg.numAttrs = off ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// device view of an amz_env_t
struct EnvDev {
    int64_t B;
    uint32_t lane_offset;
    uint4 *st;
    uint4 *mask;
    uint32_t *board;  // [16][B]
    int *err;
    // device iteration counter (CUDA-graph replay): when set, the reset / rollout key
    // prefixes passed in are the ROOT stream's, and the kernels derive the iteration's
    // streams root.fold_in(*iter).fold_in(0) (lane levels) and .fold_in(1) (auto-reset)
    const uint32_t *iter = nullptr;
    // work counter of the persistent large-batch dynamics (the launch's last fetch re-zeroes it)
    uint32_t *work = nullptr;
    // finished k_dyn warps per 128-lane group [ceil(B / 128)] (zeroed before each launch):
    // the render takes a group's tiles once its warps are done, beside k_dyn's tail
    uint32_t *gdone = nullptr;
    // render tiles past their wait per group [ceil(B / 128)]: the last one re-zeroes both
    // counters for the next rollout (no memset between the reset and k_dyn)
    uint32_t *gpass = nullptr;
};

// numpy pairwise summation schedule (numpy/_core/src/umath/loops_utils.h.src
// pairwise_sum): leaves of <= 128 elements, summed with 8 accumulators, combined
// bottom-up.  adds[i] = combines to perform after pushing leaf i.
constexpr int kMaxLeaves = 64;
struct PairwisePlan {
    int n_leaves;
    int leaf_end[kMaxLeaves];
    uint8_t adds[kMaxLeaves];
};
int make_pairwise_plan(int n, PairwisePlan &plan);

int launch_sample_levels(const Geo &G, const amz_seed_t &prefix, uint32_t lane0, const uint32_t *ids, int64_t n,
                         amz_level_t *out, cudaStream_t s);
int launch_mutate_levels(const Geo &G, const amz_seed_t &prefix, uint32_t lane0, int64_t n, const amz_level_t *par,
                         const int32_t *pidx, int n_edits, amz_level_t *out, cudaStream_t s);
int launch_teacher_reset(const Geo &G, int64_t B, uint4 *mask, uint4 *st, uint8_t *grid, float *phase,
                         int64_t *n_placed, cudaStream_t s);
int launch_teacher_step(const Geo &G, int64_t B, uint4 *mask, uint4 *st, const int64_t *actions, uint8_t *grid,
                        float *phase, int64_t *n_placed, uint8_t *done, int64_t *times, int *err, cudaStream_t s);
int launch_teacher_levels(int64_t B, const uint4 *mask, const uint4 *st, amz_level_t *out, int *err, cudaStream_t s);
int launch_policy_head(const void *logits, int dtype, int64_t B, int A, uint64_t k0, uint64_t k1,
                       const amz_seed_t *prefix_dev, const uint32_t *step_dev, int greedy, int64_t lane0, int64_t *act64,
                       uint8_t *act8, double *logp, cudaStream_t s);
int launch_copy_h2d(void *dst, const void *src, size_t bytes, int ctas, cudaStream_t s);
int launch_iter_advance(uint32_t *iter, uint32_t by, cudaStream_t s);
int launch_env_reset_dr(const Geo &G, const EnvDev &E, const amz_seed_t &prefix, const amz_seed_t *wrap,
                        amz_level_t *spec, uint32_t *spec_step, uint8_t *view, int64_t *dirs, cudaStream_t s);
int launch_level_metrics(const Geo &G, const amz_level_t *lv, int64_t n, int32_t *n_walls, int32_t *spl,
                         uint8_t *solvable, double *passable, cudaStream_t s);
int launch_check_levels(const Geo &G, const amz_level_t *lv, int64_t n, unsigned long long *first_bad,
                        cudaStream_t s);
int launch_env_reset(const Geo &G, const EnvDev &E, const amz_level_t *lv, const int64_t *lanes, int64_t n,
                     uint8_t *view, int64_t *dirs, cudaStream_t s);
int launch_env_observe(const Geo &G, const EnvDev &E, uint8_t *view, int64_t *dirs, cudaStream_t s);
int launch_env_levels(const EnvDev &E, amz_level_t *out, cudaStream_t s);
int launch_env_state(const EnvDev &E, int32_t *out, cudaStream_t s);
int launch_env_set_state(const EnvDev &E, const int32_t *in, cudaStream_t s);
int launch_env_step(const Geo &G, const EnvDev &E, const void *actions, int adtype, int mode,
                    const amz_seed_t &wrap, uint32_t step_idx, const uint32_t *step_dev, const amz_seed_t *wrap_dev,
                    uint8_t *view, int64_t *dirs, double *reward,
                    uint8_t *done, double *solved, int64_t *times, const int *term_in, int *term_out,
                    cudaStream_t s);
// poses [ceil(T/4)][B][4] (uint4 per lane per 4 steps), epochs [(T+1)*B][20], final_pose [B]: rollout scratch (amz_rollout.cu)
int launch_env_rollout(const Geo &G, const EnvDev &E, int T, const uint8_t *actions, int mode,
                       const amz_seed_t &wrap, uint32_t step0, uint8_t *view, uint8_t *dirs, double *reward,
                       uint8_t *done, uint8_t *fview, uint8_t *fdir, uint32_t *poses, uint32_t *epochs,
                       uint32_t *final_pose, amz_level_t *spec, uint32_t *spec_step, int spec_ready,
                       cudaStream_t s);
int launch_gae_score(int T, int64_t B, const double *r, const double *v, const uint8_t *d, const double *last,
                     double gamma, double lam, const double *prior, int score_fn, int disc, double *adv,
                     double *ret, double *scores, double *maxret, const amz_episode_stats_t *stats,
                     cudaStream_t s, int do_gae = 1);
// values (and last values) as the policy's float32, widened exactly in the kernel
int launch_gae_score_v32(int T, int64_t B, const double *r, const float *v, const uint8_t *d, const float *last,
                         double gamma, double lam, const double *prior, int score_fn, int disc, double *adv,
                         double *ret, double *scores, double *maxret, const amz_episode_stats_t *stats,
                         cudaStream_t s);

// PLR buffer (amz_plr.cu)
struct PlrDev {
    int64_t K;
    amz_level_t *levels;
    double *score;
    double *maxret;
    int64_t *last;
    int64_t *seq;
    int64_t *meta;  // [0] size, [1] next_seq
};
struct UpdScratch {
    int32_t *init_match;  // [n]
    int32_t *twin_first;  // [n]
    int32_t *keyslot;     // [n] current slot of the key group led by this candidate (or -1)
    int32_t *rel;         // [n] compacted relevant candidate ids
    uint32_t *chash;      // [hsize] candidate hash table (index + 1)
    int64_t cap;
};
int launch_plr_sample(const PlrDev &D, int32_t *rank, const amz_seed_t &key, int64_t n, double omr, double rho,
                      const double *lut, int prop, double inv_beta, int64_t iter, int32_t *slots, amz_level_t *levels,
                      double *maxret, double *score, int *err, cudaStream_t s);
int launch_plr_prepare(const PlrDev &D, const amz_level_t *cand, int64_t n, const UpdScratch &W, cudaStream_t s);
int launch_plr_update(const PlrDev &D, const amz_level_t *cand, const double *cs, const double *cm, int64_t n,
                      int64_t iter, const UpdScratch &W, int *err, cudaStream_t s, int prepared = 0);
int launch_plr_digest(const PlrDev &D, int64_t *out, cudaStream_t s);
int launch_top_q(const double *scores, int64_t n, int q, int32_t *out, cudaStream_t s);

}  // namespace amz
