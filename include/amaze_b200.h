/*
 * amaze_b200.h -- C ABI of the B200-native AMaze / PLR hot path (libamaze_b200.so).
 *
 * Plain pointers and sizes only.  Every pointer named *_dev is a device pointer owned
 * by the caller (torch tensors in the Python layer); the library owns only the opaque
 * handles it allocates (amz_env_t, amz_plr_t) and frees them in *_destroy.  All
 * launches are asynchronous on the caller's stream (`stream` is a cudaStream_t, NULL =
 * legacy default stream); no call makes a hidden device synchronisation except the
 * ones documented as "synchronous".
 *
 * Return value: 0 on success or one of the negative AMZ_E* codes below, which the
 * Python shim maps 1:1 onto the reference's exception classes
 * (/root/reference/pkg/src/autocurricula/errors.py:4-34).  amz_last_error() returns a
 * thread-local message for the last failing call.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/autocurricula):
 *   amz_seed_prefix          rng.py:33-50            (RngStream key -> SeedSequence state)
 *   amz_sample_levels        amaze/generator.py:36-52, amaze/env.py:175-176
 *   amz_mutate_levels        amaze/generator.py:55-84
 *   amz_env_*                amaze/env.py:237-364 (MazeStateBatch, step_batch, observe_batch),
 *                            env/batch.py:78-115 (VectorBatchEnv),
 *                            env/wrappers.py:20-78 (AutoResetWrapper)
 *   amz_env_rollout          the env side of agents/rollout.py:120-179 with an action stream
 *   amz_gae_score(_v32)      agents/gae.py:8-37, agents/rollout.py:155-189,
 *                            runners/scoring.py:18-63
 *   amz_plr_*                the PLR level buffer runners/buffer.py imported at
 *                            runners/scoring.py:14 but absent from the reference;
 *                            semantics restated from SPEC.md:332-377,427-433
 */
#ifndef AMAZE_B200_H
#define AMAZE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMZ_ABI_VERSION 1

/* error codes -> errors.py classes */
#define AMZ_OK 0
#define AMZ_ECONFIG -1     /* ConfigError        */
#define AMZ_ELEVEL -2      /* LevelError         */
#define AMZ_ECONTRACT -3   /* ContractViolation  */
#define AMZ_ESHAPE -4      /* ShapeError         */
#define AMZ_ECUDA -5       /* RunnerFault (CUDA runtime failure) */
#define AMZ_EFAULT -6      /* RunnerFault        */

/* auto-reset modes (env/wrappers.py:16-17); NONE = bare VectorBatchEnv stepping */
#define AMZ_RESET_NONE 0
#define AMZ_RESET_RESAMPLE 1
#define AMZ_RESET_HOME 2

/* score functions (runners/scoring.py:59-62) */
#define AMZ_SCORE_MAXMC 0
#define AMZ_SCORE_PVL 1
/* flags or-ed into score_fn: keep the unclamped mean (score_pvl/score_maxmc themselves
 * do not clamp); take prior_max as the final max return (skip the episode pass) */
#define AMZ_SCORE_NOCLAMP 0x100
#define AMZ_SCORE_PRIOR_FINAL 0x200

/* One level, 32 bytes.  Interior cell (r, c) (1 <= r <= H-2, 1 <= c <= W-2) is wall
 * iff bit (r-1)*(W-2) + (c-1) of walls[] (little-endian words) is set; the border is
 * always wall.  Mirrors MazeLevel (amaze/level.py:33-80). */
typedef struct amz_level {
    uint32_t walls[4];
    uint8_t agent_r, agent_c, agent_dir, goal_r, goal_c;
    uint8_t pad[3];
    uint32_t pad2[2];
} amz_level_t;

/* StaticParams (env/core.py:24-52).  Supported here: 3 <= H, W <= 16 with
 * (H-2)*(W-2) <= 128, agent_view_size odd in [3, 9], max_episode_steps <= 65535. */
typedef struct amz_params {
    int32_t height, width, max_episode_steps, agent_view_size, wall_budget, see_through_walls;
} amz_params_t;

/* numpy SeedSequence state after absorbing the assembled entropy of a key PREFIX;
 * the device appends the per-lane suffix words (lane, or step and lane). */
typedef struct amz_seed {
    uint32_t pool[4];
    uint32_t hash_const;
    uint32_t n_words; /* words absorbed so far (diagnostic) */
} amz_seed_t;

/* per-lane completed-episode statistics (agents/rollout.py:155-189) */
typedef struct amz_episode_stats {
    int64_t *episodes;    /* [B] */
    double *mean_return;  /* [B] */
    double *max_return;   /* [B] */
    double *solved_rate;  /* [B] */
} amz_episode_stats_t;

typedef struct amz_env amz_env_t;
typedef struct amz_plr amz_plr_t;
typedef struct amz_teacher amz_teacher_t;

int amz_abi_version(void);
const char *amz_last_error(void);
int amz_validate_params(const amz_params_t *p);

/* Pinned host staging memory for the trajectory feed (the reference keeps these arrays
 * in numpy memory, agents/rollout.py:19-70): 2 MB transparent-huge-page mappings
 * registered with cudaHostRegister (portable), falling back to cudaHostAlloc; the
 * host->device copies run at the PCIe rate from it where CPU-written 4 KB pinned pages
 * read at a quarter to a half of it.  AMZ_HOST_ALLOC=cuda forces cudaHostAlloc.  Free
 * with amz_host_free.  bytes = 0 gives NULL. */
int amz_host_alloc(size_t bytes, void **out);
int amz_host_free(void *p);

/* Host-side key setup.  run = SeedSequence run entropy as u32 words (numpy's
 * _int_to_uint32_array), key = RngStream key prefix words.  The full spawn key is
 * prefix ++ suffix with a non-empty suffix, so the run entropy is zero-padded to 4. */
int amz_seed_prefix(const uint32_t *run, int n_run, const uint32_t *key, int n_key, amz_seed_t *out);
/* Host only: the first Generator.random() of the stream (numpy's Philox of the key's
 * SeedSequence: (first u64 >> 11) * 2^-53) -- the replay decision of
 * buffer_sample_decision without building a numpy Generator. */
int amz_stream_uniform(const amz_seed_t *prefix, double *out_host);

/* DR levels: out[i] = sample_random_level(key = prefix ++ [lane_ids ? lane_ids[i] : lane0 + i]). */
int amz_sample_levels(const amz_params_t *p, const amz_seed_t *prefix, uint32_t lane0,
                      const uint32_t *lane_ids_dev, int64_t n, amz_level_t *out_dev, void *stream);

/* ACCEL: out[i] = mutate_level(key = prefix ++ [lane0 + i], parents[parent_idx ? parent_idx[i] : i],
 * n_edits).  n_edits >= 1 (generator.py:63-64 -> AMZ_ECONTRACT). */
int amz_mutate_levels(const amz_params_t *p, const amz_seed_t *prefix, uint32_t lane0, int64_t n,
                      const amz_level_t *parents_dev, const int32_t *parent_idx_dev, int n_edits,
                      amz_level_t *out_dev, void *stream);

/* Validate levels on device; *bad_index_host = first invalid index or -1 (synchronous). */
/* PAIRED level designer, batched (amaze/teacher.py:36-159): n_lanes design episodes
 * of wall_budget + 2 steps.  Observations per lane: grid u8 [H][W] tile codes,
 * phase f32 [4] one-hot, n_placed i64 (phase/n_placed may be NULL); step also writes
 * done u8 and time i64 (may be NULL).  Actions are int64 interior cell indices
 * (row-major).  Contract violations (terminal lane, action out of range) are flagged on
 * the device and raised by amz_teacher_check (synchronous) as AMZ_ECONTRACT.
 * amz_teacher_levels decodes every (finished) lane into a level record (synchronous). */
int amz_teacher_create(const amz_params_t *p, int64_t n_lanes, amz_teacher_t **out);
int amz_teacher_destroy(amz_teacher_t *t);
int amz_teacher_reset(amz_teacher_t *t, uint8_t *grid_dev, float *phase_dev, int64_t *n_placed_dev, void *stream);
int amz_teacher_step(amz_teacher_t *t, const int64_t *actions_dev, uint8_t *grid_dev, float *phase_dev,
                     int64_t *n_placed_dev, uint8_t *done_dev, int64_t *time_dev, void *stream);
int amz_teacher_check(amz_teacher_t *t, void *stream);
int amz_teacher_levels(amz_teacher_t *t, amz_level_t *levels_dev, void *stream);

/* Policy hand-off (agents/rollout.py:145-152 sample_actions + agents/ppo.py:82-96,136-138):
 * logits [B][A] (dtype 0 = f32, 1 = f64; A <= 16) -> action (int64 and/or u8, any NULL)
 * and its log-softmax probability (f64, may be NULL).  Sampling uses u = the (lane0+i)-th
 * double of the generator whose SeedSequence state after its whole key is `key`
 * (e.g. RngStream.fold_in(t)), as numpy's Generator.random(B) hands them out;
 * greedy = argmax (key may be NULL). */
int amz_policy_head(const void *logits, int dtype, int64_t B, int A, const amz_seed_t *key, int greedy,
                    int64_t lane0, int64_t *actions, uint8_t *actions_u8, double *log_probs, void *stream);

/* The same for CUDA-graph replay: prefix_dev (device amz_seed_t: the rollout stream's
 * prefix) and step_dev (device u32 t) are read at run time; the generator is
 * prefix ++ [t]. */
int amz_policy_head_dev(const void *logits, int dtype, int64_t B, int A, const amz_seed_t *prefix_dev,
                        const uint32_t *step_dev, int greedy, int64_t lane0, int64_t *actions, uint8_t *actions_u8,
                        double *log_probs, void *stream);

/* Curriculum metrics of n levels (amaze/metrics.py:21-31 env_metrics, BFS of
 * amaze/pathfinding.py:116-135): interior wall count, agent->goal shortest path length
 * (0 if unsolvable), solvable flag, passable ratio (float64, bit-exact).  Any output
 * pointer may be NULL.  Async on `stream`. */
int amz_level_metrics(const amz_params_t *p, const amz_level_t *levels, int64_t n, int32_t *n_walls,
                      int32_t *shortest_path, uint8_t *solvable, double *passable, void *stream);

int amz_check_levels(const amz_params_t *p, const amz_level_t *levels_dev, int64_t n,
                     int64_t *bad_index_host, void *stream);

/* ---- batched environment (lane SoA resident in HBM) ---- */
int amz_env_create(const amz_params_t *p, int64_t n_lanes, amz_env_t **out);
int amz_env_destroy(amz_env_t *env);
int64_t amz_env_lanes(const amz_env_t *env);
/* Global index of local lane 0 (multi-GPU lane sharding: RESAMPLE keys use global lanes). */
int amz_env_set_lane_offset(amz_env_t *env, uint32_t offset);

/* Reset lanes to levels and render their observations (env/batch.py:91-96,107-115).
 * lanes_dev == NULL: all n_lanes lanes, levels_dev[n_lanes];
 * otherwise lanes_dev[n] lane ids with levels_dev[n].  view_dev [n][V][V] u8,
 * dir_dev [n] int64 (either may be NULL). */
/* VectorBatchEnv.reset fused with DR level generation: lane l plays the level of key
 * prefix ++ [lane_offset + l] (amaze/generator.py:36-52).  With `wrap` (the auto-reset
 * wrapper's key) the lanes' timeout levels for the first RESAMPLE rollout (step0 = 0,
 * same key) are prepared in the same launch.  view/dir may be NULL. */
int amz_env_reset_dr(amz_env_t *env, const amz_seed_t *prefix, const amz_seed_t *wrap, uint8_t *view_dev,
                     int64_t *dir_dev, void *stream);
int amz_env_reset_to_levels(amz_env_t *env, const amz_level_t *levels_dev, const int64_t *lanes_dev,
                            int64_t n, uint8_t *view_dev, int64_t *dir_dev, void *stream);

/* One step of every lane (amaze/env.py:320-364 + env/wrappers.py:59-78).
 * actions_dev [B] with dtype code action_dtype (0=u8, 1=i32, 2=i64).
 * mode AMZ_RESET_RESAMPLE draws lane l's new level from key wrap ++ [step_idx, l].
 * Outputs [B]: view u8[V][V] (post-auto-reset obs), dir i64, reward f64, done u8,
 * solved f64, time i64; any output may be NULL.  In mode NONE a step on terminal lanes
 * leaves the state untouched and raises AMZ_ECONTRACT at the next amz_env_check(). */
int amz_env_step(amz_env_t *env, const void *actions_dev, int action_dtype, int mode,
                 const amz_seed_t *wrap, uint32_t step_idx, uint8_t *view_dev, int64_t *dir_dev,
                 double *reward_dev, uint8_t *done_dev, double *solved_dev, int64_t *time_dev,
                 void *stream);

/* amz_env_step for CUDA-graph replay: the auto-reset key prefix (wrap_dev, a device
 * amz_seed_t) and the env step index (step_dev, a device u32 the captured graph
 * advances) are read at run time, so one captured step serves every step of every
 * rollout.  Auto-reset modes only (RESAMPLE / HOME; wrap_dev may be NULL for HOME). */
int amz_env_step_dev(amz_env_t *env, const void *actions_dev, int action_dtype, int mode,
                     const amz_seed_t *wrap_dev, const uint32_t *step_dev, uint8_t *view_dev, int64_t *dir_dev,
                     double *reward_dev, uint8_t *done_dev, double *solved_dev, int64_t *time_dev, void *stream);

/* T fused steps with an action stream actions_dev u8 [T][B] (time-major).
 * Writes the trajectory the way agents/rollout.py stores it: view [T][B][V][V] and
 * dir u8 [T][B] are the observations BEFORE each step, reward f64 [T][B], done u8 [T][B];
 * final_view [B][V][V] / final_dir u8 [B] the observation after the last step
 * (RolloutCursor.obs).  Keys: step t of this call uses wrap ++ [step0 + t, lane]. */
int amz_env_rollout(amz_env_t *env, int T, const uint8_t *actions_dev, int mode, const amz_seed_t *wrap,
                    uint32_t step0, uint8_t *view_dev, uint8_t *dir_dev, double *reward_dev,
                    uint8_t *done_dev, uint8_t *final_view_dev, uint8_t *final_dir_dev, void *stream);

/* Render the current observation of every lane (observe_batch, amaze/env.py:352-364). */
/* CUDA-graph replay of the DR iteration (reset -> rollout): the key streams come from a
 * device iteration counter iter_dev (u32) instead of host-computed prefixes, so one
 * captured graph serves every iteration.  root = the run's root stream prefix;
 * iteration it = *iter_dev uses lane levels root.fold_in(it).fold_in(0) + (lane,) and
 * auto-reset keys root.fold_in(it).fold_in(1) + (step, lane) -- the same streams as
 * amz_env_reset_dr / amz_env_rollout called with the prefixes of
 * AutoResetWrapper.reset(root.fold_in(it)) (env/wrappers.py:43-56).  The rollout starts
 * at step 0 in RESAMPLE mode.  amz_iter_advance adds `by` to the counter on the stream. */
int amz_env_reset_dr_iter(amz_env_t *env, const amz_seed_t *root, const uint32_t *iter_dev, uint8_t *view_dev,
                          int64_t *dir_dev, void *stream);
int amz_env_rollout_iter(amz_env_t *env, int T, const uint8_t *actions_dev, const amz_seed_t *root,
                         const uint32_t *iter_dev, uint8_t *view_dev, uint8_t *dir_dev, double *reward_dev,
                         uint8_t *done_dev, uint8_t *final_view_dev, uint8_t *final_dir_dev, void *stream);
int amz_iter_advance(uint32_t *iter_dev, uint32_t by, void *stream);
/* Host -> device copy by a kernel (`ctas` CTAs of 256 threads, 0 = 64) reading pinned host
 * memory (amz_host_alloc) through its unified address: the input feed of a captured
 * DR-iteration graph (graph.DRIterationGraph), at the PCIe link rate beside the step's
 * kernels.  Both buffers 16-byte aligned. */
int amz_copy_h2d(void *dst_dev, const void *src_host, size_t bytes, int ctas, void *stream);
/* Device -> host by the same kernel (`ctas` CTAs, 0 = 8) storing into pinned host memory
 * through its unified address: the result read-back of a captured DR-iteration graph
 * without a copy-engine node (which would queue behind the next step's H2D). */
int amz_copy_d2h(void *dst_host, const void *src_dev, size_t bytes, int ctas, void *stream);

int amz_env_observe(amz_env_t *env, uint8_t *view_dev, int64_t *dir_dev, void *stream);

/* lane_levels (env/batch.py:104-105): each lane's level (its reset-time pose). */
int amz_env_levels(amz_env_t *env, amz_level_t *out_dev, void *stream);

/* Episode state per lane: pos (r, c), dir, time, terminal -> out_dev [B][5] int32. */
int amz_env_state(amz_env_t *env, int32_t *out_dev, void *stream);

/* Overwrite the dynamic state (state_at/from_states, amaze/env.py:279-303): in_dev [B][5] int32. */
int amz_env_set_state(amz_env_t *env, const int32_t *in_dev, void *stream);

/* Synchronous: returns AMZ_ECONTRACT if a step hit terminal lanes since the last check. */
int amz_env_check(amz_env_t *env, void *stream);

/* ---- GAE + regret scores (time-major [T][B]) ---- */
/* adv/ret [T][B] f64 (agents/gae.py), scores/max_ret [B], stats optional.
 * prior_max_dev [B] or NULL (= 0).  dones as u8. */
int amz_gae_score(int T, int64_t B, const double *rewards_dev, const double *values_dev,
                  const uint8_t *dones_dev, const double *last_value_dev, double gamma, double lam,
                  const double *prior_max_dev, int score_fn, int maxmc_discounted, double *adv_dev,
                  double *ret_dev, double *scores_dev, double *max_ret_dev,
                  const amz_episode_stats_t *stats, void *stream);

/* amz_gae_score with values and last values as float32: the reference's values are the
 * policy's float32 outputs widened by `value.double()` (agents/ppo.py:96), so passing them
 * unwidened gives bit-identical results and halves the value bytes read (and copied). */
int amz_gae_score_v32(int T, int64_t B, const double *rewards_dev, const float *values_dev,
                      const uint8_t *dones_dev, const float *last_value_dev, double gamma, double lam,
                      const double *prior_max_dev, int score_fn, int maxmc_discounted, double *adv_dev,
                      double *ret_dev, double *scores_dev, double *max_ret_dev,
                      const amz_episode_stats_t *stats, void *stream);

/* lane_scores with caller-supplied advantages (runners/scoring.py:34-63): episode
 * stats + running max + MaxMC/PVL means, no GAE pass.  adv_dev needed for PVL only. */
int amz_lane_scores(int T, int64_t B, const double *rewards_dev, const double *values_dev,
                    const uint8_t *dones_dev, const double *adv_dev, double gamma, const double *prior_max_dev,
                    int score_fn, int maxmc_discounted, double *scores_dev, double *max_ret_dev,
                    const amz_episode_stats_t *stats, void *stream);

/* ---- PLR level buffer (device-resident; oracle/plr_np.py) ----
 * Capacity K <= 4096 (paper: 4000).  Slots 0..size-1 are valid. */
int amz_plr_create(int64_t capacity, amz_plr_t **out);
int amz_plr_destroy(amz_plr_t *plr);

/* buffer_update: for each of the n candidates IN ORDER: an identical
 * level (walls + pose) present -> score/max_return updated in place; else insert while
 * not full; else replace the (score, last_sampled, seq)-minimum iff score > its score.
 * New entries get last_sampled = insert iteration = iter. */
int amz_plr_update(amz_plr_t *plr, const amz_level_t *levels_dev, const double *scores_dev,
                   const double *max_ret_dev, int64_t n, int64_t iter, void *stream);
/* Build the twin table of the next update's candidates ahead of it (it depends on the
 * candidate levels only), e.g. on a side stream while the candidates are being rolled
 * out and scored; the next amz_plr_update with the same levels pointer and count skips
 * that work.  The caller orders the streams: the update must wait for this call's stream,
 * and this call for the previous update. */
int amz_plr_prepare(amz_plr_t *plr, const amz_level_t *levels_dev, int64_t n, void *stream);

/* buffer_sample_levels, rank prioritisation: n draws with replacement
 * = numpy Generator(key).choice(size, n, p=P), P = (1-rho) P_S + rho P_C,
 * P_S = w/sum(w), w = rank_lut_dev[rank-1] ((1/rank)^(1/beta), ranks by score desc then
 * older insertion), P_C = (iter-last_sampled)/sum (P = P_S if that sum is 0).  key = the
 * stream's full SeedSequence state (no suffix word).  Outputs slots [n] i32 and the
 * drawn levels / max returns / scores (each optional); drawn entries get
 * last_sampled = iter.  An empty buffer raises AMZ_ECONTRACT at amz_plr_size(). */
int amz_plr_sample(amz_plr_t *plr, const amz_seed_t *key, int64_t n, double rho, const double *rank_lut_dev,
                   int64_t iter, int32_t *slots_dev, amz_level_t *levels_dev, double *max_ret_dev,
                   double *score_dev, void *stream);

/* buffer_sample_levels with proportional prioritisation: P_S ~
 * score^(1/temperature) (numpy's np.power; CUDA's pow is within 2 ulp of it, so draws
 * equal the oracle's except where a uniform falls inside that rounding of a cdf
 * boundary), mixed with the staleness term like amz_plr_sample.  NaN probabilities
 * (a negative score, or every score 0: numpy's choice raises) give AMZ_ECONTRACT at
 * amz_plr_size(). */
int amz_plr_sample_proportional(amz_plr_t *plr, const amz_seed_t *key, int64_t n, double rho, double temperature,
                                int64_t iter, int32_t *slots_dev, amz_level_t *levels_dev, double *max_ret_dev,
                                double *score_dev, void *stream);

/* ACCEL parent choice: indices of the q highest scores (ties -> lower index). */
int amz_plr_top_q(const double *scores_dev, int64_t n, int q, int32_t *out_dev, void *stream);

/* Synchronous: current size; reports a deferred empty-buffer sampling error. */
int amz_plr_size(amz_plr_t *plr, int64_t *size_host, void *stream);

/* Replica drift check (the analogue of the shard-sync check at agents/ppo.py:322-328):
 * a 64-bit digest of the valid slots and meta written to out_dev[0] (device int64),
 * asynchronously on `stream`; equal buffers give equal digests. */
int amz_plr_digest(amz_plr_t *plr, int64_t *out_dev, void *stream);

/* Device-to-device copy of the whole buffer state (checkpoint / drift checks):
 * levels [K], score [K], max_return [K], last_sampled [K] i64, seq [K] i64,
 * meta [2] i64 = (size, next_seq).  Any output may be NULL for export. */
int amz_plr_export(amz_plr_t *plr, amz_level_t *levels_dev, double *score_dev, double *max_ret_dev,
                   int64_t *last_sampled_dev, int64_t *seq_dev, int64_t *meta_dev, void *stream);
int amz_plr_import(amz_plr_t *plr, const amz_level_t *levels_dev, const double *score_dev,
                   const double *max_ret_dev, const int64_t *last_sampled_dev, const int64_t *seq_dev,
                   const int64_t *meta_dev, void *stream);

#ifdef __cplusplus
}
#endif
#endif
