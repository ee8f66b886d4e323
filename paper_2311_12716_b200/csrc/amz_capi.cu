// amz_capi.cu -- extern "C" entry points of libamaze_b200.so (include/amaze_b200.h).
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>

#include <mutex>
#include <new>
#include <unordered_map>

#include "amz_internal.h"

using namespace amz;

static thread_local char g_err[512];

static int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

static int cuda_status(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(AMZ_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return 0;
}

#define AMZ_CHECK_CUDA(call, what)                                                      \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) return fail(AMZ_ECUDA, "%s: %s", what, cudaGetErrorString(e_)); \
    } while (0)

// Every handle remembers the device it was created on; an entry point that takes a
// handle makes that device current for the call (and restores the caller's), so a handle
// keeps working when another device is current.
struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev && dev >= 0)
            cudaSetDevice(dev);
        else
            prev = -1;
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
static int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

struct amz_env {
    int device;
    amz_params_t p;
    Geo G;
    EnvDev E;
    int *term;  // [2] terminal-lane counters (mode NONE)
    int parity;
    // rollout scratch (grown on demand): per-step pose records, per-epoch level boards
    uint32_t *poses = nullptr;
    uint32_t *epochs = nullptr;
    uint32_t *final_pose = nullptr;
    amz_level_t *spec = nullptr;   // speculative timeout levels [B]
    uint32_t *spec_step = nullptr; // [B]
    int64_t rollout_T = 0;
    // timeout levels prepared by a fused DR reset for the next RESAMPLE rollout with this
    // wrapper key starting at step 0 (consumed by that rollout, dropped by anything else)
    bool spec_ready = false;
    amz_seed_t spec_wrap{};
    const uint32_t *spec_iter = nullptr;  // the iteration counter the prepared levels are keyed by
};

struct amz_plr {
    int device;
    PlrDev D;
    int32_t *rank = nullptr;  // [K] sampler scratch: rank - 1 of every entry
    UpdScratch W;
    int *err;
    // candidates whose twin table amz_plr_prepare already built (consumed by the update)
    const amz_level_t *prep_cand = nullptr;
    int64_t prep_n = -1;
};

static int plr_scratch(amz_plr *b, int64_t n, cudaStream_t s) {
    if (n <= b->W.cap) return 0;
    int64_t cap = 1024;
    while (cap < n) cap <<= 1;
    cudaFreeAsync(b->W.init_match, s);
    cudaFreeAsync(b->W.twin_first, s);
    cudaFreeAsync(b->W.keyslot, s);
    cudaFreeAsync(b->W.rel, s);
    cudaFreeAsync(b->W.chash, s);
    cudaError_t e = cudaMallocAsync((void **)&b->W.init_match, cap * 4, s);
    if (e == cudaSuccess) e = cudaMallocAsync((void **)&b->W.twin_first, cap * 4, s);
    if (e == cudaSuccess) e = cudaMallocAsync((void **)&b->W.keyslot, cap * 4, s);
    if (e == cudaSuccess) e = cudaMallocAsync((void **)&b->W.rel, cap * 4, s);
    if (e == cudaSuccess) e = cudaMallocAsync((void **)&b->W.chash, cap * 2 * 4, s);
    if (e != cudaSuccess) {
        b->W.cap = 0;
        return fail(AMZ_ECUDA, "plr scratch: %s", cudaGetErrorString(e));
    }
    b->W.cap = cap;
    return 0;
}

extern "C" {

int amz_abi_version(void) { return AMZ_ABI_VERSION; }

const char *amz_last_error(void) { return g_err; }

int amz_validate_params(const amz_params_t *p) {
    if (!p) return fail(AMZ_ECONFIG, "null params");
    // StaticParams.validate (env/core.py:35-48)
    if (p->height < 3 || p->width < 3)
        return fail(AMZ_ECONFIG, "grid must be at least 3x3, got %dx%d", p->height, p->width);
    if (p->agent_view_size < 3 || p->agent_view_size % 2 == 0)
        return fail(AMZ_ECONFIG, "agent_view_size must be odd and >= 3, got %d", p->agent_view_size);
    if (p->max_episode_steps < 1)
        return fail(AMZ_ECONFIG, "max_episode_steps must be >= 1, got %d", p->max_episode_steps);
    const int max_walls = (p->height - 2) * (p->width - 2) - 2;
    if (p->wall_budget < 0 || p->wall_budget > max_walls)
        return fail(AMZ_ECONFIG, "wall_budget must be in [0, %d] for a %dx%d grid, got %d", max_walls, p->height,
                    p->width, p->wall_budget);
    // limits of this implementation
    if (p->height > 16 || p->width > 16 || (p->height - 2) * (p->width - 2) > 128)
        return fail(AMZ_ECONFIG, "grid %dx%d exceeds the 16x16 / 128-interior-cell limit", p->height, p->width);
    if (p->agent_view_size > 9) return fail(AMZ_ECONFIG, "agent_view_size %d > 9 unsupported", p->agent_view_size);
    if (p->max_episode_steps > 65535)
        return fail(AMZ_ECONFIG, "max_episode_steps %d > 65535 unsupported", p->max_episode_steps);
    return 0;
}

// Pinned host memory.  Preferred: an anonymous mapping backed by 2 MB transparent huge
// pages, registered with cudaHostRegister.  On the B200 hosts measured, the GPU reads
// CPU-written cudaHostAlloc (4 KB) pages at 11-25 GB/s (copy engine / copy kernel) while
// the same bytes on 2 MB pages stream at 49-53 GB/s: each 4 KB page costs the DMA path a
// translation.  Falls back to cudaHostAlloc when THP or registration is unavailable (or
// AMZ_HOST_ALLOC=cuda).
namespace {
constexpr size_t kHuge = size_t(2) << 20;
std::mutex g_host_mu;
std::unordered_map<void *, size_t> g_host_maps;  // THP blocks -> mapped length

void *thp_alloc(size_t bytes) {
    const char *mode = getenv("AMZ_HOST_ALLOC");
    if (mode && strcmp(mode, "cuda") == 0) return nullptr;
    const size_t len = (bytes + kHuge - 1) & ~(kHuge - 1);
    void *raw = mmap(nullptr, len + kHuge, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (raw == MAP_FAILED) return nullptr;
    const uintptr_t r = (uintptr_t)raw, a = (r + kHuge - 1) & ~(uintptr_t)(kHuge - 1);
    if (a > r) munmap(raw, a - r);  // trim to a 2 MB-aligned [a, a + len)
    if (r + len + kHuge > a + len) munmap((void *)(a + len), r + len + kHuge - (a + len));
    void *p = (void *)a;
#ifdef MADV_HUGEPAGE
    madvise(p, len, MADV_HUGEPAGE);
#endif
    memset(p, 0, len);  // fault the huge pages in before pinning
    if (cudaHostRegister(p, len, cudaHostRegisterPortable) != cudaSuccess) {
        cudaGetLastError();
        munmap(p, len);
        return nullptr;
    }
    std::lock_guard<std::mutex> lk(g_host_mu);
    g_host_maps[p] = len;
    return p;
}
}  // namespace

int amz_host_alloc(size_t bytes, void **out) {
    if (!out) return fail(AMZ_ECONFIG, "null argument");
    *out = nullptr;
    if (bytes == 0) return 0;
    if ((*out = thp_alloc(bytes)) != nullptr) return 0;
    if (cudaHostAlloc(out, bytes, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return fail(AMZ_ECUDA, "cudaHostAlloc of %zu bytes failed", bytes);
    }
    return 0;
}

int amz_host_free(void *p) {
    if (!p) return 0;
    size_t len = 0;
    {
        std::lock_guard<std::mutex> lk(g_host_mu);
        auto it = g_host_maps.find(p);
        if (it != g_host_maps.end()) {
            len = it->second;
            g_host_maps.erase(it);
        }
    }
    if (len) {
        const bool ok = cudaHostUnregister(p) == cudaSuccess;
        if (!ok) cudaGetLastError();
        munmap(p, len);
        return ok ? 0 : fail(AMZ_ECUDA, "cudaHostUnregister failed");
    }
    if (cudaFreeHost(p) != cudaSuccess) {
        cudaGetLastError();
        return fail(AMZ_ECUDA, "cudaFreeHost failed");
    }
    return 0;
}

int amz_seed_prefix(const uint32_t *run, int n_run, const uint32_t *key, int n_key, amz_seed_t *out) {
    if (!out || n_run < 1 || (n_key > 0 && !key) || !run) return fail(AMZ_ECONFIG, "bad seed prefix arguments");
    seed_prefix_host(run, n_run, key, n_key, *out);
    return 0;
}

int amz_stream_uniform(const amz_seed_t *prefix, double *out) {
    if (!prefix || !out) return fail(AMZ_ECONFIG, "null argument");
    uint64_t k0, k1, o0, o1, o2, o3;
    seed_key(*prefix, k0, k1);
    philox_block(1ull, k0, k1, o0, o1, o2, o3);  // numpy pre-increments the counter
    *out = (double)(o0 >> 11) * (1.0 / 9007199254740992.0);
    return 0;
}

int amz_sample_levels(const amz_params_t *p, const amz_seed_t *prefix, uint32_t lane0, const uint32_t *lane_ids,
                      int64_t n, amz_level_t *out, void *stream) {
    int rc = amz_validate_params(p);
    if (rc) return rc;
    if (!prefix || (n > 0 && !out)) return fail(AMZ_ECONFIG, "null argument");
    rc = launch_sample_levels(make_geo(*p), *prefix, lane0, lane_ids, n, out, (cudaStream_t)stream);
    return rc ? rc : cuda_status("sample_levels");
}

int amz_mutate_levels(const amz_params_t *p, const amz_seed_t *prefix, uint32_t lane0, int64_t n,
                      const amz_level_t *parents, const int32_t *pidx, int n_edits, amz_level_t *out, void *stream) {
    int rc = amz_validate_params(p);
    if (rc) return rc;
    if (n_edits < 1) return fail(AMZ_ECONTRACT, "n_mutations must be >= 1, got %d", n_edits);
    if (!prefix || (n > 0 && (!out || !parents))) return fail(AMZ_ECONFIG, "null argument");
    rc = launch_mutate_levels(make_geo(*p), *prefix, lane0, n, parents, pidx, n_edits, out, (cudaStream_t)stream);
    return rc ? rc : cuda_status("mutate_levels");
}

int amz_check_levels(const amz_params_t *p, const amz_level_t *lv, int64_t n, int64_t *bad, void *stream) {
    int rc = amz_validate_params(p);
    if (rc) return rc;
    if (!bad) return fail(AMZ_ECONFIG, "null argument");
    *bad = -1;
    if (n <= 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long *d = nullptr, h = ~0ull;
    AMZ_CHECK_CUDA(cudaMallocAsync((void **)&d, sizeof(h), s), "check_levels alloc");
    cudaMemcpyAsync(d, &h, sizeof(h), cudaMemcpyHostToDevice, s);
    launch_check_levels(make_geo(*p), lv, n, d, s);
    cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d, s);
    AMZ_CHECK_CUDA(cudaStreamSynchronize(s), "check_levels");
    *bad = h == ~0ull ? -1 : (int64_t)h;
    return 0;
}

// ---- PAIRED level designer (amaze/teacher.py) ----
struct amz_teacher {
    int device;
    amz_params_t p;
    Geo G;
    int64_t B;
    uint4 *mask = nullptr;
    uint4 *st = nullptr;
    int *err = nullptr;
};

int amz_teacher_create(const amz_params_t *p, int64_t n_lanes, amz_teacher_t **out) {
    int rc = amz_validate_params(p);
    if (rc) return rc;
    if (!out || n_lanes < 1) return fail(AMZ_ESHAPE, "n_lanes must be >= 1, got %lld", (long long)n_lanes);
    amz_teacher *t = new (std::nothrow) amz_teacher();
    if (!t) return fail(AMZ_EFAULT, "out of host memory");
    t->device = current_device();
    t->p = *p;
    t->G = make_geo(*p);
    t->B = n_lanes;
    cudaError_t err = cudaMalloc((void **)&t->mask, (size_t)n_lanes * sizeof(uint4));
    if (err == cudaSuccess) err = cudaMalloc((void **)&t->st, (size_t)n_lanes * sizeof(uint4));
    if (err == cudaSuccess) err = cudaMalloc((void **)&t->err, sizeof(int));
    if (err == cudaSuccess) err = cudaMemset(t->err, 0, sizeof(int));
    if (err != cudaSuccess) {
        cudaFree(t->mask);
        cudaFree(t->st);
        cudaFree(t->err);
        delete t;
        return fail(AMZ_ECUDA, "teacher alloc: %s", cudaGetErrorString(err));
    }
    *out = t;
    return 0;
}

int amz_teacher_destroy(amz_teacher_t *t) {
    if (!t) return 0;
    DevGuard guard_(t->device);
    cudaFree(t->mask);
    cudaFree(t->st);
    cudaFree(t->err);
    delete t;
    return 0;
}

int amz_teacher_reset(amz_teacher_t *t, uint8_t *grid, float *phase, int64_t *n_placed, void *stream) {
    if (!t || !grid) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(t->device);
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(t->err, 0, sizeof(int), s);
    launch_teacher_reset(t->G, t->B, t->mask, t->st, grid, phase, n_placed, s);
    return cuda_status("teacher_reset");
}

int amz_teacher_step(amz_teacher_t *t, const int64_t *actions, uint8_t *grid, float *phase, int64_t *n_placed,
                     uint8_t *done, int64_t *times, void *stream) {
    if (!t || !actions || !grid) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(t->device);
    launch_teacher_step(t->G, t->B, t->mask, t->st, actions, grid, phase, n_placed, done, times, t->err,
                        (cudaStream_t)stream);
    return cuda_status("teacher_step");
}

static int teacher_err(amz_teacher_t *t, cudaStream_t s) {
    DevGuard guard_(t->device);
    int h = 0;
    cudaMemcpyAsync(&h, t->err, sizeof(int), cudaMemcpyDeviceToHost, s);
    AMZ_CHECK_CUDA(cudaStreamSynchronize(s), "teacher check");
    if (h) cudaMemsetAsync(t->err, 0, sizeof(int), s);
    if (h & 1) return fail(AMZ_ECONTRACT, "step called on a terminal design state");
    if (h & 2) return fail(AMZ_ECONTRACT, "design action outside interior range [0, %d)", t->G.ni);
    if (h & 4) return fail(AMZ_ECONTRACT, "no free cell left for the agent");
    if (h & 8) return fail(AMZ_ECONTRACT, "design sequence not finished");
    return 0;
}

int amz_teacher_check(amz_teacher_t *t, void *stream) {
    if (!t) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(t->device);
    return teacher_err(t, (cudaStream_t)stream);
}

int amz_teacher_levels(amz_teacher_t *t, amz_level_t *out, void *stream) {
    if (!t || !out) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(t->device);
    cudaStream_t s = (cudaStream_t)stream;
    launch_teacher_levels(t->B, t->mask, t->st, out, t->err, s);
    return teacher_err(t, s);
}

int amz_policy_head_dev(const void *logits, int dtype, int64_t B, int A, const amz_seed_t *prefix_dev,
                        const uint32_t *step_dev, int greedy, int64_t lane0, int64_t *actions, uint8_t *actions_u8,
                        double *log_probs, void *stream) {
    if (B < 0) return fail(AMZ_ESHAPE, "lanes must be >= 0, got %lld", (long long)B);
    if (A < 1 || A > 16) return fail(AMZ_ESHAPE, "action count must be in [1, 16], got %d", A);
    if (dtype != 0 && dtype != 1) return fail(AMZ_ECONFIG, "logits dtype code must be 0 (f32) or 1 (f64)");
    if (B > 0 && !logits) return fail(AMZ_ECONFIG, "null argument");
    if (!greedy && (!prefix_dev || !step_dev)) return fail(AMZ_ECONFIG, "sampling needs a key prefix and a step counter");
    int rc = launch_policy_head(logits, dtype, B, A, 0, 0, prefix_dev, step_dev, greedy, lane0, actions, actions_u8,
                                log_probs, (cudaStream_t)stream);
    if (rc) return fail(rc, "policy_head: bad shape");
    AMZ_CHECK_CUDA(cudaGetLastError(), "policy_head launch");
    return 0;
}

int amz_policy_head(const void *logits, int dtype, int64_t B, int A, const amz_seed_t *key, int greedy,
                    int64_t lane0, int64_t *actions, uint8_t *actions_u8, double *log_probs, void *stream) {
    if (B < 0) return fail(AMZ_ESHAPE, "lanes must be >= 0, got %lld", (long long)B);
    if (A < 1 || A > 16) return fail(AMZ_ESHAPE, "action count must be in [1, 16], got %d", A);
    if (dtype != 0 && dtype != 1) return fail(AMZ_ECONFIG, "logits dtype code must be 0 (f32) or 1 (f64)");
    if (B > 0 && !logits) return fail(AMZ_ECONFIG, "null argument");
    if (!greedy && !key) return fail(AMZ_ECONFIG, "sampling needs a generator key");
    uint64_t k0 = 0, k1 = 0;
    if (key) seed_key(*key, k0, k1);
    int rc = launch_policy_head(logits, dtype, B, A, k0, k1, nullptr, nullptr, greedy, lane0, actions, actions_u8,
                                log_probs, (cudaStream_t)stream);
    if (rc) return fail(rc, "policy_head: bad shape");
    AMZ_CHECK_CUDA(cudaGetLastError(), "policy_head launch");
    return 0;
}

int amz_level_metrics(const amz_params_t *p, const amz_level_t *lv, int64_t n, int32_t *n_walls, int32_t *spl,
                      uint8_t *solvable, double *passable, void *stream) {
    int rc = amz_validate_params(p);
    if (rc) return rc;
    if (n < 0) return fail(AMZ_ESHAPE, "n must be >= 0, got %lld", (long long)n);
    if (n > 0 && !lv) return fail(AMZ_ECONFIG, "null argument");
    launch_level_metrics(make_geo(*p), lv, n, n_walls, spl, solvable, passable, (cudaStream_t)stream);
    AMZ_CHECK_CUDA(cudaGetLastError(), "level_metrics launch");
    return 0;
}

int amz_env_create(const amz_params_t *p, int64_t n_lanes, amz_env_t **out) {
    int rc = amz_validate_params(p);
    if (rc) return rc;
    if (!out || n_lanes < 1) return fail(AMZ_ESHAPE, "n_lanes must be >= 1, got %lld", (long long)n_lanes);
    amz_env *e = new (std::nothrow) amz_env();
    if (!e) return fail(AMZ_EFAULT, "out of host memory");
    e->device = current_device();
    e->p = *p;
    e->G = make_geo(*p);
    e->E.B = n_lanes;
    e->E.lane_offset = 0;
    e->parity = 0;
    size_t b = (size_t)n_lanes;
    cudaError_t err = cudaMalloc((void **)&e->E.st, b * sizeof(uint4));
    if (err == cudaSuccess) err = cudaMalloc((void **)&e->E.mask, b * sizeof(uint4));
    if (err == cudaSuccess) err = cudaMalloc((void **)&e->E.board, b * 16 * sizeof(uint32_t));
    if (err == cudaSuccess) err = cudaMalloc((void **)&e->E.err, 4 * sizeof(int));
    if (err == cudaSuccess) err = cudaMalloc((void **)&e->term, 2 * sizeof(int));
    if (err == cudaSuccess) err = cudaMalloc((void **)&e->final_pose, b * sizeof(uint32_t));
    if (err == cudaSuccess) err = cudaMalloc((void **)&e->spec, b * sizeof(amz_level_t));
    if (err == cudaSuccess) err = cudaMalloc((void **)&e->spec_step, b * sizeof(uint32_t));
    if (err == cudaSuccess) err = cudaMalloc((void **)&e->E.work, sizeof(uint32_t));
    if (err == cudaSuccess) err = cudaMalloc((void **)&e->E.gdone, ((b + 127) / 128) * sizeof(uint32_t));
    if (err == cudaSuccess) err = cudaMalloc((void **)&e->E.gpass, ((b + 127) / 128) * sizeof(uint32_t));
    if (err == cudaSuccess) err = cudaMemset(e->E.work, 0, sizeof(uint32_t));
    if (err == cudaSuccess) err = cudaMemset(e->E.gdone, 0, ((b + 127) / 128) * sizeof(uint32_t));
    if (err == cudaSuccess) err = cudaMemset(e->E.gpass, 0, ((b + 127) / 128) * sizeof(uint32_t));
    if (err == cudaSuccess) err = cudaMemset(e->E.err, 0, 4 * sizeof(int));
    if (err == cudaSuccess) err = cudaMemset(e->term, 0, 2 * sizeof(int));
    if (err == cudaSuccess) err = cudaMemset(e->E.st, 0, b * sizeof(uint4));
    if (err == cudaSuccess) err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
        amz_env_destroy(e);
        return fail(AMZ_ECUDA, "env alloc: %s", cudaGetErrorString(err));
    }
    *out = e;
    return 0;
}

int amz_env_destroy(amz_env_t *e) {
    if (!e) return 0;
    DevGuard guard_(e->device);
    cudaFree(e->E.st);
    cudaFree(e->E.mask);
    cudaFree(e->E.board);
    cudaFree(e->E.err);
    cudaFree(e->term);
    cudaFree(e->final_pose);
    cudaFree(e->spec);
    cudaFree(e->spec_step);
    cudaFree(e->E.work);
    cudaFree(e->E.gdone);
    cudaFree(e->E.gpass);
    cudaFree(e->poses);
    cudaFree(e->epochs);
    delete e;
    return 0;
}

int64_t amz_env_lanes(const amz_env_t *e) { return e ? e->E.B : -1; }

int amz_env_set_lane_offset(amz_env_t *e, uint32_t offset) {
    if (!e) return fail(AMZ_ECONFIG, "null env");
    DevGuard guard_(e->device);
    e->E.lane_offset = offset;
    e->spec_ready = false;
    return 0;
}

int amz_env_reset_dr(amz_env_t *e, const amz_seed_t *prefix, const amz_seed_t *wrap, uint8_t *view, int64_t *dirs,
                     void *stream) {
    if (!e || !prefix) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(e->device);
    cudaStream_t s = (cudaStream_t)stream;
    int rc = launch_env_reset_dr(e->G, e->E, *prefix, wrap, e->spec, e->spec_step, view, dirs, s);
    if (rc) return fail(rc, "reset: unsupported agent_view_size");
    cudaMemsetAsync(e->term, 0, 2 * sizeof(int), s);
    e->spec_ready = wrap != nullptr;
    e->spec_iter = nullptr;
    if (wrap) e->spec_wrap = *wrap;
    return cuda_status("env_reset_dr");
}

int amz_env_reset_dr_iter(amz_env_t *e, const amz_seed_t *root, const uint32_t *iter_dev, uint8_t *view,
                          int64_t *dirs, void *stream) {
    if (!e || !root || !iter_dev) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(e->device);
    cudaStream_t s = (cudaStream_t)stream;
    EnvDev E = e->E;
    E.iter = iter_dev;
    int rc = launch_env_reset_dr(e->G, E, *root, root, e->spec, e->spec_step, view, dirs, s);
    if (rc) return fail(rc, "reset: unsupported agent_view_size");
    cudaMemsetAsync(e->term, 0, 2 * sizeof(int), s);
    e->spec_ready = true;
    e->spec_iter = iter_dev;
    e->spec_wrap = *root;
    return cuda_status("env_reset_dr_iter");
}

int amz_copy_h2d(void *dst_dev, const void *src_host, size_t bytes, int ctas, void *stream) {
    if (!dst_dev || !src_host) return fail(AMZ_ECONFIG, "null argument");
    if ((((uintptr_t)dst_dev) | ((uintptr_t)src_host)) & 15u) return fail(AMZ_ECONFIG, "copy buffers must be 16-byte aligned");
    if (bytes == 0) return 0;
    launch_copy_h2d(dst_dev, src_host, bytes, ctas > 0 ? ctas : 64, (cudaStream_t)stream);
    return cuda_status("copy_h2d");
}

int amz_copy_d2h(void *dst_host, const void *src_dev, size_t bytes, int ctas, void *stream) {
    if (!dst_host || !src_dev) return fail(AMZ_ECONFIG, "null argument");
    if ((((uintptr_t)dst_host) | ((uintptr_t)src_dev)) & 15u) return fail(AMZ_ECONFIG, "copy buffers must be 16-byte aligned");
    if (bytes == 0) return 0;
    launch_copy_h2d(dst_host, src_dev, bytes, ctas > 0 ? ctas : 8, (cudaStream_t)stream);  // same kernel, UVA both ways
    return cuda_status("copy_d2h");
}

int amz_iter_advance(uint32_t *iter_dev, uint32_t by, void *stream) {
    if (!iter_dev) return fail(AMZ_ECONFIG, "null argument");
    launch_iter_advance(iter_dev, by, (cudaStream_t)stream);
    return cuda_status("iter_advance");
}

int amz_env_reset_to_levels(amz_env_t *e, const amz_level_t *lv, const int64_t *lanes, int64_t n, uint8_t *view,
                            int64_t *dirs, void *stream) {
    if (!e || !lv) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(e->device);
    e->spec_ready = false;
    if (!lanes && n != e->E.B) return fail(AMZ_ESHAPE, "expected %lld levels, got %lld", (long long)e->E.B, (long long)n);
    cudaStream_t s = (cudaStream_t)stream;
    int rc = launch_env_reset(e->G, e->E, lv, lanes, n, view, dirs, s);
    if (rc) return fail(rc, "reset: unsupported agent_view_size");
    if (!lanes) cudaMemsetAsync(e->term, 0, 2 * sizeof(int), s);
    return cuda_status("env_reset");
}

static int env_step_impl(amz_env_t *e, const void *actions, int adtype, int mode, const amz_seed_t *wrap,
                         uint32_t step_idx, const uint32_t *step_dev, const amz_seed_t *wrap_dev, uint8_t *view,
                         int64_t *dirs, double *reward, uint8_t *done, double *solved, int64_t *times,
                         void *stream) {
    if (!e || !actions) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(e->device);
    if (adtype < 0 || adtype > 2) return fail(AMZ_ECONTRACT, "bad action dtype code %d", adtype);
    if (mode < AMZ_RESET_NONE || mode > AMZ_RESET_HOME) return fail(AMZ_ECONTRACT, "unknown auto-reset mode %d", mode);
    if (mode == AMZ_RESET_RESAMPLE && !wrap && !wrap_dev) return fail(AMZ_ECONFIG, "RESAMPLE needs a wrapper key");
    cudaStream_t s = (cudaStream_t)stream;
    amz_seed_t w = wrap ? *wrap : amz_seed_t{};
    e->spec_ready = false;
    int *tin = e->term + e->parity, *tout = e->term + (e->parity ^ 1);
    if (mode == AMZ_RESET_NONE) {
        cudaMemsetAsync(tout, 0, sizeof(int), s);
        e->parity ^= 1;
    }
    int rc = launch_env_step(e->G, e->E, actions, adtype, mode, w, step_idx, step_dev, wrap_dev, view, dirs, reward,
                             done, solved, times,
                             tin, tout, s);
    if (rc) return fail(rc, "step: unsupported agent_view_size");
    return cuda_status("env_step");
}

int amz_env_step(amz_env_t *e, const void *actions, int adtype, int mode, const amz_seed_t *wrap, uint32_t step_idx,
                 uint8_t *view, int64_t *dirs, double *reward, uint8_t *done, double *solved, int64_t *times,
                 void *stream) {
    DevGuard guard_(e->device);
    return env_step_impl(e, actions, adtype, mode, wrap, step_idx, nullptr, nullptr, view, dirs, reward, done, solved,
                         times, stream);
}

int amz_env_step_dev(amz_env_t *e, const void *actions, int adtype, int mode, const amz_seed_t *wrap_dev,
                     const uint32_t *step_dev, uint8_t *view, int64_t *dirs, double *reward, uint8_t *done,
                     double *solved, int64_t *times, void *stream) {
    DevGuard guard_(e->device);
    if (!step_dev) return fail(AMZ_ECONFIG, "null step counter");
    if (mode == AMZ_RESET_NONE) return fail(AMZ_ECONTRACT, "the device-counter step needs an auto-reset mode");
    if (mode == AMZ_RESET_RESAMPLE && !wrap_dev) return fail(AMZ_ECONFIG, "RESAMPLE needs a wrapper key");
    return env_step_impl(e, actions, adtype, mode, nullptr, 0u, step_dev, wrap_dev, view, dirs, reward, done, solved,
                         times, stream);
}

static int env_rollout_impl(amz_env_t *e, int T, const uint8_t *actions, int mode, const amz_seed_t *wrap,
                            uint32_t step0, const uint32_t *iter_dev, uint8_t *view, uint8_t *dirs, double *reward,
                            uint8_t *done, uint8_t *fview, uint8_t *fdir, void *stream);

int amz_env_rollout(amz_env_t *e, int T, const uint8_t *actions, int mode, const amz_seed_t *wrap, uint32_t step0,
                    uint8_t *view, uint8_t *dirs, double *reward, uint8_t *done, uint8_t *fview, uint8_t *fdir,
                    void *stream) {
    return env_rollout_impl(e, T, actions, mode, wrap, step0, nullptr, view, dirs, reward, done, fview, fdir, stream);
}

int amz_env_rollout_iter(amz_env_t *e, int T, const uint8_t *actions, const amz_seed_t *root,
                         const uint32_t *iter_dev, uint8_t *view, uint8_t *dirs, double *reward, uint8_t *done,
                         uint8_t *fview, uint8_t *fdir, void *stream) {
    if (!iter_dev || !root) return fail(AMZ_ECONFIG, "null argument");
    return env_rollout_impl(e, T, actions, AMZ_RESET_RESAMPLE, root, 0u, iter_dev, view, dirs, reward, done, fview,
                            fdir, stream);
}

static int env_rollout_impl(amz_env_t *e, int T, const uint8_t *actions, int mode, const amz_seed_t *wrap,
                            uint32_t step0, const uint32_t *iter_dev, uint8_t *view, uint8_t *dirs, double *reward,
                            uint8_t *done, uint8_t *fview, uint8_t *fdir, void *stream) {
    if (!e || !actions || !view || !dirs || !reward || !done) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(e->device);
    if (T < 1) return fail(AMZ_ECONTRACT, "rollout length must be >= 1, got %d", T);
    if (mode != AMZ_RESET_RESAMPLE && mode != AMZ_RESET_HOME)
        return fail(AMZ_ECONTRACT, "rollout needs an auto-resetting env (mode %d)", mode);
    if (mode == AMZ_RESET_RESAMPLE && !wrap) return fail(AMZ_ECONFIG, "RESAMPLE needs a wrapper key");
    amz_seed_t w = wrap ? *wrap : amz_seed_t{};
    cudaStream_t s = (cudaStream_t)stream;
    if (T > e->rollout_T) {
        cudaFreeAsync(e->poses, s);
        cudaFreeAsync(e->epochs, s);
        e->poses = nullptr;
        e->epochs = nullptr;
        const size_t b = (size_t)e->E.B;
        cudaError_t er = cudaMallocAsync((void **)&e->poses, (((size_t)T + 3) / 4) * 4 * b * sizeof(uint32_t), s);
        if (er == cudaSuccess) er = cudaMallocAsync((void **)&e->epochs, ((size_t)T + 1) * b * 20 * sizeof(uint32_t), s);
        if (er != cudaSuccess) {
            e->rollout_T = 0;
            return fail(AMZ_ECUDA, "rollout scratch: %s", cudaGetErrorString(er));
        }
        e->rollout_T = T;
    }
    const bool ready = e->spec_ready && mode == AMZ_RESET_RESAMPLE && step0 == 0 && e->spec_iter == iter_dev &&
                       memcmp(&e->spec_wrap, &w, sizeof(w)) == 0;
    e->spec_ready = false;
    EnvDev E = e->E;
    E.iter = iter_dev;
    int rc = launch_env_rollout(e->G, E, T, actions, mode, w, step0, view, dirs, reward, done, fview, fdir,
                                e->poses, e->epochs, e->final_pose, e->spec, e->spec_step, ready ? 1 : 0, s);
    if (rc) return fail(rc, "rollout: unsupported agent_view_size");
    return cuda_status("env_rollout");
}

int amz_env_observe(amz_env_t *e, uint8_t *view, int64_t *dirs, void *stream) {
    if (!e) return fail(AMZ_ECONFIG, "null env");
    DevGuard guard_(e->device);
    int rc = launch_env_observe(e->G, e->E, view, dirs, (cudaStream_t)stream);
    if (rc) return fail(rc, "observe: unsupported agent_view_size");
    return cuda_status("env_observe");
}

int amz_env_levels(amz_env_t *e, amz_level_t *out, void *stream) {
    if (!e || !out) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(e->device);
    launch_env_levels(e->E, out, (cudaStream_t)stream);
    return cuda_status("env_levels");
}

int amz_env_state(amz_env_t *e, int32_t *out, void *stream) {
    if (!e || !out) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(e->device);
    launch_env_state(e->E, out, (cudaStream_t)stream);
    return cuda_status("env_state");
}

int amz_env_set_state(amz_env_t *e, const int32_t *in, void *stream) {
    if (!e || !in) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(e->device);
    e->spec_ready = false;
    launch_env_set_state(e->E, in, (cudaStream_t)stream);
    return cuda_status("env_set_state");
}

int amz_env_check(amz_env_t *e, void *stream) {
    if (!e) return fail(AMZ_ECONFIG, "null env");
    DevGuard guard_(e->device);
    cudaStream_t s = (cudaStream_t)stream;
    int h = 0;
    AMZ_CHECK_CUDA(cudaMemcpyAsync(&h, e->E.err, sizeof(int), cudaMemcpyDeviceToHost, s), "env_check");
    AMZ_CHECK_CUDA(cudaStreamSynchronize(s), "env_check");
    if (h) {
        cudaMemsetAsync(e->E.err, 0, sizeof(int), s);
        cudaStreamSynchronize(s);
        if (h & 2) return fail(AMZ_ECONTRACT, "reset_to_levels: lane index out of range");
        return fail(AMZ_ECONTRACT, "step_batch called with terminal lanes");
    }
    return 0;
}

int amz_gae_score(int T, int64_t B, const double *r, const double *v, const uint8_t *d, const double *last,
                  double gamma, double lam, const double *prior, int score_fn, int disc, double *adv, double *ret,
                  double *scores, double *maxret, const amz_episode_stats_t *stats, void *stream) {
    if (T < 1) return fail(AMZ_ECONTRACT, "cannot score an empty trajectory slice");
    if (B < 0) return fail(AMZ_ESHAPE, "negative lane count");
    if (!r || !v || !d || !last || !adv || !ret) return fail(AMZ_ECONFIG, "null argument");
    if ((score_fn & 0xFF) != AMZ_SCORE_MAXMC && (score_fn & 0xFF) != AMZ_SCORE_PVL)
        return fail(AMZ_ECONFIG, "unknown score_fn %d", score_fn);
    if ((score_fn & AMZ_SCORE_PRIOR_FINAL) && !prior) return fail(AMZ_ECONFIG, "PRIOR_FINAL needs prior_max");
    int rc = launch_gae_score(T, B, r, v, d, last, gamma, lam, prior, score_fn, disc, adv, ret, scores, maxret, stats,
                              (cudaStream_t)stream);
    if (rc) return fail(rc, "gae_score: T=%d too long for the pairwise schedule", T);
    return cuda_status("gae_score");
}

int amz_gae_score_v32(int T, int64_t B, const double *r, const float *v, const uint8_t *d, const float *last,
                      double gamma, double lam, const double *prior, int score_fn, int disc, double *adv,
                      double *ret, double *scores, double *maxret, const amz_episode_stats_t *stats, void *stream) {
    if (T < 1) return fail(AMZ_ECONTRACT, "cannot score an empty trajectory slice");
    if (B < 0) return fail(AMZ_ESHAPE, "negative lane count");
    if (!r || !v || !d || !last || !adv || !ret) return fail(AMZ_ECONFIG, "null argument");
    if ((score_fn & 0xFF) != AMZ_SCORE_MAXMC && (score_fn & 0xFF) != AMZ_SCORE_PVL)
        return fail(AMZ_ECONFIG, "unknown score_fn %d", score_fn);
    if ((score_fn & AMZ_SCORE_PRIOR_FINAL) && !prior) return fail(AMZ_ECONFIG, "PRIOR_FINAL needs prior_max");
    int rc = launch_gae_score_v32(T, B, r, v, d, last, gamma, lam, prior, score_fn, disc, adv, ret, scores, maxret,
                                  stats, (cudaStream_t)stream);
    if (rc) return fail(rc, "gae_score: T=%d too long for the pairwise schedule", T);
    return cuda_status("gae_score_v32");
}

int amz_lane_scores(int T, int64_t B, const double *r, const double *v, const uint8_t *d, const double *adv,
                    double gamma, const double *prior, int score_fn, int disc, double *scores, double *maxret,
                    const amz_episode_stats_t *stats, void *stream) {
    if (T < 1) return fail(AMZ_ECONTRACT, "cannot score an empty trajectory slice");
    if (B < 0) return fail(AMZ_ESHAPE, "negative lane count");
    if (!r || !v || !d || !scores || !maxret || (score_fn == AMZ_SCORE_PVL && !adv))
        return fail(AMZ_ECONFIG, "null argument");
    if ((score_fn & 0xFF) != AMZ_SCORE_MAXMC && (score_fn & 0xFF) != AMZ_SCORE_PVL)
        return fail(AMZ_ECONFIG, "unknown score_fn %d", score_fn);
    if ((score_fn & AMZ_SCORE_PRIOR_FINAL) && !prior) return fail(AMZ_ECONFIG, "PRIOR_FINAL needs prior_max");
    int rc = launch_gae_score(T, B, r, v, d, nullptr, gamma, 1.0, prior, score_fn, disc, (double *)adv, nullptr,
                              scores, maxret, stats, (cudaStream_t)stream, 0);
    if (rc) return fail(rc, "lane_scores: T=%d too long for the pairwise schedule", T);
    return cuda_status("lane_scores");
}

int amz_plr_create(int64_t capacity, amz_plr_t **out) {
    if (!out) return fail(AMZ_ECONFIG, "null argument");
    if (capacity < 1 || capacity > 4096) return fail(AMZ_ECONFIG, "buffer_size must be in [1, 4096], got %lld",
                                                     (long long)capacity);
    amz_plr *b = new (std::nothrow) amz_plr();
    if (!b) return fail(AMZ_EFAULT, "out of host memory");
    b->device = current_device();
    b->D.K = capacity;
    size_t K = (size_t)capacity;
    cudaError_t e = cudaMalloc((void **)&b->D.levels, K * sizeof(amz_level_t));
    if (e == cudaSuccess) e = cudaMalloc((void **)&b->D.score, K * 8);
    if (e == cudaSuccess) e = cudaMalloc((void **)&b->D.maxret, K * 8);
    if (e == cudaSuccess) e = cudaMalloc((void **)&b->D.last, K * 8);
    if (e == cudaSuccess) e = cudaMalloc((void **)&b->D.seq, K * 8);
    if (e == cudaSuccess) e = cudaMalloc((void **)&b->D.meta, 2 * 8);
    if (e == cudaSuccess) e = cudaMalloc((void **)&b->err, 4 * sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc((void **)&b->rank, K * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemset(b->D.meta, 0, 16);
    if (e == cudaSuccess) e = cudaMemset(b->err, 0, 4 * sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(b->D.levels, 0, K * sizeof(amz_level_t));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        amz_plr_destroy(b);
        return fail(AMZ_ECUDA, "plr alloc: %s", cudaGetErrorString(e));
    }
    *out = b;
    return 0;
}

int amz_plr_destroy(amz_plr_t *b) {
    if (!b) return 0;
    DevGuard guard_(b->device);
    cudaDeviceSynchronize();
    cudaFree(b->D.levels);
    cudaFree(b->D.score);
    cudaFree(b->D.maxret);
    cudaFree(b->D.last);
    cudaFree(b->D.seq);
    cudaFree(b->D.meta);
    cudaFree(b->err);
    cudaFree(b->rank);
    cudaFree(b->W.init_match);
    cudaFree(b->W.twin_first);
    cudaFree(b->W.keyslot);
    cudaFree(b->W.rel);
    cudaFree(b->W.chash);
    delete b;
    return 0;
}

int amz_plr_update(amz_plr_t *b, const amz_level_t *levels, const double *scores, const double *max_ret, int64_t n,
                   int64_t iter, void *stream) {
    if (!b || (n > 0 && (!levels || !scores || !max_ret))) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(b->device);
    if (n < 0) return fail(AMZ_ESHAPE, "negative candidate count");
    if (n > ((int64_t)1 << 30)) return fail(AMZ_ESHAPE, "too many candidates");
    cudaStream_t s = (cudaStream_t)stream;
    const int prepared = b->prep_cand == levels && b->prep_n == n && n > 0;
    b->prep_cand = nullptr;
    b->prep_n = -1;
    if (!prepared) {
        int rc = plr_scratch(b, n, s);
        if (rc) return rc;
    }
    launch_plr_update(b->D, levels, scores, max_ret, n, iter, b->W, b->err, s, prepared);
    return cuda_status("plr_update");
}

int amz_plr_prepare(amz_plr_t *b, const amz_level_t *levels, int64_t n, void *stream) {
    if (!b || (n > 0 && !levels)) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(b->device);
    if (n < 0) return fail(AMZ_ESHAPE, "negative candidate count");
    if (n > ((int64_t)1 << 30)) return fail(AMZ_ESHAPE, "too many candidates");
    cudaStream_t s = (cudaStream_t)stream;
    int rc = plr_scratch(b, n, s);
    if (rc) return rc;
    launch_plr_prepare(b->D, levels, n, b->W, s);
    b->prep_cand = levels;
    b->prep_n = n;
    return cuda_status("plr_prepare");
}

int amz_plr_sample(amz_plr_t *b, const amz_seed_t *key, int64_t n, double rho, const double *lut, int64_t iter,
                   int32_t *slots, amz_level_t *levels, double *max_ret, double *score, void *stream) {
    if (!b || !key || !lut || (n > 0 && !slots)) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(b->device);
    if (rho < 0.0 || rho > 1.0) return fail(AMZ_ECONFIG, "staleness_coef must be in [0, 1], got %g", rho);
    if (n <= 0) return 0;
    launch_plr_sample(b->D, b->rank, *key, n, 1.0 - rho, rho, lut, 0, 0.0, iter, slots, levels, max_ret, score,
                      b->err, (cudaStream_t)stream);
    return cuda_status("plr_sample");
}

int amz_plr_sample_proportional(amz_plr_t *b, const amz_seed_t *key, int64_t n, double rho, double temperature,
                                int64_t iter, int32_t *slots, amz_level_t *levels, double *max_ret, double *score,
                                void *stream) {
    if (!b || !key || (n > 0 && !slots)) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(b->device);
    if (rho < 0.0 || rho > 1.0) return fail(AMZ_ECONFIG, "staleness_coef must be in [0, 1], got %g", rho);
    if (!(temperature > 0.0)) return fail(AMZ_ECONFIG, "temperature must be > 0, got %g", temperature);
    if (n <= 0) return 0;
    launch_plr_sample(b->D, b->rank, *key, n, 1.0 - rho, rho, nullptr, 1, 1.0 / temperature, iter, slots, levels,
                      max_ret, score, b->err, (cudaStream_t)stream);
    return cuda_status("plr_sample_proportional");
}

int amz_plr_top_q(const double *scores, int64_t n, int q, int32_t *out, void *stream) {
    if (!scores || !out) return fail(AMZ_ECONFIG, "null argument");
    if (q < 1 || q > 64 || q > n) return fail(AMZ_ECONFIG, "subsample size q=%d must be in [1, min(64, %lld)]", q,
                                              (long long)n);
    launch_top_q(scores, n, q, out, (cudaStream_t)stream);
    return cuda_status("plr_top_q");
}

int amz_plr_size(amz_plr_t *b, int64_t *size, void *stream) {
    if (!b || !size) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(b->device);
    cudaStream_t s = (cudaStream_t)stream;
    int64_t meta[2];
    int err = 0;
    AMZ_CHECK_CUDA(cudaMemcpyAsync(meta, b->D.meta, 16, cudaMemcpyDeviceToHost, s), "plr_size");
    AMZ_CHECK_CUDA(cudaMemcpyAsync(&err, b->err, sizeof(int), cudaMemcpyDeviceToHost, s), "plr_size");
    AMZ_CHECK_CUDA(cudaStreamSynchronize(s), "plr_size");
    *size = meta[0];
    if (err) {
        cudaMemsetAsync(b->err, 0, sizeof(int), s);
        cudaStreamSynchronize(s);
        if (err & 4)
            return fail(AMZ_ECONTRACT, "buffer_update refused: last_sampled / seq spans exceed a 64-bit tie key");
        if (err & 8)
            return fail(AMZ_ECONTRACT, "proportional sampling: NaN probabilities (a negative score, or every score 0)");
        return fail(AMZ_ECONTRACT, "sampled from an empty level buffer");
    }
    return 0;
}

int amz_plr_digest(amz_plr_t *b, int64_t *out_dev, void *stream) {
    if (!b || !out_dev) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(b->device);
    launch_plr_digest(b->D, out_dev, (cudaStream_t)stream);
    return cuda_status("plr_digest");
}

int amz_plr_export(amz_plr_t *b, amz_level_t *levels, double *score, double *max_ret, int64_t *last, int64_t *seq,
                   int64_t *meta, void *stream) {
    if (!b) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(b->device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t K = (size_t)b->D.K;
    if (levels) cudaMemcpyAsync(levels, b->D.levels, K * sizeof(amz_level_t), cudaMemcpyDeviceToDevice, s);
    if (score) cudaMemcpyAsync(score, b->D.score, K * 8, cudaMemcpyDeviceToDevice, s);
    if (max_ret) cudaMemcpyAsync(max_ret, b->D.maxret, K * 8, cudaMemcpyDeviceToDevice, s);
    if (last) cudaMemcpyAsync(last, b->D.last, K * 8, cudaMemcpyDeviceToDevice, s);
    if (seq) cudaMemcpyAsync(seq, b->D.seq, K * 8, cudaMemcpyDeviceToDevice, s);
    if (meta) cudaMemcpyAsync(meta, b->D.meta, 16, cudaMemcpyDeviceToDevice, s);
    return cuda_status("plr_export");
}

int amz_plr_import(amz_plr_t *b, const amz_level_t *levels, const double *score, const double *max_ret,
                   const int64_t *last, const int64_t *seq, const int64_t *meta, void *stream) {
    if (!b || !levels || !score || !max_ret || !last || !seq || !meta) return fail(AMZ_ECONFIG, "null argument");
    DevGuard guard_(b->device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t K = (size_t)b->D.K;
    cudaMemcpyAsync(b->D.levels, levels, K * sizeof(amz_level_t), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(b->D.score, score, K * 8, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(b->D.maxret, max_ret, K * 8, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(b->D.last, last, K * 8, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(b->D.seq, seq, K * 8, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(b->D.meta, meta, 16, cudaMemcpyDeviceToDevice, s);
    return cuda_status("plr_import");
}

}  // extern "C"
