// amz_teacher.cu -- the PAIRED level-designer decision process, batched (SURVEY §8f
// row 3; amaze/teacher.py:36-159).  A lane builds one maze in wall_budget + 2 steps:
// aimed wall placements (no-op on a wall), then the goal (clears a wall under it), then
// the agent (first free non-goal cell at or after the aimed one in the wrapping
// row-major interior scan).  The design reuses the 128-bit interior mask of amz_level_t,
// so a finished lane decodes to a level record with no conversion.
//
// Lane state (SoA): mask[B] uint4 (interior walls) and st[B] uint4:
//   x = n_placed | phase << 16;  y = goal r | c << 8 | has_goal << 16;
//   z = agent r | c << 8 | has_agent << 16;  w = time | terminal << 31.
#include <cuda_runtime.h>
#include <stdint.h>

#include "amz_internal.h"
#include "amz_level.cuh"

namespace amz {

enum { kPhaseWalls = 0, kPhaseGoal = 1, kPhaseAgent = 2, kPhaseDone = 3 };

// teacher_observe (amaze/teacher.py:100-107): grid u8 [H][W] tile codes (wall 1, goal 2),
// phase f32 one-hot [4], n_placed i64
__device__ __forceinline__ void teacher_observe(const Geo &G, const Mask &m, uint4 st, uint8_t *grid, float *phase,
                                                int64_t *n_placed) {
    const int ph = (int)(st.x >> 16), np_ = (int)(st.x & 0xFFFFu);
    const bool hg = (st.y >> 16) & 1u;
    const int gr = st.y & 0xFF, gc = (st.y >> 8) & 0xFF;
    for (int r = 0; r < G.H; r++) {
        const uint32_t row =
            (r == 0 || r == G.H - 1) ? 0xFFFFu : (1u | (mask_bits(m, (r - 1) * G.iw, G.iw) << 1) | (1u << (G.W - 1)));
        for (int c = 0; c < G.W; c++) {
            uint8_t code = (uint8_t)((row >> c) & 1u);
            if (hg && r == gr && c == gc) code = 2;
            grid[r * G.W + c] = code;
        }
    }
    if (phase)
        for (int k = 0; k < 4; k++) phase[k] = k == ph ? 1.0f : 0.0f;
    if (n_placed) *n_placed = np_;
}

__global__ void k_teacher_reset(Geo G, int64_t B, uint4 *__restrict__ mask, uint4 *__restrict__ st,
                                uint8_t *__restrict__ grid, float *__restrict__ phase, int64_t *__restrict__ n_placed) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= B) return;
    Mask m;
    m.w[0] = m.w[1] = m.w[2] = m.w[3] = 0u;
    const int ph = G.budget > 0 ? kPhaseWalls : kPhaseGoal;
    const uint4 s = make_uint4((uint32_t)ph << 16, 0u, 0u, 0u);
    mask[l] = make_uint4(0u, 0u, 0u, 0u);
    st[l] = s;
    teacher_observe(G, m, s, grid + l * G.H * G.W, phase ? phase + 4 * l : nullptr, n_placed ? n_placed + l : nullptr);
}

// first set bit of the 128-bit mask at or after bit k, wrapping; -1 if empty
__device__ __forceinline__ int mask_next_wrap(const Mask &m, int k, int n) {
    for (int pass = 0; pass < 2; pass++) {
        const int lo = pass == 0 ? k : 0, hi = pass == 0 ? n : k;
        for (int w = lo >> 5; w < 4 && w * 32 < hi; w++) {
            uint32_t bits = mask_word(m, w);
            if (w == (lo >> 5)) bits &= ~0u << (lo & 31);
            const int top = hi - w * 32;
            if (top < 32) bits &= (top <= 0) ? 0u : ((1u << top) - 1u);
            if (bits) return w * 32 + __ffs(bits) - 1;
        }
    }
    return -1;
}

__global__ void k_teacher_step(Geo G, int64_t B, uint4 *__restrict__ mask, uint4 *__restrict__ st,
                               const int64_t *__restrict__ actions, uint8_t *__restrict__ grid,
                               float *__restrict__ phase, int64_t *__restrict__ n_placed, uint8_t *__restrict__ done,
                               int64_t *__restrict__ times, int *__restrict__ err) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= B) return;
    uint4 s = st[l];
    const uint4 mw = mask[l];
    Mask m;
    m.w[0] = mw.x;
    m.w[1] = mw.y;
    m.w[2] = mw.z;
    m.w[3] = mw.w;
    const int64_t a = actions[l];
    bool bad = false;
    if (s.w >> 31) {  // teacher_step on a finished design (amaze/teacher.py:61-62)
        atomicOr(err, 1);
        bad = true;
    } else if (a < 0 || a >= G.ni) {  // _cell_of (amaze/teacher.py:52-57)
        atomicOr(err, 2);
        bad = true;
    }
    if (!bad) {
        const int i = (int)a;
        const int ph = (int)(s.x >> 16);
        int np_ = (int)(s.x & 0xFFFFu), nph = ph;
        if (ph == kPhaseWalls) {
            mask_set(m, i, 1u);
            np_++;
            nph = np_ >= G.budget ? kPhaseGoal : kPhaseWalls;
        } else if (ph == kPhaseGoal) {
            m.w[i >> 5] &= ~(1u << (i & 31));
            s.y = (uint32_t)(1 + i / G.iw) | ((uint32_t)(1 + i % G.iw) << 8) | (1u << 16);
            nph = kPhaseAgent;
        } else {  // agent: first free non-goal cell at or after i, wrapping
            Mask fr;
            for (int w = 0; w < 4; w++) fr.w[w] = ~mask_word(m, w);
            const int gi = ((int)(s.y & 0xFF) - 1) * G.iw + ((int)((s.y >> 8) & 0xFF) - 1);
            fr.w[gi >> 5] &= ~(1u << (gi & 31));
            const int k = mask_next_wrap(fr, i, G.ni);
            if (k < 0) {
                atomicOr(err, 4);  // unreachable under the wall_budget bound (amaze/teacher.py:87)
            } else {
                s.z = (uint32_t)(1 + k / G.iw) | ((uint32_t)(1 + k % G.iw) << 8) | (1u << 16);
                nph = kPhaseDone;
            }
        }
        const uint32_t t = (s.w & 0x7FFFFFFFu) + 1u;
        s.x = (uint32_t)np_ | ((uint32_t)nph << 16);
        s.w = t | ((nph == kPhaseDone) ? 0x80000000u : 0u);
        mask[l] = make_uint4(m.w[0], m.w[1], m.w[2], m.w[3]);
        st[l] = s;
    }
    teacher_observe(G, m, s, grid + l * G.H * G.W, phase ? phase + 4 * l : nullptr, n_placed ? n_placed + l : nullptr);
    if (done) done[l] = (uint8_t)(s.w >> 31);
    if (times) times[l] = (int64_t)(s.w & 0x7FFFFFFFu);
}

// decode_teacher_level (amaze/teacher.py:90-97): agent faces north
__global__ void k_teacher_levels(int64_t B, const uint4 *__restrict__ mask, const uint4 *__restrict__ st,
                                 amz_level_t *__restrict__ out, int *__restrict__ err) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= B) return;
    const uint4 s = st[l];
    if (!(s.w >> 31)) {
        atomicOr(err, 8);
        return;
    }
    const uint4 mw = mask[l];
    Mask m;
    m.w[0] = mw.x;
    m.w[1] = mw.y;
    m.w[2] = mw.z;
    m.w[3] = mw.w;
    store_level(out + l, m, (int)(s.z & 0xFF), (int)((s.z >> 8) & 0xFF), 0, (int)(s.y & 0xFF), (int)((s.y >> 8) & 0xFF));
}

int launch_teacher_reset(const Geo &G, int64_t B, uint4 *mask, uint4 *st, uint8_t *grid, float *phase,
                         int64_t *n_placed, cudaStream_t s) {
    if (B <= 0) return 0;
    k_teacher_reset<<<(unsigned)((B + 127) / 128), 128, 0, s>>>(G, B, mask, st, grid, phase, n_placed);
    return 0;
}
int launch_teacher_step(const Geo &G, int64_t B, uint4 *mask, uint4 *st, const int64_t *actions, uint8_t *grid,
                        float *phase, int64_t *n_placed, uint8_t *done, int64_t *times, int *err, cudaStream_t s) {
    if (B <= 0) return 0;
    k_teacher_step<<<(unsigned)((B + 127) / 128), 128, 0, s>>>(G, B, mask, st, actions, grid, phase, n_placed, done,
                                                               times, err);
    return 0;
}
int launch_teacher_levels(int64_t B, const uint4 *mask, const uint4 *st, amz_level_t *out, int *err, cudaStream_t s) {
    if (B <= 0) return 0;
    k_teacher_levels<<<(unsigned)((B + 127) / 128), 128, 0, s>>>(B, mask, st, out, err);
    return 0;
}

}  // namespace amz
