// amz_metrics.cu -- per-level curriculum metrics on packed levels:
// env_metrics (amaze/metrics.py:21-31) = interior wall count, agent -> goal shortest
// path length by single-source grid BFS (amaze/pathfinding.py:116-135), solvable flag,
// passable ratio 1 - mean(interior walls) in float64.
//
// One thread per level.  The grid lives in 16 registers of row bits (bit c = column
// c); a BFS wave is the 4-neighbour dilation (f << 1 | f >> 1 | f[r-1] | f[r+1]) masked
// by free and unvisited cells -- ~5 integer ops per row, no memory traffic -- and the
// search stops at the first wave that contains the goal.
#include <cuda_runtime.h>
#include <stdint.h>

#include "amz_internal.h"
#include "amz_level.cuh"

namespace amz {

__global__ void __launch_bounds__(128) k_level_metrics(Geo G, const amz_level_t *__restrict__ lv, int64_t n,
                                                       int32_t *__restrict__ n_walls, int32_t *__restrict__ spl,
                                                       uint8_t *__restrict__ solvable,
                                                       double *__restrict__ passable) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Mask m;
    int ar, ac, ad, gr, gc;
    load_level(lv + i, m, ar, ac, ad, gr, gc);
    const uint32_t full = (1u << G.W) - 1u;
    uint32_t fr[16], f[16], vis[16];
#pragma unroll
    for (int r = 0; r < 16; r++) {
        uint32_t wall;
        if (r == 0 || r == G.H - 1)
            wall = full;
        else if (r < G.H - 1)
            wall = 1u | (mask_bits(m, (r - 1) * G.iw, G.iw) << 1) | (1u << (G.W - 1));
        else
            wall = full;  // rows past the grid: nothing to reach
        fr[r] = ~wall & full;
        f[r] = (r == ar) ? (1u << ac) : 0u;
        vis[r] = f[r];
    }
    int nw = __popc(m.w[0]) + __popc(m.w[1]) + __popc(m.w[2]) + __popc(m.w[3]);
    int d = -1;
    const bool src_free = (fr[ar & 15] >> ac) & 1u;
    if (src_free) {
        for (int dd = 0;; dd++) {
            uint32_t at_goal = 0u, any = 0u;
#pragma unroll
            for (int r = 0; r < 16; r++) {
                at_goal |= (r == gr) ? (f[r] >> gc) & 1u : 0u;
                any |= f[r];
            }
            if (at_goal) {
                d = dd;
                break;
            }
            if (!any) break;
            uint32_t g2[16];
#pragma unroll
            for (int r = 0; r < 16; r++) {
                const uint32_t up = r > 0 ? f[r - 1] : 0u, dn = r < 15 ? f[r + 1] : 0u;
                g2[r] = ((f[r] << 1) | (f[r] >> 1) | up | dn) & fr[r] & ~vis[r];
            }
#pragma unroll
            for (int r = 0; r < 16; r++) {
                f[r] = g2[r];
                vis[r] |= g2[r];
            }
        }
    }
    if (n_walls) n_walls[i] = nw;
    if (spl) spl[i] = d >= 0 ? d : 0;
    if (solvable) solvable[i] = d >= 0;
    // 1.0 - interior.mean(): the bool mean is an exact count over ni, then one division
    if (passable) passable[i] = __dsub_rn(1.0, __ddiv_rn((double)nw, (double)G.ni));
}

int launch_level_metrics(const Geo &G, const amz_level_t *lv, int64_t n, int32_t *n_walls, int32_t *spl,
                         uint8_t *solvable, double *passable, cudaStream_t s) {
    if (n <= 0) return 0;
    k_level_metrics<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(G, lv, n, n_walls, spl, solvable, passable);
    return 0;
}

}  // namespace amz
