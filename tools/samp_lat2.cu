// phase timing of warp_sample_level<true> (tools only): build with -DAMZ_SAMP_PROF
#include <cstdio>
#include "amz_internal.h"
#include "amz_rng.cuh"
#include "amz_sampler.cuh"
using namespace amz;
__global__ void k_lat(Geo G, amz_seed_t pre, int n, long long *out) {
    __shared__ WarpSampler X;
    long long acc[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < n; i++) {
        amz_seed_t sd = pre;
        seed_absorb(sd, 1000u + i);
        seed_absorb(sd, 7u);
        uint64_t k0, k1;
        seed_key(sd, k0, k1);
        for (int k = 0; k < 6; k++) if (threadIdx.x == 0) g_samp_prof[k] = 0;
        __syncwarp();
        Mask m;
        int ar, ac, ad, gr, gc;
        warp_sample_level<true>(k0, k1, G, X, m, ar, ac, ad, gr, gc);
        __syncwarp();
        for (int k = 1; k < 6; k++) acc[k] += g_samp_prof[k] - g_samp_prof[k - 1];
        if (m.w[0] == 12345 && ar == 99) out[7] = 1;
    }
    if (threadIdx.x == 0) for (int k = 1; k < 6; k++) out[k] = acc[k] / n;
}
int main() {
    amz_params_t p{13, 13, 250, 5, 60, 1};
    Geo G = make_geo(p);
    uint32_t run[1] = {5}, key[1] = {1};
    amz_seed_t pre;
    seed_prefix_host(run, 1, key, 1, pre);
    long long *d;
    cudaMalloc(&d, 64);
    k_lat<<<1, 32>>>(G, pre, 200, d);
    long long h[8];
    cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("stage %lld, nw draw %lld, jacobi %lld, track %lld, tail %lld\n", h[1], h[2], h[3], h[4], h[5]);
    return 0;
}
