// Latency of one warp-cooperative level sample, phase by phase (tools only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I paper_2311_12716_b200/csrc \
//      -o tools/_prof/samp_lat tools/samp_lat.cu
#include <cstdio>
#include "amz_internal.h"
#include "amz_rng.cuh"
#include "amz_sampler.cuh"
using namespace amz;

__global__ void k_lat(Geo G, amz_seed_t pre, int n, long long *out, int track) {
    __shared__ WarpSampler X;
    long long tot_seed = 0, tot_samp = 0;
    for (int i = 0; i < n; i++) {
        long long t0 = clock64();
        amz_seed_t sd = pre;
        seed_absorb(sd, 1000u + i);
        seed_absorb(sd, 7u);
        uint64_t k0, k1;
        seed_key(sd, k0, k1);
        k0 = __shfl_sync(0xFFFFFFFFu, k0, 0);
        long long t1 = clock64();
        Mask m;
        int ar, ac, ad, gr, gc;
        if (track) warp_sample_level<true>(k0, k1, G, X, m, ar, ac, ad, gr, gc);
        else warp_sample_level<false>(k0, k1, G, X, m, ar, ac, ad, gr, gc);
        long long t2 = clock64();
        tot_seed += t1 - t0;
        tot_samp += t2 - t1;
        if (m.w[0] == 12345 && ar == 99) out[3] = 1;  // keep results live
    }
    if (threadIdx.x == 0) { out[0] = tot_seed / n; out[1] = tot_samp / n; }
}

int main() {
    amz_params_t p{13, 13, 250, 5, 60, 1};
    Geo G = make_geo(p);
    uint32_t run[1] = {5}, key[1] = {1};
    amz_seed_t pre;
    seed_prefix_host(run, 1, key, 1, pre);
    long long *d;
    cudaMalloc(&d, 64);
    for (int track = 0; track < 2; track++) {
        k_lat<<<1, 32>>>(G, pre, 200, d, track);
        long long h[4];
        cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        printf("track=%d seed cycles %lld, sample cycles %lld\n", track, h[0], h[1]);
    }
    return 0;
}
