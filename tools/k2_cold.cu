// K2 cold-cache microbenchmark (tools/, not product): launches rotate over 32 distinct 88 MB tiles
// (2.8 GB > 126 MB L2) so every launch streams from HBM, as in the decode.  Compares the L2
// prefetch modes for small launches (1 - 8 segments) and reports the combine time.
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/k2_cold tools/k2_cold.cu
#include <cstdio>
#include <vector>

#include "../paper_2408_10284_b200/csrc/kernels/expert_ffn.cu"

using namespace adapmoe;

__global__ void fill(uint16_t* w, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        w[i] = 0x3c00 + (uint16_t)((i * 2654435761u) & 0x3ff) - 0x200;
}

int main() {
    const int D = 4096, Ft = 3584, NT = 32;
    const size_t tile_elems = (size_t)3 * Ft * D, tile_bytes = tile_elems * 2;
    uint16_t* w;
    cudaMalloc(&w, tile_bytes * NT);
    fill<<<148 * 8, 256>>>(w, tile_elems * NT);
    double* x;
    cudaMalloc(&x, D * 8);
    cudaMemset(x, 0, D * 8);
    float *part, *out;
    cudaMalloc(&part, (size_t)8 * kFfnMaxCtas * kFfnSlotsPerCta * D * 4);
    cudaMalloc(&out, D * 4);
    double* sc;
    cudaMalloc(&sc, 64 * 8);
    cudaMemset(sc, 0, 64 * 8);
    cudaEvent_t a, b, c;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventCreate(&c);
    for (int nseg : {1, 2, 4, 8, 16}) {
        for (int mode : {0}) {
            double sum_ms = 0, sum_c = 0;
            int n = 0;
            for (int rep = 0; rep < 24; ++rep) {
                FfnLaunch p;
                p.n_seg = nseg;
                p.d = D;
                p.ft = Ft;
                p.x = x;
                p.partial = part;
                (void)mode;  // L2 prefetch modes measured slower and removed (profiles/r1_k2_variants.txt)
                for (int s = 0; s < nseg; ++s) {
                    const uint16_t* t = w + ((rep * nseg + s) % NT) * tile_elems;
                    p.seg[s].gate_up = t;
                    p.seg[s].down_t = t + (size_t)2 * Ft * D;
                }
                CombineArgs ca;
                ca.x = x;
                ca.scores = sc;
                ca.out = out;
                ca.ranks = 1;
                ca.d = D;
                ca.ft = Ft;
                ca.n_refs = nseg;
                for (int s = 0; s < nseg; ++s) {
                    ca.refs[s] = FfnPartialRef{part, ffn_grid(p, 148), nseg, s, 0};
                    ffn_partial_range(ca.refs[s], Ft);
                }
                cudaEventRecord(a);
                launch_ffn(p, 148, 0);
                cudaEventRecord(b);
                launch_combine(ca, 0);
                cudaEventRecord(c);
                cudaEventSynchronize(c);
                float ms, mc;
                cudaEventElapsedTime(&ms, a, b);
                cudaEventElapsedTime(&mc, b, c);
                if (rep >= 4) {
                    sum_ms += ms;
                    sum_c += mc;
                    ++n;
                }
            }
            const double bytes = (double)nseg * tile_bytes;
            printf("K2 cold nseg=%2d l2_mode=%d: mean %.1f us = %.0f GB/s | combine %.1f us  (%s)\n", nseg, mode,
                   sum_ms / n * 1e3, bytes / (sum_ms / n * 1e-3) / 1e9, sum_c / n * 1e3,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
