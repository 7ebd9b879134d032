// K2 fixed-cost decomposition (tools/, not product): event-timed empty kernel, then ffn_rows_kernel
// over one segment with growing ffn rows (cold: rotating 32 distinct tiles), d = 4096.
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/k2_floor tools/k2_floor.cu
#include <cstdio>

#include "../paper_2408_10284_b200/csrc/kernels/expert_ffn.cu"

using namespace adapmoe;

__global__ void empty_kernel() {}

int main() {
    const int D = 4096, NT = 32, FMAX = 3584;
    const size_t tile_elems = (size_t)3 * FMAX * D;
    uint16_t* w;
    cudaMalloc(&w, tile_elems * 2 * NT);
    cudaMemset(w, 0x3c, tile_elems * 2 * NT);
    double* x;
    cudaMalloc(&x, D * 8);
    cudaMemset(x, 0, D * 8);
    float* part;
    cudaMalloc(&part, (size_t)kFfnMaxCtas * kFfnSlotsPerCta * D * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto&& fn) {
        double s = 0;
        for (int rep = 0; rep < 44; ++rep) {
            cudaEventRecord(a);
            fn(rep);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep >= 4) s += ms;
        }
        return s / 40 * 1e3;
    };
    printf("empty kernel <<<148, 512>>>: %.2f us\n", timeit([&](int) { empty_kernel<<<148, 512>>>(); }));
    for (int ft : {148, 296, 592, 1184, 2368, 3584}) {
        const double us = timeit([&](int rep) {
            FfnLaunch p;
            p.n_seg = 1;
            p.d = D;
            p.ft = ft;
            p.x = x;
            p.partial = part;
            const uint16_t* t = w + (rep % NT) * tile_elems;
            p.seg[0].gate_up = t;
            p.seg[0].down_t = t + (size_t)2 * ft * D;
            launch_ffn(p, 148, 0);
        });
        const double bytes = 3.0 * ft * D * 2;
        printf("K2 nseg=1 ft=%4d (%5.1f rows/CTA, %5.1f MB): %6.2f us = %5.0f GB/s (%s)\n", ft, ft / 148.0, bytes / 1e6,
               us, bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
