// Microbenchmark (tools/, not product): fp64 DADD chain latency and throughput on the GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, const double* p, int n, int active) {
    double acc = 0.0;
    if (threadIdx.x < active) {
#pragma unroll 8
        for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, p[i & 255]);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void chain_f32(float* out, const float* p, int n) {
    float acc = 0.0f;
#pragma unroll 8
    for (int i = 0; i < n; ++i) acc = __fadd_rn(acc, p[i & 255]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void thru(double* out, double a, int n) {
    double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
    for (int i = 0; i < n; ++i) {
        x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
        x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, a); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, a);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

int main() {
    double *out, *p;
    float *outf, *pf;
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&p, 256 * 8);
    cudaMalloc(&outf, 1 << 24);
    cudaMalloc(&pf, 256 * 4);
    cudaMemset(p, 0, 256 * 8);
    cudaMemset(pf, 0, 256 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int n = 1 << 16;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int active : {1, 8, 32}) {
        for (int warps : {1, 4}) {
            chain<<<1, 32 * warps>>>(out, p, n, active);
            cudaEventRecord(a);
            chain<<<1, 32 * warps>>>(out, p, n, active);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("dadd chain: active lanes %2d warps %d: %.2f ns/step (%.1f cycles at %d MHz)\n", active, warps,
                   ms * 1e6 / n, ms * 1e-3 / n * clk * 1e3, clk / 1000);
        }
    }
    chain_f32<<<1, 32>>>(outf, pf, n);
    cudaEventRecord(a);
    chain_f32<<<1, 32>>>(outf, pf, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("fadd chain: %.2f ns/step\n", ms * 1e6 / n);
    for (int blocks : {148, 148 * 8}) {
        thru<<<blocks, 256>>>(out, 1.0, 1024);
        cudaEventRecord(a);
        thru<<<blocks, 256>>>(out, 1.0, 1024);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double flops = double(blocks) * 256 * 1024 * 8;
        printf("dadd throughput (%d blocks): %.1f GFLOP/s\n", blocks, flops / (ms * 1e-3) / 1e9);
    }
    return 0;
}
