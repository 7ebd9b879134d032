// Launch-overhead probe (tools/, not product): CUDA-event time of empty launches under different
// shared-memory configurations, to separate launch cost from the K2 kernel's own time.
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/launch_probe tools/launch_probe.cu
#include <cstdio>
__global__ void spin(long long ns) {
    extern __shared__ unsigned char sm[];
    long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < ns);
    if (ns < 0) sm[0] = 1;
}
__global__ void empty(int f) {
    extern __shared__ unsigned char sm[];
    if (f < 0) sm[threadIdx.x] = 1;
}
int main() {
    cudaFuncSetAttribute(empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    struct Case { const char* name; int grid, block, smem, spin_smem, carve; };
    Case cases[] = {{"events only", 0, 0, 0, 0, -1},
                    {"empty 1x32 0KB", 1, 32, 0, 0, -1},
                    {"empty 148x288 0KB", 148, 288, 0, 0, -1},
                    {"empty 148x288 192KB (spin 0KB)", 148, 288, 192 * 1024, 0, -1},
                    {"empty 148x288 192KB (spin 192KB)", 148, 288, 192 * 1024, 192 * 1024, -1},
                    {"empty 148x288 0KB, carveout 100 both", 148, 288, 0, 0, 100},
                    {"empty 148x288 192KB, carveout 100 both", 148, 288, 192 * 1024, 0, 100},
                    {"empty 148x512 64KB (spin 0KB)", 148, 512, 64 * 1024, 0, -1}};
    for (const Case& c : cases) {
        if (c.carve >= 0) {
            cudaFuncSetAttribute(empty, cudaFuncAttributePreferredSharedMemoryCarveout, c.carve);
            cudaFuncSetAttribute(spin, cudaFuncAttributePreferredSharedMemoryCarveout, c.carve);
        }
        for (int busy = 0; busy < 2; ++busy) {
            double sum = 0;
            int n = 0;
            for (int r = 0; r < 40; ++r) {
                if (busy) spin<<<1, 32, c.spin_smem, s>>>(20000);
                cudaEventRecord(a, s);
                if (c.grid) empty<<<c.grid, c.block, c.smem, s>>>(1);
                cudaEventRecord(b, s);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (r >= 5) { sum += ms; ++n; }
            }
            printf("%-42s %s: %6.2f us (%s)\n", c.name, busy ? "busy" : "idle", sum / n * 1e3, cudaGetErrorString(cudaGetLastError()));
        }
    }
    // back-to-back chain: 20 empty 192KB kernels alternating with 0KB kernels, events at the ends
    for (int alt = 0; alt < 2; ++alt) {
        spin<<<1, 32, 0, s>>>(50000);
        cudaEventRecord(a, s);
        for (int k = 0; k < 20; ++k) {
            empty<<<148, 288, 192 * 1024, s>>>(1);
            if (alt) empty<<<128, 512, 0, s>>>(1);
        }
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("chain of 20 x (192KB kernel%s): %.2f us per 192KB launch\n", alt ? " + 0KB kernel" : "", ms * 1e3 / 20);
    }
    return 0;
}
