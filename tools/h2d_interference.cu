// How a concurrent host-to-device copy slows an HBM-streaming kernel (tools/, not product).
// A read-only streaming kernel (16-byte non-caching loads) over 704 MB of a 2 GB buffer (rotating
// offsets, so every launch streams from HBM) is timed with CUDA events: alone; beside a 512 MB pinned
// H2D copy into a DRAM-sized destination; beside the same bytes copied as 32 x 16 MB pieces into one
// 16 MB destination (which stays in the 126 MB L2); and beside a device-to-device write stream of the
// same rate budget (a kernel writing 512 MB), to separate "PCIe traffic" from "DRAM writes".
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/h2d_interference tools/h2d_interference.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

__global__ void __launch_bounds__(512) stream_read(const uint4* p, size_t n16, unsigned* out) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * 512ull + threadIdx.x; i < n16; i += 512ull * gridDim.x) {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(p + i));
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void __launch_bounds__(256) stream_write(uint4* p, size_t n16) {
    for (size_t i = blockIdx.x * 256ull + threadIdx.x; i < n16; i += 256ull * gridDim.x)
        p[i] = make_uint4(static_cast<unsigned>(i), 1, 2, 3);
}

int main() {
    const size_t buf = 2ull << 30, win = 704ull << 20, copy = 512ull << 20, small = 16ull << 20;
    uint4* d;
    CK(cudaMalloc(&d, buf));
    CK(cudaMemset(d, 1, buf));
    unsigned* out;
    CK(cudaMalloc(&out, 4));
    void *h, *dst_big, *dst_small;
    CK(cudaMallocHost(&h, copy));
    CK(cudaMalloc(&dst_big, copy));
    CK(cudaMalloc(&dst_small, small));
    uint4* wbuf;
    CK(cudaMalloc(&wbuf, copy));
    cudaStream_t ks, cs;
    CK(cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    auto launch = [&](int r) {
        const size_t off = (static_cast<size_t>(r) * (win + (64ull << 20))) % (buf - win);
        CK(cudaEventRecord(a, ks));
        stream_read<<<sms * 2, 512, 0, ks>>>(d + off / 16, win / 16, out);
        CK(cudaEventRecord(b, ks));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        return ms * 1e3f;
    };
    const char* names[] = {"alone", "beside 512 MB H2D -> 512 MB buffer (DRAM)",
                           "beside 32 x 16 MB H2D -> one 16 MB buffer (L2-resident)",
                           "beside a 512 MB device write kernel (8 CTAs, ~H2D rate)"};
    for (int mode = 0; mode < 4; ++mode) {
        std::vector<float> t;
        for (int r = 0; r < 13; ++r) {
            CK(cudaDeviceSynchronize());
            if (mode == 1) CK(cudaMemcpyAsync(dst_big, h, copy, cudaMemcpyHostToDevice, cs));
            if (mode == 2)
                for (int k = 0; k < 32; ++k)
                    CK(cudaMemcpyAsync(dst_small, static_cast<char*>(h) + (k % 32) * small, small, cudaMemcpyHostToDevice, cs));
            if (mode == 3) stream_write<<<8, 256, 0, cs>>>(wbuf, copy / 16);
            if (mode) {  // let the background traffic start
                cudaEvent_t s;
                CK(cudaEventCreate(&s));
                CK(cudaEventRecord(s, cs));
                for (int spin = 0; spin < 200000; ++spin) asm volatile("" ::: "memory");
                CK(cudaEventDestroy(s));
            }
            const float us = launch(r);
            if (r >= 3) t.push_back(us);
            CK(cudaStreamSynchronize(cs));
        }
        std::sort(t.begin(), t.end());
        std::printf("%-60s median %7.1f us  best %7.1f us  = %5.0f GB/s\n", names[mode], t[t.size() / 2], t[0],
                    win / (t[t.size() / 2] * 1e-6) / 1e9);
    }
    return 0;
}
