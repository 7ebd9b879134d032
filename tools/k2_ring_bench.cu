// K2 A/B microbenchmark (tools/, not product): the TMA-ring kernel (ffn_ring_kernel, default) vs the
// LDG row-owner kernel (ffn_rows_kernel) on cold launches of 1-16 (expert, tile) segments.  Launches
// rotate over distinct tiles (> 2.5 GB >> 126 MB L2) so every launch streams from HBM, as in the
// decode.  Each case also checks that both kernels produce the same layer output (combine).
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/k2_ring_bench tools/k2_ring_bench.cu
//   tools/bin/k2_ring_bench [d] [ft]        (default 4096 3584: one 8x7B tile of 88 MB)
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define ADAPMOE_K2_TRACE 1
#include "../paper_2408_10284_b200/csrc/kernels/expert_ffn.cu"

using namespace adapmoe;

__global__ void fill(uint16_t* w, size_t n, uint32_t salt) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)(i * 2654435761u) ^ salt;
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        h ^= h >> 15;
        const float v = ((int)(h & 0xffff) - 32768) * (1.0f / 32768.0f) * 0.02f;
        w[i] = (uint16_t)(__float_as_uint(v) >> 16);
    }
}

__global__ void fill_x(double* x, int d) {
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < d; i += blockDim.x * gridDim.x) x[i] = sin(0.37 * i) * 1.5;
}

static void launch_variant(int variant, const FfnLaunch& p, int sms, cudaStream_t s) {
    const int grid = ffn_grid(p, sms);
    if (variant == 0) {
        const ring::Geometry geo = ring::geometry(p.d);
        const size_t smem = (size_t)geo.stages * geo.stage_bytes;
        const int dv = (p.d / 8 + ring::kConsumers - 1) / ring::kConsumers;
        auto fn = dv <= 1 ? ffn_ring_kernel<1> : dv <= 2 ? ffn_ring_kernel<2> : dv <= 3 ? ffn_ring_kernel<3>
                : dv <= 4 ? ffn_ring_kernel<4> : dv <= 6 ? ffn_ring_kernel<6> : ffn_ring_kernel<8>;
        static bool once = (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ring::kRingBytes), true); (void)once;
        fn<<<grid, ring::kThreads, smem, s>>>(p);
    } else {
        const size_t smem = (size_t)p.d * 4;
        auto fn = p.d <= 4096 ? ffn_rows_kernel<1> : p.d <= 8192 ? ffn_rows_kernel<2> : ffn_rows_kernel<4>;
        static bool once = (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024), true); (void)once;
        fn<<<grid, kThreads, smem, s>>>(p);
    }
}


__global__ void spin_kernel(long long ns) {
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > ns) break;
    }
}
__global__ void __launch_bounds__(ring::kThreads, 1) empty_kernel(const __grid_constant__ FfnLaunch p) {
    extern __shared__ unsigned char sm[];
    if (threadIdx.x == 0 && p.n_seg < 0) sm[0] = 1;
}
__global__ void __launch_bounds__(ring::kThreads, 1) xload_kernel(const __grid_constant__ FfnLaunch p) {
    const int v = threadIdx.x;
    float s = 0;
    if (v < p.d / 8)
        for (int e = 0; e < 8; ++e) s += (float)__ldg(p.x + 8 * v + e);
    if (s == 12345.f) p.partial[blockIdx.x] = s;
}

// time one launch with the stream kept busy before it (no host latency inside the events)
template <class F>
static double timed(F&& launch, int reps, bool busy) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double sum = 0;
    for (int r = 0; r < reps; ++r) {
        if (busy) spin_kernel<<<1, 32>>>(30000);
        cudaEventRecord(a);
        launch(r);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 3) sum += ms;
    }
    return sum / (reps - 3) * 1e3;
}

static int probe(int D, int Ft, uint16_t* w, int NT, double* x, float* part) {
    const size_t tile_elems = (size_t)3 * Ft * D;
    auto mk = [&](int nseg, int r, bool hot) {
        FfnLaunch p;
        p.n_seg = nseg; p.d = D; p.ft = Ft; p.x = x; p.partial = part;
        for (int s = 0; s < nseg; ++s) {
            const uint16_t* t = w + ((hot ? s : (r * nseg + s)) % NT) * tile_elems;
            p.seg[s].gate_up = t; p.seg[s].down_t = t + (size_t)2 * Ft * D;
        }
        return p;
    };
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ring::kRingBytes);
    for (bool busy : {false, true}) {
        printf("-- stream %s before each launch\n", busy ? "busy (30 us spin)" : "idle");
        printf("empty 148x288 192KB smem : %6.1f us\n", timed([&](int r) { FfnLaunch p = mk(1, r, false); empty_kernel<<<148, ring::kThreads, ring::kRingBytes>>>(p); }, 20, busy));
        printf("x load only              : %6.1f us\n", timed([&](int r) { FfnLaunch p = mk(1, r, false); xload_kernel<<<148, ring::kThreads, 0>>>(p); }, 20, busy));
        for (int nseg : {1, 4}) {
            for (int variant : {0, 1}) {
                for (bool hot : {false, true}) {
                    const double us = timed([&](int r) { FfnLaunch p = mk(nseg, r, hot); launch_variant(variant, p, 148, 0); }, 20, busy);
                    printf("%s nseg=%d %s : %6.1f us = %5.0f GB/s\n", variant == 0 ? "ring" : "rows", nseg, hot ? "hot " : "cold", us,
                           nseg * tile_elems * 2 / (us * 1e-6) / 1e9);
                }
            }
        }
    }
    // idle gaps before each launch (GPU idle, host sleeping): does a sparse launch pattern (the
    // link-bound decode computes ~10 % of the time) slow the kernel down?
    for (int gap_us : {0, 200, 1000, 5000, 10000}) {
        for (bool h2d : {false, true}) {
            static void* hsrc = nullptr;
            static void* ddst = nullptr;
            static cudaStream_t cs;
            if (!hsrc) {
                cudaMallocHost(&hsrc, 256 << 20);
                cudaMalloc(&ddst, 256 << 20);
                cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
            }
            double sum = 0;
            int n = 0;
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            for (int r = 0; r < 16; ++r) {
                if (h2d) cudaMemcpyAsync(ddst, hsrc, 256 << 20, cudaMemcpyHostToDevice, cs);  // ~4.6 ms of link traffic
                if (gap_us) {
                    auto t0 = std::chrono::steady_clock::now();
                    while (std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(gap_us)) {}
                }
                FfnLaunch p = mk(8, r, false);
                cudaEventRecord(a);
                launch_variant(0, p, 148, 0);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (r >= 3) { sum += ms; ++n; }
                cudaStreamSynchronize(cs);
            }
            printf("ring nseg=8 after %5d us idle%s: %6.1f us\n", gap_us, h2d ? " (+ concurrent 256 MB H2D)" : "", sum / n * 1e3);
        }
    }
    // per-CTA timeline of one cold ring launch (globaltimer, ns)
    for (int nseg : {1, 4}) {
        for (int r = 0; r < 6; ++r) {
            spin_kernel<<<1, 32>>>(30000);
            long long t_host0;
            FfnLaunch p = mk(nseg, r + 7, false);
            launch_variant(0, p, 148, 0);
            cudaDeviceSynchronize();
            (void)t_host0;
        }
        unsigned long long tr[kFfnMaxCtas][4];
        cudaMemcpyFromSymbol(tr, k2_trace, sizeof tr);
        const int grid = ffn_grid(mk(nseg, 0, false), 148);
        unsigned long long t0 = ~0ull, t_end = 0;
        for (int c = 0; c < grid; ++c) { t0 = std::min(t0, tr[c][0]); t_end = std::max(t_end, tr[c][2]); }
        std::vector<double> st, fs, en;
        for (int c = 0; c < grid; ++c) { st.push_back((tr[c][0] - t0) * 1e-3); fs.push_back((tr[c][1] - tr[c][0]) * 1e-3); en.push_back((tr[c][2] - t0) * 1e-3); }
        auto q = [](std::vector<double> v, double f) { std::sort(v.begin(), v.end()); return v[(size_t)(f * (v.size() - 1))]; };
        printf("ring nseg=%d per-CTA (us): start spread p50 %.2f max %.2f | first stage after start p50 %.2f max %.2f | end p0 %.2f p50 %.2f p90 %.2f max %.2f\n",
               nseg, q(st, .5), q(st, 1), q(fs, .5), q(fs, 1), q(en, 0), q(en, .5), q(en, .9), q(en, 1));
    }
    return 0;
}

int main(int argc, char** argv) {
    const int D = argc > 1 ? atoi(argv[1]) : 4096, Ft = argc > 2 ? atoi(argv[2]) : 3584;
    const size_t tile_elems = (size_t)3 * Ft * D, tile_bytes = tile_elems * 2;
    const int NT = (int)std::max<size_t>(24, (size_t)(3ull << 30) / tile_bytes);
    uint16_t* w;
    if (cudaMalloc(&w, tile_bytes * NT) != cudaSuccess) {
        printf("alloc failed\n");
        return 1;
    }
    fill<<<148 * 8, 256>>>(w, tile_elems * NT, 0x1234567u);
    double* x;
    cudaMalloc(&x, D * 8);
    fill_x<<<16, 256>>>(x, D);
    float *part, *out[2];
    cudaMalloc(&part, (size_t)kFfnMaxCtas * kFfnSlotsPerCta * D * 4);
    cudaMalloc(&out[0], D * 4);
    cudaMalloc(&out[1], D * 4);
    double* sc;
    cudaMalloc(&sc, 64 * 8);
    cudaMemset(sc, 0, 64 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    printf("d=%d ft=%d tile=%.1f MB, %d distinct tiles\n", D, Ft, tile_bytes / 1e6, NT);
    if (argc > 3) return probe(D, Ft, w, NT, x, part);
    for (int nseg : {1, 2, 3, 4, 7, 8, 16, 32}) {
        double mean_us[2] = {0, 0};
        for (int variant : {0, 1}) {
            double sum_ms = 0;
            int n = 0;
            for (int rep = 0; rep < 28; ++rep) {
                FfnLaunch p;
                p.n_seg = nseg;
                p.d = D;
                p.ft = Ft;
                p.x = x;
                p.partial = part;
                for (int s = 0; s < nseg; ++s) {
                    const uint16_t* t = w + ((rep * nseg + s) % NT) * tile_elems;
                    p.seg[s].gate_up = t;
                    p.seg[s].down_t = t + (size_t)2 * Ft * D;
                }
                cudaEventRecord(a);
                launch_variant(variant, p, 148, 0);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep >= 4) {
                    sum_ms += ms;
                    ++n;
                }
                if (rep == 0) {  // layer output of rep 0 through the shared combine
                    CombineArgs ca;
                    ca.x = x;
                    ca.scores = sc;
                    ca.out = out[variant];
                    ca.ranks = 1;
                    ca.d = D;
                    ca.ft = Ft;
                    ca.n_refs = nseg;
                    for (int s = 0; s < nseg; ++s) {
                        ca.refs[s] = FfnPartialRef{part, ffn_grid(p, 148), nseg, s, 0};
                        ffn_partial_range(ca.refs[s], Ft);
                    }
                    launch_combine(ca, 0);
                    cudaDeviceSynchronize();
                }
            }
            mean_us[variant] = sum_ms / n * 1e3;
        }
        std::vector<float> y0(D), y1(D);
        cudaMemcpy(y0.data(), out[0], D * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(y1.data(), out[1], D * 4, cudaMemcpyDeviceToHost);
        double md = 0, mx = 0;
        for (int j = 0; j < D; ++j) {
            md = std::max(md, (double)std::fabs(y0[j] - y1[j]));
            mx = std::max(mx, (double)std::fabs(y1[j]));
        }
        const double bytes = (double)nseg * tile_bytes;
        printf("nseg=%2d (%7.1f MB): ring %7.1f us = %5.0f GB/s | rows %7.1f us = %5.0f GB/s | max|dy|/max|y| %.2e  (%s)\n",
               nseg, bytes / 1e6, mean_us[0], bytes / (mean_us[0] * 1e-6) / 1e9, mean_us[1],
               bytes / (mean_us[1] * 1e-6) / 1e9, md / mx, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
