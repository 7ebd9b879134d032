// Microbenchmark (tools/, not product): K2 expert streaming bandwidth in isolation, at the
// Mixtral-8x7B tile shape (d 4096, ffn/tiles 3584 -> 88 MB per (expert, tile) segment).
// Built in several variants by tools/ffn_microbench.sh (-DADAPMOE_FFN_WARPS, _STAGE_KB, _BATCH).
// Also times a plain LDG-streaming GEMV over the same bytes as a no-TMA reference point.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2408_10284_b200/csrc/kernels/expert_ffn.cu"

using namespace adapmoe;

__global__ void fill_kernel(uint16_t* w, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        w[i] = 0x3c00 + (uint16_t)((i * 2654435761u) & 0x3ff) - 0x200;  // |w| ~ 2^-7..2^-6
}

__global__ void fill_x(double* x, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = ((i * 37) % 101) / 101.0 - 0.5;
}

// plain LDG streaming GEMV over 4096-wide rows (no TMA, no smem staging of weights)
__global__ void __launch_bounds__(256) ldg_gemv2(const uint4* __restrict__ w, const double* __restrict__ x, float* y,
                                                 long long rows) {
    __shared__ float xs[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) xs[i] = (float)x[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x / 32);
    for (long long r = blockIdx.x * (long long)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
        const uint4* row = w + r * 512;
        int4 v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = ptx::ld_stream(reinterpret_cast<const int4*>(row + lane + 32 * j));
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const float* xv = xs + (lane + 32 * j) * 8;
            const unsigned a = v[j].x, b = v[j].y, c = v[j].z, d = v[j].w;
            acc += __uint_as_float(a << 16) * xv[0] + __uint_as_float(a & 0xffff0000u) * xv[1] +
                   __uint_as_float(b << 16) * xv[2] + __uint_as_float(b & 0xffff0000u) * xv[3] +
                   __uint_as_float(c << 16) * xv[4] + __uint_as_float(c & 0xffff0000u) * xv[5] +
                   __uint_as_float(d << 16) * xv[6] + __uint_as_float(d & 0xffff0000u) * xv[7];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) y[r] = acc;
    }
}

int main_v3();
int main_v4();
int main() {
    if (getenv("FFN_V3")) return main_v3();
    if (getenv("FFN_V4")) return main_v4();
    const int D = 4096, Ft = 3584;
    const size_t tile_elems = (size_t)3 * Ft * D, tile_bytes = tile_elems * 2;
    const int max_seg = 16;
    uint16_t* w;
    cudaMalloc(&w, tile_bytes * max_seg);
    fill_kernel<<<148 * 8, 256>>>(w, tile_elems * max_seg);
    double* x;
    cudaMalloc(&x, D * 8);
    fill_x<<<1, 256>>>(x, D);
    float *h, *y;
    cudaMalloc(&h, (size_t)max_seg * Ft * 4);
    cudaMalloc(&y, (size_t)max_seg * D * 4 + (size_t)max_seg * 3 * Ft * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float* part;
    cudaMalloc(&part, (size_t)kFfnMaxCtas * kFfnSlotsPerCta * D * 4);
    for (int nseg : {1, 4, 8, 16}) {
        FfnLaunch p;
        p.n_seg = nseg;
        p.d = D;
        p.ft = Ft;
        p.x = x;
        p.partial = part;
        // (the L2 prefetch option was removed from the product kernel: measured slower)
        for (int s = 0; s < nseg; ++s) {
            const uint16_t* t = w + s * tile_elems;
            p.seg[s].gate_up = t;
            p.seg[s].down_t = t + (size_t)2 * Ft * D;
        }
        float best = 1e9, sum = 0;
        const int reps = 10;
        for (int r = 0; r < reps + 3; ++r) {
            cudaEventRecord(a);
            launch_ffn(p, sms, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 3) {
                best = ms < best ? ms : best;
                sum += ms;
            }
        }
        const double bytes = (double)nseg * tile_bytes;
        printf("  product ffn_rows nseg=%2d (%.0f MB): best %.1f us = %.0f GB/s, mean %.0f GB/s  err=%s\n", nseg,
               bytes / 1e6, best * 1e3, bytes / (best * 1e-3) / 1e9, bytes / (sum / reps * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    for (int nseg : {1, 4, 16}) {
        const long long rows = (long long)nseg * tile_elems / 4096;
        float best = 1e9;
        for (int r = 0; r < 8; ++r) {
            cudaEventRecord(a);
            ldg_gemv2<<<sms * 4, 256>>>(reinterpret_cast<const uint4*>(w), x, y, rows);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 2) best = ms < best ? ms : best;
        }
        const double bytes = (double)rows * 4096 * 2;
        printf("  ldg_gemv  nseg=%2d (%.0f MB): best %.1f us = %.0f GB/s\n", nseg, bytes / 1e6, best * 1e3,
               bytes / (best * 1e-3) / 1e9);
    }
    return 0;
}

// ---- v3 candidate: LDG-streaming fused SwiGLU, no smem ring, warp-independent -------------------
namespace v3 {
constexpr int kWarps = 8;
struct Seg { const uint4* gate_up; const uint4* down; float* h; float* y; };
struct Launch { int n_seg; int d, ft; const float* x32; unsigned* counters; Seg seg[32]; };

__device__ __forceinline__ float dot8(uint4 w, float4 a, float4 b, float acc) {
    acc = __fmaf_rn(__uint_as_float(w.x << 16), a.x, acc);
    acc = __fmaf_rn(__uint_as_float(w.x & 0xffff0000u), a.y, acc);
    acc = __fmaf_rn(__uint_as_float(w.y << 16), a.z, acc);
    acc = __fmaf_rn(__uint_as_float(w.y & 0xffff0000u), a.w, acc);
    acc = __fmaf_rn(__uint_as_float(w.z << 16), b.x, acc);
    acc = __fmaf_rn(__uint_as_float(w.z & 0xffff0000u), b.y, acc);
    acc = __fmaf_rn(__uint_as_float(w.w << 16), b.z, acc);
    acc = __fmaf_rn(__uint_as_float(w.w & 0xffff0000u), b.w, acc);
    return acc;
}

template <int U>
__global__ void __launch_bounds__(32 * kWarps, 2) fused(const __grid_constant__ Launch p) {
    const int lane = threadIdx.x & 31;
    const long long gw = (long long)blockIdx.x * kWarps + (threadIdx.x >> 5);
    const long long W = (long long)gridDim.x * kWarps;
    const int D = p.d, Ft = p.ft;
    const long long ta = (long long)p.n_seg * Ft;       // row pairs
    const long long tb = (long long)p.n_seg * D;        // down rows
    const int vpr_a = D / 8, vpr_b = Ft / 8;             // uint4 per row
    // phase A: contiguous block of row pairs per warp
    for (long long u = ta * gw / W; u < ta * (gw + 1) / W; ++u) {
        const int s = (int)(u / Ft), r = (int)(u % Ft);
        const uint4* w1 = p.seg[s].gate_up + (size_t)r * 2 * vpr_a;
        const uint4* w3 = w1 + vpr_a;
        float a = 0.f, b = 0.f;
        for (int j0 = lane; j0 < vpr_a; j0 += 32 * U) {
            uint4 q1[U], q3[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int j = j0 + 32 * k;
                q1[k] = j < vpr_a ? make_uint4(0,0,0,0) : make_uint4(0,0,0,0);
                if (j < vpr_a) {
                    int4 t1 = ptx::ld_stream(reinterpret_cast<const int4*>(w1 + j));
                    int4 t3 = ptx::ld_stream(reinterpret_cast<const int4*>(w3 + j));
                    q1[k] = make_uint4(t1.x, t1.y, t1.z, t1.w);
                    q3[k] = make_uint4(t3.x, t3.y, t3.z, t3.w);
                } else {
                    q3[k] = make_uint4(0,0,0,0);
                }
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int j = j0 + 32 * k;
                if (j < vpr_a) {
                    const float4 xa = __ldg(reinterpret_cast<const float4*>(p.x32 + j * 8));
                    const float4 xb = __ldg(reinterpret_cast<const float4*>(p.x32 + j * 8 + 4));
                    a = dot8(q1[k], xa, xb, a);
                    b = dot8(q3[k], xa, xb, b);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        if (lane == 0) {
            p.seg[s].h[r] = a / (1.0f + expf(-a)) * b;
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.counters + s) : "memory");
        }
    }
    // phase B
    int ready = -1;
    for (long long u = tb * gw / W; u < tb * (gw + 1) / W; ++u) {
        const int s = (int)(u / D), r = (int)(u % D);
        if (s != ready) {
            if (lane == 0) {
                unsigned v;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.counters + s) : "memory");
                } while (v < (unsigned)Ft);
            }
            __syncwarp();
            ready = s;
        }
        const uint4* w2 = p.seg[s].down + (size_t)r * vpr_b;
        const float* h = p.seg[s].h;
        float acc = 0.f;
        for (int j0 = lane; j0 < vpr_b; j0 += 32 * U) {
            uint4 q[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int j = j0 + 32 * k;
                if (j < vpr_b) {
                    int4 t = ptx::ld_stream(reinterpret_cast<const int4*>(w2 + j));
                    q[k] = make_uint4(t.x, t.y, t.z, t.w);
                } else q[k] = make_uint4(0,0,0,0);
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int j = j0 + 32 * k;
                if (j < vpr_b) {
                    const float4 ha = __ldcg(reinterpret_cast<const float4*>(h + j * 8));
                    const float4 hb = __ldcg(reinterpret_cast<const float4*>(h + j * 8 + 4));
                    acc = dot8(q[k], ha, hb, acc);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) p.seg[s].y[r] = acc;
    }
}
}  // namespace v3

int main_v3() {
    const int D = 4096, Ft = 3584;
    const size_t tile_elems = (size_t)3 * Ft * D, tile_bytes = tile_elems * 2;
    const int max_seg = 16;
    uint16_t* w;
    cudaMalloc(&w, tile_bytes * max_seg);
    fill_kernel<<<148 * 8, 256>>>(w, tile_elems * max_seg);
    float *x32, *h, *y;
    cudaMalloc(&x32, D * 4);
    cudaMemset(x32, 0, D * 4);
    cudaMalloc(&h, (size_t)max_seg * Ft * 4);
    cudaMalloc(&y, (size_t)max_seg * D * 4);
    unsigned* counters;
    cudaMalloc(&counters, 64 * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int U : {4, 8}) {
        for (int per_sm : {1, 2}) {
            for (int nseg : {1, 4, 16}) {
                v3::Launch p;
                p.n_seg = nseg; p.d = D; p.ft = Ft; p.x32 = x32; p.counters = counters;
                for (int s = 0; s < nseg; ++s) {
                    const uint16_t* t = w + s * tile_elems;
                    p.seg[s].gate_up = reinterpret_cast<const uint4*>(t);
                    p.seg[s].down = reinterpret_cast<const uint4*>(t + (size_t)2 * Ft * D);
                    p.seg[s].h = h + (size_t)s * Ft;
                    p.seg[s].y = y + (size_t)s * D;
                }
                float best = 1e9;
                for (int r = 0; r < 10; ++r) {
                    cudaMemsetAsync(counters, 0, 64 * 4);
                    cudaEventRecord(a);
                    if (U == 4) v3::fused<4><<<sms * per_sm, 32 * v3::kWarps>>>(p);
                    else v3::fused<8><<<sms * per_sm, 32 * v3::kWarps>>>(p);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (r >= 3) best = ms < best ? ms : best;
                }
                const double bytes = (double)nseg * tile_bytes;
                printf("  v3 U=%d ctas/sm=%d nseg=%2d (%.0f MB): best %.1f us = %.0f GB/s err=%s\n", U, per_sm, nseg,
                       bytes / 1e6, best * 1e3, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}

// ---- v4 candidate: row-owner LDG kernel (W2 stored transposed per tile), no cross-CTA dependency ----
namespace v4 {
constexpr int kThreads = 512, kWarps = 16, kChunk = 16;
struct Seg { const uint4* gate_up; const uint4* down_t; };
struct Launch { int n_seg; int d, ft; const float* x32; float* partial; Seg seg[32]; };

template <int U, bool PF>
__global__ void __launch_bounds__(kThreads, 1) rows(const __grid_constant__ Launch p) {
    __shared__ float xs[4096];
    __shared__ float hs[2][kChunk];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = p.d, Ft = p.ft, vpr = D / 8;
    for (int i = tid; i < D; i += kThreads) xs[i] = p.x32[i];
    const long long TR = (long long)p.n_seg * Ft;
    const long long r_lo = TR * blockIdx.x / gridDim.x, r_hi = TR * (blockIdx.x + 1) / gridDim.x;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int cur_seg = (int)(r_lo / Ft), slot = 0;
    __syncthreads();
    int parity = 0;
    for (long long c0 = r_lo; c0 < r_hi; parity ^= 1) {
        const int s = (int)(c0 / Ft), r0 = (int)(c0 % Ft);
        const int n = (int)min((long long)min(kChunk, Ft - r0), r_hi - c0);
        if (s != cur_seg) {  // flush partial of the previous segment
            float* dst = p.partial + ((size_t)blockIdx.x * 2 + slot) * D + tid * 8;
            *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
            *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
            for (int k = 0; k < 8; ++k) acc[k] = 0.f;
            cur_seg = s;
            ++slot;
        }
        if (PF && tid == 0) {  // prefetch the next chunk into L2
            const long long c1 = c0 + n;
            if (c1 < r_hi) {
                const int s1 = (int)(c1 / Ft), q0 = (int)(c1 % Ft);
                const int n1 = (int)min((long long)min(kChunk, Ft - q0), r_hi - c1);
                ptx::bulk_prefetch_l2(p.seg[s1].gate_up + (size_t)q0 * 2 * vpr, n1 * 2u * D * 2u);
                ptx::bulk_prefetch_l2(p.seg[s1].down_t + (size_t)q0 * vpr, n1 * (unsigned)D * 2u);
            }
        }
        // phase 1: warp w -> h of row r0 + w
        if (warp < n) {
            const uint4* w1 = p.seg[s].gate_up + (size_t)(r0 + warp) * 2 * vpr;
            const uint4* w3 = w1 + vpr;
            float a = 0.f, b = 0.f;
            for (int j0 = lane; j0 < vpr; j0 += 32 * U) {
                int4 q1[U], q3[U];
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    q1[k] = ptx::ld_stream(reinterpret_cast<const int4*>(w1 + j0 + 32 * k));
                    q3[k] = ptx::ld_stream(reinterpret_cast<const int4*>(w3 + j0 + 32 * k));
                }
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    const float* xv = xs + (j0 + 32 * k) * 8;
                    const float4 xa = *reinterpret_cast<const float4*>(xv);
                    const float4 xb = *reinterpret_cast<const float4*>(xv + 4);
                    a = v3::dot8(make_uint4(q1[k].x, q1[k].y, q1[k].z, q1[k].w), xa, xb, a);
                    b = v3::dot8(make_uint4(q3[k].x, q3[k].y, q3[k].z, q3[k].w), xa, xb, b);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                a += __shfl_xor_sync(0xffffffffu, a, o);
                b += __shfl_xor_sync(0xffffffffu, b, o);
            }
            if (lane == 0) hs[parity][warp] = a / (1.0f + expf(-a)) * b;
        }
        __syncthreads();
        // phase 2: thread t owns outputs [8t, 8t+8)
        int4 q[kChunk];
#pragma unroll
        for (int k = 0; k < kChunk; ++k)
            if (k < n) q[k] = ptx::ld_stream(reinterpret_cast<const int4*>(p.seg[s].down_t + (size_t)(r0 + k) * vpr + tid));
#pragma unroll
        for (int k = 0; k < kChunk; ++k)
            if (k < n) {
                const float h = hs[parity][k];
                const unsigned u[4] = {(unsigned)q[k].x, (unsigned)q[k].y, (unsigned)q[k].z, (unsigned)q[k].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    acc[2 * e] = __fmaf_rn(h, __uint_as_float(u[e] << 16), acc[2 * e]);
                    acc[2 * e + 1] = __fmaf_rn(h, __uint_as_float(u[e] & 0xffff0000u), acc[2 * e + 1]);
                }
            }
        c0 += n;
    }
    float* dst = p.partial + ((size_t)blockIdx.x * 2 + slot) * D + tid * 8;
    *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
}
}  // namespace v4

int main_v4() {
    const int D = 4096, Ft = 3584;
    const size_t tile_elems = (size_t)3 * Ft * D, tile_bytes = tile_elems * 2;
    const int max_seg = 16;
    uint16_t* w;
    cudaMalloc(&w, tile_bytes * max_seg);
    fill_kernel<<<148 * 8, 256>>>(w, tile_elems * max_seg);
    float *x32, *part;
    cudaMalloc(&x32, D * 4);
    cudaMemset(x32, 0, D * 4);
    cudaMalloc(&part, (size_t)148 * 2 * D * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int variant = 0; variant < 4; ++variant) {
        for (int nseg : {1, 4, 16}) {
            v4::Launch p;
            p.n_seg = nseg; p.d = D; p.ft = Ft; p.x32 = x32; p.partial = part;
            for (int s = 0; s < nseg; ++s) {
                const uint16_t* t = w + s * tile_elems;
                p.seg[s].gate_up = reinterpret_cast<const uint4*>(t);
                p.seg[s].down_t = reinterpret_cast<const uint4*>(t + (size_t)2 * Ft * D);
            }
            float best = 1e9;
            for (int r = 0; r < 10; ++r) {
                cudaEventRecord(a);
                if (variant == 0) v4::rows<4, false><<<148, v4::kThreads>>>(p);
                if (variant == 1) v4::rows<4, true><<<148, v4::kThreads>>>(p);
                if (variant == 2) v4::rows<8, false><<<148, v4::kThreads>>>(p);
                if (variant == 3) v4::rows<8, true><<<148, v4::kThreads>>>(p);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (r >= 3) best = ms < best ? ms : best;
            }
            const double bytes = (double)nseg * tile_bytes;
            printf("  v4 U=%d prefetch=%d nseg=%2d (%.0f MB): best %.1f us = %.0f GB/s err=%s\n", variant >= 2 ? 8 : 4,
                   variant & 1, nseg, bytes / 1e6, best * 1e3, bytes / (best * 1e-3) / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
