// XB12 encode / decode kernels (see xb12.hpp).  All memory-bound byte shuffles: 16 values per thread,
// 16-byte loads / stores, grid-stride over 148 x 8 CTAs.
#include <cuda_runtime.h>

#include <algorithm>

#include "xb12.hpp"

namespace adapmoe {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kGrid = 148 * 8;

__global__ void __launch_bounds__(kThreads) hist_kernel(const uint4* src, std::uint64_t n8, unsigned* hist) {
    __shared__ unsigned h[kWarps][256];  // per-warp bins: fewer same-address collisions
    for (int i = threadIdx.x; i < kWarps * 256; i += kThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    const int w = threadIdx.x >> 5;
    for (std::uint64_t g = blockIdx.x * static_cast<std::uint64_t>(kThreads) + threadIdx.x; g < n8;
         g += static_cast<std::uint64_t>(gridDim.x) * kThreads) {
        const uint4 q = src[g];
        const unsigned words[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            atomicAdd(&h[w][(words[k] >> 7) & 0xffu], 1u);
            atomicAdd(&h[w][(words[k] >> 23) & 0xffu], 1u);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += kThreads) {
        unsigned s = 0;
        for (int q = 0; q < kWarps; ++q) s += h[q][b];
        if (s) atomicAdd(&hist[b], s);
    }
}

// work[0..255] histogram -> work[256] = first exponent of the best 15-wide window, work[257] = 0
__global__ void base_kernel(unsigned* work) {
    if (threadIdx.x != 0) return;
    unsigned long long best = 0;
    unsigned best_b = 0;
    for (unsigned b = 0; b + 15 <= 256; ++b) {
        unsigned long long s = 0;
        for (unsigned e = b; e < b + 15; ++e) s += work[e];
        if (s > best) {
            best = s;
            best_b = b;
        }
    }
    work[256] = best_b;
    work[257] = 0;
}

__global__ void __launch_bounds__(kThreads) encode_kernel(const uint4* src, std::uint64_t n16, const unsigned* work,
                                                           uint4* lo, uint2* nib, unsigned long long* exc,
                                                           std::uint64_t cap, unsigned* counter) {
    const unsigned base = work[256];
    for (std::uint64_t g = blockIdx.x * static_cast<std::uint64_t>(kThreads) + threadIdx.x; g < n16;
         g += static_cast<std::uint64_t>(gridDim.x) * kThreads) {
        const uint4 a = src[2 * g], b = src[2 * g + 1];
        const unsigned words[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        unsigned lob[4] = {0, 0, 0, 0}, nb[2] = {0, 0};
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const unsigned v = (words[k >> 1] >> (16 * (k & 1))) & 0xffffu;
            unsigned c = ((v >> 7) & 0xffu) - base;  // wraps for exponents below the window
            if (c >= 15u) {
                c = 15u;
                const unsigned slot = atomicAdd(counter, 1u);
                if (slot < cap) exc[slot] = ((g * 16 + k) << 16) | v;
            }
            lob[k >> 2] |= (((v >> 8) & 0x80u) | (v & 0x7fu)) << (8 * (k & 3));
            nb[k >> 3] |= c << (4 * (k & 7));
        }
        lo[g] = make_uint4(lob[0], lob[1], lob[2], lob[3]);
        nib[g] = make_uint2(nb[0], nb[1]);
    }
}

__global__ void __launch_bounds__(kThreads) decode_kernel(const uint4* lo, const uint2* nib, unsigned base,
                                                           std::uint64_t n16, uint4* dst) {
    for (std::uint64_t g = blockIdx.x * static_cast<std::uint64_t>(kThreads) + threadIdx.x; g < n16;
         g += static_cast<std::uint64_t>(gridDim.x) * kThreads) {
        const uint4 l = lo[g];
        const uint2 c = nib[g];
        const unsigned lw[4] = {l.x, l.y, l.z, l.w}, cw[2] = {c.x, c.y};
        unsigned out[8];
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
            unsigned pair = 0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const unsigned b = (lw[(k + h) >> 2] >> (8 * ((k + h) & 3))) & 0xffu;
                const unsigned e = (base + ((cw[(k + h) >> 3] >> (4 * ((k + h) & 7))) & 0xfu)) & 0xffu;
                pair |= (((b & 0x80u) << 8) | (e << 7) | (b & 0x7fu)) << (16 * h);
            }
            out[k >> 1] = pair;
        }
        dst[2 * g] = make_uint4(out[0], out[1], out[2], out[3]);
        dst[2 * g + 1] = make_uint4(out[4], out[5], out[6], out[7]);
    }
}

__global__ void patch_kernel(const unsigned long long* exc, std::uint64_t m, std::uint16_t* dst) {
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < m;
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long e = exc[i];
        dst[e >> 16] = static_cast<std::uint16_t>(e & 0xffffu);
    }
}

int grid_for(std::uint64_t items) {
    const std::uint64_t g = (items + kThreads - 1) / kThreads;
    return static_cast<int>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(g, kGrid)));
}

}  // namespace

cudaError_t xb12_encode(const std::uint16_t* src, std::uint64_t n, std::uint8_t* lo, std::uint8_t* nib,
                        std::uint64_t* exc, std::uint64_t exc_cap, std::uint32_t* work, cudaStream_t stream) {
    if (n % 16 || !src || !lo || !nib || !work) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(work, 0, 256 * sizeof(std::uint32_t), stream);
    if (e != cudaSuccess) return e;
    hist_kernel<<<grid_for(n / 8), kThreads, 0, stream>>>(reinterpret_cast<const uint4*>(src), n / 8, work);
    base_kernel<<<1, 32, 0, stream>>>(work);
    encode_kernel<<<grid_for(n / 16), kThreads, 0, stream>>>(
        reinterpret_cast<const uint4*>(src), n / 16, work, reinterpret_cast<uint4*>(lo), reinterpret_cast<uint2*>(nib),
        reinterpret_cast<unsigned long long*>(exc), exc_cap, work + 257);
    return cudaGetLastError();
}

cudaError_t xb12_histogram(const std::uint16_t* src, std::uint64_t n, std::uint32_t* hist, cudaStream_t stream) {
    if (n % 8 || !src || !hist) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(hist, 0, 256 * sizeof(std::uint32_t), stream);
    if (e != cudaSuccess) return e;
    hist_kernel<<<grid_for(n / 8), kThreads, 0, stream>>>(reinterpret_cast<const uint4*>(src), n / 8, hist);
    return cudaGetLastError();
}

cudaError_t xb12_decode(const std::uint8_t* record, const Xb12Tile& t, std::uint16_t* dst, cudaStream_t stream) {
    if (t.format != 1 || t.n % 16) return cudaErrorInvalidValue;
    decode_kernel<<<grid_for(t.n / 16), kThreads, 0, stream>>>(reinterpret_cast<const uint4*>(record),
                                                                reinterpret_cast<const uint2*>(record + t.nib_off),
                                                                t.base, t.n / 16, reinterpret_cast<uint4*>(dst));
    if (t.n_exc)
        patch_kernel<<<grid_for(t.n_exc), kThreads, 0, stream>>>(
            reinterpret_cast<const unsigned long long*>(record + t.exc_off), t.n_exc, dst);
    return cudaGetLastError();
}

void xb12_decode_host(const std::uint8_t* record, const Xb12Tile& t, std::uint16_t* dst, std::uint64_t i0,
                      std::uint64_t count) {
    const std::uint8_t* lo = record;
    const std::uint8_t* nib = record + t.nib_off;
    for (std::uint64_t i = i0; i < i0 + count; ++i) {
        const unsigned b = lo[i];
        const unsigned c = (nib[i >> 1] >> (4 * (i & 1))) & 0xfu;
        const unsigned e = (t.base + c) & 0xffu;
        dst[i - i0] = static_cast<std::uint16_t>(((b & 0x80u) << 8) | (e << 7) | (b & 0x7fu));
    }
    // escapes inside [i0, i0 + count): binary search in the ascending list
    const std::uint64_t* exc = reinterpret_cast<const std::uint64_t*>(record + t.exc_off);
    const std::uint64_t* lo_it = std::lower_bound(exc, exc + t.n_exc, i0 << 16);
    for (const std::uint64_t* p = lo_it; p < exc + t.n_exc && (*p >> 16) < i0 + count; ++p)
        dst[(*p >> 16) - i0] = static_cast<std::uint16_t>(*p & 0xffffu);
}

}  // namespace adapmoe
