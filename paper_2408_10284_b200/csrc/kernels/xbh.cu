// XBH encode / decode (see xbh.hpp).  Encode runs once per tile when the store is built; decode
// runs on the copy engine's decode stream after each tile record lands in HBM.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "xbh.hpp"

namespace adapmoe {

// ---- host: the per-tile code --------------------------------------------------------------------

void xbh_build_code(const std::uint32_t* hist, XbhCode& c) {
    c = XbhCode{};
    // window: first of the best 15 consecutive exponents (XB12's rule, xb12.cu base_kernel)
    unsigned long long best = 0, total = 0;
    for (int e = 0; e < 256; ++e) total += hist[e];
    for (unsigned b = 0; b + 15 <= 256; ++b) {
        unsigned long long s = 0;
        for (unsigned e = b; e < b + 15; ++e) s += hist[e];
        if (s > best) {
            best = s;
            c.base = b;
        }
    }
    unsigned long long cnt[16];
    for (int s = 0; s < 15; ++s) cnt[s] = hist[c.base + s];
    cnt[15] = total - best;
    // leaves: present symbols by (count, symbol)
    struct Item {
        unsigned long long w;
        std::uint8_t n[16];
    };
    std::vector<Item> leaves;
    for (int s = 0; s < 16; ++s)
        if (cnt[s]) {
            Item it{cnt[s], {}};
            it.n[s] = 1;
            leaves.push_back(it);
        }
    std::stable_sort(leaves.begin(), leaves.end(), [](const Item& a, const Item& b) { return a.w < b.w; });
    const size_t m = leaves.size();
    if (m == 1) {
        for (int s = 0; s < 16; ++s)
            if (leaves[0].n[s]) c.len[s] = 1;
    } else if (m > 1) {
        // package-merge (coin collector) with kXbhMaxLen levels; equal weights: leaf first
        std::vector<Item> list = leaves;
        for (int level = 1; level < kXbhMaxLen; ++level) {
            std::vector<Item> pk;
            for (size_t i = 0; i + 1 < list.size(); i += 2) {
                Item p{list[i].w + list[i + 1].w, {}};
                for (int s = 0; s < 16; ++s) p.n[s] = static_cast<std::uint8_t>(list[i].n[s] + list[i + 1].n[s]);
                pk.push_back(p);
            }
            std::vector<Item> merged;
            size_t i = 0, j = 0;
            while (i < leaves.size() || j < pk.size()) {
                if (j >= pk.size() || (i < leaves.size() && leaves[i].w <= pk[j].w))
                    merged.push_back(leaves[i++]);
                else
                    merged.push_back(pk[j++]);
            }
            list.swap(merged);
        }
        for (size_t k = 0; k < 2 * m - 2; ++k)
            for (int s = 0; s < 16; ++s) c.len[s] = static_cast<std::uint8_t>(c.len[s] + list[k].n[s]);
    }
    // canonical codes by (length, symbol)
    unsigned code = 0, prev = 0;
    bool first = true;
    for (int l = 1; l <= kXbhMaxLen; ++l)
        for (int s = 0; s < 16; ++s) {
            if (c.len[s] != l) continue;
            if (!first) code = (code + 1) << (l - prev);
            first = false;
            prev = static_cast<unsigned>(l);
            c.code[s] = static_cast<std::uint16_t>(code);
        }
    for (int s = 0; s < 16; ++s) {
        if (!c.len[s]) continue;
        const unsigned sh = kXbhMaxLen - c.len[s];
        const std::uint16_t entry =
            static_cast<std::uint16_t>(((s < 15 ? c.base + s : 0u) & 0xffu) | (static_cast<unsigned>(c.len[s]) << 8));
        for (unsigned k = static_cast<unsigned>(c.code[s]) << sh; k < ((static_cast<unsigned>(c.code[s]) + 1) << sh); ++k)
            c.lut[k] = entry;
    }
}

namespace {

constexpr int kThreads = 256;
constexpr int kGrid = 148 * 8;

__device__ __forceinline__ unsigned symbol_of(unsigned v, unsigned base) {
    const unsigned s = ((v >> 7) & 0xffu) - base;  // wraps below the window
    return s < 15u ? s : 15u;
}

// bits of each segment's codes
__global__ void __launch_bounds__(kThreads) seglen_kernel(const uint4* src, std::uint64_t n, const XbhCode* code,
                                                          std::uint32_t* seglen) {
    __shared__ unsigned len[16];
    __shared__ unsigned base;
    if (threadIdx.x < 16) len[threadIdx.x] = code->len[threadIdx.x];
    if (threadIdx.x == 0) base = code->base;
    __syncthreads();
    const std::uint64_t nseg = xbh_segments(n);
    const std::uint64_t s = blockIdx.x * static_cast<std::uint64_t>(kThreads) + threadIdx.x;
    if (s >= nseg) return;
    const std::uint64_t v0 = s * kXbhSeg, v1 = std::min<std::uint64_t>(n, v0 + kXbhSeg);
    unsigned bits = 0;
    for (std::uint64_t g = v0 / 8; g < v1 / 8; ++g) {
        const uint4 q = src[g];
        const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) bits += len[symbol_of(w[k] & 0xffffu, base)] + len[symbol_of(w[k] >> 16, base)];
    }
    seglen[s] = bits;
}

// exclusive scan of seglen[0..nseg) into seg[0..nseg], seg[nseg] = total (one CTA)
__global__ void __launch_bounds__(1024) scan_kernel(const std::uint32_t* seglen, std::uint64_t nseg, std::uint32_t* seg,
                                                    std::uint32_t* work) {
    __shared__ unsigned long long part[1024];
    const std::uint64_t per = (nseg + 1023) / 1024;
    const std::uint64_t a = threadIdx.x * per, b = std::min<std::uint64_t>(nseg, a + per);
    unsigned long long sum = 0;
    for (std::uint64_t i = a; i < b; ++i) sum += seglen[i];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {  // Hillis-Steele inclusive scan
        const unsigned long long v = threadIdx.x >= off ? part[threadIdx.x - off] : 0ull;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    unsigned long long run = part[threadIdx.x] - sum;
    for (std::uint64_t i = a; i < b; ++i) {
        seg[i] = static_cast<std::uint32_t>(run);
        run += seglen[i];
    }
    if (threadIdx.x == 1023) {
        seg[nseg] = static_cast<std::uint32_t>(part[1023]);
        work[1] = static_cast<std::uint32_t>(part[1023]);
    }
}

// every segment's codes, MSB first from its bit offset (words shared with a neighbour: atomicOr
// into the zeroed bit section), and the escapes
__global__ void __launch_bounds__(kThreads) emit_kernel(const std::uint16_t* src, std::uint64_t n, const XbhCode* code,
                                                        const std::uint32_t* seg, std::uint32_t* words,
                                                        unsigned long long* exc, std::uint64_t cap, unsigned* counter) {
    __shared__ unsigned len[16], cw[16];
    __shared__ unsigned base;
    if (threadIdx.x < 16) {
        len[threadIdx.x] = code->len[threadIdx.x];
        cw[threadIdx.x] = code->code[threadIdx.x];
    }
    if (threadIdx.x == 0) base = code->base;
    __syncthreads();
    const std::uint64_t nseg = xbh_segments(n);
    const std::uint64_t s = blockIdx.x * static_cast<std::uint64_t>(kThreads) + threadIdx.x;
    if (s >= nseg) return;
    const std::uint64_t v0 = s * kXbhSeg, v1 = std::min<std::uint64_t>(n, v0 + kXbhSeg);
    const std::uint32_t p = seg[s];
    std::uint64_t w = p >> 5;
    unsigned long long acc = 0;
    unsigned nacc = p & 31u;  // bits of the first word that belong to the previous segment (zeros here)
    for (std::uint64_t i = v0; i < v1; ++i) {
        const unsigned v = src[i];
        const unsigned sym = symbol_of(v, base), l = len[sym];
        if (sym == 15u) {
            const unsigned slot = atomicAdd(counter, 1u);
            if (slot < cap) exc[slot] = (static_cast<unsigned long long>(i) << 16) | v;
        }
        acc |= static_cast<unsigned long long>(cw[sym]) << (64 - nacc - l);
        nacc += l;
        if (nacc >= 32) {
            atomicOr(&words[w++], static_cast<unsigned>(acc >> 32));
            acc <<= 32;
            nacc -= 32;
        }
    }
    if (nacc) atomicOr(&words[w], static_cast<unsigned>(acc >> 32));
}

__global__ void __launch_bounds__(kThreads) lo_kernel(const uint4* src, std::uint64_t n16, uint4* lo) {
    for (std::uint64_t g = blockIdx.x * static_cast<std::uint64_t>(kThreads) + threadIdx.x; g < n16;
         g += static_cast<std::uint64_t>(gridDim.x) * kThreads) {
        const uint4 a = src[2 * g], b = src[2 * g + 1];
        const unsigned words[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        unsigned lob[4] = {0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const unsigned v = (words[k >> 1] >> (16 * (k & 1))) & 0xffffu;
            lob[k >> 2] |= (((v >> 8) & 0x80u) | (v & 0x7fu)) << (8 * (k & 3));
        }
        lo[g] = make_uint4(lob[0], lob[1], lob[2], lob[3]);
    }
}

constexpr int kDecThreads = 128;

// One thread per 512-value segment: 64-bit bit buffer, 12-bit peek into the shared table, refilled
// by a 32-bit word whenever fewer than 24 bits remain (two codes per check).
__global__ void __launch_bounds__(kDecThreads) decode_kernel(const std::uint8_t* rec, std::uint64_t n, uint4* dst) {
    __shared__ __align__(16) std::uint16_t lut[kXbhLut];
    {
        const uint4* src = reinterpret_cast<const uint4*>(rec + xbh_lut_off(n));
        uint4* d = reinterpret_cast<uint4*>(lut);
        for (int i = threadIdx.x; i < kXbhLut / 8; i += kDecThreads) d[i] = __ldg(src + i);
    }
    __syncthreads();
    const std::uint64_t nseg = xbh_segments(n);
    const std::uint64_t s = blockIdx.x * static_cast<std::uint64_t>(kDecThreads) + threadIdx.x;
    if (s >= nseg) return;
    const std::uint32_t* seg = reinterpret_cast<const std::uint32_t*>(rec + xbh_seg_off(n));
    const std::uint32_t* words = reinterpret_cast<const std::uint32_t*>(rec + xbh_bits_off(n));
    const uint4* lo = reinterpret_cast<const uint4*>(rec);
    const std::uint32_t p = __ldg(seg + s);
    std::uint64_t nx = (p >> 5) + 2;
    unsigned long long buf =
        ((static_cast<unsigned long long>(__ldg(words + nx - 2)) << 32) | __ldg(words + nx - 1)) << (p & 31u);
    int nb = 64 - static_cast<int>(p & 31u);
    const std::uint64_t g0 = s * (kXbhSeg / 16), g1 = std::min<std::uint64_t>(n, (s + 1) * kXbhSeg) / 16;
    for (std::uint64_t g = g0; g < g1; ++g) {
        const uint4 l = __ldg(lo + g);
        const unsigned lw[4] = {l.x, l.y, l.z, l.w};
        unsigned out[8];
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
            if (nb < 24) {
                buf |= static_cast<unsigned long long>(__ldg(words + nx++)) << (32 - nb);
                nb += 32;
            }
            unsigned pair = 0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const unsigned e = lut[buf >> (64 - kXbhMaxLen)];
                const unsigned len = e >> 8;
                buf <<= len;
                nb -= static_cast<int>(len);
                const unsigned b = (lw[(k + h) >> 2] >> (8 * ((k + h) & 3))) & 0xffu;
                pair |= (((b & 0x80u) << 8) | ((e & 0xffu) << 7) | (b & 0x7fu)) << (16 * h);
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

int grid_for(std::uint64_t items, int threads = kThreads) {
    const std::uint64_t g = (items + threads - 1) / threads;
    return static_cast<int>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(g, kGrid)));
}
int grid_all(std::uint64_t items, int threads) {  // one thread per item
    return static_cast<int>(std::max<std::uint64_t>(1, (items + threads - 1) / threads));
}

}  // namespace

cudaError_t xbh_encode(const std::uint16_t* src, std::uint64_t n, const XbhCode* dcode, std::uint8_t* record,
                       std::uint64_t* exc, std::uint64_t exc_cap, std::uint32_t* seglen, std::uint32_t* work,
                       cudaStream_t stream) {
    if (n % 16 || !src || !dcode || !record || !seglen || !work) return cudaErrorInvalidValue;
    if (n * kXbhMaxLen >= (1ull << 32)) return cudaErrorInvalidValue;  // u32 bit offsets
    const std::uint64_t nseg = xbh_segments(n);
    std::uint32_t* words = reinterpret_cast<std::uint32_t*>(record + xbh_bits_off(n));
    cudaError_t e = cudaMemsetAsync(words, 0, 4 * xbh_words(n * kXbhMaxLen), stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(work, 0, kXbhWorkWords * sizeof(std::uint32_t), stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(record + xbh_lut_off(n), dcode->lut, 2 * kXbhLut, cudaMemcpyDeviceToDevice, stream);
    if (e != cudaSuccess) return e;
    lo_kernel<<<grid_for(n / 16), kThreads, 0, stream>>>(reinterpret_cast<const uint4*>(src), n / 16,
                                                          reinterpret_cast<uint4*>(record));
    seglen_kernel<<<grid_all(nseg, kThreads), kThreads, 0, stream>>>(reinterpret_cast<const uint4*>(src), n, dcode, seglen);
    std::uint32_t* seg = reinterpret_cast<std::uint32_t*>(record + xbh_seg_off(n));
    scan_kernel<<<1, 1024, 0, stream>>>(seglen, nseg, seg, work);
    emit_kernel<<<grid_all(nseg, kThreads), kThreads, 0, stream>>>(src, n, dcode, seg, words,
                                                                    reinterpret_cast<unsigned long long*>(exc), exc_cap,
                                                                    work);
    return cudaGetLastError();
}

cudaError_t xbh_decode(const std::uint8_t* record, const Xb12Tile& t, std::uint16_t* dst, cudaStream_t stream) {
    if (t.format != 2 || t.n % 16) return cudaErrorInvalidValue;
    decode_kernel<<<grid_all(xbh_segments(t.n), kDecThreads), kDecThreads, 0, stream>>>(record, t.n,
                                                                                         reinterpret_cast<uint4*>(dst));
    if (t.n_exc)
        patch_kernel<<<grid_for(t.n_exc), kThreads, 0, stream>>>(
            reinterpret_cast<const unsigned long long*>(record + t.exc_off), t.n_exc, dst);
    return cudaGetLastError();
}

void xbh_decode_host(const std::uint8_t* record, const Xb12Tile& t, std::uint16_t* dst, std::uint64_t i0,
                     std::uint64_t count) {
    const std::uint16_t* lut = reinterpret_cast<const std::uint16_t*>(record + xbh_lut_off(t.n));
    const std::uint32_t* seg = reinterpret_cast<const std::uint32_t*>(record + xbh_seg_off(t.n));
    const std::uint32_t* words = reinterpret_cast<const std::uint32_t*>(record + xbh_bits_off(t.n));
    const std::uint64_t end = i0 + count;
    for (std::uint64_t s = i0 / kXbhSeg; s * kXbhSeg < end; ++s) {
        std::uint64_t pos = seg[s];
        const std::uint64_t v1 = std::min<std::uint64_t>(end, (s + 1) * kXbhSeg);
        for (std::uint64_t i = s * kXbhSeg; i < v1; ++i) {
            const std::uint64_t w = pos >> 5;
            const unsigned long long win = (static_cast<unsigned long long>(words[w]) << 32) | words[w + 1];
            const unsigned e = lut[(win << (pos & 31)) >> (64 - kXbhMaxLen)];
            pos += e >> 8;
            if (i < i0) continue;
            const unsigned b = record[i];
            dst[i - i0] = static_cast<std::uint16_t>(((b & 0x80u) << 8) | ((e & 0xffu) << 7) | (b & 0x7fu));
        }
    }
    const std::uint64_t* exc = reinterpret_cast<const std::uint64_t*>(record + t.exc_off);
    const std::uint64_t* it = std::lower_bound(exc, exc + t.n_exc, i0 << 16);
    for (; it < exc + t.n_exc && (*it >> 16) < end; ++it) dst[(*it >> 16) - i0] = static_cast<std::uint16_t>(*it & 0xffffu);
}

}  // namespace adapmoe
