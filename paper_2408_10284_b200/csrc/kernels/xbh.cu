// XBH encode / decode (see xbh.hpp).  Encode runs once per tile when the store is built; decode
// runs on the copy engine's decode stream after each tile record lands in HBM.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <vector>

#include "xbh.hpp"

namespace adapmoe {

static_assert(offsetof(XbhCode, mlut) == offsetof(XbhCode, lut) + 2 * kXbhLut, "lut and mlut are copied as one block");

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
    std::vector<std::uint16_t> sym_lut(kXbhLut, 0);  // symbol | length << 8 of the 12-bit peek
    for (int s = 0; s < 16; ++s) {
        if (!c.len[s]) continue;
        const unsigned sh = kXbhMaxLen - c.len[s];
        const std::uint16_t entry =
            static_cast<std::uint16_t>(((s < 15 ? c.base + s : 0u) & 0xffu) | (static_cast<unsigned>(c.len[s]) << 8));
        for (unsigned k = static_cast<unsigned>(c.code[s]) << sh; k < ((static_cast<unsigned>(c.code[s]) + 1) << sh); ++k) {
            c.lut[k] = entry;
            sym_lut[k] = static_cast<std::uint16_t>(s | (c.len[s] << 8));
        }
    }
    // multi-code table: follow the peek through up to 5 codes that end inside its 12 bits; entry =
    // symbols (4 bits each, bits 0-19) | count << 20 | first code's length << 23 | total length
    // << 27.  A peek without a code (length 0) never occurs in a stream and ends the walk.
    for (unsigned i = 0; i < static_cast<unsigned>(kXbhLut); ++i) {
        unsigned len = 0, syms = 0, first_len = 0, cnt = 0;
        for (int k = 0; k < kXbhMultiCodes && len < static_cast<unsigned>(kXbhMaxLen); ++k) {
            const unsigned e = sym_lut[(i << len) & (kXbhLut - 1)], l = e >> 8;
            if (l == 0 || len + l > static_cast<unsigned>(kXbhMaxLen)) break;
            syms |= (e & 15u) << (4 * k);
            if (k == 0) first_len = l;
            ++cnt;
            len += l;
        }
        c.mlut[i] = syms | (cnt << 20) | (first_len << 23) | (len << 27);
    }
}

namespace {

constexpr int kThreads = 256;
constexpr int kGrid = 148 * 8;

__device__ __forceinline__ unsigned symbol_of(unsigned v, unsigned base) {
    const unsigned s = ((v >> 7) & 0xffu) - base;  // wraps below the window
    return s < 15u ? s : 15u;
}

// ---- encode: 512 values per thread ----------------------------------------------------------------

// bits of each encoder segment's codes
__global__ void __launch_bounds__(kThreads) seglen_kernel(const uint4* src, std::uint64_t n, const XbhCode* code,
                                                          std::uint32_t* seglen) {
    __shared__ unsigned len[16];
    __shared__ unsigned base;
    if (threadIdx.x < 16) len[threadIdx.x] = code->len[threadIdx.x];
    if (threadIdx.x == 0) base = code->base;
    __syncthreads();
    const std::uint64_t s = blockIdx.x * static_cast<std::uint64_t>(kThreads) + threadIdx.x;
    if (s >= xbh_enc_segments(n)) return;
    const std::uint64_t v0 = s * kXbhEncSeg, v1 = std::min<std::uint64_t>(n, v0 + kXbhEncSeg);
    unsigned bits = 0;
    for (std::uint64_t g = v0 / 8; g < v1 / 8; ++g) {
        const uint4 q = src[g];
        const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) bits += len[symbol_of(w[k] & 0xffffu, base)] + len[symbol_of(w[k] >> 16, base)];
    }
    seglen[s] = bits;
}

// exclusive scan of seglen[0..nseg) in place, seglen[nseg] = total = work[1] (one CTA)
__global__ void __launch_bounds__(1024) scan_kernel(std::uint32_t* seglen, std::uint64_t nseg, std::uint32_t* work) {
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
        const unsigned l = seglen[i];
        seglen[i] = static_cast<std::uint32_t>(run);
        run += l;
    }
    if (threadIdx.x == 1023) {
        seglen[nseg] = static_cast<std::uint32_t>(part[1023]);
        work[1] = static_cast<std::uint32_t>(part[1023]);
    }
}

// every segment's codes, MSB first from its bit offset (words shared with a neighbour: atomicOr into
// the zeroed bit section); for each code that is the first to start in its 128-bit chunk, the
// chunk's gap (and, for a block's first chunk, the block's base value index); the escapes
__global__ void __launch_bounds__(kThreads) emit_kernel(const std::uint16_t* src, std::uint64_t n, const XbhCode* code,
                                                        const std::uint32_t* seg, std::uint32_t* words,
                                                        std::uint32_t* gaps, std::uint32_t* bases,
                                                        unsigned long long* exc, std::uint64_t cap, unsigned* counter) {
    __shared__ unsigned len[16], cw[16];
    __shared__ unsigned base;
    if (threadIdx.x < 16) {
        len[threadIdx.x] = code->len[threadIdx.x];
        cw[threadIdx.x] = code->code[threadIdx.x];
    }
    if (threadIdx.x == 0) base = code->base;
    __syncthreads();
    const std::uint64_t s = blockIdx.x * static_cast<std::uint64_t>(kThreads) + threadIdx.x;
    if (s >= xbh_enc_segments(n)) return;
    const std::uint64_t v0 = s * kXbhEncSeg, v1 = std::min<std::uint64_t>(n, v0 + kXbhEncSeg);
    std::uint64_t pos = seg[s];
    // start of the previous code (the last of the previous segment); "none" before value 0
    std::uint64_t prev = v0 ? pos - len[symbol_of(src[v0 - 1], base)] : ~0ull;
    std::uint64_t w = pos >> 5;
    unsigned long long acc = 0;
    unsigned nacc = pos & 31u;  // bits of the first word that belong to the previous segment (zeros here)
    for (std::uint64_t i = v0; i < v1; ++i) {
        const unsigned v = src[i];
        const unsigned sym = symbol_of(v, base), l = len[sym];
        if (sym == 15u) {
            const unsigned slot = atomicAdd(counter, 1u);
            if (slot < cap) exc[slot] = (static_cast<unsigned long long>(i) << 16) | v;
        }
        const std::uint64_t c = pos / kXbhChunkBits;
        if (prev == ~0ull || prev / kXbhChunkBits != c) {  // first code starting in chunk c
            atomicOr(&gaps[c >> 3], static_cast<unsigned>(pos - c * kXbhChunkBits) << (4 * (c & 7)));
            if (c % kXbhBlockChunks == 0) bases[c / kXbhBlockChunks] = static_cast<std::uint32_t>(i);
        }
        prev = pos;
        pos += l;
        acc |= static_cast<unsigned long long>(cw[sym]) << (64 - nacc - l);
        nacc += l;
        if (nacc >= 32) {
            atomicOr(&words[w++], static_cast<unsigned>(acc >> 32));
            acc <<= 32;
            nacc -= 32;
        }
    }
    if (nacc) atomicOr(&words[w], static_cast<unsigned>(acc >> 32));
    if (v1 == n) {  // the last code may run into a final chunk where no code starts: its gap points at
                    // the end of the codes (a decode walk from there takes nothing); a block opening
                    // there holds no values (base n)
        const std::uint64_t cl = (pos + kXbhChunkBits - 1) / kXbhChunkBits - 1;
        if (prev / kXbhChunkBits != cl) {
            atomicOr(&gaps[cl >> 3], static_cast<unsigned>(pos - cl * kXbhChunkBits) << (4 * (cl & 7)));
            if (cl % kXbhBlockChunks == 0) bases[cl / kXbhBlockChunks] = static_cast<std::uint32_t>(n);
        }
    }
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

// ---- decode: one thread per 128-bit chunk, one CTA pass per block of 256 chunks --------------------
//  stage: the block's 1024 code words (+8 look-ahead) into shared memory (one pad word per 32: the
//         lanes' chunks are 4 words apart) — prefetched into registers during the previous block's
//         merge — and the gap of each thread's chunk;
//  walk:  each thread walks its chunk once from its gap with the multi-code table (up to 5, ~4 codes
//         per 12-bit lookup while the lookup's codes all start inside the chunk, then one code per
//         lookup until the next chunk's first code), queueing 4-bit symbols in a 64-bit fifo that
//         spills 8 at a time into the thread's slot (17-word stride: conflict-free spills);
//  scan:  the CTA turns code counts into the first block-relative value index of every chunk;
//  compact: each thread ORs its slot's symbols into a zeroed block-wide nibble buffer at its
//         position (value j at nibble j + (v0 & 15): 16-value groups stay word-aligned);
//  merge: per 16-value group of the block's value range, 8 bytes of symbols (+ the window base =
//         exponent; escapes are patched afterwards) join the lo bytes into bf16: 16-byte lo loads,
//         32-byte stores (element stores for the two partial groups at the range ends, which the
//         neighbouring blocks share); the merge zeroes the nibble words it read.
constexpr int kDecThreads = static_cast<int>(kXbhBlockChunks);
constexpr std::uint64_t kDecBlocksPerCta = 2;
constexpr int kDecWords = static_cast<int>(kXbhBlockBits / 32);  // 1024
constexpr int kDecStage = (kDecWords + 8 + (kDecWords + 8) / 32 + 1 + 3) / 4 * 4;  // padded, 16-byte multiple
constexpr int kDecSlot = static_cast<int>(kXbhChunkBits) / 8 + 1;  // <= 128 codes per chunk, 8 per word, + pad
constexpr int kDecSlotWords = kDecThreads * kDecSlot + 4;         // + the gather's read-ahead past the last slot
constexpr int kDecNibWords = (static_cast<int>(kXbhBlockBits) + 32) / 8 + 2;  // the block's symbols, 8 per word
constexpr size_t kDecSmem = sizeof(std::uint32_t) * (kXbhLut + kDecStage + 2 * (kDecThreads / 32) + kDecSlotWords +
                                                     kDecNibWords);

__device__ __forceinline__ unsigned padw(unsigned w) { return w + (w >> 5); }

__global__ void __launch_bounds__(kDecThreads) decode_kernel(const std::uint8_t* rec, std::uint64_t n,
                                                             std::uint64_t bits, unsigned base_exp, std::uint16_t* dst) {
    extern __shared__ __align__(16) std::uint32_t sm[];
    std::uint32_t* mlut = sm;
    std::uint32_t* sw = sm + kXbhLut;
    std::uint32_t* wsum = sw + kDecStage;
    std::uint32_t* slots = wsum + 2 * (kDecThreads / 32);  // [thread][kDecSlot] symbol nibbles
    std::uint32_t* nib = slots + kDecSlotWords;  // compacted: block-relative value j at nibble j + (v0 & 15)
    for (int i = threadIdx.x; i < kDecNibWords; i += kDecThreads) nib[i] = 0;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const std::uint32_t* words = reinterpret_cast<const std::uint32_t*>(rec + xbh_bits_off(n));
    const std::uint32_t* gaps = reinterpret_cast<const std::uint32_t*>(rec + xbh_gap_off(n, bits));
    const std::uint32_t* bases = reinterpret_cast<const std::uint32_t*>(rec + xbh_base_off(n, bits));
    const uint4* lo = reinterpret_cast<const uint4*>(rec);
    const std::uint64_t chunks = xbh_chunks(bits), blocks = xbh_blocks(bits);
    {
        const uint4* src = reinterpret_cast<const uint4*>(rec + xbh_mlut_off(n));
        for (int i = t; i < kXbhLut / 4; i += kDecThreads) reinterpret_cast<uint4*>(mlut)[i] = __ldg(src + i);
    }
    const unsigned base4 = (base_exp & 0xffu) * 0x01010101u;
    const std::uint64_t nwords = xbh_words(bits);  // the bit section's words (codes + zero padding)
    uint4 pw, px = make_uint4(0, 0, 0, 0);
    std::uint32_t pg = 0;
    auto prefetch = [&](std::uint64_t b) {
        const std::uint64_t q = b * (kDecWords / 4) + t;  // uint4 index in the bit section
        const uint4* src = reinterpret_cast<const uint4*>(words);
        pw = 4 * q + 4 <= nwords ? __ldg(src + q) : make_uint4(0, 0, 0, 0);
        if (t < 2) px = 4 * (q + kDecThreads) + 4 <= nwords ? __ldg(src + q + kDecThreads) : make_uint4(0, 0, 0, 0);
        const std::uint64_t c = b * kXbhBlockChunks + t;
        pg = c < chunks ? __ldg(gaps + (c >> 3)) : 0u;
    };
    auto peek = [&](unsigned pos) {  // 12 bits at `pos` of the staged block
        const unsigned w = pos >> 5;
        return __funnelshift_l(sw[padw(w + 1)], sw[padw(w)], pos & 31u) >> (32 - kXbhMaxLen);
    };
    std::uint32_t* slot = slots + t * kDecSlot;
    // kDecBlocksPerCta consecutive blocks per CTA: short-lived CTAs, so a higher-priority kernel (the
    // FFN on the compute stream) waiting for SM space gets it within one CTA's lifetime
    std::uint64_t b = static_cast<std::uint64_t>(blockIdx.x) * kDecBlocksPerCta;
    const std::uint64_t b_end = std::min<std::uint64_t>(blocks, b + kDecBlocksPerCta);
    if (b < b_end) prefetch(b);
    for (; b < b_end; ++b) {
        __syncthreads();  // the previous block's merge is done with sw / slots / nib
        {
            const unsigned w = 4u * t;  // 4 words, none crossing a pad (w % 32 <= 28)
            sw[padw(w)] = pw.x, sw[padw(w) + 1] = pw.y, sw[padw(w) + 2] = pw.z, sw[padw(w) + 3] = pw.w;
            if (t < 2) {
                const unsigned x = 4u * (kDecThreads + t);
                sw[padw(x)] = px.x, sw[padw(x) + 1] = px.y, sw[padw(x) + 2] = px.z, sw[padw(x) + 3] = px.w;
            }
        }
        const std::uint64_t c = b * kXbhBlockChunks + t;
        const unsigned end = static_cast<unsigned>(t + 1) * static_cast<unsigned>(kXbhChunkBits);
        const std::uint64_t rem = bits - b * kXbhBlockBits;  // codes start below this in the block
        const unsigned stop = c < chunks ? (end < rem ? end : static_cast<unsigned>(rem)) : 0u;
        unsigned pos =
            static_cast<unsigned>(t) * static_cast<unsigned>(kXbhChunkBits) + ((pg >> (4 * (c & 7))) & 15u);
        const std::uint64_t v0 = __ldg(bases + b), v1 = __ldg(bases + b + 1);
        __syncthreads();
        // walk: symbols into the slot (a lookup adds <= 5 symbols: the fifo holds <= 12 before a spill)
        unsigned nf = 0, sp = 0;
        unsigned long long fifo = 0;
        auto spill = [&]() {
            if (nf >= 8) {
                slot[sp++] = static_cast<std::uint32_t>(fifo);
                fifo >>= 32;
                nf -= 8;
            }
        };
        auto take_all = [&]() {  // every code of the lookup (<= 5) starts inside the chunk
            const unsigned e = mlut[peek(pos)];
            fifo |= static_cast<unsigned long long>(e & 0xfffffu) << (4 * nf);  // unused symbol nibbles are zero
            nf += (e >> 20) & 7u;
            pos += e >> 27;
        };
        while (pos + kXbhMaxLen <= stop) {
            take_all();
            spill();
        }
        while (pos < stop) {  // the chunk's last codes, one per lookup: stop where the next chunk's first code starts
            const unsigned e = mlut[peek(pos)];
            fifo |= static_cast<unsigned long long>(e & 15u) << (4 * nf);
            nf += 1;
            pos += (e >> 23) & 15u;
            spill();
        }
        const unsigned cnt = 8 * sp + nf;
        if (nf) slot[sp] = static_cast<std::uint32_t>(fifo);
        // scan: this chunk's first block-relative value
        unsigned incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        unsigned before = 0;
#pragma unroll
        for (int w = 0; w < kDecThreads / 32; ++w) before += w < warp ? wsum[w] : 0u;
        // compact: this chunk's cnt symbols to nibbles [o, o + cnt) of the block buffer (words shared with
        // the neighbouring chunks: atomicOr into the zeroed buffer)
        {
            const unsigned o = before + incl - cnt + static_cast<unsigned>(v0 & 15);
            const unsigned sh = 4 * (o & 7);
            std::uint32_t* d = nib + (o >> 3);
            for (unsigned w = 0; 8 * w < cnt; ++w) {
                const unsigned rest = cnt - 8 * w;  // symbols left, the slot's stale tail masked off
                const std::uint32_t x = rest >= 8 ? slot[w] : slot[w] & ((1u << (4 * rest)) - 1u);
                atomicOr(d + w, x << sh);
                if (sh) atomicOr(d + w + 1, x >> (32 - sh));
            }
        }
        __syncthreads();
        // merge
        const std::uint64_t gs = v0 >> 4, ge = (v1 + 15) >> 4;  // 16-value groups touching [v0, v1)
        if (b + 1 < b_end) prefetch(b + 1);
        for (std::uint64_t g = gs + t; g < ge; g += kDecThreads) {
            const uint4 l = __ldg(lo + g);
            // the group's 16 symbols (values of other blocks at the range ends are masked on store)
            const uint2 sy2 = *reinterpret_cast<const uint2*>(nib + 2 * (g - gs));
            nib[2 * (g - gs)] = 0;  // zeroed for the next block
            nib[2 * (g - gs) + 1] = 0;
            const unsigned long long sy = (static_cast<unsigned long long>(sy2.y) << 32) | sy2.x;
            const unsigned sx = static_cast<unsigned>(sy), sz = static_cast<unsigned>(sy >> 32);
            const unsigned ew[4] = {  // nibbles -> bytes + window base: symbols 4q .. 4q+3
                __vadd4(__byte_perm(sx & 0x0f0f0f0fu, (sx >> 4) & 0x0f0f0f0fu, 0x5140), base4),
                __vadd4(__byte_perm(sx & 0x0f0f0f0fu, (sx >> 4) & 0x0f0f0f0fu, 0x7362), base4),
                __vadd4(__byte_perm(sz & 0x0f0f0f0fu, (sz >> 4) & 0x0f0f0f0fu, 0x5140), base4),
                __vadd4(__byte_perm(sz & 0x0f0f0f0fu, (sz >> 4) & 0x0f0f0f0fu, 0x7362), base4)};
            const unsigned lw[4] = {l.x, l.y, l.z, l.w};
            unsigned out[8];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const unsigned lp0 = __byte_perm(lw[q], 0, 0x4140), ep0 = __byte_perm(ew[q], 0, 0x4140);
                const unsigned lp1 = __byte_perm(lw[q], 0, 0x4342), ep1 = __byte_perm(ew[q], 0, 0x4342);
                out[2 * q] = ((lp0 & 0x00800080u) << 8) | (ep0 << 7) | (lp0 & 0x007f007fu);
                out[2 * q + 1] = ((lp1 & 0x00800080u) << 8) | (ep1 << 7) | (lp1 & 0x007f007fu);
            }
            if (g * 16 >= v0 && g * 16 + 16 <= v1) {
                uint4* d = reinterpret_cast<uint4*>(dst + g * 16);
                d[0] = make_uint4(out[0], out[1], out[2], out[3]);
                d[1] = make_uint4(out[4], out[5], out[6], out[7]);
            } else {  // a range end: only this block's values
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const std::uint64_t v = g * 16 + k;
                    if (v >= v0 && v < v1) dst[v] = static_cast<std::uint16_t>(out[k >> 1] >> (16 * (k & 1)));
                }
            }
        }
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
                       std::uint32_t* gaps, std::uint32_t* bases, std::uint64_t* exc, std::uint64_t exc_cap,
                       std::uint32_t* seglen, std::uint32_t* work, cudaStream_t stream) {
    if (n % 16 || !src || !dcode || !record || !gaps || !bases || !seglen || !work) return cudaErrorInvalidValue;
    if (n * kXbhMaxLen >= (1ull << 32)) return cudaErrorInvalidValue;  // u32 bit offsets
    const std::uint64_t nseg = xbh_enc_segments(n);
    std::uint32_t* words = reinterpret_cast<std::uint32_t*>(record + xbh_bits_off(n));
    cudaError_t e = cudaMemsetAsync(words, 0, 4 * xbh_words(n * kXbhMaxLen), stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(gaps, 0, 4 * xbh_gap_words(n * kXbhMaxLen), stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(work, 0, kXbhWorkWords * sizeof(std::uint32_t), stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(record + xbh_lut_off(n), dcode->lut, 6 * kXbhLut, cudaMemcpyDeviceToDevice, stream);
    if (e != cudaSuccess) return e;
    lo_kernel<<<grid_for(n / 16), kThreads, 0, stream>>>(reinterpret_cast<const uint4*>(src), n / 16,
                                                          reinterpret_cast<uint4*>(record));
    seglen_kernel<<<grid_all(nseg, kThreads), kThreads, 0, stream>>>(reinterpret_cast<const uint4*>(src), n, dcode, seglen);
    scan_kernel<<<1, 1024, 0, stream>>>(seglen, nseg, work);
    emit_kernel<<<grid_all(nseg, kThreads), kThreads, 0, stream>>>(src, n, dcode, seglen, words, gaps, bases,
                                                                    reinterpret_cast<unsigned long long*>(exc), exc_cap,
                                                                    work);
    return cudaGetLastError();
}

cudaError_t xbh_decode(const std::uint8_t* record, const Xb12Tile& t, std::uint16_t* dst, cudaStream_t stream) {
    if (t.format != 2 || t.n % 16) return cudaErrorInvalidValue;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    static std::atomic<unsigned long long> configured{0};  // one bit per device: > 48 KB dynamic smem opted in
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!(configured.load() >> dev & 1ull)) {
        e = cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kDecSmem));
        if (e != cudaSuccess) return e;
        configured.fetch_or(1ull << dev);
    }
    const std::uint64_t blocks = xbh_blocks(t.code_bits);
    const int grid = static_cast<int>(std::max<std::uint64_t>(1, (blocks + kDecBlocksPerCta - 1) / kDecBlocksPerCta));
    decode_kernel<<<grid, kDecThreads, kDecSmem, stream>>>(record, t.n, t.code_bits, t.base, dst);
    if (t.n_exc)
        patch_kernel<<<grid_for(t.n_exc), kThreads, 0, stream>>>(
            reinterpret_cast<const unsigned long long*>(record + t.exc_off), t.n_exc, dst);
    return cudaGetLastError();
}

void xbh_decode_host(const std::uint8_t* record, const Xb12Tile& t, std::uint16_t* dst, std::uint64_t i0,
                     std::uint64_t count) {
    if (!count) return;
    const std::uint16_t* lut = reinterpret_cast<const std::uint16_t*>(record + xbh_lut_off(t.n));
    const std::uint32_t* words = reinterpret_cast<const std::uint32_t*>(record + xbh_bits_off(t.n));
    const std::uint32_t* gaps = reinterpret_cast<const std::uint32_t*>(record + xbh_gap_off(t.n, t.code_bits));
    const std::uint32_t* bases = reinterpret_cast<const std::uint32_t*>(record + xbh_base_off(t.n, t.code_bits));
    const std::uint64_t blocks = xbh_blocks(t.code_bits);
    // the last block whose first code is at or before value i0
    const std::uint64_t b = static_cast<std::uint64_t>(std::upper_bound(bases, bases + blocks, i0) - bases) - 1;
    std::uint64_t pos = b * kXbhBlockBits + (gaps[(b * kXbhBlockChunks) >> 3] & 15u);
    const std::uint64_t end = i0 + count;
    for (std::uint64_t i = bases[b]; i < end; ++i) {
        const std::uint64_t w = pos >> 5;
        const unsigned long long win = (static_cast<unsigned long long>(words[w]) << 32) | words[w + 1];
        const unsigned e = lut[(win << (pos & 31)) >> (64 - kXbhMaxLen)];
        pos += e >> 8;
        if (i < i0) continue;
        const unsigned lb = record[i];
        dst[i - i0] = static_cast<std::uint16_t>(((lb & 0x80u) << 8) | ((e & 0xffu) << 7) | (lb & 0x7fu));
    }
    const std::uint64_t* exc = reinterpret_cast<const std::uint64_t*>(record + t.exc_off);
    const std::uint64_t* it = std::lower_bound(exc, exc + t.n_exc, i0 << 16);
    for (; it < exc + t.n_exc && (*it >> 16) < end; ++it) dst[(*it >> 16) - i0] = static_cast<std::uint16_t>(*it & 0xffffu);
}

}  // namespace adapmoe
