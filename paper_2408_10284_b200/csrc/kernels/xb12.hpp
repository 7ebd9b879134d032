// XB12 — lossless exponent-coded bf16 for the host-link copies of offloaded expert tiles.
//
// The decode at any budget below L*N moves ~19 GB of expert weights per token over a 55 GB/s PCIe
// link and runs at that link's bound (the FFN is ~2 % of the step), so the bytes on the link are
// the cost.  bf16 weights spend 8 bits on an exponent whose distribution is narrow (random-init
// and trained LLM weights alike: 15 consecutive exponents hold all but ~1e-4 of a tile's values), so
// the host store keeps each tile as
//   lo  [n]   u8 : sign << 7 | mantissa(7)
//   nib [n/2] u8 : 4-bit code c of value i in nibble i & 1 of byte i / 2 (low nibble first);
//                  exponent = base + c for c < 15; c == 15 = escape
//   exc [m]   u64: (index << 16) | bf16 bits of each escaped value, index ascending
// i.e. 12 bits per value + 8 bytes per escape (75.0 % of the bytes at 8x7B), and the GPU restores
// the exact bf16 bits in HBM (decode + patch kernels, ~15 us per 88 MB tile) after the tile lands,
// before anything reads it.  A tile with more than n / 64 escapes stays raw bf16.  Bit-exact by
// construction: every value is either reconstructed from its own sign / exponent / mantissa or
// patched with its original bits.
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>

#ifdef __CUDACC__
#define XB_HD __host__ __device__
#else
#define XB_HD
#endif

namespace adapmoe {

struct Xb12Tile {
    int format = 0;               // 0 raw bf16 (the record is the tile), 1 XB12, 2 XBH (xbh.hpp)
    std::uint32_t base = 0;       // first exponent of the 15-exponent window
    std::uint64_t n = 0;          // values in the tile
    std::uint64_t n_exc = 0;      // escaped values
    std::uint64_t nib_off = 0;    // byte offsets inside the record (lo at 0); XBH: the segment table
    std::uint64_t exc_off = 0;
    std::uint64_t bytes = 0;      // record bytes (256-aligned)
    std::uint64_t code_bits = 0;  // XBH: total bits of the exponent codes
};

constexpr std::uint64_t kXb12Align = 256;
XB_HD inline std::uint64_t xb12_align(std::uint64_t v, std::uint64_t a = 16) { return (v + a - 1) / a * a; }
// record layout for n values with m escapes
inline void xb12_layout(Xb12Tile& t) {
    t.nib_off = xb12_align(t.n);
    t.exc_off = xb12_align(t.nib_off + t.n / 2);
    t.bytes = xb12_align(t.exc_off + t.n_exc * 8, kXb12Align);
}

// Encode (device): histogram of the tile's exponents -> best 15-exponent window (device-side, no
// host sync) -> lo / nib streams + escapes appended through an atomic counter (unordered; the host
// sorts them).  n % 16 == 0.  `work` holds 256 histogram bins + base + counter (u32).
cudaError_t xb12_encode(const std::uint16_t* src, std::uint64_t n, std::uint8_t* lo, std::uint8_t* nib,
                        std::uint64_t* exc, std::uint64_t exc_cap, std::uint32_t* work, cudaStream_t stream);
constexpr int kXb12WorkWords = 258;  // hist[256], base, escape count

// Exponent histogram of n bf16 values (n % 8 == 0) into hist[256] (zeroed here).
cudaError_t xb12_histogram(const std::uint16_t* src, std::uint64_t n, std::uint32_t* hist, cudaStream_t stream);

// Decode (device): dst[i] = bf16 of (lo, nib) for every i, then the escapes patched.
cudaError_t xb12_decode(const std::uint8_t* record, const Xb12Tile& t, std::uint16_t* dst, cudaStream_t stream);

// Host restatements (CPU consumers of the store, tests).
void xb12_decode_host(const std::uint8_t* record, const Xb12Tile& t, std::uint16_t* dst, std::uint64_t i0,
                      std::uint64_t count);

}  // namespace adapmoe
