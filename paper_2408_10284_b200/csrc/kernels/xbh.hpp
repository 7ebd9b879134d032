// XBH — lossless bf16 with Huffman-coded exponents, for the host-link copies of offloaded expert
// tiles (format 2 of the store; XB12, format 1, is the fixed 4-bit exponent code of xb12.hpp).
//
// The budget-64 decode runs at the PCIe link's bound, so link bytes are the step time.  XB12 spends
// 4 bits on each exponent; the exponents of weight tiles carry ~2.5 bits of entropy (random-init and
// trained LLM weights alike: two or three exponents hold most values, each lower one about half as
// many), so XBH codes them with a per-tile canonical Huffman code:
//   lo   [n]        u8  : sign << 7 | mantissa(7)                                   at 0
//   lut  [4096]     u16 : decode table, entry = exponent | code length << 8         at lut_off = align(n)
//   seg  [n_seg+1]  u32 : bit offset of each 512-value segment's codes; [n_seg] = total bits
//                                                                                   at seg_off = lut_off + 8192
//   bits [words]    u32 : the codes, MSB first, segments back to back (+2 zero words of padding)
//                                                                                   at bits_off = align(seg_off + 4 (n_seg+1))
//   exc  [m]        u64 : (index << 16) | bf16 bits of each escaped value, index ascending
//                                                                                   at exc_off
// Symbols: exponent base + s for s < 15 (the tile's best 15-exponent window, as XB12), s = 15 =
// escape (the value's bits are patched from `exc`).  Code lengths are length-limited Huffman
// (package-merge, <= kXbhMaxLen bits) over the 16 symbol counts, codes canonical by (length,
// symbol), so a record is a pure function of the tile.  ~10.6 bits per value at 8x7B (66 % of bf16,
// XB12 75 %).  Decode: one thread per segment walks its bit string through the shared-memory table
// (12-bit peek), merges each exponent with its lo byte and stores 32-byte runs of bf16; escapes are
// patched afterwards.  Bit-exact by construction, like XB12.
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>

#include "xb12.hpp"

namespace adapmoe {

constexpr int kXbhMaxLen = 12;        // longest code: the decode table has 2^12 entries
constexpr int kXbhLut = 1 << kXbhMaxLen;
constexpr std::uint64_t kXbhSeg = 512;  // values per independently decodable segment

XB_HD inline std::uint64_t xbh_segments(std::uint64_t n) { return (n + kXbhSeg - 1) / kXbhSeg; }
// Sections that depend only on n (Xb12Tile fields: nib_off = seg_off; lut and bits offsets derived).
XB_HD inline std::uint64_t xbh_lut_off(std::uint64_t n) { return xb12_align(n); }
XB_HD inline std::uint64_t xbh_seg_off(std::uint64_t n) { return xbh_lut_off(n) + 2 * kXbhLut; }
XB_HD inline std::uint64_t xbh_bits_off(std::uint64_t n) { return xb12_align(xbh_seg_off(n) + 4 * (xbh_segments(n) + 1)); }
XB_HD inline std::uint64_t xbh_words(std::uint64_t total_bits) { return (total_bits + 31) / 32 + 2; }
// record layout for n values, total_bits of codes and t.n_exc escapes (t.n, t.n_exc set)
inline void xbh_layout(Xb12Tile& t, std::uint64_t total_bits) {
    t.nib_off = xbh_seg_off(t.n);
    t.exc_off = xb12_align(xbh_bits_off(t.n) + 4 * xbh_words(total_bits));
    t.bytes = xb12_align(t.exc_off + t.n_exc * 8, kXb12Align);
}

// The per-tile code, built on the host from the exponent histogram (hist[256]): window base,
// lengths / canonical codes of the 16 symbols (0 = symbol absent) and the decode table.
struct XbhCode {
    std::uint32_t base = 0;
    std::uint8_t len[16] = {};
    std::uint16_t code[16] = {};
    std::uint16_t lut[kXbhLut] = {};
};
void xbh_build_code(const std::uint32_t* hist, XbhCode& c);

// Encode (device), given the tile's code (device copy of XbhCode, `dcode`):
//   record: lo, lut, seg and bits sections (bits zeroed here); exc: escapes, unordered, through the
//   counter work[0]; work[1] = total bits.  `seglen` scratch: n_seg + 1 u32.
cudaError_t xbh_encode(const std::uint16_t* src, std::uint64_t n, const XbhCode* dcode, std::uint8_t* record,
                       std::uint64_t* exc, std::uint64_t exc_cap, std::uint32_t* seglen, std::uint32_t* work,
                       cudaStream_t stream);
constexpr int kXbhWorkWords = 2;
// Upper bound of the encoder's record region for n values (lo + lut + seg + 12 bits per value).
inline std::uint64_t xbh_region_bytes(std::uint64_t n) {
    return xb12_align(xbh_bits_off(n) + 4 * xbh_words(n * kXbhMaxLen));
}

// Decode (device): dst[i] = bf16 of value i for every i, then the escapes patched.
cudaError_t xbh_decode(const std::uint8_t* record, const Xb12Tile& t, std::uint16_t* dst, cudaStream_t stream);

// Host restatement: values [i0, i0 + count) of a record.
void xbh_decode_host(const std::uint8_t* record, const Xb12Tile& t, std::uint16_t* dst, std::uint64_t i0,
                     std::uint64_t count);

}  // namespace adapmoe
