// XBH — lossless bf16 with Huffman-coded exponents, for the host-link copies of offloaded expert
// tiles (format 2 of the store; XB12, format 1, is the fixed 4-bit exponent code of xb12.hpp).
//
// The budget-64 decode runs at the PCIe link's bound, so link bytes are the step time.  XB12 spends
// 4 bits on each exponent; the exponents of weight tiles carry ~2.5 bits of entropy (random-init and
// trained LLM weights alike: two or three exponents hold most values, each lower one about half as
// many), so XBH codes them with a per-tile canonical Huffman code.  Record of a tile of n values:
//   lo   [n]        u8  : sign << 7 | mantissa(7)                                   at 0
//   lut  [4096]     u16 : single-code table of the 12-bit peek: exponent | length << 8   at lut_off = align(n)
//   mlut [4096]     u32 : multi-code table: up to 5 consecutive codes inside the peek — symbols
//                         (4 bits each, bits 0-19), count (20-22), the first code's length (23-26),
//                         total length (27-30)                                      at mlut_off = lut_off + 8 KB
//   hdr             2 u64: total code bits, escapes                                  at hdr_off = mlut_off + 16 KB
//   bits [words]    u32 : the codes, MSB first, back to back (+8 zero words)         at bits_off = hdr_off + 16
//   gaps [chunks]   4 bit: per 128-bit chunk of `bits`, the offset of the first code starting in it
//                         (<= 11: a code is <= 12 bits; a final chunk that only holds the end of the
//                         last code points at the end of the codes), 8 per u32, low nibble first
//                                                                                   at gap_off
//   base [blocks+1] u32 : per block of 256 chunks, the index of the value whose code starts first in
//                         it (n for a final block without one); [blocks] = n          at base_off
//   exc  [m]        u64 : (index << 16) | bf16 bits of each escaped value, index ascending   at exc_off
// Symbols: exponent base + s for s < 15 (the tile's best 15-exponent window, as XB12), s = 15 =
// escape (the value's bits are patched from `exc`).  Code lengths are length-limited Huffman
// (package-merge, <= kXbhMaxLen bits) over the 16 symbol counts, codes canonical by (length,
// symbol), so a record is a pure function of the tile.  ~10.6 bits per value at 8x7B (66 % of bf16,
// XB12 75 %).  The chunk gaps make every 128 bits of codes an independent unit of decoding (~50
// codes; ~880k units in an 88 MB tile): one GPU thread per chunk counts its codes, a CTA scan turns
// counts into output positions, the thread decodes again into a shared exponent buffer and the CTA
// merges exponents with the lo bytes into bf16 (the DFloat11 scheme).  Host decoders walk the
// single-code table from a block start.  Bit-exact by construction, like XB12.
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>

#include "xb12.hpp"

namespace adapmoe {

constexpr int kXbhMaxLen = 12;        // longest code: the decode tables have 2^12 entries
constexpr int kXbhLut = 1 << kXbhMaxLen;
constexpr int kXbhMultiCodes = 5;     // codes per multi-code table entry
constexpr std::uint64_t kXbhChunkBits = 128;  // unit of independent decoding
constexpr std::uint64_t kXbhBlockChunks = 256;  // chunks per output-base entry (one decode CTA pass)
constexpr std::uint64_t kXbhBlockBits = kXbhChunkBits * kXbhBlockChunks;

XB_HD inline std::uint64_t xbh_chunks(std::uint64_t bits) { return (bits + kXbhChunkBits - 1) / kXbhChunkBits; }
XB_HD inline std::uint64_t xbh_blocks(std::uint64_t bits) { return (bits + kXbhBlockBits - 1) / kXbhBlockBits; }
XB_HD inline std::uint64_t xbh_lut_off(std::uint64_t n) { return xb12_align(n); }
XB_HD inline std::uint64_t xbh_mlut_off(std::uint64_t n) { return xbh_lut_off(n) + 2 * kXbhLut; }
XB_HD inline std::uint64_t xbh_hdr_off(std::uint64_t n) { return xbh_mlut_off(n) + 4 * kXbhLut; }
XB_HD inline std::uint64_t xbh_bits_off(std::uint64_t n) { return xbh_hdr_off(n) + 16; }
// code words + 8 zero words (a decode block reads up to 8 words past its 32 Kbit span)
XB_HD inline std::uint64_t xbh_words(std::uint64_t bits) { return (bits + 31) / 32 + 8; }
XB_HD inline std::uint64_t xbh_gap_off(std::uint64_t n, std::uint64_t bits) {
    return xb12_align(xbh_bits_off(n) + 4 * xbh_words(bits));
}
XB_HD inline std::uint64_t xbh_gap_words(std::uint64_t bits) { return (xbh_chunks(bits) + 7) / 8; }
XB_HD inline std::uint64_t xbh_base_off(std::uint64_t n, std::uint64_t bits) {
    return xb12_align(xbh_gap_off(n, bits) + 4 * xbh_gap_words(bits));
}
// record layout for t.n values, `bits` of codes and t.n_exc escapes (Xb12Tile: nib_off = hdr_off)
inline void xbh_layout(Xb12Tile& t, std::uint64_t bits) {
    t.code_bits = bits;
    t.nib_off = xbh_hdr_off(t.n);
    t.exc_off = xb12_align(xbh_base_off(t.n, bits) + 4 * (xbh_blocks(bits) + 1));
    t.bytes = xb12_align(t.exc_off + t.n_exc * 8, kXb12Align);
}

// The per-tile code, built on the host from the exponent histogram (hist[256]): window base,
// lengths / canonical codes of the 16 symbols (0 = symbol absent) and the decode tables.
struct XbhCode {
    std::uint32_t base = 0;
    std::uint8_t len[16] = {};
    std::uint16_t code[16] = {};
    std::uint16_t lut[kXbhLut] = {};
    std::uint32_t mlut[kXbhLut] = {};
};
void xbh_build_code(const std::uint32_t* hist, XbhCode& c);

// Encode (device), given the tile's code (device copy of XbhCode, `dcode`), into scratch sections:
//   record: lo, lut, mlut and bits (zeroed here) at their record offsets (hdr not written);
//   gaps: >= xbh_gap_words(n * kXbhMaxLen) u32 (zeroed here); bases: >= xbh_blocks(n * kXbhMaxLen)
//   u32; exc: escapes, unordered, through the counter work[0]; work[1] = total code bits.
//   `seglen`: xbh_enc_segments(n) + 1 u32 of scratch.
constexpr std::uint64_t kXbhEncSeg = 512;  // values per encoder thread
XB_HD inline std::uint64_t xbh_enc_segments(std::uint64_t n) { return (n + kXbhEncSeg - 1) / kXbhEncSeg; }
cudaError_t xbh_encode(const std::uint16_t* src, std::uint64_t n, const XbhCode* dcode, std::uint8_t* record,
                       std::uint32_t* gaps, std::uint32_t* bases, std::uint64_t* exc, std::uint64_t exc_cap,
                       std::uint32_t* seglen, std::uint32_t* work, cudaStream_t stream);
constexpr int kXbhWorkWords = 2;
// Upper bound of the encoder's record region for n values (lo + tables + hdr + 12 bits per value).
inline std::uint64_t xbh_region_bytes(std::uint64_t n) {
    return xb12_align(xbh_bits_off(n) + 4 * xbh_words(n * kXbhMaxLen));
}

// Decode (device): dst[i] = bf16 of value i for every i, then the escapes patched.
cudaError_t xbh_decode(const std::uint8_t* record, const Xb12Tile& t, std::uint16_t* dst, cudaStream_t stream);

// Host restatement: values [i0, i0 + count) of a record (walks the single-code table from the
// block whose first code precedes i0).
void xbh_decode_host(const std::uint8_t* record, const Xb12Tile& t, std::uint16_t* dst, std::uint64_t i0,
                     std::uint64_t count);

}  // namespace adapmoe
