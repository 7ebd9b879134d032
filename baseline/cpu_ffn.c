/* CPU expert-FFN decode baseline — builder-written, NOT the reference.
 *
 * The reference (moesim) charges expert compute as ticks and does no FFN arithmetic
 * (/root/reference/proj/include/moesim/simulator.hpp:446-462), so its timed CPU path moves no
 * weights.  BASELINE.md §4.3 asks for a CPU SwiGLU of the same decode next to it: this file computes
 * one MoE layer, out = x + sum_e w_e * SwiGLU_e(x), for the selected experts of a (token, layer),
 * reading the expert weights in place from the engine's pinned host store (moe_expert_host_ptr;
 * tile-major bf16 layout of paper_2408_10284_b200/csrc/kernels/expert_ffn.hpp), fp32 accumulation,
 * ffn rows split over OpenMP threads (each thread a private partial of y, summed in thread order).
 * Used only by bench.py's cpu_baseline_ffn leg.
 *   gcc -O3 -march=x86-64-v3 -fopenmp -fPIC -shared -o baseline/libcpu_ffn.so baseline/cpu_ffn.c -lm
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline float bf16(uint16_t v) {
    union { uint32_t u; float f; } c;
    c.u = (uint32_t)v << 16;
    return c.f;
}

/* XB12 / XBH records (paper_2408_10284_b200/csrc/kernels/xb12.hpp, xbh.hpp) decoded on the fly: values
 * [i0, i0 + n) of one tile record into bf16 (pairs share a nibble byte: vectorisable), then the
 * escapes that fall in the range (ascending list, binary search). */
typedef struct {
    const uint8_t* rec;
    int32_t format; /* 0 raw bf16, 1 XB12, 2 XBH */
    uint32_t base;
    int64_t n_exc, nib_off, exc_off;
    int64_t n; /* values in the tile */
} tile_rec;

/* XBH (kernels/xbh.hpp): sections at offsets derived from n and the header's code-bit count; the
 * walk starts at the last block whose first code precedes i0 (block value bases + chunk gaps) and
 * follows the single-code table. */
#define XBH_MAXLEN 12
#define XBH_BLOCK_BITS (256 * 128)
static int64_t al16(int64_t v) { return (v + 15) / 16 * 16; }
static void decode_xbh(const tile_rec* t, int64_t i0, int64_t n, uint16_t* dst) {
    const int64_t N = t->n, lut_off = al16(N), hdr_off = lut_off + 6 * (1 << XBH_MAXLEN); /* lut u16 + mlut u32 */
    const int64_t bits = (int64_t)((const uint64_t*)(t->rec + hdr_off))[0];
    const int64_t bits_off = hdr_off + 16, words = (bits + 31) / 32 + 8, chunks = (bits + 127) / 128;
    const int64_t gap_off = al16(bits_off + 4 * words), base_off = al16(gap_off + 4 * ((chunks + 7) / 8));
    const int64_t blocks = (bits + XBH_BLOCK_BITS - 1) / XBH_BLOCK_BITS;
    const uint16_t* lut = (const uint16_t*)(t->rec + lut_off);
    const uint32_t* w = (const uint32_t*)(t->rec + bits_off);
    const uint32_t* gaps = (const uint32_t*)(t->rec + gap_off);
    const uint32_t* bases = (const uint32_t*)(t->rec + base_off);
    int64_t lo_b = 0, hi_b = blocks; /* last block with bases[b] <= i0 */
    while (hi_b - lo_b > 1) {
        const int64_t m = (lo_b + hi_b) / 2;
        if ((int64_t)bases[m] <= i0) lo_b = m; else hi_b = m;
    }
    uint64_t pos = (uint64_t)lo_b * XBH_BLOCK_BITS + (gaps[(lo_b * 256) >> 3] & 15u);
    const int64_t end = i0 + n;
    for (int64_t i = bases[lo_b]; i < end; ++i) {
        const uint64_t win = ((uint64_t)w[pos >> 5] << 32) | w[(pos >> 5) + 1];
        const uint32_t e = lut[(win << (pos & 31)) >> (64 - XBH_MAXLEN)];
        pos += e >> 8;
        if (i < i0) continue;
        const uint32_t b = t->rec[i];
        dst[i - i0] = (uint16_t)(((b & 0x80u) << 8) | ((e & 0xffu) << 7) | (b & 0x7fu));
    }
}

static void decode_range(const tile_rec* t, int64_t i0, int64_t n, uint16_t* dst) {
    if (t->format == 0) {
        memcpy(dst, (const uint16_t*)t->rec + i0, (size_t)n * 2);
        return;
    }
    if (t->format == 2) {
        decode_xbh(t, i0, n, dst);
    } else {
        const uint8_t* lo = t->rec + i0;
        const uint8_t* nib = t->rec + t->nib_off + i0 / 2; /* i0 even */
        const uint32_t base = t->base;
        for (int64_t j = 0; j < n / 2; ++j) {
            const uint32_t c = nib[j], b0 = lo[2 * j], b1 = lo[2 * j + 1];
            const uint32_t e0 = (base + (c & 15u)) & 0xffu, e1 = (base + (c >> 4)) & 0xffu;
            dst[2 * j] = (uint16_t)(((b0 & 0x80u) << 8) | (e0 << 7) | (b0 & 0x7fu));
            dst[2 * j + 1] = (uint16_t)(((b1 & 0x80u) << 8) | (e1 << 7) | (b1 & 0x7fu));
        }
    }
    const uint64_t* exc = (const uint64_t*)(t->rec + t->exc_off);
    int64_t a = 0, b = t->n_exc;
    while (a < b) { /* first escape with index >= i0 */
        const int64_t m = (a + b) / 2;
        if ((int64_t)(exc[m] >> 16) < i0) a = m + 1; else b = m;
    }
    for (; a < t->n_exc && (int64_t)(exc[a] >> 16) < i0 + n; ++a) dst[(exc[a] >> 16) - i0] = (uint16_t)(exc[a] & 0xffffu);
}

/* The same layer as cpu_moe_layer over coded stores (XB12 / XBH records, or raw tiles):
 * recs[k * tiles + t] = tile t of selected expert k. */
int cpu_moe_layer_xb12(const void* const* recs, const int32_t* formats, const uint32_t* bases, const int64_t* n_exc,
                       const int64_t* nib_off, const int64_t* exc_off, const double* weights, int n_experts, int D,
                       int F, int tiles, const double* x_in, float* out, int threads) {
    if (D <= 0 || F <= 0 || tiles <= 0 || F % tiles || n_experts < 0 || threads <= 0 || D % 2) return 1;
    const int Ft = F / tiles;
    float* x = (float*)malloc(sizeof(float) * D);
    float* part = (float*)calloc((size_t)threads * D, sizeof(float));
    uint16_t* rows = (uint16_t*)malloc(sizeof(uint16_t) * 3 * (size_t)D * threads);
    if (!x || !part || !rows) return 2;
    for (int j = 0; j < D; ++j) x[j] = (float)x_in[j];
    for (int j = 0; j < D; ++j) out[j] = x[j];
    for (int k = 0; k < n_experts; ++k) {
        memset(part, 0, sizeof(float) * (size_t)threads * D);
#pragma omp parallel num_threads(threads)
        {
            const int t = omp_get_thread_num(), nt = omp_get_num_threads();
            float* y = part + (size_t)t * D;
            uint16_t* w1 = rows + (size_t)3 * D * t;
            uint16_t* w3 = w1 + D;
            uint16_t* w2 = w3 + D;
            const int r0 = (int)((long long)F * t / nt), r1 = (int)((long long)F * (t + 1) / nt);
            for (int r = r0; r < r1; ++r) {
                const int ti = r / Ft, rr = r % Ft;
                const size_t q = (size_t)k * tiles + ti;
                const tile_rec tr = {(const uint8_t*)recs[q], formats[q], bases[q], n_exc[q], nib_off[q], exc_off[q],
                                     (int64_t)3 * Ft * D};
                decode_range(&tr, (int64_t)rr * 2 * D, 2 * (int64_t)D, w1); /* W1 row then W3 row */
                decode_range(&tr, (int64_t)2 * Ft * D + (int64_t)rr * D, D, w2);
                float a = 0.0f, b = 0.0f;
#pragma omp simd reduction(+ : a, b)
                for (int j = 0; j < D; ++j) {
                    a += bf16(w1[j]) * x[j];
                    b += bf16(w3[j]) * x[j];
                }
                const float h = a / (1.0f + expf(-a)) * b;
#pragma omp simd
                for (int j = 0; j < D; ++j) y[j] += h * bf16(w2[j]);
            }
        }
        const float w = (float)weights[k];
        for (int t = 0; t < threads; ++t) {
            const float* y = part + (size_t)t * D;
            for (int j = 0; j < D; ++j) out[j] += w * y[j];
        }
    }
    free(x);
    free(part);
    free(rows);
    return 0;
}

/* experts[k]: tile-major block of the k-th selected expert; weights[k]: its combine weight. */
int cpu_moe_layer(const void* const* experts, const double* weights, int n_experts, int D, int F, int tiles,
                  const double* x_in, float* out, int threads) {
    if (D <= 0 || F <= 0 || tiles <= 0 || F % tiles || n_experts < 0 || threads <= 0) return 1;
    const int Ft = F / tiles;
    const size_t tile_elems = (size_t)3 * Ft * D;
    float* x = (float*)malloc(sizeof(float) * D);
    float* part = (float*)calloc((size_t)threads * D, sizeof(float));
    if (!x || !part) return 2;
    for (int j = 0; j < D; ++j) x[j] = (float)x_in[j];
    for (int j = 0; j < D; ++j) out[j] = x[j];
    for (int k = 0; k < n_experts; ++k) {
        const uint16_t* base = (const uint16_t*)experts[k];
        memset(part, 0, sizeof(float) * (size_t)threads * D);
#pragma omp parallel num_threads(threads)
        {
            const int t = omp_get_thread_num(), nt = omp_get_num_threads();
            float* y = part + (size_t)t * D;
            const int r0 = (int)((long long)F * t / nt), r1 = (int)((long long)F * (t + 1) / nt);
            for (int r = r0; r < r1; ++r) {
                const uint16_t* tile = base + (size_t)(r / Ft) * tile_elems;
                const uint16_t* w1 = tile + (size_t)(r % Ft) * 2 * D;
                const uint16_t* w3 = w1 + D;
                const uint16_t* w2 = tile + (size_t)2 * Ft * D + (size_t)(r % Ft) * D;
                float a = 0.0f, b = 0.0f;
#pragma omp simd reduction(+ : a, b)
                for (int j = 0; j < D; ++j) {
                    a += bf16(w1[j]) * x[j];
                    b += bf16(w3[j]) * x[j];
                }
                const float h = a / (1.0f + expf(-a)) * b;
#pragma omp simd
                for (int j = 0; j < D; ++j) y[j] += h * bf16(w2[j]);
            }
        }
        const float w = (float)weights[k];
        for (int t = 0; t < threads; ++t) {
            const float* y = part + (size_t)t * D;
            for (int j = 0; j < D; ++j) out[j] += w * y[j];
        }
    }
    free(x);
    free(part);
    return 0;
}
