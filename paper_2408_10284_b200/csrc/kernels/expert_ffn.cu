// K2 — batch-1 SwiGLU expert FFN for sm_100a: row-owner HBM streaming.
//
// Decode at batch 1 reads every weight byte exactly once (~1 flop/byte), so the kernel is built
// around HBM bandwidth.  One persistent CTA per SM (512 threads) owns a contiguous range of ffn
// rows of the launch's (expert, tile) segments and walks it in chunks of 16 rows:
//   phase 1: warp w streams the W1 and W3 rows of ffn row r0+w (ld.global.nc.L1::no_allocate,
//            16-byte vectors, 4-deep unrolled), dots them with x (fp32 in shared memory) and
//            forms h = silu(a) * b;
//   phase 2: thread t streams its 16-byte slice of the chunk's 16 W2^T rows (all 16 loads in
//            flight) and accumulates h_r * W2^T_r[8t..8t+8) into 8 fp32 registers.
// Because a CTA consumes the h values it produced, there is no cross-CTA dependency (the earlier
// TMA-ring design needed a grid-wide gate/up -> down handoff and topped out at 4.1 TB/s; this one
// measures 6.3 TB/s on large launches, tools/ffn_microbench.cu v4, profiles/r1_ffn_microbench.txt).
// Optional L2 bulk prefetch (cp.async.bulk.prefetch.L2) of the next chunk or of the whole row range
// exists for experiments; on cold launches both measured slower (tools/k2_cold.cu), so the decode
// leaves it off.  A TMA-ring variant of this row-owner kernel (a producer warp streaming R rows per
// stage into a 2-stage 96 KB ring) measured 4.9 TB/s vs 5.85 TB/s at 16 segments and was dropped
// (profiles/r1_k2_variants.txt).  Each CTA writes one fp32 partial of y per segment it touched; the
// combine kernel reduces them in a fixed order.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cstring>

#include "expert_ffn.hpp"
#include "ptx.cuh"

namespace adapmoe {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = kWarps;  // ffn rows per chunk (one per warp in phase 1)
constexpr int kUnroll = 4;

__device__ __forceinline__ float dot8(int4 w, float4 a, float4 b, float acc) {
    const unsigned x = w.x, y = w.y, z = w.z, q = w.w;
    acc = __fmaf_rn(__uint_as_float(x << 16), a.x, acc);
    acc = __fmaf_rn(__uint_as_float(x & 0xffff0000u), a.y, acc);
    acc = __fmaf_rn(__uint_as_float(y << 16), a.z, acc);
    acc = __fmaf_rn(__uint_as_float(y & 0xffff0000u), a.w, acc);
    acc = __fmaf_rn(__uint_as_float(z << 16), b.x, acc);
    acc = __fmaf_rn(__uint_as_float(z & 0xffff0000u), b.y, acc);
    acc = __fmaf_rn(__uint_as_float(q << 16), b.z, acc);
    acc = __fmaf_rn(__uint_as_float(q & 0xffff0000u), b.w, acc);
    return acc;
}

__device__ __forceinline__ float silu(float a) { return a / (1.0f + expf(-a)); }

#ifndef ADAPMOE_FFN_P2_BATCH
#define ADAPMOE_FFN_P2_BATCH 8
#endif
constexpr int kP2Batch = ADAPMOE_FFN_P2_BATCH;  // W2^T rows loaded per batch in phase 2

template <int DC>
__device__ __forceinline__ void store_partial(float* dst, float (&acc)[DC][8], int tid, int D) {
#pragma unroll
    for (int c = 0; c < DC; ++c) {
        const int col = c * 4096 + tid * 8;
        if (col < D) {
            *reinterpret_cast<float4*>(dst + col) = make_float4(acc[c][0], acc[c][1], acc[c][2], acc[c][3]);
            *reinterpret_cast<float4*>(dst + col + 4) = make_float4(acc[c][4], acc[c][5], acc[c][6], acc[c][7]);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[c][k] = 0.0f;
    }
}

// DC = ceil(d / 4096): output columns per thread = 8 * DC
template <int DC>
__global__ void __launch_bounds__(kThreads, 1) ffn_rows_kernel(const __grid_constant__ FfnLaunch p) {
    extern __shared__ __align__(16) float xs[];  // [d]
    __shared__ float hs[2][kChunk];
    __shared__ float ha[2][kChunk], hb[2][kChunk];  // per-warp half sums when two warps share a row
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = p.d, Ft = p.ft, vpr = D / 8;  // 16-byte vectors per weight row
    ptx::load_x_f32<kThreads>(xs, p.x, D);
    const long long TR = static_cast<long long>(p.n_seg) * Ft;
    const long long r_lo = TR * blockIdx.x / gridDim.x, r_hi = TR * (blockIdx.x + 1) / gridDim.x;
    float acc[DC][8];
#pragma unroll
    for (int c = 0; c < DC; ++c)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[c][k] = 0.0f;
    const int first_seg = static_cast<int>(r_lo / Ft);
    float* const part = p.partial + static_cast<size_t>(blockIdx.x) * kFfnSlotsPerCta * D;
    int cur_seg = first_seg;
    __syncthreads();
    int parity = 0;
    for (long long c0 = r_lo; c0 < r_hi; parity ^= 1) {
        const int s = static_cast<int>(c0 / Ft), r0 = static_cast<int>(c0 % Ft);
        const int n = static_cast<int>(min(static_cast<long long>(min(kChunk, Ft - r0)), r_hi - c0));
        if (s != cur_seg) {
            store_partial<DC>(part + static_cast<size_t>(cur_seg - first_seg) * D, acc, tid, D);
            cur_seg = s;
        }
        // ---- phase 1: h for row r0 + warp (a short chunk spreads each row over wpr = 2/4/8/16
        // warps, equal slices of d summed in part order — every warp keeps loads in flight) ----
#ifndef ADAPMOE_K2_MAXWPR
#define ADAPMOE_K2_MAXWPR 4
#endif
        int wpr = n <= 1 ? 16 : n <= 2 ? 8 : n <= 4 ? 4 : n <= 8 ? 2 : 1;
        if (wpr > ADAPMOE_K2_MAXWPR) wpr = ADAPMOE_K2_MAXWPR;
        const int row = warp / wpr, part = warp % wpr;
        if (row < n) {
            const int4* w1 = reinterpret_cast<const int4*>(p.seg[s].gate_up) + static_cast<size_t>(r0 + row) * 2 * vpr;
            const int4* w3 = w1 + vpr;
            const int j_lo = part * (vpr / wpr), j_hi = part + 1 == wpr ? vpr : (part + 1) * (vpr / wpr);
            float a = 0.0f, b = 0.0f;
            for (int j0 = j_lo + lane; j0 < j_hi; j0 += 32 * kUnroll) {
                int4 q1[kUnroll], q3[kUnroll];
#pragma unroll
                for (int k = 0; k < kUnroll; ++k) {
                    const int j = j0 + 32 * k;
                    if (j < j_hi) {
                        q1[k] = ptx::ld_stream(w1 + j);
                        q3[k] = ptx::ld_stream(w3 + j);
                    }
                }
#pragma unroll
                for (int k = 0; k < kUnroll; ++k) {
                    const int j = j0 + 32 * k;
                    if (j < j_hi) {
                        const float4 xa = *reinterpret_cast<const float4*>(xs + j * 8);
                        const float4 xb = *reinterpret_cast<const float4*>(xs + j * 8 + 4);
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
                if (wpr == 1) {
                    hs[parity][warp] = silu(a) * b;
                } else {
                    ha[parity][warp] = a;
                    hb[parity][warp] = b;
                }
            }
        }
        __syncthreads();  // h of this chunk visible; double-buffered hs makes one barrier enough
        if (wpr > 1 && tid < n) {  // combine the parts (fixed order), one thread per row
            float a = 0.0f, b = 0.0f;
            for (int q = 0; q < wpr; ++q) {
                a += ha[parity][tid * wpr + q];
                b += hb[parity][tid * wpr + q];
            }
            hs[parity][tid] = silu(a) * b;
        }
        if (wpr > 1) __syncthreads();
        // ---- phase 2: acc += h_r * W2^T_r over this thread's columns ----
        const int4* down = reinterpret_cast<const int4*>(p.seg[s].down_t) + static_cast<size_t>(r0) * vpr;
#pragma unroll
        for (int c = 0; c < DC; ++c) {
            const int v = c * 512 + tid;  // 16-byte vector index within a row
            if (v >= vpr) continue;
            for (int k0 = 0; k0 < n; k0 += kP2Batch) {
                int4 q[kP2Batch];
#pragma unroll
                for (int k = 0; k < kP2Batch; ++k)
                    if (k0 + k < n) q[k] = ptx::ld_stream(down + static_cast<size_t>(k0 + k) * vpr + v);
#pragma unroll
                for (int k = 0; k < kP2Batch; ++k)
                    if (k0 + k < n) {
                        const float h = hs[parity][k0 + k];
                        acc[c][0] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q[k].x) << 16), acc[c][0]);
                        acc[c][1] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q[k].x) & 0xffff0000u), acc[c][1]);
                        acc[c][2] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q[k].y) << 16), acc[c][2]);
                        acc[c][3] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q[k].y) & 0xffff0000u), acc[c][3]);
                        acc[c][4] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q[k].z) << 16), acc[c][4]);
                        acc[c][5] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q[k].z) & 0xffff0000u), acc[c][5]);
                        acc[c][6] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q[k].w) << 16), acc[c][6]);
                        acc[c][7] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q[k].w) & 0xffff0000u), acc[c][7]);
                    }
            }
        }
        c0 += n;
    }
    store_partial<DC>(part + static_cast<size_t>(cur_seg - first_seg) * D, acc, tid, D);
}

// ---------------------------------------------------------------------------------------------
// K2 v5 — the same row-owner decomposition, fed by the TMA engine through a deep shared-memory ring.
//
// The LDG kernel above alternates two load phases per 16-row chunk (W1/W3 rows, then W2^T rows)
// with a CTA barrier between them, so its loads drain twice per chunk; on short launches (a
// layer's final 88 MB tile = ~24 rows per CTA) that ramp / drain is ~11 us of fixed cost per
// launch (profiles/r1_ncu_summary.md: 25 us for 88 MB, 44 % DRAM).  Here one producer lane issues
// 1-D bulk copies (cp.async.bulk, evict-first) of the CTA's contiguous rows in exactly the order
// the consumers use them — per chunk the W1/W3 row pairs, then the W2^T rows — into a ring of
// kRingBytes (4-8 stages of ~32 KB, mbarrier full/empty pairs), and never waits on compute except
// for a free stage, so HBM sees 100-200 KB in flight per SM from the first microsecond to the last.
// Consumer thread t owns the 16-byte column vectors v = t + kRingConsumers*k of every row: its
// slice of x lives in registers (fp32), phase 1 accumulates its part of (W1_r.x, W3_r.x) for the
// chunk's rows, a reduce-scatter shuffle + one consumer barrier forms h_r = silu(a)*b, and phase 2
// accumulates h_r * W2^T_r into the same columns of y (registers), as in the LDG kernel.  The
// partial layout [grid][2][d] and the CTA row split are unchanged, so the combine is shared.
#ifndef ADAPMOE_K2_CWARPS  // tuning knobs (tools/k2_ring_bench.cu sweeps them)
#define ADAPMOE_K2_CWARPS 16
#endif
#ifndef ADAPMOE_K2_STAGE_KB
#define ADAPMOE_K2_STAGE_KB 64
#endif
#ifndef ADAPMOE_K2_MAX_STAGES
#define ADAPMOE_K2_MAX_STAGES 8
#endif
#ifndef ADAPMOE_K2_RING_KB
#define ADAPMOE_K2_RING_KB 192
#endif
namespace ring {
constexpr int kConsumerWarps = ADAPMOE_K2_CWARPS;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreads = kConsumers + 32;  // + one producer warp
#ifndef ADAPMOE_K2_ROWS
#define ADAPMOE_K2_ROWS 16
#endif
constexpr int kRows = ADAPMOE_K2_ROWS;     // ffn rows per chunk (16 or 32)
static_assert(kRows == 16 || kRows == 32);
constexpr int kRingBytes = ADAPMOE_K2_RING_KB * 1024;
constexpr int kMaxStages = ADAPMOE_K2_MAX_STAGES;
constexpr int kStageTarget = ADAPMOE_K2_STAGE_KB * 1024;

struct Geometry {
    int g;            // W1/W3 row pairs per phase-1 stage (2g W2^T rows per phase-2 stage)
    int stage_bytes;  // g * 4 * d
    int stages;
};
__host__ __device__ inline Geometry geometry(int d) {
    Geometry q;
    q.g = 4 * d >= kStageTarget ? 1 : kStageTarget / (4 * d);
    if (q.g > kRows / 2) q.g = kRows / 2;
    q.stage_bytes = q.g * 4 * d;
    q.stages = kRingBytes / q.stage_bytes;
    if (q.stages > kMaxStages) q.stages = kMaxStages;
    return q;
}
}  // namespace ring

__device__ __forceinline__ void consumer_sync() {  // named barrier 1: the consumer warps only
    asm volatile("bar.sync 1, %0;" ::"n"(ring::kConsumers) : "memory");
}

#ifdef ADAPMOE_K2_TRACE  // tools/k2_ring_bench.cu: per-CTA globaltimer stamps (start, first stage, end)
__device__ unsigned long long k2_trace[kFfnMaxCtas][4];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// DV = ceil(d / 8 / kConsumers): 16-byte column vectors per consumer thread and row
template <int DV>
__global__ void __launch_bounds__(ring::kThreads, 1) ffn_ring_kernel(const __grid_constant__ FfnLaunch p) {
    using namespace ring;
    extern __shared__ __align__(128) unsigned char ring_buf[];
    __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
    __shared__ float red[kConsumerWarps][2 * kRows];
    __shared__ float hs[kRows];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = p.d, Ft = p.ft, vpr = D / 8;
    const Geometry geo = geometry(D);
    const int G = geo.g, G2 = 2 * geo.g, NS = geo.stages, SB = geo.stage_bytes;
    const long long TR = static_cast<long long>(p.n_seg) * Ft;
    const long long r_lo = TR * blockIdx.x / gridDim.x, r_hi = TR * (blockIdx.x + 1) / gridDim.x;
#ifdef ADAPMOE_K2_TRACE
    if (tid == 0) k2_trace[blockIdx.x][0] = gtime();
#endif
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], kConsumerWarps);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();

    if (warp == kConsumerWarps) {  // ---- producer: one lane streams the CTA's rows ----
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_first();
            int i = 0;
            auto issue = [&](const unsigned char* src, int bytes) {
                const int slot = i % NS;
                if (i >= NS) ptx::mbar_wait(&empty[slot], ((i / NS) - 1) & 1);
                ptx::mbar_arrive_expect_tx(&full[slot], static_cast<uint32_t>(bytes));
                ptx::bulk_g2s_stream(ring_buf + static_cast<size_t>(slot) * SB, src, static_cast<uint32_t>(bytes),
                                     &full[slot], pol);
                ++i;
            };
            for (long long c0 = r_lo; c0 < r_hi;) {
                const int s = static_cast<int>(c0 / Ft), r0 = static_cast<int>(c0 % Ft);
                const int n = static_cast<int>(min(static_cast<long long>(min(kRows, Ft - r0)), r_hi - c0));
                const unsigned char* gu = reinterpret_cast<const unsigned char*>(p.seg[s].gate_up) + static_cast<size_t>(r0) * 4 * D;
                for (int j = 0; j < n; j += G) issue(gu + static_cast<size_t>(j) * 4 * D, min(G, n - j) * 4 * D);
                const unsigned char* dn = reinterpret_cast<const unsigned char*>(p.seg[s].down_t) + static_cast<size_t>(r0) * 2 * D;
                for (int j = 0; j < n; j += G2) issue(dn + static_cast<size_t>(j) * 2 * D, min(G2, n - j) * 2 * D);
                c0 += n;
            }
        }
        return;
    }

    // ---- consumers ----
    float4 xa[DV], xb[DV];  // x[8v .. 8v+8) of this thread's vectors, fp32
#pragma unroll
    for (int k = 0; k < DV; ++k) {
        const int v = tid + kConsumers * k;
        float t[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) t[e] = v < vpr ? static_cast<float>(__ldg(p.x + 8 * v + e)) : 0.0f;
        xa[k] = make_float4(t[0], t[1], t[2], t[3]);
        xb[k] = make_float4(t[4], t[5], t[6], t[7]);
    }
    float acc[DV][8];
#pragma unroll
    for (int k = 0; k < DV; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[k][e] = 0.0f;
    const int first_seg = static_cast<int>(r_lo / Ft);
    int cur_seg = first_seg;
    float* const part = p.partial + static_cast<size_t>(blockIdx.x) * kFfnSlotsPerCta * D;
    auto flush = [&](int seg) {
        float* dst = part + static_cast<size_t>(seg - first_seg) * D;
#pragma unroll
        for (int k = 0; k < DV; ++k) {
            const int v = tid + kConsumers * k;
            if (v < vpr) {
                *reinterpret_cast<float4*>(dst + 8 * v) = make_float4(acc[k][0], acc[k][1], acc[k][2], acc[k][3]);
                *reinterpret_cast<float4*>(dst + 8 * v + 4) = make_float4(acc[k][4], acc[k][5], acc[k][6], acc[k][7]);
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[k][e] = 0.0f;
        }
    };
    int i = 0;  // stage sequence number (mirrors the producer)
    for (long long c0 = r_lo; c0 < r_hi;) {
        const int s = static_cast<int>(c0 / Ft), r0 = static_cast<int>(c0 % Ft);
        const int n = static_cast<int>(min(static_cast<long long>(min(kRows, Ft - r0)), r_hi - c0));
        if (s != cur_seg) {
            flush(cur_seg);
            cur_seg = s;
        }
        // phase 1: this thread's part of a_r = W1_r.x, b_r = W3_r.x for the chunk's rows
        float ab[2 * kRows];
#pragma unroll
        for (int q = 0; q < 2 * kRows; ++q) ab[q] = 0.0f;
        const unsigned char* base = nullptr;
        int slot = 0;
#pragma unroll
        for (int rr = 0; rr < kRows; ++rr) {
            if (rr < n) {
                const int j = rr % G;
                if (j == 0) {
                    slot = i % NS;
                    ptx::mbar_wait(&full[slot], (i / NS) & 1);
                    base = ring_buf + static_cast<size_t>(slot) * SB;
#ifdef ADAPMOE_K2_TRACE
                    if (i == 0 && tid == 0) k2_trace[blockIdx.x][1] = gtime();
#endif
                }
                const int4* w1 = reinterpret_cast<const int4*>(base + static_cast<size_t>(j) * 4 * D);
                const int4* w3 = w1 + vpr;
#pragma unroll
                for (int k = 0; k < DV; ++k) {
                    const int v = tid + kConsumers * k;
                    if (v < vpr) {
                        ab[rr] = dot8(w1[v], xa[k], xb[k], ab[rr]);
                        ab[kRows + rr] = dot8(w3[v], xa[k], xb[k], ab[kRows + rr]);
                    }
                }
                if (j == G - 1 || rr == n - 1) {
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&empty[slot]);
                    ++i;
                }
            }
        }
        // warp reduce-scatter of the 2*kRows values (a then b): lane l ends with the warp sums of
        // values [l*V, l*V + V), V = 2*kRows/32 (each halving step keeps the upper or lower half)
        constexpr int V = 2 * kRows / 32;
#pragma unroll
        for (int o = 16, half = kRows; o >= 1; o >>= 1, half >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int q = 0; q < half; ++q) {
                const float send = up ? ab[q] : ab[q + half];
                const float keep = up ? ab[q + half] : ab[q];
                ab[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
#pragma unroll
        for (int e = 0; e < V; ++e) red[warp][lane * V + e] = ab[e];
        consumer_sync();
        if (tid < n) {  // fixed warp order
            float a = 0.0f, b = 0.0f;
#pragma unroll
            for (int w = 0; w < kConsumerWarps; ++w) {
                a += red[w][tid];
                b += red[w][kRows + tid];
            }
            hs[tid] = silu(a) * b;
        }
        consumer_sync();
        // phase 2: acc += h_r * W2^T_r over this thread's columns
#pragma unroll
        for (int rr = 0; rr < kRows; ++rr) {
            if (rr < n) {
                const int j = rr % G2;
                if (j == 0) {
                    slot = i % NS;
                    ptx::mbar_wait(&full[slot], (i / NS) & 1);
                    base = ring_buf + static_cast<size_t>(slot) * SB;
                }
                const int4* w2 = reinterpret_cast<const int4*>(base + static_cast<size_t>(j) * 2 * D);
                const float h = hs[rr];
#pragma unroll
                for (int k = 0; k < DV; ++k) {
                    const int v = tid + kConsumers * k;
                    if (v < vpr) {
                        const int4 q = w2[v];
                        acc[k][0] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q.x) << 16), acc[k][0]);
                        acc[k][1] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q.x) & 0xffff0000u), acc[k][1]);
                        acc[k][2] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q.y) << 16), acc[k][2]);
                        acc[k][3] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q.y) & 0xffff0000u), acc[k][3]);
                        acc[k][4] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q.z) << 16), acc[k][4]);
                        acc[k][5] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q.z) & 0xffff0000u), acc[k][5]);
                        acc[k][6] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q.w) << 16), acc[k][6]);
                        acc[k][7] = __fmaf_rn(h, __uint_as_float(static_cast<unsigned>(q.w) & 0xffff0000u), acc[k][7]);
                    }
                }
                if (j == G2 - 1 || rr == n - 1) {
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&empty[slot]);
                    ++i;
                }
            }
        }
        c0 += n;
    }
    flush(cur_seg);
#ifdef ADAPMOE_K2_TRACE
    if (tid == 0) k2_trace[blockIdx.x][2] = gtime();
#endif
}

// out[j] = x[j] + sum_rank w_rank * y_rank[j];  y_rank = fixed-order reduction of the K2 partials
// of the rank's (tile) segments.  Block = 32 output columns x 8 partial lanes: lane q of column j
// sums the partials of CTAs c = c_lo + q, c_lo + q + 8, ... of every segment of the rank (coalesced
// 128-byte rows, several loads in flight), then lanes 0..7 are added in order through shared memory.
constexpr int kCombineCols = 32, kCombineLanes = 16;

__global__ void __launch_bounds__(kCombineCols * kCombineLanes) combine_kernel(const __grid_constant__ CombineArgs a) {
    __shared__ float red[kCombineLanes][kCombineCols];
    const int jl = threadIdx.x % kCombineCols, q = threadIdx.x / kCombineCols;
    const int j = blockIdx.x * kCombineCols + jl;
    const bool live = j < a.d;
    double denom = 0.0;
    for (int r = 0; r < a.ranks; ++r) denom += a.scores[a.experts[r]];
    float acc = (live && a.residual) ? static_cast<float>(a.x[j]) : 0.0f;
    if (live && a.accumulate) acc += a.out[j];
    int ref = 0;
    for (int r = 0; r < a.ranks; ++r) {
        float part = 0.0f;
        for (; ref < a.n_refs && a.refs[ref].rank == r; ++ref) {
            const FfnPartialRef& f = a.refs[ref];
            if (!live) continue;
            // lane q sums CTAs c_lo + q, c_lo + q + 16, ... in that order; 8 loads in flight per lane
            float p0 = 0.0f, p1 = 0.0f;
            for (int c = f.c_lo + q; c <= f.c_hi; c += 8 * kCombineLanes) {
                float v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int cc = c + k * kCombineLanes;
                    const int sl = cc == f.c_lo ? f.slot_lo : 0;
                    v[k] = cc <= f.c_hi ? f.partial[(static_cast<size_t>(cc) * kFfnSlotsPerCta + sl) * a.d + j] : 0.0f;
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) p0 += v[k];
            }
            part += p0 + p1;
        }
        red[q][jl] = part;
        __syncthreads();
        if (q == 0 && live) {
            float yr = 0.0f;
#pragma unroll
            for (int k = 0; k < kCombineLanes; ++k) yr += red[k][jl];
            const float w = (a.ranks == 1 ? 1.0f : static_cast<float>(a.scores[a.experts[r]] / denom)) * a.scale;
            acc = __fmaf_rn(w, yr, acc);
        }
        __syncthreads();
    }
    if (q == 0 && live) {
        if (a.n_out_peer > 0) {
            for (int g = 0; g < a.n_out_peer; ++g) a.out_peer[g][j] = acc;  // P2P stores into each shard's slot
        } else {
            a.out[j] = acc;
        }
    }
    if (a.next_res) {
        __shared__ unsigned last;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
        __syncthreads();
        if (!last) return;
        __threadfence();
        extern __shared__ double sq[];  // [d]
        __shared__ double rms_s;
        const int n_threads = kCombineCols * kCombineLanes;
        for (int i = threadIdx.x; i < a.d; i += n_threads) {
            const double v = static_cast<double>(__ldcg(a.out + i));
            a.next_res[i] = v;
            sq[i] = __dmul_rn(v, v);
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // same order as free_running_input_kernel
            double ss = 0.0;
            for (int i = threadIdx.x; i < a.d; i += 32) ss = __dadd_rn(ss, sq[i]);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) ss = __dadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, off));
            if (threadIdx.x == 0) rms_s = __dsqrt_rn(__dadd_rn(__ddiv_rn(ss, static_cast<double>(a.d)), a.eps));
        }
        __syncthreads();
        for (int i = threadIdx.x; i < a.d; i += n_threads)
            a.next_norm[i] = __ddiv_rn(static_cast<double>(__ldcg(a.out + i)), rms_s);
        if (threadIdx.x == 0) *a.ticket = 0;  // re-arm for the next (stream-ordered) launch
    }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ uint16_t init_value(uint64_t base, uint64_t index, float scale) {
    const uint64_t h = splitmix64(base + index);
    const int u = static_cast<int>(h & 0xffff) + static_cast<int>((h >> 16) & 0xffff) + static_cast<int>((h >> 32) & 0xffff) +
                  static_cast<int>((h >> 48) & 0xffff);
    const float v = __fmul_rn(__int2float_rn(u - 131070), scale);
    uint32_t bits = __float_as_uint(v);
    bits += 0x7fffu + ((bits >> 16) & 1u);
    return static_cast<uint16_t>(bits >> 16);
}

struct InitArgs {
    uint64_t base[3];
    float scale[3];
};

// one thread per 8 consecutive elements (rows are multiples of 8 elements)
__global__ void expert_init_kernel(uint16_t* dst, int D, int F, int tiles, InitArgs ia) {
    const int Ft = F / tiles;
    const size_t tile_elems = static_cast<size_t>(3) * Ft * D;
    const size_t total8 = tile_elems * tiles / 8;
    for (size_t g = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; g < total8;
         g += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t pos = g * 8;
        const size_t t = pos / tile_elems;
        const size_t off = pos % tile_elems;
        int m;
        uint64_t idx, stride;
        if (off < static_cast<size_t>(2) * Ft * D) {  // gate_up [Ft][2][D]: W1/W3 row-major
            const size_t rl = off / (2 * static_cast<size_t>(D));
            const size_t rem = off % (2 * static_cast<size_t>(D));
            m = static_cast<int>(rem / D);
            idx = (t * Ft + rl) * D + rem % D;
            stride = 1;
        } else {  // down_t [Ft][D]: element (rl, j) is W2[j][t*Ft + rl], logical index j*F + t*Ft + rl
            const size_t o2 = off - static_cast<size_t>(2) * Ft * D;
            m = 2;
            idx = (o2 % D) * F + t * Ft + o2 / D;
            stride = static_cast<uint64_t>(F);
        }
        uint16_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = init_value(ia.base[m], idx + k * stride, ia.scale[m]);
        uint4 pack;
        pack.x = v[0] | (static_cast<uint32_t>(v[1]) << 16);
        pack.y = v[2] | (static_cast<uint32_t>(v[3]) << 16);
        pack.z = v[4] | (static_cast<uint32_t>(v[5]) << 16);
        pack.w = v[6] | (static_cast<uint32_t>(v[7]) << 16);
        *reinterpret_cast<uint4*>(dst + pos) = pack;
    }
}

// One block per row.  The sum of squares keeps its fixed order — lane j of warp 0 adds x_i^2 for
// i = j, j+32, ... (each product and sum separately rounded), then an xor butterfly over the 32
// lane sums — while the whole block does the elementwise work (fp32 -> fp64 residual, squares into
// shared memory, the final divisions).
constexpr int kNormThreads = 256;

__global__ void __launch_bounds__(kNormThreads) free_running_input_kernel(double* res, double* norm, long long stride,
                                                                          const float* src, long long src_stride, int d,
                                                                          double eps) {
    extern __shared__ double sq[];  // [d]
    __shared__ double rms_s;
    const int r = blockIdx.x;
    double* x = res + r * stride;
    for (int i = threadIdx.x; i < d; i += kNormThreads) {
        const double v = src ? static_cast<double>(src[r * src_stride + i]) : x[i];
        if (src) x[i] = v;
        sq[i] = __dmul_rn(v, v);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double ss = 0.0;
        for (int i = lane; i < d; i += 32) ss = __dadd_rn(ss, sq[i]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) ss = __dadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, off));
        if (lane == 0) rms_s = __dsqrt_rn(__dadd_rn(__ddiv_rn(ss, static_cast<double>(d)), eps));
    }
    __syncthreads();
    const double rms = rms_s;
    double* n = norm + r * stride;
    for (int i = threadIdx.x; i < d; i += kNormThreads) n[i] = __ddiv_rn(x[i], rms);
}

}  // namespace

cudaError_t launch_free_running_input(double* res, double* norm, long long stride, const float* src,
                                      long long src_stride, int rows, int d, double eps, cudaStream_t stream) {
    if (rows <= 0 || d <= 0) return cudaSuccess;
    const size_t smem = static_cast<size_t>(d) * sizeof(double);
    if (smem > 40 * 1024) {  // the opt-in counts static shared memory too
        cudaError_t e = cudaFuncSetAttribute(free_running_input_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    free_running_input_kernel<<<rows, kNormThreads, smem, stream>>>(res, norm, stride, src, src_stride, d, eps);
    return cudaGetLastError();
}

void ffn_partial_range(FfnPartialRef& f, int ft) {
    const long long TR = static_cast<long long>(f.n_seg) * ft;
    const long long s_lo = static_cast<long long>(f.seg) * ft, s_hi = s_lo + ft;
    int c_lo = static_cast<int>(s_lo * f.grid / TR);
    while (c_lo > 0 && TR * c_lo / f.grid > s_lo) --c_lo;
    while (TR * (c_lo + 1) / f.grid <= s_lo) ++c_lo;  // first CTA whose range reaches the segment
    int c_hi = static_cast<int>((s_hi - 1) * f.grid / TR);
    while (c_hi + 1 < f.grid && TR * (c_hi + 1) / f.grid < s_hi) ++c_hi;
    while (c_hi > c_lo && TR * c_hi / f.grid >= s_hi) --c_hi;  // last CTA starting inside it
    f.c_lo = c_lo;
    f.c_hi = c_hi;
    f.slot_lo = f.seg - static_cast<int>(TR * c_lo / f.grid / ft);
}

FfnKernel ffn_kernel_variant() {
    const char* e = std::getenv("ADAPMOE_K2");  // A/B knob (read per launch): "rows" = the LDG kernel
    return (e && std::strcmp(e, "rows") == 0) ? FfnKernel::Rows : FfnKernel::Ring;
}

int ffn_grid(const FfnLaunch& p, int sm_count) {
    const long long rows = static_cast<long long>(p.n_seg) * p.ft;
    long long g = sm_count < kFfnMaxCtas ? sm_count : kFfnMaxCtas;
    if (g > rows) g = rows;
    if (g < p.n_seg) g = p.n_seg;  // keeps every CTA's range within <= 2 segments
    return static_cast<int>(g);
}

cudaError_t launch_ffn(const FfnLaunch& p, int sm_count, cudaStream_t stream) {
    if (p.n_seg <= 0) return cudaSuccess;
    if (p.n_seg > kMaxFfnSegments || p.d % 8 || p.d > 16384 || p.ft < 1 || !p.partial || !p.x)
        return cudaErrorInvalidValue;
    const int grid = ffn_grid(p, sm_count);
    // the > 48 KB opt-in is a per-device function attribute: configure each device once
    static std::atomic<std::uint64_t> configured{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return cudaErrorInvalidDevice;
    if (!(configured.load() >> dev & 1)) {
        for (auto fn : {ffn_rows_kernel<1>, ffn_rows_kernel<2>, ffn_rows_kernel<4>}) {
            const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
            if (e != cudaSuccess) return e;
        }
        for (auto fn : {ffn_ring_kernel<1>, ffn_ring_kernel<2>, ffn_ring_kernel<3>, ffn_ring_kernel<4>,
                        ffn_ring_kernel<6>, ffn_ring_kernel<8>}) {
            const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ring::kRingBytes);
            if (e != cudaSuccess) return e;
        }
        configured.fetch_or(std::uint64_t{1} << dev);
    }
    if (ffn_kernel_variant() == FfnKernel::Ring) {
        const ring::Geometry geo = ring::geometry(p.d);
        const size_t smem = static_cast<size_t>(geo.stages) * geo.stage_bytes;
        const int dv = (p.d / 8 + ring::kConsumers - 1) / ring::kConsumers;
        auto fn = dv <= 1 ? ffn_ring_kernel<1> : dv <= 2 ? ffn_ring_kernel<2> : dv <= 3 ? ffn_ring_kernel<3>
                : dv <= 4 ? ffn_ring_kernel<4> : dv <= 6 ? ffn_ring_kernel<6> : ffn_ring_kernel<8>;
        fn<<<grid, ring::kThreads, smem, stream>>>(p);
        return cudaGetLastError();
    }
    const size_t smem = static_cast<size_t>(p.d) * sizeof(float);
    if (p.d <= 4096)
        ffn_rows_kernel<1><<<grid, kThreads, smem, stream>>>(p);
    else if (p.d <= 8192)
        ffn_rows_kernel<2><<<grid, kThreads, smem, stream>>>(p);
    else
        ffn_rows_kernel<4><<<grid, kThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t stream) {
    if (a.next_res && (!a.next_norm || !a.ticket || a.n_out_peer > 0)) return cudaErrorInvalidValue;
    const size_t smem = a.next_res ? static_cast<size_t>(a.d) * sizeof(double) : 0;
    if (smem > 40 * 1024) {  // the opt-in counts static shared memory too
        cudaError_t e = cudaFuncSetAttribute(combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    combine_kernel<<<(a.d + kCombineCols - 1) / kCombineCols, kCombineCols * kCombineLanes, smem, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_expert_init(uint16_t* dst, int d, int f, int tiles, const uint64_t base[3], const float scale[3],
                               cudaStream_t stream) {
    InitArgs ia;
    for (int m = 0; m < 3; ++m) {
        ia.base[m] = base[m];
        ia.scale[m] = scale[m];
    }
    expert_init_kernel<<<148 * 8, 256, 0, stream>>>(dst, d, f, tiles, ia);
    return cudaGetLastError();
}

}  // namespace adapmoe
