// K2 — batch-1 SwiGLU expert FFN for sm_100a: TMA-staged HBM streaming, gate/up and down fused.
//
// Decode at batch 1 reads every weight byte exactly once (~1 flop/byte), so the kernel is built
// around HBM bandwidth: one persistent CTA per SM.  Warp 0 (one lane) streams contiguous blocks
// of R weight rows into a shared-memory ring with cp.async.bulk (TMA engine; SASS UBLKCP),
// completing on mbarriers, with an L2 evict-first policy since every byte is used once.  Sixteen
// consumer warps turn each staged block into R dot products (R rows x 16/R column parts per row)
// against an fp32 vector in shared memory: bf16 -> fp32 by shift, fp32 FMA, warp-shuffle
// reduction, fixed-order combination of column parts.
//
// Work list of one launch = every phase-A unit (R rows of W1/W3 pairs) of every segment, then
// every phase-B unit (R rows of W2_t); each CTA owns one contiguous range of A units and one of B
// units and runs its A units first.  Every h value is published with its own release-add on the segment's
// counter; a phase-B unit of segment s waits (acquire) until all Ft values of s are published,
// then stages h_s (no fences, no extra CTA barrier).  The producer never waits on that
// dependency — it keeps prefetching W2 rows — so the gate/up -> down transition costs no HBM idle
// time.  Every CTA is co-resident (grid <= #SMs, 1 CTA/SM), so the cross-CTA wait cannot deadlock.
#include <cuda_runtime.h>

#include "expert_ffn.hpp"
#include "ptx.cuh"

namespace adapmoe {

namespace {

#ifndef ADAPMOE_FFN_WARPS
#define ADAPMOE_FFN_WARPS 8
#endif
#ifndef ADAPMOE_FFN_STAGE_KB
#define ADAPMOE_FFN_STAGE_KB 64
#endif
#ifndef ADAPMOE_FFN_BATCH
#define ADAPMOE_FFN_BATCH 4
#endif
#ifndef ADAPMOE_FFN_SPLIT
#define ADAPMOE_FFN_SPLIT 0
#endif
#ifndef ADAPMOE_FFN_L2AHEAD
#define ADAPMOE_FFN_L2AHEAD 0
#endif
constexpr int kL2Ahead = ADAPMOE_FFN_L2AHEAD;
constexpr int kConsumerWarps = ADAPMOE_FFN_WARPS;  // tuning knobs (tools/ffn_microbench.sh)
constexpr int kThreads = 32 * (1 + kConsumerWarps);
constexpr int kMaxStages = 8;
constexpr int kSmemBudget = 226 * 1024;
constexpr int kHeader = 2048;  // barriers + partial dots

struct Geometry {
    int ra, rb;          // rows per stage, phase A (even) / phase B
    int wpr_a, wpr_b;    // consumer warps per row
    int stages;
    size_t stage_bytes;  // ring slot size
    size_t vec_a, vec_b;  // fp32 vector bytes
    size_t smem;
};

__host__ __device__ inline int rows_for(int cols, int min_rows) {
    int r = kConsumerWarps;
    while (r > min_rows && static_cast<size_t>(r) * cols * 2 > ADAPMOE_FFN_STAGE_KB * 1024) r /= 2;
    return r;
}

__host__ __device__ inline Geometry geometry(int d, int ft) {
    Geometry g{};
    g.ra = rows_for(d, 2);
    g.rb = rows_for(ft, 1);
    g.wpr_a = kConsumerWarps / g.ra;
    g.wpr_b = kConsumerWarps / g.rb;
    const size_t a = static_cast<size_t>(g.ra) * d * 2, b = static_cast<size_t>(g.rb) * ft * 2;
    g.stage_bytes = ((a > b ? a : b) + 127) & ~size_t(127);
    g.vec_a = (static_cast<size_t>(d) * 4 + 127) & ~size_t(127);
    g.vec_b = (static_cast<size_t>(ft) * 4 + 127) & ~size_t(127);
    int st = static_cast<int>((kSmemBudget - kHeader - g.vec_a - g.vec_b) / g.stage_bytes);
    g.stages = st > kMaxStages ? kMaxStages : st;
    g.smem = kHeader + g.vec_a + g.vec_b + g.stages * g.stage_bytes;
    return g;
}

__device__ __forceinline__ float silu(float a) { return a / (1.0f + expf(-a)); }

__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps) : "memory"); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// dot of `len` bf16 (starting at row) with fp32 vec; lane handles 4-element groups lane*4 + 128*j,
// so a warp reads 256 contiguous weight bytes and 512 contiguous vector bytes per step
__device__ __forceinline__ float row_dot(const unsigned char* row, const float* vec, int len, int lane) {
    constexpr int kBatch = ADAPMOE_FFN_BATCH;  // weight + vector loads issued before the math
    float acc = 0.0f;
    for (int k0 = lane * 4; k0 < len; k0 += 128 * kBatch) {
        uint2 w[kBatch];
        float4 v[kBatch];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const int k = k0 + 128 * b;
            if (k < len) {
                w[b] = *reinterpret_cast<const uint2*>(row + static_cast<size_t>(k) * 2);
                v[b] = *reinterpret_cast<const float4*>(vec + k);
            } else {
                w[b] = make_uint2(0u, 0u);
                v[b] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            acc = __fmaf_rn(__uint_as_float(w[b].x << 16), v[b].x, acc);
            acc = __fmaf_rn(__uint_as_float(w[b].x & 0xffff0000u), v[b].y, acc);
            acc = __fmaf_rn(__uint_as_float(w[b].y << 16), v[b].z, acc);
            acc = __fmaf_rn(__uint_as_float(w[b].y & 0xffff0000u), v[b].w, acc);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    return acc;
}

struct Unit {
    int phase;  // 0 = A, 1 = B
    int seg;
    int r0;
    int rows;
};

// CTA b owns a contiguous range of phase-A units and a contiguous range of phase-B units (so it
// streams contiguous HBM and stages h for at most a couple of segments); i-th unit of the CTA:
__device__ __forceinline__ int cta_unit(int i, int total_a, int total_b, int b, int G) {
    const int a0 = static_cast<int>((static_cast<long long>(total_a) * b) / G);
    const int a1 = static_cast<int>((static_cast<long long>(total_a) * (b + 1)) / G);
    if (i < a1 - a0) return a0 + i;
    const int b0 = static_cast<int>((static_cast<long long>(total_b) * b) / G);
    const int b1 = static_cast<int>((static_cast<long long>(total_b) * (b + 1)) / G);
    const int j = i - (a1 - a0);
    return j < b1 - b0 ? total_a + b0 + j : -1;
}

__device__ __forceinline__ Unit unit_at(int u, const FfnLaunch& p, const Geometry& g, int units_a_per_seg,
                                        int units_b_per_seg) {
    Unit x;
    const int total_a = units_a_per_seg * p.n_seg;
    if (u < total_a) {
        x.phase = 0;
        x.seg = u / units_a_per_seg;
        x.r0 = (u % units_a_per_seg) * g.ra;
        x.rows = min(g.ra, 2 * p.ft - x.r0);
    } else {
        const int v = u - total_a;
        x.phase = 1;
        x.seg = v / units_b_per_seg;
        x.r0 = (v % units_b_per_seg) * g.rb;
        x.rows = min(g.rb, p.d - x.r0);
    }
    return x;
}

__global__ void __launch_bounds__(kThreads, 1) ffn_kernel(const __grid_constant__ FfnLaunch p) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const Geometry geo = geometry(p.d, p.ft);
    const int NS = geo.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kMaxStages;
    float* partial = reinterpret_cast<float*>(smem + 128);  // [kMaxStages][kConsumerWarps]
    float* vec_a = reinterpret_cast<float*>(smem + kHeader);
    float* vec_b = reinterpret_cast<float*>(smem + kHeader + geo.vec_a);
    unsigned char* ring = smem + kHeader + geo.vec_a + geo.vec_b;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ua = (2 * p.ft + geo.ra - 1) / geo.ra;  // phase-A units per segment
    const int ub = (p.d + geo.rb - 1) / geo.rb;       // phase-B units per segment
    const int total_a = ua * p.n_seg, total_b = ub * p.n_seg;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], kConsumerWarps);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t policy = ptx::policy_evict_first();
            // L2 prefetch runs kL2Ahead units ahead of the smem ring: more bytes in flight per SM
            // than shared memory can hold, so the ring's bulk copies hit L2 instead of HBM
            auto prefetch = [&](int j) {
                const int v = cta_unit(j, total_a, total_b, blockIdx.x, gridDim.x);
                if (v < 0) return;
                const Unit y = unit_at(v, p, geo, ua, ub);
                const int c = y.phase == 0 ? p.d : p.ft;
                const std::uint16_t* b = y.phase == 0 ? p.seg[y.seg].gate_up : p.seg[y.seg].down;
                ptx::bulk_prefetch_l2(b + static_cast<size_t>(y.r0) * c, static_cast<uint32_t>(y.rows) * c * 2u);
            };
            for (int j = NS; j < NS + kL2Ahead; ++j) prefetch(j);
            for (int i = 0;; ++i) {
                const int u = cta_unit(i, total_a, total_b, blockIdx.x, gridDim.x);
                if (u < 0) break;
                const Unit x = unit_at(u, p, geo, ua, ub);
                const int st = i % NS;
                if (kL2Ahead > 0) prefetch(i + NS + kL2Ahead);
                if (i >= NS) ptx::mbar_wait(&empty[st], ((i / NS) - 1) & 1);
                const int cols = x.phase == 0 ? p.d : p.ft;
                const std::uint16_t* base = x.phase == 0 ? p.seg[x.seg].gate_up : p.seg[x.seg].down;
                const uint32_t bytes = static_cast<uint32_t>(x.rows) * cols * 2u;
                ptx::mbar_arrive_expect_tx(&full[st], bytes);
#if ADAPMOE_FFN_SPLIT
                // one bulk copy per row: more copies in flight per SM than one big copy
                for (int r = 0; r < x.rows; ++r)
                    ptx::bulk_g2s_stream(ring + st * geo.stage_bytes + static_cast<size_t>(r) * cols * 2,
                                         base + static_cast<size_t>(x.r0 + r) * cols, cols * 2u, &full[st], policy);
#else
                ptx::bulk_g2s_stream(ring + st * geo.stage_bytes, base + static_cast<size_t>(x.r0) * cols, bytes,
                                     &full[st], policy);
#endif
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    const int cw = warp - 1;  // 0..15
    const int ctid = threadIdx.x - 32;
    for (int i = ctid; i < p.d; i += 32 * kConsumerWarps) vec_a[i] = static_cast<float>(p.x[i]);
    consumer_bar();
    int vec_seg = -1;
    for (int i = 0;; ++i) {
        const int u = cta_unit(i, total_a, total_b, blockIdx.x, gridDim.x);
        if (u < 0) break;
        const Unit x = unit_at(u, p, geo, ua, ub);
        const int R = x.phase == 0 ? geo.ra : geo.rb;
        const int WPR = x.phase == 0 ? geo.wpr_a : geo.wpr_b;
        const int C = x.phase == 0 ? p.d : p.ft;
        if (x.phase == 1 && vec_seg != x.seg) {
            // wait until every phase-A unit of this segment has published its h values
            if (ctid == 0) {
                const unsigned* cnt = p.counters + x.seg;
                while (ld_acquire(cnt) < static_cast<unsigned>(p.ft)) __nanosleep(32);
            }
            consumer_bar();
            const float* h = p.seg[x.seg].h;
            for (int k = ctid; k < p.ft; k += 32 * kConsumerWarps) vec_b[k] = __ldcg(h + k);
            vec_seg = x.seg;
            consumer_bar();
        }
        const int st = i % NS;
        const int row = cw / WPR, part = cw % WPR;
        const int part_len = C / WPR;
        ptx::mbar_wait(&full[st], (i / NS) & 1);
        float dot = 0.0f;
        if (row < x.rows) {
            const unsigned char* rp = ring + st * geo.stage_bytes + (static_cast<size_t>(row) * C + part * part_len) * 2;
            dot = row_dot(rp, (x.phase == 0 ? vec_a : vec_b) + part * part_len, part_len, lane);
        }
        if (lane == 0) {
            partial[st * kConsumerWarps + cw] = dot;
            ptx::mbar_arrive(&empty[st]);
        }
        consumer_bar();
        if (part == 0 && lane == 0 && row < x.rows) {
            float v = 0.0f;
            for (int q = 0; q < WPR; ++q) v += partial[st * kConsumerWarps + row * WPR + q];
            if (x.phase == 0) {
                if ((row & 1) == 0) {
                    float b = 0.0f;
                    for (int q = 0; q < WPR; ++q) b += partial[st * kConsumerWarps + (row + 1) * WPR + q];
                    p.seg[x.seg].h[(x.r0 + row) >> 1] = silu(v) * b;
                    red_release_add(p.counters + x.seg, 1u);  // publishes this h value (release)
                }
            } else {
                p.seg[x.seg].y[x.r0 + row] = v;
            }
        }
        (void)R;
    }
}

__global__ void combine_kernel(CombineArgs a) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= a.d) return;
    double denom = 0.0;
    for (int r = 0; r < a.ranks; ++r) denom += a.scores[a.experts[r]];
    float acc = static_cast<float>(a.x[j]);
    for (int r = 0; r < a.ranks; ++r) {
        const float w = a.ranks == 1 ? 1.0f : static_cast<float>(a.scores[a.experts[r]] / denom);
        float yr = 0.0f;
        for (int t = 0; t < a.tiles; ++t) yr += a.y[(static_cast<size_t>(r) * a.tiles + t) * a.d + j];
        acc = __fmaf_rn(w, yr, acc);
    }
    a.out[j] = acc;
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
        uint64_t idx;
        if (off < static_cast<size_t>(2) * Ft * D) {
            const size_t rl = off / (2 * static_cast<size_t>(D));
            const size_t rem = off % (2 * static_cast<size_t>(D));
            m = static_cast<int>(rem / D);
            idx = (t * Ft + rl) * D + rem % D;
        } else {
            const size_t o2 = off - static_cast<size_t>(2) * Ft * D;
            m = 2;
            idx = (o2 / Ft) * F + t * Ft + o2 % Ft;
        }
        uint16_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = init_value(ia.base[m], idx + k, ia.scale[m]);
        uint4 pack;
        pack.x = v[0] | (static_cast<uint32_t>(v[1]) << 16);
        pack.y = v[2] | (static_cast<uint32_t>(v[3]) << 16);
        pack.z = v[4] | (static_cast<uint32_t>(v[5]) << 16);
        pack.w = v[6] | (static_cast<uint32_t>(v[7]) << 16);
        *reinterpret_cast<uint4*>(dst + pos) = pack;
    }
}

}  // namespace

cudaError_t launch_ffn(const FfnLaunch& p, int sm_count, cudaStream_t stream) {
    if (p.n_seg <= 0) return cudaSuccess;
    if (p.n_seg > kMaxFfnSegments || p.d % 64 || p.ft % 32 || p.d > 16384 || p.ft > 16384 || !p.counters)
        return cudaErrorInvalidValue;
    const Geometry g = geometry(p.d, p.ft);
    if (g.stages < 2 || (p.d / g.wpr_a) % 4 || (p.ft / g.wpr_b) % 4) return cudaErrorInvalidValue;
    const long long units = static_cast<long long>(p.n_seg) * ((2 * p.ft + g.ra - 1) / g.ra + (p.d + g.rb - 1) / g.rb);
    const int grid = static_cast<int>(units < sm_count ? units : sm_count);
    static bool set = false;
    if (!set) {
        cudaFuncSetAttribute(ffn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
        set = true;
    }
    ffn_kernel<<<grid, kThreads, g.smem, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t stream) {
    combine_kernel<<<(a.d + 255) / 256, 256, 0, stream>>>(a);
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
