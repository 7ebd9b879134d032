// K2 — batch-1 SwiGLU expert FFN for sm_100a: TMA-staged HBM streaming.
//
// Decode at batch 1 reads every weight byte exactly once (~1 flop/byte), so the kernel is built
// around HBM bandwidth, not math: one persistent CTA per SM; warp 0 (one elected lane) streams
// contiguous blocks of R weight rows into a 2-4 stage shared-memory ring with cp.async.bulk (the
// TMA engine; SASS UBLKCP) completing on mbarriers, with an L2 evict-first policy because every
// byte is used once; warps 1..8 turn each staged block into R dot products against a vector held
// in shared memory as fp32 (bf16 -> fp32 by shift, fp32 FMA, warp-shuffle reduction), and release
// the slot.  Row blocks are contiguous in HBM (expert_ffn.hpp layout), so every bulk copy is a
// single 2*R*cols-byte transfer.  Pass A fuses the SwiGLU gate: the W1 and W3 rows of an ffn
// index sit next to each other, so silu(a)*b is formed in the same stage that produced a and b.
#include <cuda_runtime.h>

#include "expert_ffn.hpp"
#include "ptx.cuh"

namespace adapmoe {

namespace {

constexpr int kConsumerWarps = 8;
constexpr int kThreads = 32 * (1 + kConsumerWarps);
constexpr int kMaxStages = 4;
constexpr int kSmemBudget = 227 * 1024 - 1024;  // leave room for static shared memory

struct PassGeometry {
    int rows_per_stage;  // R (8, 4 or 2)
    int warps_per_row;   // 8 / R
    int stages;
    size_t vec_bytes;
    size_t stage_bytes;
    size_t smem;
};

__host__ __device__ inline PassGeometry geometry(int cols) {
    PassGeometry g{};
    g.rows_per_stage = 8;
    while (g.rows_per_stage > 2 && static_cast<size_t>(g.rows_per_stage) * cols * 2 > 64 * 1024) g.rows_per_stage /= 2;
    g.warps_per_row = kConsumerWarps / g.rows_per_stage;
    g.vec_bytes = (static_cast<size_t>(cols) * 4 + 127) & ~size_t(127);
    g.stage_bytes = (static_cast<size_t>(g.rows_per_stage) * cols * 2 + 127) & ~size_t(127);
    const size_t header = 1024;  // barriers + partial dots
    int st = static_cast<int>((kSmemBudget - header - g.vec_bytes) / g.stage_bytes);
    g.stages = st > kMaxStages ? kMaxStages : st;
    g.smem = header + g.vec_bytes + g.stages * g.stage_bytes;
    return g;
}

__device__ __forceinline__ float silu(float a) { return a / (1.0f + expf(-a)); }

__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps) : "memory"); }

__device__ __forceinline__ float dot_bf16x8(uint4 w, const float* v) {
    const float4 a = *reinterpret_cast<const float4*>(v);
    const float4 b = *reinterpret_cast<const float4*>(v + 4);
    float s = 0.0f;
    s = __fmaf_rn(__uint_as_float(w.x << 16), a.x, s);
    s = __fmaf_rn(__uint_as_float(w.x & 0xffff0000u), a.y, s);
    s = __fmaf_rn(__uint_as_float(w.y << 16), a.z, s);
    s = __fmaf_rn(__uint_as_float(w.y & 0xffff0000u), a.w, s);
    s = __fmaf_rn(__uint_as_float(w.z << 16), b.x, s);
    s = __fmaf_rn(__uint_as_float(w.z & 0xffff0000u), b.y, s);
    s = __fmaf_rn(__uint_as_float(w.w << 16), b.z, s);
    s = __fmaf_rn(__uint_as_float(w.w & 0xffff0000u), b.w, s);
    return s;
}

template <bool kSwiglu>
__global__ void __launch_bounds__(kThreads, 1) ffn_pass_kernel(const __grid_constant__ FfnLaunch p) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const PassGeometry geo = geometry(p.cols);
    const int R = geo.rows_per_stage, WPR = geo.warps_per_row, NS = geo.stages, C = p.cols;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kMaxStages;
    float* partial = reinterpret_cast<float*>(smem + 128);  // [kMaxStages][8]
    float* vec = reinterpret_cast<float*>(smem + 1024);
    unsigned char* ring = smem + 1024 + geo.vec_bytes;

    // unit = R consecutive rows of one segment
    __shared__ int seg_units[kMaxFfnSegments + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        seg_units[0] = 0;
        for (int s = 0; s < p.n_seg; ++s) seg_units[s + 1] = seg_units[s] + (p.seg[s].rows_count + R - 1) / R;
        for (int s = 0; s < NS; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], kConsumerWarps);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const int total = seg_units[p.n_seg];
    const int u_begin = static_cast<int>((static_cast<long long>(total) * blockIdx.x) / gridDim.x);
    const int u_end = static_cast<int>((static_cast<long long>(total) * (blockIdx.x + 1)) / gridDim.x);

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t policy = ptx::policy_evict_first();
            int s = 0;
            while (s + 1 < p.n_seg && seg_units[s + 1] <= u_begin) ++s;
            for (int u = u_begin, i = 0; u < u_end; ++u, ++i) {
                while (seg_units[s + 1] <= u) ++s;
                const int local = u - seg_units[s];
                const int r0 = local * R;
                const int rows = min(R, p.seg[s].rows_count - r0);
                const int st = i % NS;
                if (i >= NS) ptx::mbar_wait(&empty[st], ((i / NS) - 1) & 1);
                const uint32_t bytes = static_cast<uint32_t>(rows) * C * 2u;
                ptx::mbar_arrive_expect_tx(&full[st], bytes);
                ptx::bulk_g2s_stream(ring + st * geo.stage_bytes, p.seg[s].rows + static_cast<size_t>(r0) * C, bytes,
                                     &full[st], policy);
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    const int cw = warp - 1;                 // 0..7
    const int row_in_stage = cw / WPR;
    const int part = cw % WPR;
    const int part_len = C / WPR;
    const int col0 = part * part_len;
    const int ctid = threadIdx.x - 32;
    if (kSwiglu) {
        for (int i = ctid; i < C; i += 32 * kConsumerWarps) vec[i] = static_cast<float>(p.x[i]);
    }
    int s = 0;
    while (s + 1 < p.n_seg && seg_units[s + 1] <= u_begin) ++s;
    int vec_seg = -1;
    for (int u = u_begin, i = 0; u < u_end; ++u, ++i) {
        while (seg_units[s + 1] <= u) ++s;
        if (!kSwiglu && vec_seg != s) {
            consumer_bar();  // everyone is done with the previous vector
            for (int k = ctid; k < C; k += 32 * kConsumerWarps) vec[k] = p.seg[s].vec[k];
            vec_seg = s;
            consumer_bar();  // new vector visible
        }
        if (kSwiglu && i == 0) consumer_bar();  // x staged
        const int local = u - seg_units[s];
        const int r0 = local * R;
        const int rows = min(R, p.seg[s].rows_count - r0);
        const int st = i % NS;
        ptx::mbar_wait(&full[st], (i / NS) & 1);
        float acc = 0.0f;
        if (row_in_stage < rows) {
            const unsigned char* row = ring + st * geo.stage_bytes + static_cast<size_t>(row_in_stage) * C * 2;
#pragma unroll 4
            for (int k = col0 + lane * 8; k < col0 + part_len; k += 256) {
                const uint4 w = *reinterpret_cast<const uint4*>(row + static_cast<size_t>(k) * 2);
                acc += dot_bf16x8(w, vec + k);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        __syncwarp();
        if (lane == 0) {
            partial[st * 8 + cw] = acc;
            ptx::mbar_arrive(&empty[st]);
        }
        consumer_bar();
        // one lane per row (pair) finalizes, summing column parts in fixed order
        if (part == 0 && lane == 0 && row_in_stage < rows) {
            float dot = 0.0f;
            for (int q = 0; q < WPR; ++q) dot += partial[st * 8 + row_in_stage * WPR + q];
            if (kSwiglu) {
                if ((row_in_stage & 1) == 0) {
                    float b = 0.0f;
                    for (int q = 0; q < WPR; ++q) b += partial[st * 8 + (row_in_stage + 1) * WPR + q];
                    p.seg[s].out[(r0 + row_in_stage) >> 1] = silu(dot) * b;
                }
            } else {
                p.seg[s].out[r0 + row_in_stage] = dot;
            }
        }
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

cudaError_t launch_ffn_pass(const FfnLaunch& p, int sm_count, cudaStream_t stream) {
    if (p.n_seg <= 0) return cudaSuccess;
    if (p.n_seg > kMaxFfnSegments || p.cols % 8 != 0 || p.cols > 16384) return cudaErrorInvalidValue;
    const PassGeometry g = geometry(p.cols);
    if (g.stages < 2 || (p.cols / g.warps_per_row) % 8 != 0) return cudaErrorInvalidValue;
    long long units = 0;
    for (int s = 0; s < p.n_seg; ++s) units += (p.seg[s].rows_count + g.rows_per_stage - 1) / g.rows_per_stage;
    const int grid = static_cast<int>(units < sm_count ? units : sm_count);
    if (p.swiglu) {
        static bool set = false;
        if (!set) {
            cudaFuncSetAttribute(ffn_pass_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);  // NOLINT
            set = true;
        }
        ffn_pass_kernel<true><<<grid, kThreads, g.smem, stream>>>(p);
    } else {
        static bool set = false;
        if (!set) {
            cudaFuncSetAttribute(ffn_pass_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);  // NOLINT
            set = true;
        }
        ffn_pass_kernel<false><<<grid, kThreads, g.smem, stream>>>(p);
    }
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
