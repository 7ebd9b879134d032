// K3 — grouped SwiGLU expert FFN on tcgen05 tensor cores (see grouped_ffn.hpp for the design).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "grouped_ffn.hpp"
#include "ptx.cuh"

namespace adapmoe {

namespace {

constexpr int kBK = 64;                 // K elements per pipeline stage (one 128-byte swizzle row)
constexpr int kABytes = 128 * kBK * 2;  // 16 KB: 128 M rows x 64 K
constexpr int kSmemBudget = 200 * 1024;

// ---- tcgen05 / TMA PTX ------------------------------------------------------------------------
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                       uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(ptx::smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(ptx::smem_addr(bar)), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// UMMA shared-memory descriptor: 128-byte swizzle, version 1 (sm_100), base offset 0 (atoms are
// 1024-byte aligned).  K-major: LBO unused (1), SBO = 1024 B between 8-row groups.  MN-major:
// LBO = byte stride between 64-element MN blocks, SBO = 1024 B between 8-row K groups.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, A K-major (0) or MN-major (1), B K-major.
__device__ __forceinline__ uint32_t instr_desc(int m, int n, bool a_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn_major ? 1u : 0u) << 15) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     ptx::smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint16_t to_bf16(float f) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// ---- unit decoding --------------------------------------------------------------------------
struct Unit {
    int seg, entry;
    int t;          // gate/up: tile
    int m;          // M tile
    int kb0, kb1;   // K blocks [kb0, kb1) (down: relative to the segment's first tile)
};

template <int PHASE>
__device__ __forceinline__ Unit decode_unit(const GroupedLaunch& p, int u) {
    Unit x;
    int s = 0;
    while (s + 1 < p.n_seg && p.unit_prefix[s + 1] <= u) ++s;
    const int r = u - p.unit_prefix[s];
    x.seg = s;
    x.entry = p.seg[s].entry;
    if (PHASE == 0) {
        const int mt = (2 * p.ft) / 128;
        x.t = p.seg[s].t0 + r / mt;
        x.m = r % mt;
        x.kb0 = 0;
        x.kb1 = p.d / kBK;
    } else {
        x.t = 0;
        x.m = r / p.kc;
        const int c = r % p.kc;
        const int kb = (p.seg[s].t1 - p.seg[s].t0) * (p.ft / kBK);
        x.kb0 = kb * c / p.kc;
        x.kb1 = kb * (c + 1) / p.kc;
    }
    return x;
}

// PHASE 0: gate/up + SwiGLU -> H.   PHASE 1: down -> fp32 partials.
template <int PHASE>
__global__ void __launch_bounds__(kGThreads, 1) grouped_kernel(const __grid_constant__ GroupedLaunch p) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem =
        reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    __shared__ __align__(8) uint64_t full[kGMaxStages], empty[kGMaxStages], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base_sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NP = p.np_stride;
    const int b_bytes = NP * 128;
    const int stage_bytes = kABytes + b_bytes;
    const int S = p.stages;
    uint32_t tmem_cols = 32;
    while (tmem_cols < static_cast<uint32_t>(2 * NP)) tmem_cols <<= 1;

    if (warp == 0 && lane == 0) {
        prefetch_map(&p.map_a);
        prefetch_map(&p.map_b);
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 128);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_addr(&tmem_base_sh)),
                     "r"(tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer =====
            const uint64_t pol_w = ptx::policy_evict_first();  // weights: streamed once
            const uint64_t pol_b = policy_evict_last();        // activations: re-read by every unit
            int stage = 0;
            uint32_t phase = 0;
            for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
                const Unit x = decode_unit<PHASE>(p, u);
                const GEntry& e = p.ent[x.entry];
                const int nb = e.np / 16;
                for (int kb = x.kb0; kb < x.kb1; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    unsigned char* sa = smem + static_cast<size_t>(stage) * stage_bytes;
                    unsigned char* sb = sa + kABytes;
                    ptx::mbar_arrive_expect_tx(&full[stage], kABytes + nb * 16 * 128);
                    int kcol;
                    if (PHASE == 0) {
                        const long long row = e.slot_row + static_cast<long long>(x.t) * 3 * p.ft + x.m * 128;
                        kcol = kb * kBK;
                        tma_2d(sa, &p.map_a, kcol, static_cast<int>(row), &full[stage], pol_w);
                    } else {
                        const int f = p.seg[x.seg].t0 * p.ft + kb * kBK;  // global ffn index of the K block
                        const int t = f / p.ft;
                        const long long row = e.slot_row + static_cast<long long>(t) * 3 * p.ft + 2 * p.ft + (f - t * p.ft);
                        tma_2d(sa, &p.map_a, x.m * 128, static_cast<int>(row), &full[stage], pol_w);
                        tma_2d(sa + kABytes / 2, &p.map_a, x.m * 128 + 64, static_cast<int>(row), &full[stage], pol_w);
                        kcol = f;
                    }
                    for (int i = 0; i < nb; ++i)
                        tma_2d(sb + i * 16 * 128, &p.map_b, kcol, x.entry * NP + i * 16, &full[stage], pol_b);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ===== MMA issuer =====
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
                const Unit x = decode_unit<PHASE>(p, u);
                const int np = p.ent[x.entry].np;
                const uint32_t idesc = instr_desc(128, np, PHASE == 1);
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem + static_cast<uint32_t>(acc * NP);
                for (int kb = x.kb0; kb < x.kb1; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_base = ptx::smem_addr(smem + static_cast<size_t>(stage) * stage_bytes);
                    const uint32_t b_base = a_base + kABytes;
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        const uint64_t ad = PHASE == 0 ? smem_desc(a_base + k * 32, 16, 1024)
                                                       : smem_desc(a_base + k * 2048, kABytes / 2, 1024);
                        const uint64_t bd = smem_desc(b_base + k * 32, 16, 1024);
                        mma_bf16(d_tmem, ad, bd, idesc, (kb > x.kb0 || k > 0) ? 1u : 0u);
                    }
                    mma_commit(&empty[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else {
        // ===== epilogue: warps 2..5, TMEM lane quadrant q = warp % 4 =====
        const int q = warp & 3;
        const int row = q * 32 + lane;  // accumulator row (M index within the tile)
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
            const Unit x = decode_unit<PHASE>(p, u);
            const GEntry& e = p.ent[x.entry];
            ptx::mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * NP);
            for (int c0 = 0; c0 < e.np; c0 += 16) {
                float v[16];
                tmem_ld16(taddr + c0, v);
                if (PHASE == 0) {
                    // rows 2r / 2r+1 of the tile hold W1 / W3 of ffn row r: pair lanes exchange; the
                    // even lane finishes columns c0..c0+7, the odd lane c0+8..c0+15
                    float w[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) w[i] = __shfl_xor_sync(0xffffffffu, v[i], 1);
                    const bool odd = lane & 1;
                    const int fr = (x.m * 128 + row) >> 1;
                    const int f = x.t * p.ft + fr;
                    uint16_t* hrow = p.h + static_cast<size_t>(x.entry) * NP * p.f + f;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int col = c0 + (odd ? 8 : 0) + i;
                        const float a = odd ? w[8 + i] : v[i];
                        const float b = odd ? v[8 + i] : w[i];
                        const float h = a / (1.0f + __expf(-a)) * b;
                        if (col < e.n) hrow[static_cast<size_t>(col) * p.f] = to_bf16(h);
                        else if (col < e.np) hrow[static_cast<size_t>(col) * p.f] = 0;
                    }
                } else {
                    float* dst = p.partial + static_cast<size_t>(u) * NP * 128 + row;
#pragma unroll
                    for (int i = 0; i < 16; ++i) dst[static_cast<size_t>(c0 + i) * 128] = v[i];
                }
            }
            tc_fence_before();
            ptx::mbar_arrive(&tempty[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols) : "memory");
    }
}

// ---- gather / combine -----------------------------------------------------------------------
__global__ void gather_kernel(const __grid_constant__ GatherArgs a) {
    const int rows = a.n_entries * a.np_stride;
    for (int r = blockIdx.x; r < rows; r += gridDim.x) {
        const int e = r / a.np_stride, i = r % a.np_stride;
        const int n = a.first[e + 1] - a.first[e];
        uint16_t* dst = a.x + static_cast<size_t>(r) * a.d;
        if (i < n) {
            const double* src = a.acts + static_cast<long long>(a.stream[a.first[e] + i]) * a.stream_stride;
            for (int c = threadIdx.x * 2; c < a.d; c += blockDim.x * 2) {
                const double2 v = *reinterpret_cast<const double2*>(src + c);
                const uint32_t pk = static_cast<uint32_t>(to_bf16(static_cast<float>(v.x))) |
                                    (static_cast<uint32_t>(to_bf16(static_cast<float>(v.y))) << 16);
                *reinterpret_cast<uint32_t*>(dst + c) = pk;
            }
        } else {
            for (int c = threadIdx.x * 2; c < a.d; c += blockDim.x * 2) *reinterpret_cast<uint32_t*>(dst + c) = 0u;
        }
    }
}

// one block per (stream, 128 output columns); thread = column
__global__ void __launch_bounds__(128) gcombine_kernel(const __grid_constant__ GCombineArgs a) {
    const int b = blockIdx.y;
    const int j = blockIdx.x * 128 + threadIdx.x;
    if (j >= a.d) return;
    const int mt = j >> 7, jl = j & 127;
    const double* sc = a.scores + b * a.score_stride;
    int ranks = 0;
    double denom = 0.0;
    for (int r = 0; r < a.top_k; ++r) {
        const int ex = a.pair_expert[b * a.top_k + r];
        if (ex < 0) break;
        denom += sc[ex];
        ++ranks;
    }
    float acc = a.residual ? static_cast<float>(a.acts[b * a.stream_stride + j]) : 0.0f;
    for (int r = 0; r < ranks; ++r) {
        const int pi = b * a.top_k + r;
        const int e = a.pair_entry[pi], col = a.pair_col[pi];
        float y = 0.0f;
        for (int q = a.ref_first[e]; q < a.ref_first[e + 1]; ++q) {
            const GCombineRef& f = a.refs[q];
            const float* base = f.partial + (static_cast<size_t>(f.unit0 + mt * f.kc) * a.np_stride + col) * 128 + jl;
            for (int c = 0; c < f.kc; ++c) y += base[static_cast<size_t>(c) * a.np_stride * 128];
        }
        const float w = ranks == 1 ? 1.0f : static_cast<float>(sc[a.pair_expert[pi]] / denom);
        acc = __fmaf_rn(w, y, acc);
    }
    if (a.n_out_peer > 0) {
        for (int g = 0; g < a.n_out_peer; ++g) a.out_peer[g][b * a.out_stride + j] = acc;  // P2P stores
    } else {
        a.out[b * a.out_stride + j] = acc;
    }
}

int stages_for(int np) {
    const int stage = kABytes + np * 128;
    int s = kSmemBudget / stage;
    return s > kGMaxStages ? kGMaxStages : (s < 2 ? 2 : s);
}

size_t smem_for(const GroupedLaunch& p) {
    return static_cast<size_t>(p.stages) * (kABytes + p.np_stride * 128) + 1024;
}

}  // namespace

cudaError_t make_tensor_map_2d(CUtensorMap* map, const void* base, std::uint64_t rows, std::uint64_t cols,
                               std::uint32_t box_cols, std::uint32_t box_rows) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !f) return e != cudaSuccess ? e : cudaErrorNotSupported;
        fn = reinterpret_cast<Fn>(f);
    }
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t elem[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, elem,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

void grouped_plan_gate_up(GroupedLaunch& p) {
    const int mt = (2 * p.ft) / 128;
    p.unit_prefix[0] = 0;
    for (int s = 0; s < p.n_seg; ++s) p.unit_prefix[s + 1] = p.unit_prefix[s] + (p.seg[s].t1 - p.seg[s].t0) * mt;
    p.units = p.unit_prefix[p.n_seg];
    int np_max = 16;
    for (int s = 0; s < p.n_seg; ++s) np_max = p.ent[p.seg[s].entry].np > np_max ? p.ent[p.seg[s].entry].np : np_max;
    p.stages = stages_for(p.np_stride);
    p.kc = 1;
}

void grouped_plan_down(GroupedLaunch& p, int sm_count) {
    const int mt = p.d / 128;
    // K chunks per (segment, M tile): the smallest kc whose unit count fills the grid's waves to
    // >= 95 % (bounded by the K blocks of the shortest segment)
    int min_kb = 1 << 30, base = 0;
    for (int s = 0; s < p.n_seg; ++s) {
        const int kb = (p.seg[s].t1 - p.seg[s].t0) * (p.ft / kBK);
        min_kb = kb < min_kb ? kb : min_kb;
        base += mt;
    }
    int best = 1;
    double best_eff = 0.0;
    for (int kc = 1; kc <= min_kb && kc <= 16; ++kc) {
        const int units = base * kc;
        const int waves = (units + sm_count - 1) / sm_count;
        const double eff = static_cast<double>(units) / (static_cast<double>(waves) * sm_count);
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = kc;
        }
        if (eff >= 0.95) break;
    }
    p.kc = best;
    p.unit_prefix[0] = 0;
    for (int s = 0; s < p.n_seg; ++s) p.unit_prefix[s + 1] = p.unit_prefix[s] + mt * p.kc;
    p.units = p.unit_prefix[p.n_seg];
    p.stages = stages_for(p.np_stride);
}

int grouped_grid(const GroupedLaunch& p, int sm_count) { return p.units < sm_count ? p.units : sm_count; }

template <int PHASE>
static cudaError_t launch_phase(const GroupedLaunch& p, int sm_count, cudaStream_t stream) {
    if (p.units <= 0) return cudaSuccess;
    if (p.d % 128 || p.ft % kBK || p.np_stride % 16 || p.np_stride > 256 || p.n_seg > kGMaxSegs) return cudaErrorInvalidValue;
    const size_t smem = smem_for(p);
    cudaError_t e = cudaFuncSetAttribute(grouped_kernel<PHASE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    grouped_kernel<PHASE><<<grouped_grid(p, sm_count), kGThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_grouped_gate_up(const GroupedLaunch& p, int sm_count, cudaStream_t stream) {
    return launch_phase<0>(p, sm_count, stream);
}

cudaError_t launch_grouped_down(const GroupedLaunch& p, int sm_count, cudaStream_t stream) {
    return launch_phase<1>(p, sm_count, stream);
}

cudaError_t launch_grouped_gather(const GatherArgs& a, cudaStream_t stream) {
    const int rows = a.n_entries * a.np_stride;
    if (rows <= 0) return cudaSuccess;
    if (a.d % 2) return cudaErrorInvalidValue;
    gather_kernel<<<rows < 1184 ? rows : 1184, 256, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_grouped_combine(const GCombineArgs& a, cudaStream_t stream) {
    if (a.n_streams <= 0) return cudaSuccess;
    dim3 grid((a.d + 127) / 128, a.n_streams);
    gcombine_kernel<<<grid, 128, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace adapmoe
