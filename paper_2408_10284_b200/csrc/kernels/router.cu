// K1 — fused router + reuse-based pre-gate for sm_100a.
//
// Contract: every decision (selected experts, their order, the single-expert flag) is bit-identical
// to the reference's, which computes logits in fp64 in a fixed sequential order
// (GateMatrix::logits, inc/prefetch.hpp:24-35), then softmax (inc/core.hpp:205-216), the
// sensitivity rule (inc/gating.hpp:28-65) and a lowest-index-wins top-k (inc/core.hpp:192-203).
//
// Fast path (fp32 logits, fixed reduction order): one warp per (item, expert column) computes
//   F_j = butterfly(sum over lanes of a lane-sequential fp32 FMA chain of x32_i * w32_ij)
// and, alongside, A_j = same over |x32_i||w32_ij|.  Standard forward-error bounds give
//   |L_ref_j - F_j| <= B_j = ((m+3) u32 + (d+1) u64) * A_j * (1 + 1e-4),   m = chain length,
// so the reference's logit lies in [F_j - B_j, F_j + B_j].  The decision is *certified* when every
// gap it depends on (ranks 1..K+1 strictly separated; the single-expert test's perturbation
// interval entirely on one side of tau, with the reference's own softmax rounding added) is
// decided the same way for every logit vector in that box.  Certified items are final.
// Exact path (uncertified items, kRouteExact, kRouteEmitLogits): the reference's exact fp64
// sequential logits — products x_i * w_ij (each rounded) computed in parallel by the whole CTA
// into shared memory chunk by chunk, one lane per column adding them in index order with
// separately rounded fp64 adds — followed by the reference decision procedure.  Skipping x_i == 0
// (reference) and adding the +-0 product are identical for finite weights.
#include <cuda_runtime.h>

#include <cmath>

#include "router.hpp"

namespace adapmoe {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kChunkRows = 128;
constexpr int kMaxN = 64;

// reference decision on exact scores (or logits -> softmax), shared by the exact path
__device__ void decide_exact(const RouteItem& it, const double* logits, const RouteParams& p, const RouteOutputs& o) {
    const int N = p.n;
    if (it.flags & kRouteEmitLogits) {
        for (int j = 0; j < N; ++j) o.scores[it.out * N + j] = logits[j];
        o.count[it.out] = 0;
        o.single[it.out] = 0;
        return;
    }
    double s[kMaxN];
    if (it.gate == nullptr) {
        for (int j = 0; j < N; ++j) s[j] = it.scores[j];
    } else {
        double l[kMaxN];
        for (int j = 0; j < N; ++j) l[j] = (it.flags & kRouteDivConc) ? __ddiv_rn(logits[j], p.concentration) : logits[j];
        double mx = l[0];
        for (int j = 1; j < N; ++j)
            if (l[j] > mx) mx = l[j];
        double sum = 0.0;
        for (int j = 0; j < N; ++j) {
            s[j] = exp(__dsub_rn(l[j], mx));
            sum = __dadd_rn(sum, s[j]);
        }
        for (int j = 0; j < N; ++j) s[j] = __ddiv_rn(s[j], sum);
    }
    int take = p.k;
    int single = (p.k == 1);
    double pert = 0.0;
    if (it.flags & kRouteAdaptive) {
        double s1 = -1.0, s2 = -1.0;
        for (int j = 0; j < N; ++j) {
            if (s[j] > s1) {
                s2 = s1;
                s1 = s[j];
            } else if (s[j] > s2) {
                s2 = s[j];
            }
        }
        const double alpha = __ddiv_rn(s1, __dadd_rn(s1, s2));
        const double gap = __dsub_rn(1.0, alpha);
        pert = __dmul_rn(__dmul_rn(gap, gap), it.fisher);
        single = pert <= p.tau;
        take = single ? 1 : p.k;
    }
    uint64_t used = 0;
    for (int r = 0; r < p.k; ++r) {
        int pick = -1;
        if (r < take) {
            for (int j = 0; j < N; ++j) {
                if ((used >> j) & 1ull) continue;
                if (pick < 0 || s[j] > s[pick]) pick = j;
            }
            used |= 1ull << pick;
        }
        o.selected[it.out * p.k + r] = pick;
    }
    o.count[it.out] = take;
    o.single[it.out] = single;
    if (o.perturbation) o.perturbation[it.out] = pert;
    if (o.scores && (it.flags & kRouteEmitScores))
        for (int j = 0; j < N; ++j) o.scores[it.out * N + j] = s[j];
}

// Certified decision from fp32 logits F with error radii B.  Returns false if not certified.
__device__ bool decide_certified(const RouteItem& it, const float* F32, const float* A32, int chain_len,
                                 const RouteParams& p, const RouteOutputs& o) {
    const int N = p.n, K = p.k;
    const double e_fast = (chain_len + 3) * 0x1.0p-24;
    const double e_ref = (p.d + 1) * 0x1.0p-53;
    double F[kMaxN], B[kMaxN];
    for (int j = 0; j < N; ++j) {
        F[j] = static_cast<double>(F32[j]);
        B[j] = (e_fast + e_ref) * static_cast<double>(A32[j]) * (1.0 + 1e-4) + 1e-300;
        if (it.flags & kRouteDivConc) {
            F[j] = F[j] / p.concentration;
            B[j] = B[j] / p.concentration + fabs(F[j]) * 0x1.0p-50;
        }
        if (!isfinite(F[j]) || !isfinite(B[j])) return false;
    }
    // rank order of the top min(K+1, N) by F desc (index asc on ties); each consecutive pair must be
    // strictly separated by the radii plus a floor that also covers the reference's exp rounding
    int order[kMaxN];
    uint64_t used = 0;
    const int need = K + 1 < N ? K + 1 : N;
    for (int r = 0; r < need; ++r) {
        int pick = -1;
        for (int j = 0; j < N; ++j) {
            if ((used >> j) & 1ull) continue;
            if (pick < 0 || F[j] > F[pick]) pick = j;
        }
        used |= 1ull << pick;
        order[r] = pick;
    }
    for (int r = 0; r + 1 < need; ++r) {
        const int a = order[r], b = order[r + 1];
        const double floor_gap = 1e-9 * fmax(1.0, fabs(F[a]));
        if (!((F[a] - B[a]) - (F[b] + B[b]) > floor_gap)) return false;
    }
    int take = K;
    int single = (K == 1);
    double pert = 0.0;
    if (it.flags & kRouteAdaptive) {
        // alpha = s1/(s1+s2) = 1/(1+exp(-(L1-L2))) exactly; gap = 1 - alpha = 1/(1+exp(L1-L2))
        const int a = order[0], b = order[1];
        const double d_lo = (F[a] - B[a]) - (F[b] + B[b]);
        const double d_hi = (F[a] + B[a]) - (F[b] - B[b]);
        // reference rounding of alpha is a few ulps of 1: widen gap by 1e-15 absolute; ours 1e-12 rel
        const double g_max = (1.0 / (1.0 + exp(d_lo))) * (1.0 + 1e-12) + 1e-15;
        const double g_min = fmax((1.0 / (1.0 + exp(d_hi))) * (1.0 - 1e-12) - 1e-15, 0.0);
        const double p_max = g_max * g_max * it.fisher * (1.0 + 1e-12);
        const double p_min = g_min * g_min * it.fisher * (1.0 - 1e-12);
        if (it.fisher == 0.0) {
            single = 1;  // reference: gap*gap*0 == 0 <= tau
        } else if (p_max < p.tau) {
            single = 1;
        } else if (p_min > p.tau) {
            single = 0;
        } else {
            return false;
        }
        take = single ? 1 : K;
        const double g = 1.0 / (1.0 + exp(F[a] - F[b]));
        pert = g * g * it.fisher;  // estimate (exact value needs the exact path)
    }
    for (int r = 0; r < K; ++r) o.selected[it.out * K + r] = r < take ? order[r] : -1;
    o.count[it.out] = take;
    o.single[it.out] = single;
    if (o.perturbation) o.perturbation[it.out] = pert;
    return true;
}

__global__ void __launch_bounds__(kThreads) route_kernel(const RouteGroup* __restrict__ groups, RouteParams p, RouteOutputs o) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int D = p.d, N = p.n;
    float* x32 = reinterpret_cast<float*>(smem);                                   // [D]
    double* prod = reinterpret_cast<double*>(smem + ((static_cast<size_t>(D) * 4 + 15) & ~size_t(15)));  // [2][chunk][32]
    __shared__ RouteGroup g;
    __shared__ float F[kMaxRouteItems][kMaxN], A[kMaxRouteItems][kMaxN];
    __shared__ int need_exact[kMaxRouteItems];
    __shared__ double exact_logits[kMaxRouteItems][kMaxN];
    __shared__ int n_exact;
    __shared__ int exact_item[kMaxRouteItems];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) g = groups[blockIdx.x];
    __syncthreads();
    const bool vec4 = (D % 4 == 0);
    const int chain_len = vec4 ? 4 * ((D + 127) / 128) + 5 : (D + 31) / 32 + 5;

    // ---- fast path: fp32 logits, fixed order ----
    bool any_gate = false;
    for (int s = 0; s < g.n_items; ++s) any_gate |= (g.items[s].gate != nullptr && !(g.items[s].flags & (kRouteExact | kRouteEmitLogits)));
    if (any_gate) {
        for (int i = tid; i < D; i += kThreads) x32[i] = static_cast<float>(g.x[i]);
        __syncthreads();
        const int pairs = g.n_items * N;
        for (int pr = warp; pr < pairs; pr += kWarps) {
            const int s = pr / N, j = pr % N;
            const RouteItem& it = g.items[s];
            if (it.gate == nullptr || (it.flags & (kRouteExact | kRouteEmitLogits))) continue;
            const float* w = it.gate32 + static_cast<size_t>(j) * D;
            float acc = 0.0f, asum = 0.0f;
            if (vec4) {
                // batches of 8 independent 16-byte loads per lane; the accumulation order (lane-
                // sequential over i, then the butterfly) is unchanged by the batching
                constexpr int kB = 8;
                for (int i0 = lane * 4; i0 < D; i0 += 128 * kB) {
                    float4 wv[kB];
#pragma unroll
                    for (int b = 0; b < kB; ++b)
                        wv[b] = (i0 + 128 * b < D) ? __ldg(reinterpret_cast<const float4*>(w + i0 + 128 * b))
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int b = 0; b < kB; ++b) {
                        const int i = i0 + 128 * b;
                        if (i >= D) break;
                        const float4 xv = *reinterpret_cast<const float4*>(x32 + i);
                        acc = __fmaf_rn(xv.x, wv[b].x, acc);
                        acc = __fmaf_rn(xv.y, wv[b].y, acc);
                        acc = __fmaf_rn(xv.z, wv[b].z, acc);
                        acc = __fmaf_rn(xv.w, wv[b].w, acc);
                        asum = __fmaf_rn(fabsf(xv.x), fabsf(wv[b].x), asum);
                        asum = __fmaf_rn(fabsf(xv.y), fabsf(wv[b].y), asum);
                        asum = __fmaf_rn(fabsf(xv.z), fabsf(wv[b].z), asum);
                        asum = __fmaf_rn(fabsf(xv.w), fabsf(wv[b].w), asum);
                    }
                }
            } else {
                for (int i = lane; i < D; i += 32) {
                    acc = __fmaf_rn(x32[i], w[i], acc);
                    asum = __fmaf_rn(fabsf(x32[i]), fabsf(w[i]), asum);
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
                asum = __fadd_rn(asum, __shfl_xor_sync(0xffffffffu, asum, off));
            }
            if (lane == 0) {
                F[s][j] = acc;
                A[s][j] = asum;
            }
        }
    }
    __syncthreads();
    // ---- certify (one thread per item) ----
    if (tid < g.n_items) {
        const RouteItem& it = g.items[tid];
        int exact = 0;
        if (it.gate == nullptr) {
            decide_exact(it, nullptr, p, o);  // stored scores: the reference's own inputs
        } else if (it.flags & (kRouteExact | kRouteEmitLogits)) {
            exact = 1;
        } else if (!decide_certified(it, F[tid], A[tid], chain_len, p, o)) {
            exact = 1;
        }
        need_exact[tid] = exact;
        if (o.exact_used) o.exact_used[it.out] = exact;
    }
    __syncthreads();
    if (tid == 0) {
        int ne = 0;
        for (int s = 0; s < g.n_items; ++s)
            if (need_exact[s]) exact_item[ne++] = s;
        n_exact = ne;
    }
    __syncthreads();
    const int NE = n_exact;
    if (NE == 0) return;

    // ---- exact path: reference-order fp64 logits for the items that need them ----
    const int chains = NE * N;  // <= 4 * 64
    const int lanes_per_pass = 32;
    for (int c0 = 0; c0 < chains; c0 += lanes_per_pass) {
        const int cn = min(lanes_per_pass, chains - c0);
        double acc = 0.0;
        for (int r0 = 0; r0 < D; r0 += kChunkRows) {
            const int rows = min(kChunkRows, D - r0);
            double* buf = prod + static_cast<size_t>((r0 / kChunkRows) & 1) * kChunkRows * 32;
            // all threads: products for this chunk (each product rounded to fp64 on its own)
            for (int q = tid; q < rows * cn; q += kThreads) {
                const int r = q / cn, c = c0 + q % cn;
                const RouteItem& it = g.items[exact_item[c / N]];
                buf[r * 32 + (q % cn)] = __dmul_rn(g.x[r0 + r], it.gate[static_cast<size_t>(r0 + r) * N + (c % N)]);
            }
            __syncthreads();
            if (warp == 0 && lane < cn) {
#pragma unroll 8
                for (int r = 0; r < rows; ++r) acc = __dadd_rn(acc, buf[r * 32 + lane]);
            }
            // the double buffer lets the next chunk's products proceed while warp 0 sums; the
            // barrier at the top of the next-but-one chunk protects reuse
        }
        __syncthreads();
        if (warp == 0 && lane < cn) {
            const int c = c0 + lane;
            exact_logits[c / N][c % N] = acc;
        }
        __syncthreads();
    }
    if (tid < NE) {
        const int s = exact_item[tid];
        decide_exact(g.items[s], exact_logits[tid], p, o);
    }
}

__global__ void transpose_kernel(const double* src, float* dst, int d, int n, int count) {
    const size_t total = static_cast<size_t>(count) * d * n;
    for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t m = idx / (static_cast<size_t>(d) * n);
        const size_t rem = idx % (static_cast<size_t>(d) * n);
        const size_t i = rem / n, j = rem % n;
        dst[m * d * n + j * d + i] = static_cast<float>(src[idx]);
    }
}

}  // namespace

cudaError_t launch_route(const RouteGroup* d_groups, int n_groups, int /*max_gate_items*/, const RouteParams& p,
                         const RouteOutputs& out, cudaStream_t stream) {
    if (n_groups <= 0) return cudaSuccess;
    if (p.n < 2 || p.n > kMaxN || p.k < 1 || p.k > p.n || p.d < 1) return cudaErrorInvalidValue;
    const size_t smem = ((static_cast<size_t>(p.d) * 4 + 15) & ~size_t(15)) + 2ull * kChunkRows * 32 * 8;
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    static size_t configured = 0;
    if (smem > configured) {
        cudaFuncSetAttribute(route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(200 * 1024));
        configured = 200 * 1024;
    }
    route_kernel<<<n_groups, kThreads, smem, stream>>>(d_groups, p, out);
    return cudaGetLastError();
}

cudaError_t launch_gate_transpose(const double* src, float* dst, int d, int n, int count, cudaStream_t stream) {
    const size_t total = static_cast<size_t>(count) * d * n;
    const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 16));
    transpose_kernel<<<blocks, 256, 0, stream>>>(src, dst, d, n, count);
    return cudaGetLastError();
}

}  // namespace adapmoe
