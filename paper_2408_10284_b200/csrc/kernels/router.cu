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

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "ptx.cuh"
#include "router.hpp"

namespace adapmoe {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kChunkRows = 128;
constexpr int kMaxN = 64;

// ---- warp-cooperative decisions: lane j holds expert columns j and j + 32 (N <= 64) ------------
constexpr unsigned kFull = 0xffffffffu;

// the value of column idx (uniform idx), read from its owner lane
__device__ __forceinline__ double col(double v0, double v1, int idx) {
    return __shfl_sync(kFull, idx < 32 ? v0 : v1, idx & 31);
}

// best column among those not in `used` (64-bit mask, uniform): larger value, then lower index
__device__ __forceinline__ int warp_best(double v0, double v1, int N, uint64_t used, int lane) {
    double v = 0.0;
    int i = -1;
    if (lane < N && !((used >> lane) & 1ull)) {
        v = v0;
        i = lane;
    }
    if (lane + 32 < N && !((used >> (lane + 32)) & 1ull) && (i < 0 || v1 > v)) {
        v = v1;
        i = lane + 32;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(kFull, v, off);
        const int oi = __shfl_xor_sync(kFull, i, off);
        if (oi >= 0 && (i < 0 || ov > v || (ov == v && oi < i))) {
            v = ov;
            i = oi;
        }
    }
    return i;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, off));
    return v;
}

// The reference decision on exact scores (or logits -> softmax, inc/core.hpp:205-216), whole warp.
// softmax: max-subtract, exp, sequential index-order sum (every lane adds the same N terms in
// order), divide; normalized_top1_share's (first, second) pair (inc/gating.hpp:28-42, duplicates of
// the maximum make second == first); sensitivity rule (inc/gating.hpp:46-64); top-k with the
// lowest-index tie rule (inc/core.hpp:192-203).
__device__ void decide_exact(const RouteItem& it, const double* logits, const RouteParams& p, const RouteOutputs& o,
                             int lane) {
    const int N = p.n;
    const bool h0 = lane < N, h1 = lane + 32 < N;
    if (it.flags & kRouteEmitLogits) {
        if (h0) o.scores[it.out * N + lane] = logits[lane];
        if (h1) o.scores[it.out * N + lane + 32] = logits[lane + 32];
        if (lane == 0) {
            o.count[it.out] = 0;
            o.single[it.out] = 0;
        }
        return;
    }
    double s0 = 0.0, s1 = 0.0;
    if (it.gate == nullptr) {
        if (h0) s0 = it.scores[lane];
        if (h1) s1 = it.scores[lane + 32];
    } else {
        double l0 = -INFINITY, l1 = -INFINITY;
        if (h0) l0 = (it.flags & kRouteDivConc) ? __ddiv_rn(logits[lane], p.concentration) : logits[lane];
        if (h1) l1 = (it.flags & kRouteDivConc) ? __ddiv_rn(logits[lane + 32], p.concentration) : logits[lane + 32];
        const double mx = warp_max(fmax(l0, l1));
        const double e0 = h0 ? exp(__dsub_rn(l0, mx)) : 0.0;
        const double e1 = h1 ? exp(__dsub_rn(l1, mx)) : 0.0;
        double sum = 0.0;
        for (int j = 0; j < N; ++j) sum = __dadd_rn(sum, col(e0, e1, j));
        s0 = __ddiv_rn(e0, sum);
        s1 = __ddiv_rn(e1, sum);
    }
    int take = p.k;
    int single = (p.k == 1);
    double pert = 0.0;
    if (it.flags & kRouteAdaptive) {
        const double first = warp_max(fmax(h0 ? s0 : -1.0, h1 ? s1 : -1.0));
        const int n_first = __popc(__ballot_sync(kFull, h0 && s0 == first)) + __popc(__ballot_sync(kFull, h1 && s1 == first));
        const double second = n_first >= 2 ? first
                                            : warp_max(fmax((h0 && s0 < first) ? s0 : -1.0, (h1 && s1 < first) ? s1 : -1.0));
        const double alpha = __ddiv_rn(first, __dadd_rn(first, second));
        const double gap = __dsub_rn(1.0, alpha);
        pert = __dmul_rn(__dmul_rn(gap, gap), it.fisher);
        single = pert <= p.tau;
        take = single ? 1 : p.k;
    }
    uint64_t used = 0;
    for (int r = 0; r < p.k; ++r) {
        int pick = -1;
        if (r < take) {
            pick = warp_best(s0, s1, N, used, lane);
            used |= 1ull << pick;
        }
        if (lane == 0) o.selected[it.out * p.k + r] = pick;
    }
    if (lane == 0) {
        o.count[it.out] = take;
        o.single[it.out] = single;
        if (o.perturbation) o.perturbation[it.out] = pert;
    }
    if (o.scores && (it.flags & kRouteEmitScores)) {
        if (h0) o.scores[it.out * N + lane] = s0;
        if (h1) o.scores[it.out * N + lane + 32] = s1;
    }
}

// Certified decision from fp32 logits F with error radii B, whole warp.  Returns false (uniform) if
// not certified.
__device__ bool decide_certified(const RouteItem& it, const float* F32, const float* A32, int chain_len,
                                 const RouteParams& p, const RouteOutputs& o, int lane) {
    const int N = p.n, K = p.k;
    const double e_fast = (chain_len + 3) * 0x1.0p-24;
    const double e_ref = (p.d + 1) * 0x1.0p-53;
    double F0 = 0.0, B0 = 0.0, F1 = 0.0, B1 = 0.0;
    bool ok = true;
    auto load = [&](int j, double& Fj, double& Bj) {
        Fj = static_cast<double>(F32[j]);
        Bj = (e_fast + e_ref) * static_cast<double>(A32[j]) * (1.0 + 1e-4) + 1e-300;
        if (it.flags & kRouteDivConc) {
            Fj = Fj / p.concentration;
            Bj = Bj / p.concentration + fabs(Fj) * 0x1.0p-50;
        }
        ok &= isfinite(Fj) && isfinite(Bj);
    };
    if (lane < N) load(lane, F0, B0);
    if (lane + 32 < N) load(lane + 32, F1, B1);
    if (!__all_sync(kFull, ok)) return false;
    // rank order of the top min(K+1, N) by F desc (index asc on ties); each consecutive pair must be
    // strictly separated by the radii plus a floor that also covers the reference's exp rounding
    int order[kMaxN + 1];
    uint64_t used = 0;
    const int need = K + 1 < N ? K + 1 : N;
    for (int r = 0; r < need; ++r) {
        order[r] = warp_best(F0, F1, N, used, lane);
        used |= 1ull << order[r];
    }
    for (int r = 0; r + 1 < need; ++r) {
        const int a = order[r], b = order[r + 1];
        const double Fa = col(F0, F1, a), Ba = col(B0, B1, a), Fb = col(F0, F1, b), Bb = col(B0, B1, b);
        const double floor_gap = 1e-9 * fmax(1.0, fabs(Fa));
        if (!((Fa - Ba) - (Fb + Bb) > floor_gap)) return false;
    }
    int take = K;
    int single = (K == 1);
    double pert = 0.0;
    if (it.flags & kRouteAdaptive) {
        // alpha = s1/(s1+s2) = 1/(1+exp(-(L1-L2))) exactly; gap = 1 - alpha = 1/(1+exp(L1-L2))
        const int a = order[0], b = order[1];
        const double Fa = col(F0, F1, a), Ba = col(B0, B1, a), Fb = col(F0, F1, b), Bb = col(B0, B1, b);
        const double d_lo = (Fa - Ba) - (Fb + Bb);
        const double d_hi = (Fa + Ba) - (Fb - Bb);
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
        const double g = 1.0 / (1.0 + exp(Fa - Fb));
        pert = g * g * it.fisher;  // estimate (exact value needs the exact path)
    }
    if (lane == 0) {
        for (int r = 0; r < K; ++r) o.selected[it.out * K + r] = r < take ? order[r] : -1;
        o.count[it.out] = take;
        o.single[it.out] = single;
        if (o.perturbation) o.perturbation[it.out] = pert;
    }
    if (o.scores && (it.flags & kRouteEmitScores)) {
        // softmax of the (concentration-scaled) fp32 logits: combine weights for the free-running
        // decode (the decision above is certified; these values are within ~1e-7 of the reference's)
        const double mx = warp_max(fmax(lane < N ? F0 : -INFINITY, lane + 32 < N ? F1 : -INFINITY));
        const double e0 = lane < N ? exp(F0 - mx) : 0.0, e1 = lane + 32 < N ? exp(F1 - mx) : 0.0;
        double sum = 0.0;
        for (int j = 0; j < N; ++j) sum += col(e0, e1, j);
        if (lane < N) o.scores[it.out * N + lane] = e0 / sum;
        if (lane + 32 < N) o.scores[it.out * N + lane + 32] = e1 / sum;
    }
    return true;
}

// Fast-path dot of one (item, column) over x rows [i_lo, i_hi) (fp32, lane-sequential FMA chains in
// batches of 8 float4 loads, then the xor butterfly): returns the warp's (F, A) in every lane.
__device__ __forceinline__ void fast_dot(const float* __restrict__ w, const float* x32, int i_lo, int i_hi, bool vec4,
                                         int lane, float& acc_out, float& asum_out) {
    float acc = 0.0f, asum = 0.0f;
    if (vec4) {
        constexpr int kB = 8;
        for (int i0 = i_lo + lane * 4; i0 < i_hi; i0 += 128 * kB) {
            float4 wv[kB];
#pragma unroll
            for (int b = 0; b < kB; ++b)
                wv[b] = (i0 + 128 * b < i_hi) ? __ldg(reinterpret_cast<const float4*>(w + i0 + 128 * b))
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int b = 0; b < kB; ++b) {
                const int i = i0 + 128 * b;
                if (i >= i_hi) break;
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
        for (int i = i_lo + lane; i < i_hi; i += 32) {
            acc = __fmaf_rn(x32[i], w[i], acc);
            asum = __fmaf_rn(fabsf(x32[i]), fabsf(w[i]), asum);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
        asum = __fadd_rn(asum, __shfl_xor_sync(0xffffffffu, asum, off));
    }
    acc_out = acc;
    asum_out = asum;
}

__device__ __forceinline__ bool fast_item(const RouteItem& it, const RouteParams& p) {
    return it.gate != nullptr && !(it.flags & (kRouteExact | kRouteEmitLogits)) && !p.force_exact;
}

// Certification + exact fallback for one group, all threads of the CTA (F/A in shared memory).
__device__ void finish_group(const RouteGroup& g, float (*F)[kMaxN], float (*A)[kMaxN], int chain_len,
                             const RouteParams& p, const RouteOutputs& o, double* prod) {
    __shared__ int need_exact[kMaxRouteItems];
    __shared__ double exact_logits[kMaxRouteItems][kMaxN];
    __shared__ int n_exact;
    __shared__ int exact_item[kMaxRouteItems];
    const int D = p.d, N = p.n;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // ---- certify (one warp per item) ----
    if (warp < g.n_items) {
        const RouteItem& it = g.items[warp];
        int exact = 0;
        if (it.gate == nullptr) {
            decide_exact(it, nullptr, p, o, lane);  // stored scores: the reference's own inputs
        } else if ((it.flags & (kRouteExact | kRouteEmitLogits)) || p.force_exact) {
            exact = 1;
        } else if (!decide_certified(it, F[warp], A[warp], chain_len, p, o, lane)) {
            exact = 1;
        }
        if (lane == 0) {
            need_exact[warp] = exact;
            if (o.exact_used) o.exact_used[it.out] = exact;
        }
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
    if (warp < NE) {
        const RouteItem& it = g.items[exact_item[warp]];
        decide_exact(it, exact_logits[warp], p, o, lane);
        // queue the exact logits for the host's libm-exp decision (RouteOutputs::host_entries)
        if (o.host_entries && o.exact_used && !(it.flags & kRouteEmitLogits)) {
            unsigned idx = 0;
            if (lane == 0) idx = atomicAdd(o.host_counter, 1u);
            idx = __shfl_sync(kFull, idx, 0);
            if (idx < static_cast<unsigned>(o.host_cap)) {
                double* e = o.host_entries + static_cast<size_t>(idx) * (2 + N);
                if (lane == 0) {
                    e[0] = static_cast<double>(it.flags);
                    e[1] = it.fisher;
                }
                if (lane < N) e[2 + lane] = exact_logits[warp][lane];
                if (lane + 32 < N) e[2 + lane + 32] = exact_logits[warp][lane + 32];
                if (lane == 0) o.exact_used[it.out] = 2 + static_cast<int>(idx);
            } else if (lane == 0) {
                o.exact_used[it.out] = -1;
            }
        }
    }
}

__device__ __forceinline__ int chain_length(int D) {
    return (D % 4 == 0) ? 4 * ((D + 127) / 128) + 5 : (D + 31) / 32 + 5;
}

__global__ void __launch_bounds__(kThreads) route_kernel(const RouteGroup* __restrict__ groups, RouteParams p, RouteOutputs o) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int D = p.d, N = p.n;
    float* x32 = reinterpret_cast<float*>(smem);                                   // [D]
    double* prod = reinterpret_cast<double*>(smem + ((static_cast<size_t>(D) * 4 + 15) & ~size_t(15)));  // [2][chunk][32]
    __shared__ RouteGroup g;
    __shared__ float F[kMaxRouteItems][kMaxN], A[kMaxRouteItems][kMaxN];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) g = groups[blockIdx.x];
    __syncthreads();
    const bool vec4 = (D % 4 == 0);

    // ---- fast path: fp32 logits, fixed order ----
    bool any_gate = false;
    for (int s = 0; s < g.n_items; ++s) any_gate |= fast_item(g.items[s], p);
    if (any_gate) {
        ptx::load_x_f32<kThreads>(x32, g.x, D);
        __syncthreads();
        const int pairs = g.n_items * N;
        for (int pr = warp; pr < pairs; pr += kWarps) {
            const int s = pr / N, j = pr % N;
            const RouteItem& it = g.items[s];
            if (!fast_item(it, p)) continue;
            float acc, asum;
            fast_dot(it.gate32 + static_cast<size_t>(j) * D, x32, 0, D, vec4, lane, acc, asum);
            if (lane == 0) {
                F[s][j] = acc;
                A[s][j] = asum;
            }
        }
    }
    __syncthreads();
    finish_group(g, F, A, chain_length(D), p, o, prod);
}

// Split variant for the per-layer decode launches (latency-bound: one group per layer at batch 1).
// Group g runs on kSplit CTAs; CTA c computes pairs c*kPairsPerCta .. +kPairsPerCta of the group's
// (item, column) pairs, two warps per pair (halves of d, combined half0 + half1 in that order), and
// publishes F / A to global scratch.  The last CTA to arrive (ticket) loads all F / A and certifies
// the decisions (and runs the rare exact fp64 fallback) exactly like route_kernel.  The fp32 chains
// are shorter than route_kernel's, so its certification radius (chain_length(d)) stays an upper bound.
constexpr int kPairsPerCta = kWarps / 2;

__global__ void __launch_bounds__(kThreads) route_split_kernel(const RouteGroup* __restrict__ groups, RouteParams p,
                                                               RouteOutputs o, RouteScratch sc, int split) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int D = p.d, N = p.n;
    float* x32 = reinterpret_cast<float*>(smem);
    double* prod = reinterpret_cast<double*>(smem + ((static_cast<size_t>(D) * 4 + 15) & ~size_t(15)));
    __shared__ RouteGroup g;
    __shared__ float F[kMaxRouteItems][kMaxN], A[kMaxRouteItems][kMaxN];
    __shared__ float half_f[kWarps], half_a[kWarps];
    __shared__ int last;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gi = blockIdx.x / split, c = blockIdx.x % split;
    if (tid == 0) g = groups[gi];
    __syncthreads();
    const bool vec4 = (D % 4 == 0);
    float* gF = sc.f + static_cast<size_t>(gi) * kMaxRouteItems * kMaxN;  // [item][column]
    float* gA = sc.a + static_cast<size_t>(gi) * kMaxRouteItems * kMaxN;
    __shared__ int fast_list[kMaxRouteItems];
    __shared__ int n_fast;
    if (tid == 0) {
        int nf = 0;
        for (int s = 0; s < g.n_items; ++s)
            if (fast_item(g.items[s], p)) fast_list[nf++] = s;
        n_fast = nf;
    }
    __syncthreads();
    const int pairs = n_fast * N;  // fast (item, column) pairs, item-major
    const int p0 = c * kPairsPerCta;
    if (p0 < pairs) {
        ptx::load_x_f32<kThreads>(x32, g.x, D);
        __syncthreads();
        const int pr = p0 + (warp >> 1), half = warp & 1;
        float acc = 0.0f, asum = 0.0f;
        const int mid = min((D / 2 + 127) / 128 * 128, D);  // half boundary on a warp-batch line
        if (pr < pairs) {
            const RouteItem& it = g.items[fast_list[pr / N]];
            fast_dot(it.gate32 + static_cast<size_t>(pr % N) * D, x32, half ? mid : 0, half ? D : mid, vec4, lane, acc,
                     asum);
        }
        if (lane == 0) {
            half_f[warp] = acc;
            half_a[warp] = asum;
        }
        __syncthreads();
        if (tid < kPairsPerCta && p0 + tid < pairs) {
            const int q = p0 + tid;
            gF[fast_list[q / N] * kMaxN + q % N] = __fadd_rn(half_f[2 * tid], half_f[2 * tid + 1]);
            gA[fast_list[q / N] * kMaxN + q % N] = __fadd_rn(half_a[2 * tid], half_a[2 * tid + 1]);
        }
    }
    // publish, then the last CTA of the group finishes it
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned t = atomicAdd(sc.tickets + gi, 1u);
        last = (t == static_cast<unsigned>(split) - 1);
        if (last) sc.tickets[gi] = 0u;  // re-arm for the next launch (stream-ordered)
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int q = tid; q < pairs; q += kThreads) {
        const int s = fast_list[q / N], j = q % N;
        F[s][j] = *reinterpret_cast<volatile float*>(gF + s * kMaxN + j);
        A[s][j] = *reinterpret_cast<volatile float*>(gA + s * kMaxN + j);
    }
    __syncthreads();
    finish_group(g, F, A, chain_length(D), p, o, prod);
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

cudaError_t launch_route(const RouteGroup* d_groups, int n_groups, int max_gate_items, const RouteParams& p,
                         const RouteOutputs& out, cudaStream_t stream, const RouteScratch* scratch) {
    if (n_groups <= 0) return cudaSuccess;
    if (p.n < 2 || p.n > kMaxN || p.k < 1 || p.k > p.n || p.d < 1) return cudaErrorInvalidValue;
    const size_t smem = ((static_cast<size_t>(p.d) * 4 + 15) & ~size_t(15)) + 2ull * kChunkRows * 32 * 8;
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    // the > 48 KB opt-in is a per-device function attribute: configure each device once
    static std::atomic<std::uint64_t> configured{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return cudaErrorInvalidDevice;
    if (!(configured.load() >> dev & 1)) {
        for (const void* fn : {reinterpret_cast<const void*>(route_kernel), reinterpret_cast<const void*>(route_split_kernel)}) {
            const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            if (e != cudaSuccess) return e;
        }
        configured.fetch_or(std::uint64_t{1} << dev);
    }
    RouteParams pp = p;
    if (const char* f = std::getenv("ADAPMOE_ROUTE_FORCE_EXACT")) pp.force_exact = std::atoi(f) != 0;
    // split when a group's gate columns would take more than one round of the CTA's warps
    const int pairs = (max_gate_items > 0 ? max_gate_items : 1) * p.n;
    const int split = (pairs + kPairsPerCta - 1) / kPairsPerCta;
    if (scratch && scratch->f && scratch->a && scratch->tickets && n_groups <= scratch->groups && split > 1 &&
        p.d >= 1024) {
        route_split_kernel<<<n_groups * split, kThreads, smem, stream>>>(d_groups, pp, out, *scratch, split);
        return cudaGetLastError();
    }
    route_kernel<<<n_groups, kThreads, smem, stream>>>(d_groups, pp, out);
    return cudaGetLastError();
}

cudaError_t launch_gate_transpose(const double* src, float* dst, int d, int n, int count, cudaStream_t stream) {
    const size_t total = static_cast<size_t>(count) * d * n;
    const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 16));
    transpose_kernel<<<blocks, 256, 0, stream>>>(src, dst, d, n, count);
    return cudaGetLastError();
}

}  // namespace adapmoe
