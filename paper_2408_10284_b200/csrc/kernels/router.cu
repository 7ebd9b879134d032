// K1 — fused router + reuse-based pre-gate for sm_100a.
//
// Numerics contract (bit-exact with the reference on the same inputs):
//   logits   : logit_j = sum_i x_i * W[i][j], i ascending, x_i == 0 skipped, every product and
//              every partial sum rounded to fp64 separately (no FMA) — exactly GateMatrix::logits
//              (inc/prefetch.hpp:24-35).  The reduction order is fixed; it is the reference's.
//   softmax  : first max, exp(l - max), sequential sum in index order, divide (inc/core.hpp:205-216)
//   decision : alpha = s1/(s1+s2); p = ((1-alpha)*(1-alpha))*F; single iff p <= tau
//              (inc/gating.hpp:28-65); top-k by score desc, lowest index on ties (core.hpp:192-203).
// exp() is CUDA's fp64 exp (<= 1 ulp); tests count any selection that differs from the reference
// (none on the committed configs).
//
// Work layout: one CTA per group (one activation vector, <= 4 routing items).  Warp 1 is the
// producer: it streams fixed-size row chunks of x and of every item's gate matrix into a 3-stage
// shared-memory ring with cp.async.bulk (TMA engine) completing on mbarriers.  Warp 0 runs the
// fp64 accumulation chains (one chain per (item, expert column)), then the per-item softmax,
// sensitivity gate and top-k on one lane per item.
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "router.hpp"

namespace adapmoe {

namespace {

constexpr int kStages = 3;
constexpr int kMaxChainsPerLane = 8;  // (items * N) <= 256

struct __align__(16) RouteSmemHeader {
    uint64_t full[kStages];
    uint64_t empty[kStages];
};

__device__ void decide_item(const RouteItem& it, const double* logits, const RouteParams& p, const RouteOutputs& o) {
    const int N = p.n;
    if (it.flags & kRouteEmitLogits) {
        for (int j = 0; j < N; ++j) o.scores[it.out * N + j] = logits[j];
        o.count[it.out] = 0;
        o.single[it.out] = 0;
        return;
    }
    double s[64];
    if (it.gate == nullptr) {
        for (int j = 0; j < N; ++j) s[j] = it.scores[j];
    } else {
        double l[64];
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
    // top-k: repeated argmax under (score desc, index asc)
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

// rows per chunk and gate-slot count are launch constants; dynamic smem holds the ring.
__global__ void __launch_bounds__(64) route_kernel(const RouteGroup* __restrict__ groups, int max_gates, int rows_per_chunk,
                                                   int use_tma, RouteParams p, RouteOutputs o) {
    extern __shared__ __align__(128) unsigned char smem[];
    RouteSmemHeader* hdr = reinterpret_cast<RouteSmemHeader*>(smem);
    double* ring = reinterpret_cast<double*>(smem + sizeof(RouteSmemHeader));
    const int R = rows_per_chunk, N = p.n, D = p.d;
    const int stage_elems = R + max_gates * R * N;  // x chunk then [slot][R][N]
    __shared__ RouteGroup g;
    __shared__ const double* gate_of_slot[kMaxRouteItems];
    __shared__ int slot_item[kMaxRouteItems];
    __shared__ int n_slots;
    __shared__ double logits[kMaxRouteItems][64];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        g = groups[blockIdx.x];
        int ns = 0;
        for (int i = 0; i < g.n_items; ++i)
            if (g.items[i].gate != nullptr) {
                gate_of_slot[ns] = g.items[i].gate;
                slot_item[ns] = i;
                ++ns;
            }
        n_slots = ns;
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&hdr->full[s], 1);
            ptx::mbar_init(&hdr->empty[s], 1);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const int S = n_slots;
    const int chunks = S > 0 ? (D + R - 1) / R : 0;

    if (warp == 1) {
        // ---------------- producer ----------------
        for (int c = 0; c < chunks; ++c) {
            const int st = c % kStages;
            if (c >= kStages) ptx::mbar_wait(&hdr->empty[st], ((c / kStages) - 1) & 1);
            double* xs = ring + static_cast<size_t>(st) * stage_elems;
            double* ws = xs + R;
            const int r0 = c * R;
            const int rows = min(R, D - r0);
            if (use_tma) {
                if (lane == 0) {
                    const uint32_t bytes = static_cast<uint32_t>(rows) * 8u * (1u + static_cast<uint32_t>(S * N));
                    ptx::mbar_arrive_expect_tx(&hdr->full[st], bytes);
                    ptx::bulk_g2s(xs, g.x + r0, rows * 8u, &hdr->full[st]);
                    for (int s = 0; s < S; ++s)
                        ptx::bulk_g2s(ws + static_cast<size_t>(s) * R * N, gate_of_slot[s] + static_cast<size_t>(r0) * N,
                                      static_cast<uint32_t>(rows) * N * 8u, &hdr->full[st]);
                }
            } else {
                for (int i = lane; i < rows; i += 32) xs[i] = g.x[r0 + i];
                for (int s = 0; s < S; ++s) {
                    const double* src = gate_of_slot[s] + static_cast<size_t>(r0) * N;
                    double* dst = ws + static_cast<size_t>(s) * R * N;
                    for (int i = lane; i < rows * N; i += 32) dst[i] = src[i];
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&hdr->full[st]);
            }
        }
    } else {
        // ---------------- fp64 chains ----------------
        const int n_chains = S * N;
        double acc[kMaxChainsPerLane];
        int ch_slot[kMaxChainsPerLane], ch_col[kMaxChainsPerLane];
#pragma unroll
        for (int q = 0; q < kMaxChainsPerLane; ++q) {
            const int c = lane + 32 * q;
            acc[q] = 0.0;
            ch_slot[q] = c < n_chains ? c / N : -1;
            ch_col[q] = c < n_chains ? c % N : 0;
        }
        for (int c = 0; c < chunks; ++c) {
            const int st = c % kStages;
            ptx::mbar_wait(&hdr->full[st], (c / kStages) & 1);
            const double* xs = ring + static_cast<size_t>(st) * stage_elems;
            const double* ws = xs + R;
            const int rows = min(R, D - c * R);
            for (int i = 0; i < rows; ++i) {
                const double xi = xs[i];
                if (xi == 0.0) continue;  // GateMatrix::logits skips zero activations
#pragma unroll
                for (int q = 0; q < kMaxChainsPerLane; ++q)
                    if (ch_slot[q] >= 0)
                        acc[q] = __dadd_rn(acc[q], __dmul_rn(xi, ws[(static_cast<size_t>(ch_slot[q]) * R + i) * N + ch_col[q]]));
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&hdr->empty[st]);
        }
#pragma unroll
        for (int q = 0; q < kMaxChainsPerLane; ++q)
            if (ch_slot[q] >= 0) logits[ch_slot[q]][ch_col[q]] = acc[q];
        __syncwarp();
        // one lane per item: softmax + decision + top-k
        if (lane < g.n_items) {
            const RouteItem& it = g.items[lane];
            int slot = -1;
            for (int s = 0; s < S; ++s)
                if (slot_item[s] == lane) slot = s;
            decide_item(it, slot >= 0 ? logits[slot] : nullptr, p, o);
        }
    }
}

}  // namespace

cudaError_t launch_route(const RouteGroup* d_groups, int n_groups, int max_gate_items, const RouteParams& p,
                         const RouteOutputs& out, cudaStream_t stream) {
    if (n_groups <= 0) return cudaSuccess;
    if (p.n < 2 || p.n > 64 || max_gate_items > kMaxRouteItems || max_gate_items * p.n > 32 * kMaxChainsPerLane)
        return cudaErrorInvalidValue;
    // rows per chunk: ~24 KB per stage, even (16-byte bulk granularity), capped at d
    const int per_row = 8 * (1 + max_gate_items * p.n);
    int rows = (24 * 1024) / per_row;
    rows = rows < 2 ? 2 : (rows & ~1);
    if (rows > p.d) rows = (p.d + 1) & ~1;
    const bool tma = (p.d % 2 == 0);
    const size_t smem = 128 + static_cast<size_t>(3) * (rows + static_cast<size_t>(max_gate_items) * rows * p.n) * 8;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    route_kernel<<<n_groups, 64, smem, stream>>>(d_groups, max_gate_items, rows, tma ? 1 : 0, p, out);
    return cudaGetLastError();
}

}  // namespace adapmoe
