// K1 — fused router + reuse-based pre-gate (host launch interface).
//
// One "group" = one activation vector x (fp64, [d]) and up to kMaxRouteItems routing items that
// read it: the actual decision for layer l (from the stored trace scores, or from logits of
// layer l's gate) plus the look-ahead predictions (x . W_{l+1..l+k}, or the first-layer gate at the
// last layer).  Each item writes its selected experts (score-descending, -1 padded to K), the
// count, the single-expert flag and the sensitivity perturbation; optionally its scores/logits.
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>

namespace adapmoe {

constexpr int kMaxRouteItems = 4;

enum RouteFlags : int {
    kRouteAdaptive = 1,     // sensitivity gate (inc/gating.hpp:56-64) instead of plain top-K
    kRouteDivConc = 2,      // logits /= concentration before softmax (inc/workload.hpp:94)
    kRouteEmitScores = 4,   // write the post-softmax scores
    kRouteEmitLogits = 8,   // write the exact fp64 logits to `scores`, skip the decision (the caller
                            // applies glibc exp: used where stored score bits must match)
    kRouteExact = 16,       // skip the fp32 fast path: exact reference-order fp64 logits
};

struct RouteItem {
    const double* gate = nullptr;    // [d][N] fp64 (reference layout); nullptr => decide from `scores`
    const float* gate32 = nullptr;   // [N][d] fp32 transposed copy (fast path)
    const double* scores = nullptr;  // [N] stored post-softmax scores (gate == nullptr)
    double fisher = 0.0;
    int flags = 0;
    int out = 0;                     // output row
};

struct RouteGroup {
    const double* x = nullptr;
    int n_items = 0;
    RouteItem items[kMaxRouteItems];
};

struct RouteOutputs {
    int* selected = nullptr;         // [rows][K]
    int* count = nullptr;            // [rows]
    int* single = nullptr;           // [rows]
    double* perturbation = nullptr;  // [rows] (may be null)
    double* scores = nullptr;        // [rows][N] (may be null; kRouteEmitScores / kRouteEmitLogits)
    // [rows] (may be null): 0 = certified fp32 fast path; 1 = exact fp64 path, decided on the device;
    // 2 + i = exact fp64 path, logits queued in host_entries[i] for the host decision (below);
    // -1 = exact path but the host queue was full (the caller must fail)
    int* exact_used = nullptr;
    // Host-decision queue.  The reference softmaxes with glibc exp (inc/core.hpp:205-216); CUDA's exp
    // can differ from it by an ulp, so a decision taken on the device from exact logits is exact only
    // in practice.  With host_entries set, every exact-path gate item (the uncertified ones, ~1 in
    // 600 look-ahead items at 8x7B) also appends [flags, fisher, logits[N]] (2 + N doubles) to this
    // pinned, device-visible array and the host re-decides it with the reference's own procedure
    // (route_host_decide): bit-exact by construction.  host_counter (device memory) must be zero
    // before the first launch that uses the queue.
    double* host_entries = nullptr;
    unsigned* host_counter = nullptr;
    int host_cap = 0;
};

struct RouteParams {
    int d = 0, n = 0, k = 0;
    double tau = 0.0;
    double concentration = 1.0;
    int force_exact = 0;  // test knob (ADAPMOE_ROUTE_FORCE_EXACT=1, read by launch_route): no fast path
};

// Scratch for the split launch (per-layer decode): per group kMaxRouteItems x kMaxN fp32 logits and
// magnitude sums, and one ticket per group (zero-initialised once; the kernel re-arms it).
struct RouteScratch {
    float* f = nullptr;
    float* a = nullptr;
    unsigned* tickets = nullptr;
    int groups = 0;  // capacity in groups
};

// Launch K1 over `n_groups` groups already resident in device memory.  max_gate_items = the most
// gate items (look-ahead / exact-logit items) any group holds.  With `scratch`, groups whose gate
// columns exceed one round of a CTA's warps are split over several CTAs (lower latency).
cudaError_t launch_route(const RouteGroup* d_groups, int n_groups, int max_gate_items, const RouteParams& p,
                         const RouteOutputs& out, cudaStream_t stream, const RouteScratch* scratch = nullptr);

// Host side of the queue: re-decide every row whose exact_used is >= 2 from its queued logits with
// the reference procedure (softmax with libm exp, sensitivity gate / top-K; policy.hpp), overwriting
// selected [rows][K], count, single and (if non-null) perturbation.  rows [row0, row1) of exact_used
// are scanned; fails (Internal) on a queue overflow (-1).
void route_host_decide(const RouteParams& p, const double* host_entries, const int* exact_used, long long row0,
                       long long row1, int* selected, int* count, int* single, double* perturbation);

// fp32 transposed copy [N][d] of a row-major fp64 [d][N] gate (device to device).
cudaError_t launch_gate_transpose(const double* src, float* dst, int d, int n, int count, cudaStream_t stream);

}  // namespace adapmoe
