// Host half of K1's exact path (kernels/router.hpp, RouteOutputs::host_entries): the items the fp32
// fast path could not certify arrive here with their exact reference-order fp64 logits, and are
// decided with the reference's own procedure and libm — softmax with std::exp (inc/core.hpp:205-216),
// optional / concentration (inc/workload.hpp:94), the sensitivity gate (inc/gating.hpp:56-64) or plain
// top-K (inc/simulator.hpp:368-373, :394-395) — so the decision bits are the reference's by
// construction, not only in practice.  Compiled without FP contraction (Makefile).
#include <string>
#include <vector>

#include "../host/policy.hpp"
#include "../kernels/router.hpp"

namespace adapmoe {

void route_host_decide(const RouteParams& p, const double* host_entries, const int* exact_used, long long row0,
                       long long row1, int* selected, int* count, int* single, double* perturbation) {
    const int N = p.n, K = p.k;
    std::vector<double> logits(N);
    for (long long row = row0; row < row1; ++row) {
        const int tag = exact_used[row];
        if (tag < 0)
            fail(Status::Internal, "router: host-decision queue overflow at row " + std::to_string(row) +
                                       " (route fewer tokens per launch: ADAPMOE_ROUTE_WINDOW)");
        if (tag < 2) continue;
        const double* e = host_entries + static_cast<size_t>(tag - 2) * (2 + N);
        const int flags = static_cast<int>(e[0]);
        const double fisher = e[1];
        for (int j = 0; j < N; ++j) logits[j] = (flags & kRouteDivConc) ? e[2 + j] / p.concentration : e[2 + j];
        const std::vector<double> scores = softmax(logits);
        int* sel = selected + row * K;
        if (flags & kRouteAdaptive) {
            const GatingDecision d = gate_decide_sensitivity(scores, fisher, p.tau, K);
            for (int r = 0; r < K; ++r) sel[r] = r < static_cast<int>(d.selected.size()) ? d.selected[r] : -1;
            count[row] = static_cast<int>(d.selected.size());
            single[row] = d.single ? 1 : 0;
            if (perturbation) perturbation[row] = d.perturbation;
        } else {
            const std::vector<int> top = top_k_indices(scores, K);
            for (int r = 0; r < K; ++r) sel[r] = top[r];
            count[row] = K;
            single[row] = K == 1;
            if (perturbation) perturbation[row] = 0.0;
        }
    }
}

}  // namespace adapmoe
