// Drop-in example (C++ host code over the C ABI only): what a maintainer of the reference's
// `moesim simulate` (proj/tools/moesim_main.cpp:291-347) links against instead of the header
// library.  It reads the reference's own artifact files (trace.jsonl, gates.json, profiles.json,
// threshold.json, allocation.json — inc/io.hpp formats), validates the trace, runs simulate_trace
// with the router on the B200 (K1) and prints the SimMetrics as one JSON line.
//
//   g++ -std=c++17 -O2 -Iinclude examples/simulate_files.cpp -Lpaper_2408_10284_b200 -ladapmoe
//       -Wl,-rpath,$PWD/paper_2408_10284_b200 -o examples/simulate_files
//   examples/simulate_files <dir> [tiles transfer compute attention gate lookahead gating prefetch seed]
//
// Exit codes are the library's (= the reference CLI's classes, moesim_main.cpp:26-40).
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "adapmoe.h"

namespace {

int die(int rc, const char* what) {
    std::fprintf(stderr, "%s: %s\n", what, moe_last_error());
    return rc;
}

bool same_model(const moe_model_spec& a, const moe_model_spec& b) {
    return a.num_layers == b.num_layers && a.experts_per_layer == b.experts_per_layer && a.top_k == b.top_k &&
           a.hidden_dim == b.hidden_dim;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <dir with trace.jsonl gates.json profiles.json threshold.json allocation.json>"
                             " [tiles transfer compute attention gate lookahead gating prefetch seed]\n", argv[0]);
        return 1;
    }
    const std::string dir = argv[1];
    auto arg = [&](int i, long long def) { return argc > i ? std::atoll(argv[i]) : def; };
    // CLI defaults of `simulate` (moesim_main.cpp:259-267)
    moe_sim_config cfg{static_cast<int32_t>(arg(2, 4)), arg(3, 2), arg(4, 1), arg(5, 8), arg(6, 1),
                       static_cast<int32_t>(arg(7, 2)), static_cast<int32_t>(arg(8, 1)), static_cast<int32_t>(arg(9, 1)),
                       1};
    const uint64_t seed = static_cast<uint64_t>(arg(10, 0));

    // trace (load_trace_checked, moesim_main.cpp:91)
    moe_trace_t tr;
    if (int rc = moe_trace_load((dir + "/trace.jsonl").c_str(), &tr)) return die(rc, "load_trace");
    moe_model_spec spec;
    int32_t T = 0;
    moe_trace_info(tr, &spec, &T);
    int64_t violations = 0;
    char first[256];
    moe_trace_validate(tr, &violations, first, sizeof first);
    if (violations) {
        std::fprintf(stderr, "trace validation failed (%lld): %s\n", static_cast<long long>(violations), first);
        moe_trace_free(tr);
        return MOE_E_VALIDATION;
    }
    const size_t L = spec.num_layers, N = spec.experts_per_layer, D = spec.hidden_dim;
    std::vector<double> acts(T * L * D), scores(T * L * N);
    moe_trace_read(tr, acts.data(), scores.data(), nullptr);
    moe_trace_free(tr);

    // gates (+ trained first-layer gate), profiles (fisher), threshold, allocation
    moe_model_spec gspec;
    int32_t has_first = 0;
    if (int rc = moe_gates_load((dir + "/gates.json").c_str(), &gspec, nullptr, nullptr, &has_first, nullptr, nullptr, nullptr))
        return die(rc, "load_gates");
    std::vector<double> gates(L * D * N), first_gate(has_first ? D * N : 0);
    moe_gates_load((dir + "/gates.json").c_str(), &gspec, gates.data(), has_first ? first_gate.data() : nullptr, &has_first,
                   nullptr, nullptr, nullptr);
    moe_model_spec pspec;
    if (int rc = moe_profiles_load((dir + "/profiles.json").c_str(), &pspec, nullptr, nullptr, nullptr))
        return die(rc, "load_profiles");
    // require_same_model (moesim_main.cpp:102-104): exit 4 on a spec mismatch between input files
    if (!same_model(spec, gspec) || !same_model(spec, pspec)) {
        std::fprintf(stderr, "simulate: model spec mismatch between input files\n");
        return MOE_E_VALIDATION;
    }
    std::vector<double> alpha(L), beta(L), fisher(L);
    moe_profiles_load((dir + "/profiles.json").c_str(), &pspec, alpha.data(), beta.data(), fisher.data());
    double tau = 0.0;
    if (int rc = moe_threshold_load((dir + "/threshold.json").c_str(), &tau, nullptr, nullptr)) return die(rc, "load_threshold");
    int32_t budget = 0, n_layers = 0;
    std::vector<int32_t> caps(L);
    if (int rc = moe_allocation_load((dir + "/allocation.json").c_str(), &budget, &n_layers, nullptr, nullptr, nullptr))
        return die(rc, "load_allocation");
    if (static_cast<size_t>(n_layers) != L) {  // simulate_trace's invalid_argument -> exit 5 (moesim_main.cpp:313-317)
        std::fprintf(stderr, "simulate: allocation has %d layers, model has %zu\n", n_layers, L);
        return MOE_E_INFEASIBLE;
    }
    moe_allocation_load((dir + "/allocation.json").c_str(), &budget, &n_layers, caps.data(), nullptr, nullptr);

    // simulate_trace with K1 on the GPU
    moe_engine_t eng;
    if (int rc = moe_engine_create(&spec, 0, &eng)) return die(rc, "engine_create");
    if (int rc = moe_load_gates(eng, gates.data(), has_first ? first_gate.data() : nullptr)) return die(rc, "load_gates");
    moe_metrics m;
    std::vector<int64_t> latency(T), per_layer(L);
    int64_t n_events = 0;
    const int rc = moe_simulate_trace(eng, acts.data(), scores.data(), T, fisher.data(), caps.data(), tau, &cfg, seed, &m,
                                      latency.data(), per_layer.data(), nullptr, 0, &n_events);
    moe_engine_destroy(eng);
    if (rc) return die(rc == MOE_E_USAGE ? MOE_E_INFEASIBLE : rc, "simulate_trace");
    std::printf("{\"tokens\": %d, \"total_latency\": %lld, \"stall_time\": %lld, \"on_demand_loads\": %lld, "
                "\"cache_hits\": %lld, \"prefetch_hits\": %lld, \"single_expert_decisions\": %lld, "
                "\"experts_activated_total\": %lld, \"timeline_events\": %lld, \"on_demand_loads_per_layer\": [",
                T, static_cast<long long>(m.total_latency), static_cast<long long>(m.stall_time),
                static_cast<long long>(m.on_demand_loads), static_cast<long long>(m.cache_hits),
                static_cast<long long>(m.prefetch_hits), static_cast<long long>(m.single_expert_decisions),
                static_cast<long long>(m.experts_activated_total), static_cast<long long>(n_events));
    for (size_t l = 0; l < L; ++l) std::printf("%s%lld", l ? ", " : "", static_cast<long long>(per_layer[l]));
    std::printf("]}\n");
    return 0;
}
