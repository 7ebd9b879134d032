// TEST INFRASTRUCTURE ONLY — not product code.
//
// Driver for the *unmodified* reference library (moesim, header-only C++20 under
// /root/reference/proj/include). It is compiled by oracle/Makefile straight from
// the read-only reference headers into oracle/_ref/moesim_ref and is used only by
// tests/ (golden generation, parity pinning) and by bench.py's reference arm.
//
// It runs the reference pipeline end to end on the reference's own functions:
//   generate_trace (inc/workload.hpp:60) -> calibrate_threshold (inc/gating.hpp:85)
//   -> [first_layer_training_pairs + train_predictive_gate (inc/workload.hpp:186,
//       inc/prefetch.hpp:194)] -> generate_profiles (inc/workload.hpp:133)
//   -> build_cost_table (inc/cache_model.hpp:189) -> dp_allocate (inc/allocator.hpp:66)
//   -> simulate_trace (inc/simulator.hpp:329)
// and dumps every intermediate as JSON (doubles printed with 17 significant
// digits, so they round-trip exactly) plus an optional raw binary blob.
//
// Predicted-expert lists are not observable from simulate_trace's result, so the
// driver re-evaluates them with the reference's own functions following the
// exact call sequence of inc/simulator.hpp:368-373 and :422-436.
//
// Build flags are pinned to -O2 -std=c++20 with no -march.

#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "moesim/allocator.hpp"
#include "moesim/cache_model.hpp"
#include "moesim/io.hpp"
#include "moesim/core.hpp"
#include "moesim/gating.hpp"
#include "moesim/prefetch.hpp"
#include "moesim/simulator.hpp"
#include "moesim/workload.hpp"

using namespace moesim;

namespace {

std::map<std::string, std::string> g_args;

std::string arg(const char* key, const char* dflt) {
    auto it = g_args.find(key);
    return it == g_args.end() ? std::string(dflt) : it->second;
}
long long argi(const char* key, long long dflt) {
    auto it = g_args.find(key);
    return it == g_args.end() ? dflt : std::stoll(it->second);
}
double argd(const char* key, double dflt) {
    auto it = g_args.find(key);
    return it == g_args.end() ? dflt : std::stod(it->second);
}
std::vector<double> argv_d(const char* key) {
    std::vector<double> out;
    auto it = g_args.find(key);
    if (it == g_args.end() || it->second.empty()) return out;
    std::string s = it->second;
    size_t pos = 0;
    while (pos <= s.size()) {
        size_t next = s.find(',', pos);
        if (next == std::string::npos) next = s.size();
        out.push_back(std::stod(s.substr(pos, next - pos)));
        pos = next + 1;
    }
    return out;
}

std::uint64_t fnv1a_bytes(const void* data, size_t n, std::uint64_t h = 0xcbf29ce484222325ull) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

struct Out {
    std::string s;
    bool first = true;
    void raw(const std::string& t) { s += t; }
    void key(const char* k) {
        if (!first) s += ",\n";
        first = false;
        s += "\"";
        s += k;
        s += "\": ";
    }
    static std::string d(double v) {
        char buf[64];
        std::snprintf(buf, sizeof buf, "%.17g", v);
        return buf;
    }
    template <typename T>
    static std::string arr(const std::vector<T>& v) {
        std::string r = "[";
        for (size_t i = 0; i < v.size(); ++i) {
            if (i) r += ",";
            if constexpr (std::is_floating_point_v<T>)
                r += d(v[i]);
            else
                r += std::to_string(v[i]);
        }
        return r + "]";
    }
};

}  // namespace

int main(int argc, char** argv) {
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        auto eq = a.find('=');
        if (eq == std::string::npos) {
            std::fprintf(stderr, "bad arg %s (want key=value)\n", a.c_str());
            return 1;
        }
        g_args[a.substr(0, eq)] = a.substr(eq + 1);
    }
    const std::string mode = arg("mode", "pipeline");

    SynthConfig cfg;
    cfg.spec = ModelSpec{static_cast<int>(argi("layers", 4)), static_cast<int>(argi("experts", 8)),
                         static_cast<int>(argi("top_k", 2)), static_cast<int>(argi("hidden", 256))};
    cfg.tokens = static_cast<int>(argi("tokens", 64));
    cfg.dirichlet_concentration = argd("concentration", 0.6);
    cfg.residual_drift = argd("drift", 0.18);
    cfg.gate_seed = static_cast<std::uint64_t>(argi("gate_seed", 99));
    cfg.token_seed = static_cast<std::uint64_t>(argi("token_seed", 5000));
    cfg.shared_gates = argi("shared_gates", 0) != 0;
    cfg.scales.fisher = argv_d("fisher_scales");
    cfg.scales.drift = argv_d("drift_scales");

    const double target = argd("target", 0.24);
    const bool train_gate = argi("train_gate", 1) != 0;
    const int train_steps = static_cast<int>(argi("train_steps", 500));
    const double train_lr = argd("train_lr", 0.1);
    const std::uint64_t train_seed = static_cast<std::uint64_t>(argi("train_seed", 0));
    const int budget = static_cast<int>(argi("budget", 16));
    const bool have_tau_override = g_args.count("tau") != 0;

    SimConfig sim;
    sim.tile_count_per_expert = static_cast<int>(argi("tiles", 4));
    sim.tile_transfer_time = argi("tile_transfer", 2);
    sim.tile_compute_time = argi("tile_compute", 1);
    sim.attention_compute_time = argi("attention", 8);
    sim.gate_compute_time = argi("gate_time", 1);
    sim.lookahead_depth = static_cast<int>(argi("lookahead", 2));
    sim.policy.adaptive_gating = argi("gating", 1) != 0;
    sim.policy.prefetch = argi("prefetch", 1) != 0;
    sim.policy.adaptive_cache = true;
    const std::uint64_t sim_seed = static_cast<std::uint64_t>(argi("seed", 0));
    const bool use_uniform = argi("uniform", 0) != 0;

    using clk = std::chrono::steady_clock;
    auto secs = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };

    auto t0 = clk::now();
    GeneratedWorkload wl = generate_trace(cfg);
    auto t1 = clk::now();
    GatingThreshold tau = have_tau_override ? GatingThreshold{argd("tau", 0.0)}
                                            : calibrate_threshold(wl.traces, wl.fisher_diag_sum, target);
    auto t2 = clk::now();
    std::optional<PredictiveGate> first_gate;
    if (train_gate && cfg.tokens >= 2) {
        auto pairs = first_layer_training_pairs(wl.traces);
        first_gate = train_predictive_gate(pairs, cfg.spec.hidden_dim, cfg.spec.experts_per_layer,
                                           TrainingConfig{train_lr, train_steps, train_seed});
    }
    auto t3 = clk::now();
    std::vector<LayerProfile> profiles = generate_profiles(wl.traces, wl.gates, tau, cfg.spec, wl.fisher_diag_sum,
                                                           first_gate ? &*first_gate : nullptr);
    auto t4 = clk::now();
    CostTable table = build_cost_table(profiles, cfg.spec);
    const int clamped = std::min(budget, cfg.spec.num_layers * cfg.spec.experts_per_layer);
    AllocationResult alloc = dp_allocate(table, clamped, cfg.spec);
    Allocation uniform = uniform_allocation(clamped, cfg.spec);
    auto t5 = clk::now();

    SimulationInputs in;
    in.traces = wl.traces;
    in.spec = cfg.spec;
    in.profiles = profiles;
    in.allocation = use_uniform ? uniform : alloc.allocation;
    in.tau = tau;
    in.gates = wl.gates;
    in.first_layer_gate = first_gate ? &*first_gate : nullptr;

    // reference timing arm: repeat simulate_trace over the first `sample` tokens
    if (mode == "bench") {
        const int sample = static_cast<int>(argi("sample_tokens", cfg.tokens));
        const int reps = static_cast<int>(argi("reps", 1));
        SimulationInputs sub = in;
        sub.traces = std::span<const TokenTrace>(wl.traces.data(), std::min<size_t>(sample, wl.traces.size()));
        std::vector<double> alphas, betas;
        for (const LayerProfile& pr : profiles) {
            alphas.push_back(pr.single_expert_prob);
            betas.push_back(pr.prefetch_accuracy);
        }
        double best = 1e30, total = 0;
        SimMetrics m{};
        size_t events = 0;
        std::uint64_t h_tl = 0;
        for (int r = 0; r < reps; ++r) {
            auto a = clk::now();
            SimResult res = simulate_trace(sub, sim, sim_seed);
            auto b = clk::now();
            best = std::min(best, secs(a, b));
            total += secs(a, b);
            m = res.metrics;
            events = res.timeline.events.size();
            if (r == 0) {  // FNV-1a of the timeline as int64 [events][8] (the layout of moe_decode_end)
                std::vector<long long> ev;
                ev.reserve(events * 8);
                for (const auto& e : res.timeline.events) {
                    ev.push_back(e.stream == Stream::Compute ? 0 : 1);
                    ev.push_back(static_cast<int>(e.kind));
                    ev.push_back(e.start);
                    ev.push_back(e.end);
                    ev.push_back(e.token);
                    ev.push_back(e.layer);
                    ev.push_back(e.expert);
                    ev.push_back(e.tile);
                }
                h_tl = fnv1a_bytes(ev.data(), ev.size() * sizeof(long long));
            }
        }
        std::printf(
            "{\"tokens\": %zu, \"reps\": %d, \"simulate_best_s\": %.9f, \"simulate_mean_s\": %.9f, "
            "\"generate_s\": %.6f, \"calibrate_s\": %.6f, \"train_s\": %.6f, \"profile_s\": %.6f, "
            "\"allocate_s\": %.6f, \"on_demand_loads\": %lld, \"metrics\": {\"total_latency\": %lld, "
            "\"stall_time\": %lld, \"on_demand_loads\": %lld, \"cache_hits\": %lld, \"prefetch_hits\": %lld, "
            "\"single_expert_decisions\": %lld, \"experts_activated_total\": %lld, \"on_demand_loads_per_layer\": %s, "
            "\"latency_per_token\": %s}, \"timeline_events\": %zu, \"hash_timeline\": \"%016" PRIx64 "\", "
            "\"tau\": %s, \"alpha\": %s, \"beta\": %s, \"capacities\": %s, \"total_cost\": %s}\n",
            sub.traces.size(), reps, best, total / reps, secs(t0, t1), secs(t1, t2), secs(t2, t3), secs(t3, t4),
            secs(t4, t5), static_cast<long long>(m.on_demand_loads), static_cast<long long>(m.total_latency),
            static_cast<long long>(m.stall_time), static_cast<long long>(m.on_demand_loads),
            static_cast<long long>(m.cache_hits), static_cast<long long>(m.prefetch_hits),
            static_cast<long long>(m.single_expert_decisions), static_cast<long long>(m.experts_activated_total),
            Out::arr(m.on_demand_loads_per_layer).c_str(), Out::arr(m.latency_per_token).c_str(), events, h_tl,
            Out::d(tau.tau).c_str(), Out::arr(alphas).c_str(), Out::arr(betas).c_str(),
            Out::arr(alloc.allocation.capacities).c_str(), Out::d(alloc.total_cost).c_str());
        return 0;
    }

    // artifact files through the reference's own io (inc/io.hpp): write every kind into dir=...
    if (mode == "save") {
        const std::string dir = arg("dir", ".");
        const auto s0 = clk::now();
        save_trace(dir + "/trace.jsonl", wl.traces, cfg.spec);
        GatesFile gf;
        gf.spec = cfg.spec;
        gf.gates = wl.gates;
        gf.first_layer_gate = first_gate;
        save_gates(dir + "/gates.json", gf);
        ProfilesFile pf{cfg.spec, profiles};
        save_profiles(dir + "/profiles.json", pf);
        save_threshold(dir + "/threshold.json", ThresholdFile{tau.tau, target, 0.25});
        save_allocation(dir + "/allocation.json", AllocationFile{alloc.allocation, alloc.total_cost, profile_hash(pf)});
        save_cost_table(dir + "/cost_table.json", table);
        const double save_s = secs(s0, clk::now());
        std::printf("{\"profile_hash\": \"%s\", \"save_s\": %.9f}\n", profile_hash(pf).c_str(), save_s);
        return 0;
    }
    // ... and read them back (dir=...), printing FNV-1a hashes of the arrays and the scalars
    if (mode == "load") {
        const std::string dir = arg("dir", ".");
        auto h = [](const void* p, size_t n, std::uint64_t v) { return fnv1a_bytes(p, n, v); };
        const auto l0 = clk::now();
        TraceFile tf = load_trace(dir + "/trace.jsonl");
        const double load_trace_s = secs(l0, clk::now());
        std::uint64_t ha = 0xcbf29ce484222325ull, hs = ha, hsel = ha;
        for (const auto& tr : tf.traces)
            for (const auto& st : tr.layers) {
                ha = h(st.activation.data(), st.activation.size() * 8, ha);
                hs = h(st.gate.scores.data(), st.gate.scores.size() * 8, hs);
                hsel = h(st.gate.selected.data(), st.gate.selected.size() * 4, hsel);
            }
        GatesFile gf = load_gates(dir + "/gates.json");
        std::uint64_t hg = 0xcbf29ce484222325ull, hfg = hg;
        for (const auto& g : gf.gates) hg = h(g.weights.data(), g.weights.size() * 8, hg);
        if (gf.first_layer_gate) hfg = h(gf.first_layer_gate->gate.weights.data(), gf.first_layer_gate->gate.weights.size() * 8, hfg);
        ProfilesFile pf = load_profiles(dir + "/profiles.json");
        ThresholdFile th = load_threshold(dir + "/threshold.json");
        AllocationFile af = load_allocation(dir + "/allocation.json");
        CostTable ct = load_cost_table(dir + "/cost_table.json");
        std::uint64_t hc = 0xcbf29ce484222325ull;
        for (const auto& row : ct.loads) hc = h(row.data(), row.size() * 8, hc);
        std::vector<double> alpha, beta, fisher;
        for (const auto& p : pf.profiles) {
            alpha.push_back(p.single_expert_prob);
            beta.push_back(p.prefetch_accuracy);
            fisher.push_back(p.fisher_diag_sum);
        }
        std::printf(
            "{\"tokens\": %zu, \"hash_activations\": \"%016" PRIx64 "\", \"hash_scores\": \"%016" PRIx64
            "\", \"hash_selected\": \"%016" PRIx64 "\", \"hash_gates\": \"%016" PRIx64 "\", \"hash_first_gate\": \"%016" PRIx64
            "\", \"first_gate_steps\": %d, \"alpha\": %s, \"beta\": %s, \"fisher\": %s, \"profile_hash\": \"%s\", "
            "\"tau\": %s, \"capacities\": %s, \"budget\": %d, \"total_cost\": %s, \"alloc_profile_hash\": \"%s\", "
            "\"hash_cost_table\": \"%016" PRIx64 "\", \"load_trace_s\": %.9f}\n",
            tf.traces.size(), ha, hs, hsel, hg, hfg, gf.first_layer_gate ? gf.first_layer_gate->config.steps : -1,
            Out::arr(alpha).c_str(), Out::arr(beta).c_str(), Out::arr(fisher).c_str(), profile_hash(pf).c_str(),
            Out::d(th.tau).c_str(), Out::arr(af.allocation.capacities).c_str(), af.allocation.budget,
            Out::d(af.total_cost).c_str(), af.profile_hash.c_str(), hc, load_trace_s);
        return 0;
    }

    // the Table-2 ablation grid (inc/simulator.hpp:476-550; CLI `compare`, moesim_main.cpp:356-378:
    // the raw --budget is passed through)
    if (mode == "compare") {
        const int jobs = static_cast<int>(argi("jobs", 1));
        const auto c0 = clk::now();
        ComparisonReport rep = compare_policies(in, sim, budget, sim_seed, jobs);
        const double compare_s = secs(c0, clk::now());
        std::string r = "{\"compare_s\": " + Out::d(compare_s) + ", \"jobs\": " + std::to_string(jobs) + ", \"rows\": [";
        for (size_t i = 0; i < rep.rows.size(); ++i) {
            const ComparisonRow& row = rep.rows[i];
            const SimMetrics& m = row.metrics;
            if (i) r += ",\n";
            r += "{\"name\": \"" + row.name + "\", \"flags\": [" + std::to_string(row.flags.adaptive_gating) + "," +
                 std::to_string(row.flags.prefetch) + "," + std::to_string(row.flags.adaptive_cache) +
                 "], \"capacities\": " + Out::arr(row.allocation.capacities) +
                 ", \"speedup_vs_baseline\": " + Out::d(row.speedup_vs_baseline) +
                 ", \"metrics\": {\"total_latency\": " + std::to_string(m.total_latency) +
                 ", \"stall_time\": " + std::to_string(m.stall_time) +
                 ", \"on_demand_loads\": " + std::to_string(m.on_demand_loads) +
                 ", \"cache_hits\": " + std::to_string(m.cache_hits) +
                 ", \"prefetch_hits\": " + std::to_string(m.prefetch_hits) +
                 ", \"single_expert_decisions\": " + std::to_string(m.single_expert_decisions) +
                 ", \"experts_activated_total\": " + std::to_string(m.experts_activated_total) +
                 ", \"latency_per_token\": " + Out::arr(m.latency_per_token) +
                 ", \"on_demand_loads_per_layer\": " + Out::arr(m.on_demand_loads_per_layer) + "}}";
        }
        r += "], \"tau\": " + Out::d(tau.tau) + "}\n";
        std::fputs(r.c_str(), stdout);
        return 0;
    }

    SimResult res = simulate_trace(in, sim, sim_seed);

    const int L = cfg.spec.num_layers, N = cfg.spec.experts_per_layer, T = cfg.tokens, D = cfg.spec.hidden_dim;

    // raw binary blob: gates [L][D][N], first gate [D][N] (if any), activations [T][L][D], scores [T][L][N]
    std::string blob = arg("blob", "");
    std::uint64_t h_gates = 0xcbf29ce484222325ull, h_act = 0xcbf29ce484222325ull, h_sc = 0xcbf29ce484222325ull,
                  h_fg = 0xcbf29ce484222325ull;
    for (const auto& g : wl.gates) h_gates = fnv1a_bytes(g.weights.data(), g.weights.size() * 8, h_gates);
    for (const auto& tr : wl.traces)
        for (const auto& st : tr.layers) {
            h_act = fnv1a_bytes(st.activation.data(), st.activation.size() * 8, h_act);
            h_sc = fnv1a_bytes(st.gate.scores.data(), st.gate.scores.size() * 8, h_sc);
        }
    if (first_gate) h_fg = fnv1a_bytes(first_gate->gate.weights.data(), first_gate->gate.weights.size() * 8, h_fg);
    if (!blob.empty()) {
        FILE* f = std::fopen(blob.c_str(), "wb");
        if (!f) return 2;
        for (const auto& g : wl.gates) std::fwrite(g.weights.data(), 8, g.weights.size(), f);
        if (first_gate) std::fwrite(first_gate->gate.weights.data(), 8, first_gate->gate.weights.size(), f);
        for (const auto& tr : wl.traces)
            for (const auto& st : tr.layers) std::fwrite(st.activation.data(), 8, st.activation.size(), f);
        for (const auto& tr : wl.traces)
            for (const auto& st : tr.layers) std::fwrite(st.gate.scores.data(), 8, st.gate.scores.size(), f);
        std::fclose(f);
    }

    // predicted lists exactly as simulate_trace evaluates them (inc/simulator.hpp:368-373, 422-436)
    const bool prefetch_on = sim.policy.prefetch && sim.lookahead_depth > 0;
    auto predicted_selection = [&](std::span<const double> activation, const GateMatrix& gate, int target_layer) {
        const std::vector<double> scores = predict_scores(activation, gate);
        if (sim.policy.adaptive_gating)
            return gate_decide_sensitivity(scores, in.profiles[target_layer], in.tau, in.spec).selected;
        return top_k_indices(scores, in.spec.top_k);
    };

    Out o;
    o.raw("{\n");
    char hx[32];
    auto hex = [&](std::uint64_t v) {
        std::snprintf(hx, sizeof hx, "\"%016" PRIx64 "\"", v);
        return std::string(hx);
    };
    o.key("spec");
    o.raw("[" + std::to_string(L) + "," + std::to_string(N) + "," + std::to_string(cfg.spec.top_k) + "," +
          std::to_string(D) + "]");
    o.key("tokens");
    o.raw(std::to_string(T));
    o.key("hash_gates");
    o.raw(hex(h_gates));
    o.key("hash_activations");
    o.raw(hex(h_act));
    o.key("hash_scores");
    o.raw(hex(h_sc));
    o.key("hash_first_gate");
    o.raw(first_gate ? hex(h_fg) : "null");
    o.key("fisher");
    o.raw(Out::arr(wl.fisher_diag_sum));
    o.key("tau");
    o.raw(Out::d(tau.tau));
    {
        std::vector<int> gen_sel;
        for (const auto& tr : wl.traces)
            for (const auto& st : tr.layers)
                for (int e : st.gate.selected) gen_sel.push_back(e);
        o.key("generated_selected");
        o.raw(Out::arr(gen_sel));
    }
    {
        std::vector<double> a, b, f;
        for (const auto& p : profiles) {
            a.push_back(p.single_expert_prob);
            b.push_back(p.prefetch_accuracy);
            f.push_back(p.fisher_diag_sum);
        }
        o.key("alpha");
        o.raw(Out::arr(a));
        o.key("beta");
        o.raw(Out::arr(b));
    }
    {
        std::vector<double> flat;
        for (const auto& row : table.loads)
            for (double v : row) flat.push_back(v);
        o.key("cost_table");
        o.raw(Out::arr(flat));
    }
    o.key("budget");
    o.raw(std::to_string(clamped));
    o.key("capacities");
    o.raw(Out::arr(alloc.allocation.capacities));
    o.key("total_cost");
    o.raw(Out::d(alloc.total_cost));
    o.key("uniform_capacities");
    o.raw(Out::arr(uniform.capacities));
    o.key("sim_capacities");
    o.raw(Out::arr(in.allocation.capacities));

    // actual decisions from stored scores (inc/simulator.hpp:390-396)
    {
        std::vector<int> sel_flat, sel_count, single;
        std::vector<double> pert;
        for (const auto& tr : wl.traces)
            for (int l = 0; l < L; ++l) {
                GatingDecision dec;
                if (sim.policy.adaptive_gating) {
                    dec = gate_decide_sensitivity(tr.layers[l].gate.scores, in.profiles[l], in.tau, in.spec);
                } else {
                    dec.selected = top_k_indices(tr.layers[l].gate.scores, in.spec.top_k);
                    dec.single = in.spec.top_k == 1;
                }
                sel_count.push_back(static_cast<int>(dec.selected.size()));
                for (int k = 0; k < cfg.spec.top_k; ++k)
                    sel_flat.push_back(k < static_cast<int>(dec.selected.size()) ? dec.selected[k] : -1);
                single.push_back(dec.single ? 1 : 0);
                pert.push_back(dec.perturbation);
            }
        o.key("decision_selected");
        o.raw(Out::arr(sel_flat));
        o.key("decision_count");
        o.raw(Out::arr(sel_count));
        o.key("decision_single");
        o.raw(Out::arr(single));
        o.key("decision_perturbation");
        o.raw(Out::arr(pert));
    }
    // predictions: per (tok, layer, depth-slot<3): target layer (-1 none), count, experts[K] (-1 pad)
    {
        std::vector<int> pred;
        for (int tok = 0; tok < T; ++tok)
            for (int l = 0; l < L; ++l) {
                std::vector<LayerPrediction> preds;
                if (prefetch_on) {
                    const auto& act = wl.traces[tok].layers[l].activation;
                    if (l + 1 < L) {
                        for (int depth = 1; depth <= sim.lookahead_depth; ++depth) {
                            const int tgt = l + depth;
                            if (tgt >= L) break;
                            preds.push_back(LayerPrediction{tgt, predicted_selection(act, wl.gates[tgt], tgt)});
                        }
                    } else if (first_gate && tok + 1 < T) {
                        preds.push_back(LayerPrediction{0, predicted_selection(act, first_gate->gate, 0)});
                    }
                }
                for (int s = 0; s < 3; ++s) {
                    if (s < static_cast<int>(preds.size())) {
                        pred.push_back(preds[s].layer);
                        pred.push_back(static_cast<int>(preds[s].experts.size()));
                        for (int k = 0; k < cfg.spec.top_k; ++k)
                            pred.push_back(k < static_cast<int>(preds[s].experts.size()) ? preds[s].experts[k] : -1);
                    } else {
                        pred.push_back(-1);
                        pred.push_back(0);
                        for (int k = 0; k < cfg.spec.top_k; ++k) pred.push_back(-1);
                    }
                }
            }
        o.key("predictions");
        o.raw(Out::arr(pred));
    }
    const SimMetrics& m = res.metrics;
    o.key("metrics");
    o.raw("{\"total_latency\": " + std::to_string(m.total_latency) + ", \"stall_time\": " +
          std::to_string(m.stall_time) + ", \"on_demand_loads\": " + std::to_string(m.on_demand_loads) +
          ", \"cache_hits\": " + std::to_string(m.cache_hits) + ", \"prefetch_hits\": " +
          std::to_string(m.prefetch_hits) + ", \"single_expert_decisions\": " +
          std::to_string(m.single_expert_decisions) + ", \"experts_activated_total\": " +
          std::to_string(m.experts_activated_total) + ", \"on_demand_loads_per_layer\": " +
          Out::arr(m.on_demand_loads_per_layer) + ", \"latency_per_token\": " + Out::arr(m.latency_per_token) + "}");
    {
        std::vector<long long> ev;
        for (const auto& e : res.timeline.events) {
            ev.push_back(e.stream == Stream::Compute ? 0 : 1);
            ev.push_back(static_cast<int>(e.kind));
            ev.push_back(e.start);
            ev.push_back(e.end);
            ev.push_back(e.token);
            ev.push_back(e.layer);
            ev.push_back(e.expert);
            ev.push_back(e.tile);
        }
        o.key("timeline");
        o.raw(Out::arr(ev));
    }
    o.raw("\n}\n");
    std::fwrite(o.s.data(), 1, o.s.size(), stdout);
    return 0;
}
