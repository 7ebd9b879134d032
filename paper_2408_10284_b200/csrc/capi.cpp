// C ABI (include/adapmoe.h) over the C++ engine.  Exceptions are caught at this boundary and
// turned into the reference CLI's exit-code classes (proj/tools/moesim_main.cpp:26-40, :738-757).
#include "../../include/adapmoe.h"

#include <cuda_runtime_api.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "host/files.hpp"
#include "host/policy.hpp"
#include "host/policy_engine.hpp"
#include "runtime/decode.hpp"
#include "runtime/engine.hpp"
#include "runtime/experts.hpp"
#include "kernels/expert_ffn.hpp"

using namespace adapmoe;

struct moe_engine {
    Engine* impl;
};

namespace {
thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
    try {
        g_last_error.clear();
        f();
        return MOE_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return static_cast<int>(e.status);
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return MOE_E_USAGE;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return MOE_E_USAGE;
    }
}

ModelSpec to_spec(const moe_model_spec* s) {
    if (!s) fail(Status::Usage, "null model spec");
    ModelSpec m{s->num_layers, s->experts_per_layer, s->top_k, s->hidden_dim};
    m.validate();
    return m;
}

SimConfig to_cfg(const moe_sim_config* c) {
    if (!c) fail(Status::Usage, "null sim config");
    SimConfig s;
    s.tile_count_per_expert = c->tile_count_per_expert;
    s.tile_transfer_time = c->tile_transfer_time;
    s.tile_compute_time = c->tile_compute_time;
    s.attention_compute_time = c->attention_compute_time;
    s.gate_compute_time = c->gate_compute_time;
    s.lookahead_depth = c->lookahead_depth;
    s.policy = PolicyFlags{c->adaptive_gating != 0, c->prefetch != 0, c->adaptive_cache != 0};
    s.validate();
    return s;
}

Engine& eng(moe_engine_t h) {
    if (!h || !h->impl) fail(Status::Usage, "null engine handle");
    return *h->impl;
}

void require(const void* p, const char* what) {
    if (!p) fail(Status::Usage, std::string("null pointer: ") + what);
}

void export_metrics(const SimMetrics& m, moe_metrics* out, int64_t* lat, int64_t* odl) {
    if (out) {
        out->total_latency = m.total_latency;
        out->stall_time = m.stall_time;
        out->on_demand_loads = m.on_demand_loads;
        out->cache_hits = m.cache_hits;
        out->prefetch_hits = m.prefetch_hits;
        out->single_expert_decisions = m.single_expert_decisions;
        out->experts_activated_total = m.experts_activated_total;
    }
    if (lat) std::memcpy(lat, m.latency_per_token.data(), m.latency_per_token.size() * sizeof(int64_t));
    if (odl)
        for (size_t l = 0; l < m.on_demand_loads_per_layer.size(); ++l) odl[l] = m.on_demand_loads_per_layer[l];
}

void export_events(const std::vector<TimelineEvent>& ev, long long total, moe_event* out, int64_t cap, int64_t* n) {
    if (n) *n = total;
    if (!out) return;
    if (static_cast<int64_t>(ev.size()) > cap) fail(Status::Usage, "events buffer too small (need " + std::to_string(ev.size()) + ")");
    for (size_t i = 0; i < ev.size(); ++i)
        out[i] = moe_event{static_cast<int64_t>(ev[i].stream), static_cast<int64_t>(ev[i].kind), ev[i].start, ev[i].end,
                           ev[i].token, ev[i].layer, ev[i].expert, ev[i].tile};
}

// Replays router outputs through the logical engine (simulate_trace's cache/transfer half).
struct Replayer {
    const ModelSpec& spec;
    const SimConfig& cfg;
    std::vector<int> caps;
    PolicyEngine pe;
    Replayer(const ModelSpec& s, int T, const int32_t* c, const SimConfig& conf, uint64_t seed, bool events)
        : spec(s), cfg(conf), caps(validated(s, c)), pe(s, conf, caps, seed, T, nullptr, events) {}
    static std::vector<int> validated(const ModelSpec& s, const int32_t* c) {
        std::vector<int> v(c, c + s.num_layers);
        Allocation a{v, 0};
        for (int t : v) a.budget += t;
        a.validate(s);
        return v;
    }
    // tokens [t0, t1) of [T][L] router outputs
    void tokens(int t0, int t1, const int32_t* sel, const int32_t* single, const int32_t* preds) {
        const int L = spec.num_layers, K = spec.top_k, PW = 2 + K;
        RouteDecision d;
        RoutePrediction p[3];
        for (int tok = t0; tok < t1; ++tok)
            for (int l = 0; l < L; ++l) {
                const size_t tl = static_cast<size_t>(tok) * L + l;
                d.count = 0;
                for (int k = 0; k < K; ++k) {
                    const int e = sel[tl * K + k];
                    if (e >= 0) d.experts[d.count++] = e;
                }
                d.single = single ? single[tl] != 0 : (cfg.policy.adaptive_gating ? d.count == 1 : K == 1);
                int np = 0;
                if (preds)
                    for (int s = 0; s < 3; ++s) {
                        const int32_t* row = preds + (tl * 3 + s) * PW;
                        if (row[0] < 0) continue;
                        p[np].target = row[0];
                        p[np].count = row[1];
                        for (int k = 0; k < row[1]; ++k) p[np].experts[k] = row[2 + k];
                        ++np;
                    }
                pe.step(tok, l, d, std::span<const RoutePrediction>(p, np));
            }
    }
    void finish(moe_metrics* metrics, int64_t* lat, int64_t* odl, moe_event* events, int64_t cap, int64_t* n_events) {
        export_metrics(pe.metrics(), metrics, lat, odl);
        export_events(pe.timeline(), pe.events_recorded(), events, cap, n_events);
    }
};

void replay(const ModelSpec& spec, int T, const int32_t* caps, const SimConfig& cfg, uint64_t seed, const int32_t* sel,
            const int32_t* single, const int32_t* preds, moe_metrics* metrics, int64_t* lat, int64_t* odl,
            moe_event* events, int64_t cap, int64_t* n_events) {
    Replayer rp(spec, T, caps, cfg, seed, events != nullptr);
    rp.tokens(0, T, sel, single, preds);
    rp.finish(metrics, lat, odl, events, cap, n_events);
}

}  // namespace

extern "C" {

const char* moe_last_error(void) { return g_last_error.c_str(); }
const char* moe_version(void) { return "adapmoe-b200 0.1.0 (sm_100a)"; }

int moe_calibrate_threshold(const moe_model_spec* spec, const double* scores, int32_t tokens, const double* fisher,
                            double target, double* tau, double* realized) {
    return guarded([&] {
        ModelSpec s = to_spec(spec);
        require(scores, "scores");
        require(fisher, "fisher");
        require(tau, "tau");
        const size_t n = static_cast<size_t>(tokens > 0 ? tokens : 0) * s.num_layers * s.experts_per_layer;
        *tau = calibrate_threshold(std::span<const double>(scores, n), tokens, s,
                                   std::span<const double>(fisher, s.num_layers), target, realized);
    });
}

int moe_build_cost_table(const moe_model_spec* spec, const double* alpha, const double* beta, double* table) {
    return guarded([&] {
        ModelSpec s = to_spec(spec);
        require(alpha, "alpha");
        require(beta, "beta");
        require(table, "table");
        for (int l = 0; l < s.num_layers; ++l) LayerProfile{alpha[l], beta[l], 0.0}.validate();
        auto t = build_cost_table(std::span<const double>(alpha, s.num_layers), std::span<const double>(beta, s.num_layers), s);
        std::memcpy(table, t.data(), t.size() * sizeof(double));
    });
}

int moe_dp_allocate(const moe_model_spec* spec, const double* table, int32_t budget, int32_t* caps, double* total) {
    return guarded([&] {
        ModelSpec s = to_spec(spec);
        require(table, "table");
        require(caps, "capacities");
        auto r = dp_allocate(std::span<const double>(table, static_cast<size_t>(s.num_layers) * (s.experts_per_layer + 1)), budget, s);
        for (int l = 0; l < s.num_layers; ++l) caps[l] = r.allocation.capacities[l];
        if (total) *total = r.total_cost;
    });
}

int moe_uniform_allocation(const moe_model_spec* spec, int32_t budget, int32_t* caps) {
    return guarded([&] {
        ModelSpec s = to_spec(spec);
        require(caps, "capacities");
        auto a = uniform_allocation(budget, s);
        for (int l = 0; l < s.num_layers; ++l) caps[l] = a.capacities[l];
    });
}

int moe_expected_cost(int32_t t, int32_t n, double alpha, double beta, double* cost) {
    return guarded([&] {
        require(cost, "cost");
        *cost = expected_cost(t, n, alpha, beta);
    });
}

int moe_tile_pipeline_latency(int32_t tiles, int64_t transfer, int64_t compute, int64_t* latency) {
    return guarded([&] {
        require(latency, "latency");
        *latency = tile_pipeline_latency(tiles, transfer, compute);
    });
}

int moe_replay_policy(const moe_model_spec* spec, int32_t tokens, const int32_t* caps, const moe_sim_config* cfg,
                      uint64_t seed, const int32_t* decisions, const int32_t* single, const int32_t* predictions,
                      moe_metrics* metrics, int64_t* lat, int64_t* odl, moe_event* events, int64_t cap,
                      int64_t* n_events) {
    return guarded([&] {
        ModelSpec s = to_spec(spec);
        SimConfig c = to_cfg(cfg);
        require(caps, "capacities");
        require(decisions, "decisions");
        replay(s, tokens, caps, c, seed, decisions, single, predictions, metrics, lat, odl, events, cap, n_events);
    });
}

int moe_engine_create(const moe_model_spec* spec, int32_t device, moe_engine_t* out) {
    return guarded([&] {
        require(out, "out");
        *out = nullptr;
        ModelSpec s = to_spec(spec);
        auto* h = new moe_engine{nullptr};
        try {
            h->impl = new Engine(s, device);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int moe_engine_destroy(moe_engine_t h) {
    return guarded([&] {
        if (!h) return;
        delete h->impl;
        delete h;
    });
}

int moe_load_gates(moe_engine_t h, const double* gates, const double* first_gate) {
    return guarded([&] {
        require(gates, "gates");
        eng(h).load_gates(gates, first_gate);
    });
}

int moe_route_trace(moe_engine_t h, const double* acts, const double* scores, int32_t T, const double* fisher, double tau,
                    const moe_sim_config* cfg, int32_t* decisions, int32_t* single, double* pert, int32_t* predictions) {
    return guarded([&] {
        Engine& e = eng(h);
        SimConfig c = to_cfg(cfg);
        require(acts, "acts");
        require(scores, "scores");
        require(fisher, "fisher");
        require(decisions, "decisions");
        if (T < 1) fail(Status::Validation, "trace holds no tokens");
        GatingThreshold{tau}.validate();
        const ModelSpec& s = e.spec();
        TraceRoutes r = e.route_trace(acts, scores, T, std::span<const double>(fisher, s.num_layers), tau, c);
        std::memcpy(decisions, r.selected.data(), r.selected.size() * sizeof(int));
        if (single) std::memcpy(single, r.single.data(), r.single.size() * sizeof(int));
        if (pert) std::memcpy(pert, r.perturbation.data(), r.perturbation.size() * sizeof(double));
        if (predictions) std::memcpy(predictions, r.predictions.data(), r.predictions.size() * sizeof(int));
    });
}

int moe_router_forward(moe_engine_t h, int32_t layer, const double* x, int32_t rows, const double* scores, double tau,
                       const double* fisher, int32_t lookahead, int32_t flags, const moe_route_out* out, void* stream) {
    return guarded([&] {
        Engine& e = eng(h);
        require(fisher, "fisher");
        require(out, "out");
        GatingThreshold{tau}.validate();
        RouteOutputs o{out->selected, out->count, out->single, out->perturbation, nullptr};
        e.router_forward(layer, x, rows, scores, tau, std::span<const double>(fisher, e.spec().num_layers), lookahead,
                         (flags & MOE_ROUTE_ADAPTIVE) != 0, o, static_cast<cudaStream_t>(stream));
    });
}

int moe_simulate_trace(moe_engine_t h, const double* acts, const double* scores, int32_t T, const double* fisher,
                       const int32_t* caps, double tau, const moe_sim_config* cfg, uint64_t seed, moe_metrics* metrics,
                       int64_t* lat, int64_t* odl, moe_event* events, int64_t cap, int64_t* n_events) {
    return guarded([&] {
        Engine& e = eng(h);
        SimConfig c = to_cfg(cfg);
        require(acts, "acts");
        require(scores, "scores");
        require(fisher, "fisher");
        require(caps, "capacities");
        if (T < 1) fail(Status::Validation, "trace holds no tokens");
        GatingThreshold{tau}.validate();
        const ModelSpec& s = e.spec();
        // the host engine replays each chunk of tokens while the GPU moves / routes the next ones
        Replayer rp(s, T, caps, c, seed, events != nullptr);
        TraceRoutes r;
        const int chunk = std::max(1, std::min(16, (T + 7) / 8));
        e.route_trace_stream(acts, scores, T, std::span<const double>(fisher, s.num_layers), tau, c, chunk, r,
                             [&](int t0, int t1) {
                                 rp.tokens(t0, t1, r.selected.data(), r.single.data(), r.predictions.data());
                             });
        rp.finish(metrics, lat, odl, events, cap, n_events);
    });
}

int moe_compare_policies(moe_engine_t h, const double* acts, const double* scores, int32_t T, const double* fisher,
                         const double* alpha, const double* beta, double tau, const moe_sim_config* cfg, int32_t budget,
                         uint64_t seed, moe_compare_row* rows, int32_t* capacities, int64_t* lat, int64_t* odl) {
    return guarded([&] {
        Engine& e = eng(h);
        SimConfig base = to_cfg(cfg);
        require(acts, "acts");
        require(scores, "scores");
        require(fisher, "fisher");
        require(alpha, "alpha");
        require(beta, "beta");
        require(rows, "rows");
        require(capacities, "capacities");
        if (T < 1) fail(Status::Validation, "trace holds no tokens");
        GatingThreshold{tau}.validate();
        const ModelSpec& s = e.spec();
        const int L = s.num_layers;
        struct Row {
            const char* name;
            bool g, p, c;
        };
        // ablation_grid (inc/simulator.hpp:476-486), in the reference's order
        const Row grid[7] = {{"baseline", false, false, false},     {"+gating", true, false, false},
                             {"+prefetch", false, true, false},     {"+gating+cache", true, false, true},
                             {"+prefetch+cache", false, true, true}, {"+gating+prefetch", true, true, false},
                             {"all", true, true, true}};
        std::map<int, TraceRoutes> routes;  // K1 once per (gating, prefetch) combination
        std::vector<double> mean(7);
        for (int i = 0; i < 7; ++i) {
            const Row& r = grid[i];
            std::vector<double> a(alpha, alpha + L), b(beta, beta + L);
            if (!r.g) std::fill(a.begin(), a.end(), 0.0);
            if (!r.p) std::fill(b.begin(), b.end(), 0.0);
            const Allocation alloc = r.c ? dp_allocate(build_cost_table(a, b, s), budget, s).allocation
                                         : uniform_allocation(budget, s);
            SimConfig c = base;
            c.policy.adaptive_gating = r.g;
            c.policy.prefetch = r.p;
            c.policy.adaptive_cache = r.c;
            const int key = (r.g ? 1 : 0) | (r.p ? 2 : 0);
            if (!routes.count(key))
                routes[key] = e.route_trace(acts, scores, T, std::span<const double>(fisher, L), tau, c);
            const TraceRoutes& tr = routes[key];
            int32_t* caps = capacities + static_cast<size_t>(i) * L;
            for (int l = 0; l < L; ++l) caps[l] = alloc.capacities[l];
            moe_compare_row& out = rows[i];
            std::memset(out.name, 0, sizeof out.name);
            std::strncpy(out.name, r.name, sizeof out.name - 1);
            out.adaptive_gating = r.g;
            out.prefetch = r.p;
            out.adaptive_cache = r.c;
            int64_t n_events = 0;
            replay(s, T, caps, c, seed, tr.selected.data(), tr.single.data(), tr.predictions.data(), &out.metrics,
                   lat ? lat + static_cast<size_t>(i) * T : nullptr, odl ? odl + static_cast<size_t>(i) * L : nullptr,
                   nullptr, 0, &n_events);
            mean[i] = static_cast<double>(out.metrics.total_latency) / static_cast<double>(T);  // SimMetrics::mean_latency
        }
        for (int i = 0; i < 7; ++i) rows[i].speedup_vs_baseline = mean[i] > 0.0 ? mean[0] / mean[i] : 1.0;
    });
}

int moe_generate_trace(moe_engine_t h, const moe_synth_config* cfg, double* gates, double* acts, double* scores,
                       int32_t* selected, double* fisher) {
    return guarded([&] {
        Engine& e = eng(h);
        require(cfg, "config");
        ModelSpec s = to_spec(&cfg->spec);
        if (!(s == e.spec())) fail(Status::Validation, "generate_trace: spec differs from the engine's");
        require(gates, "gates");
        require(acts, "acts");
        require(scores, "scores");
        require(selected, "selected");
        require(fisher, "fisher");
        e.generate_trace(cfg->tokens, cfg->dirichlet_concentration, cfg->residual_drift, cfg->gate_seed, cfg->token_seed,
                         cfg->shared_gates != 0, cfg->fisher_scales, cfg->drift_scales, gates, acts, scores, selected,
                         fisher);
    });
}

int moe_generate_profiles(moe_engine_t h, const double* acts, const double* scores, int32_t T, const double* fisher,
                          double tau, double* alpha, double* beta) {
    return guarded([&] {
        Engine& e = eng(h);
        require(acts, "acts");
        require(scores, "scores");
        require(fisher, "fisher");
        require(alpha, "alpha");
        require(beta, "beta");
        GatingThreshold{tau}.validate();
        e.generate_profiles(acts, scores, T, std::span<const double>(fisher, e.spec().num_layers), tau, alpha, beta);
    });
}

}  // extern "C"

extern "C" int moe_train_first_gate(moe_engine_t h, const double* acts, const double* scores, int32_t T, double lr,
                                    int32_t steps, uint64_t seed, double* out) {
    return guarded([&] {
        Engine& e = eng(h);
        require(acts, "acts");
        require(scores, "scores");
        require(out, "first_gate_out");
        e.train_first_gate(acts, scores, T, lr, steps, seed, out);
    });
}

// ---- physical decode ------------------------------------------------------------------------
namespace {
void export_stats(const DecodeStats& s, moe_decode_stats* out) {
    if (!out) return;
    out->tokens = s.tokens;
    out->kernels_launched = s.kernels;
    out->ffn_launches = s.ffn_launches;
    out->tile_copies = s.tile_copies;
    out->copy_bytes = s.copy_bytes;
    out->input_bytes = s.input_bytes;
    out->ffn_bytes = s.ffn_bytes;
    out->copy_busy_ms = s.copy_busy_ms;
    out->ffn_ms = s.ffn_ms;
    out->ffn_gate_up_ms = s.gate_up_ms;
    out->ffn_down_ms = s.down_ms;
    out->ffn_gate_up_bytes = s.gate_up_bytes;
    out->ffn_down_bytes = s.down_bytes;
    out->router_ms = s.router_ms;
    out->stall_ms = s.stall_ms;
    out->router_exact_items = s.router_exact;
    out->host_sync_ms = s.host_sync_ms;
    out->host_step_ms = s.host_step_ms;
    out->slots_total = s.slots_total;
    out->staging_high_water = s.staging_high_water;
    out->prefetch_copy_ms = s.prefetch_copy_ms;
    out->prefetch_stall_ms = s.prefetch_stall_ms;
    out->prefetch_tile_copies = s.prefetch_tiles;
    out->prefetch_used_copy_ms = s.prefetch_used_copy_ms;
    out->router_launches = s.router_launches;
    out->spec_launches = s.spec_launches;
    out->spec_hits = s.spec_hits;
    out->record_decode_ms = s.decode_ms;
    out->record_decodes = s.decode_launches;
    out->record_decode_bytes = s.decode_bytes;
}
}  // namespace

extern "C" {

namespace {
int experts_build(moe_engine_t h, int32_t ffn, int32_t tiles, uint64_t seed, int32_t alias, bool init_values,
                  const int32_t* owner, int32_t rank) {
    return guarded([&] {
        Engine& e = eng(h);
        if (owner && (rank < 0 || rank >= e.spec().experts_per_layer))
            fail(Status::Usage, "experts_init: shard rank out of [0, N)");
        e.session.reset();
        e.experts = std::make_unique<ExpertStore>();
        try {
            build_expert_store(e, *e.experts, ffn, tiles, seed, alias, init_values, owner, rank, e.store_format);
        } catch (...) {
            e.experts.reset();
            throw;
        }
    });
}
}  // namespace

int moe_experts_init(moe_engine_t h, int32_t ffn, int32_t tiles, uint64_t seed, int32_t alias) {
    return experts_build(h, ffn, tiles, seed, alias, true, nullptr, 0);
}

int moe_experts_init_shard(moe_engine_t h, int32_t ffn, int32_t tiles, uint64_t seed, int32_t alias,
                           const int32_t* expert_owner, int32_t rank) {
    if (!expert_owner) return experts_build(h, ffn, tiles, seed, alias, true, nullptr, 0);
    return experts_build(h, ffn, tiles, seed, alias, true, expert_owner, rank);
}

int moe_experts_alloc(moe_engine_t h, int32_t ffn, int32_t tiles) {
    return experts_build(h, ffn, tiles, 0, 0, false, nullptr, 0);
}

int moe_experts_alloc_shard(moe_engine_t h, int32_t ffn, int32_t tiles, const int32_t* expert_owner, int32_t rank) {
    return experts_build(h, ffn, tiles, 0, 0, false, expert_owner, rank);
}

int moe_experts_info(moe_engine_t h, int64_t* pinned_bytes, int32_t* stored_experts, int32_t* numa_node) {
    return guarded([&] {
        Engine& e = eng(h);
        if (!e.experts) fail(Status::Usage, "experts not initialised");
        if (pinned_bytes) *pinned_bytes = static_cast<int64_t>(e.experts->pinned_bytes());
        if (stored_experts) *stored_experts = static_cast<int32_t>(e.experts->blocks.size());
        if (numa_node) *numa_node = e.experts->numa_node;
    });
}

int moe_copy_tiles(moe_engine_t h, int32_t layer, int32_t expert, int32_t tile0, int32_t n_tiles, void* dst,
                   void* stream, void* const* tile_events) {
    return guarded([&] {
        Engine& e = eng(h);
        require(dst, "dst");
        if (!e.experts) fail(Status::Usage, "copy_tiles: experts not initialised");
        const ExpertStore& st = *e.experts;
        if (layer < 0 || layer >= st.layers || expert < 0 || expert >= st.experts) fail(Status::Usage, "ExpertRef out of range");
        if (tile0 < 0 || n_tiles < 0 || tile0 + n_tiles > st.tiles) fail(Status::Usage, "copy_tiles: tile range out of [0, tiles)");
        e.activate();
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : e.copy_stream();
        upload_expert_tiles(st, layer, expert, tile0, tile0 + n_tiles, static_cast<unsigned char*>(dst), e.copy_staging,
                            s, reinterpret_cast<cudaEvent_t const*>(tile_events));
    });
}

int moe_expert_ffn_async(moe_engine_t h, const void* expert, const double* x, float* y, int32_t rows,
                         const double* weights, int32_t accumulate, void* const* tile_events, void* stream) {
    return guarded([&] {
        Engine& e = eng(h);
        require(expert, "expert");
        require(x, "x");
        require(y, "y");
        if (rows < 0) fail(Status::Usage, "expert_ffn_async: rows must be >= 0");
        if (!e.experts) fail(Status::Usage, "expert_ffn_async: experts not initialised (shape unknown)");
        e.activate();
        const ExpertStore& st = *e.experts;
        const int D = e.spec().hidden_dim, T = st.tiles, Ft = st.ffn / T;
        cudaStream_t cs = stream ? static_cast<cudaStream_t>(stream) : e.compute_stream();
        if (tile_events)
            for (int t = 0; t < T; ++t)
                if (tile_events[t]) MOE_CUDA(cudaStreamWaitEvent(cs, static_cast<cudaEvent_t>(tile_events[t]), 0));
        int sms = 148;
        MOE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e.device()));
        e.ffn_scratch.reserve(static_cast<size_t>(kFfnMaxCtas) * kFfnSlotsPerCta * D * sizeof(float));
        const size_t gate_up = static_cast<size_t>(2) * Ft * D * 2;
        for (int b = 0; b < rows; ++b) {
            FfnLaunch p;
            p.d = D;
            p.ft = Ft;
            p.x = x + static_cast<size_t>(b) * D;
            p.partial = e.ffn_scratch.as<float>();
            for (int t = 0; t < T; ++t) {
                const unsigned char* tile = static_cast<const unsigned char*>(expert) + t * st.tile_bytes;
                p.seg[p.n_seg].gate_up = reinterpret_cast<const std::uint16_t*>(tile);
                p.seg[p.n_seg].down_t = reinterpret_cast<const std::uint16_t*>(tile + gate_up);
                ++p.n_seg;
            }
            MOE_CUDA(launch_ffn(p, sms, cs));
            CombineArgs c;
            c.x = p.x;
            c.scores = p.x;  // unread: one rank has weight 1
            c.out = y + static_cast<size_t>(b) * D;
            c.ranks = 1;
            c.d = D;
            c.ft = Ft;
            c.residual = 0;
            c.accumulate = accumulate ? 1 : 0;
            c.scale = weights ? static_cast<float>(weights[b]) : 1.0f;
            c.n_refs = T;
            for (int t = 0; t < T; ++t) {
                c.refs[t] = FfnPartialRef{p.partial, ffn_grid(p, sms), T, t, 0};
                ffn_partial_range(c.refs[t], Ft);
            }
            MOE_CUDA(launch_combine(c, cs));
        }
    });
}

int moe_experts_set_format(moe_engine_t h, int32_t format) {
    return guarded([&] {
        Engine& e = eng(h);
        if (format != kStoreBf16 && format != kStoreXb12 && format != kStoreXbh)
            fail(Status::Usage, "experts_set_format: unknown format");
        e.store_format = format;
    });
}

int moe_experts_format(moe_engine_t h, int32_t* format, int64_t* link_bytes) {
    return guarded([&] {
        Engine& e = eng(h);
        if (!e.experts) fail(Status::Usage, "experts not initialised");
        if (format) *format = e.experts->format;
        if (link_bytes) *link_bytes = static_cast<int64_t>(e.experts->link_bytes);
    });
}

int moe_expert_tile_record(moe_engine_t h, int32_t layer, int32_t expert, int32_t tile, const void** record,
                           int64_t* bytes, int32_t* format, uint32_t* base, int64_t* n_escapes, int64_t* nib_offset,
                           int64_t* esc_offset) {
    return guarded([&] {
        Engine& e = eng(h);
        if (!e.experts) fail(Status::Usage, "experts not initialised");
        const ExpertStore& st = *e.experts;
        if (layer < 0 || layer >= st.layers || expert < 0 || expert >= st.experts) fail(Status::Usage, "ExpertRef out of range");
        if (tile < 0 || tile >= st.tiles) fail(Status::Usage, "tile out of range");
        size_t b = 0;
        const unsigned char* r = st.record(layer, expert, tile, &b);
        const Xb12Tile& m = st.meta(layer, expert, tile);
        if (record) *record = r;
        if (bytes) *bytes = static_cast<int64_t>(b);
        if (format) *format = m.format;
        if (base) *base = m.base;
        if (n_escapes) *n_escapes = static_cast<int64_t>(m.n_exc);
        if (nib_offset) *nib_offset = static_cast<int64_t>(m.nib_off);
        if (esc_offset) *esc_offset = static_cast<int64_t>(m.exc_off);
    });
}

int moe_expert_host_ptr(moe_engine_t h, int32_t layer, int32_t expert, const void** ptr) {
    return guarded([&] {
        Engine& e = eng(h);
        require(ptr, "ptr");
        if (!e.experts) fail(Status::Usage, "experts not initialised");
        if (layer < 0 || layer >= e.experts->layers || expert < 0 || expert >= e.experts->experts)
            fail(Status::Usage, "ExpertRef out of range");
        if (e.experts->format != kStoreBf16)
            fail(Status::Usage, "expert_host_ptr: the store is coded (XB12 / XBH; moe_expert_tile_record gives its records)");
        *ptr = e.experts->expert(layer, expert);
    });
}

int moe_expert_set(moe_engine_t h, int32_t layer, int32_t expert, const uint16_t* w1, const uint16_t* w3,
                   const uint16_t* w2) {
    return guarded([&] {
        Engine& e = eng(h);
        require(w1, "w1");
        require(w3, "w3");
        require(w2, "w2");
        if (!e.experts) fail(Status::Usage, "expert_set: call moe_experts_alloc (or moe_experts_init) first");
        if (e.session) fail(Status::Usage, "expert_set: a decode session is active (its HBM slots hold copies)");
        set_expert_weights(e, *e.experts, layer, expert, w1, w3, w2);
    });
}

int moe_expert_bytes(moe_engine_t h, int64_t* bytes) {
    return guarded([&] {
        Engine& e = eng(h);
        require(bytes, "bytes");
        if (!e.experts) fail(Status::Usage, "experts not initialised");
        *bytes = static_cast<int64_t>(e.experts->expert_bytes);
    });
}

int moe_expert_read(moe_engine_t h, int32_t layer, int32_t expert, uint16_t* out) {
    return guarded([&] {
        Engine& e = eng(h);
        require(out, "out");
        if (!e.experts) fail(Status::Usage, "experts not initialised");
        const ModelSpec& s = e.spec();
        if (layer < 0 || layer >= s.num_layers || expert < 0 || expert >= s.experts_per_layer)
            fail(Status::Usage, "ExpertRef out of range");
        read_expert_host(*e.experts, layer, expert, out);
    });
}

int moe_decode_begin_ex(moe_engine_t h, const int32_t* caps, int32_t staging, const double* fisher, double tau,
                        const moe_sim_config* cfg, uint64_t seed, int32_t total_tokens, const moe_decode_opts* opts) {
    return guarded([&] {
        Engine& e = eng(h);
        SimConfig c = to_cfg(cfg);
        require(caps, "capacities");
        require(fisher, "fisher");
        GatingThreshold{tau}.validate();
        if (!e.experts) fail(Status::Usage, "decode_begin: call moe_experts_init first");
        const int L = e.spec().num_layers;
        const int batch = opts ? opts->batch : 1;
        const int ep_rank = opts ? opts->ep_rank : 0;
        const int ep_world = opts ? opts->ep_world : 1;
        const bool free_running = opts ? opts->free_running != 0 : false;
        const double conc = (opts && opts->dirichlet_concentration > 0.0) ? opts->dirichlet_concentration : 1.0;
        const int32_t* owner = opts ? opts->expert_owner : nullptr;
        e.session.reset();
        e.session = std::make_unique<DecodeSession>(e, std::span<const int>(caps, L), staging,
                                                    std::span<const double>(fisher, L), tau, c, seed, total_tokens,
                                                    batch, ep_rank, ep_world, free_running, conc, owner);
    });
}

int moe_decode_begin(moe_engine_t h, const int32_t* caps, int32_t staging, const double* fisher, double tau,
                     const moe_sim_config* cfg, uint64_t seed, int32_t total_tokens) {
    return moe_decode_begin_ex(h, caps, staging, fisher, tau, cfg, seed, total_tokens, nullptr);
}

int moe_decode_ep_export(moe_engine_t h, int32_t max_tokens, uint64_t* ptr, uint8_t* ipc) {
    return guarded([&] {
        Engine& e = eng(h);
        if (!e.session) fail(Status::Usage, "decode_ep_export: no session (call moe_decode_begin_ex)");
        e.session->ep_export(max_tokens, ptr, ipc);
    });
}

int moe_decode_ep_connect(moe_engine_t h, const uint64_t* ptrs, const uint8_t* ipc) {
    return guarded([&] {
        Engine& e = eng(h);
        if (!e.session) fail(Status::Usage, "decode_ep_connect: no session (call moe_decode_begin_ex)");
        e.session->ep_connect(ptrs, ipc);
    });
}

int moe_decode_tokens(moe_engine_t h, const double* acts, const double* scores, int32_t count, int32_t on_device,
                      float* hidden_out, double* gpu_ms) {
    return guarded([&] {
        Engine& e = eng(h);
        require(acts, "acts");
        require(scores, "scores");
        if (!e.session) fail(Status::Usage, "decode_tokens: no session (call moe_decode_begin)");
        const double ms = e.session->decode(acts, scores, count, on_device != 0, hidden_out);
        if (gpu_ms) *gpu_ms = ms;
    });
}

int moe_decode_end(moe_engine_t h, moe_metrics* metrics, int64_t* lat, int64_t* odl, moe_event* events, int64_t cap,
                   int64_t* n_events, moe_decode_stats* stats) {
    return guarded([&] {
        Engine& e = eng(h);
        if (!e.session) fail(Status::Usage, "decode_end: no session");
        DecodeStats s = e.session->finish();
        const PolicyEngine& pe = e.session->policy();
        export_metrics(pe.metrics(), metrics, lat, odl);
        export_events(pe.timeline(), pe.events_recorded(), events, cap, n_events);
        export_stats(s, stats);
        e.session.reset();
    });
}

int moe_decode_layer(moe_engine_t h, int32_t layer, const double* x, const double* scores, float* out,
                     int32_t add_input, void* stream) {
    return guarded([&] {
        Engine& e = eng(h);
        if (!e.session) fail(Status::Usage, "decode_layer: no session (moe_decode_begin)");
        if (layer < 0 || layer >= e.spec().num_layers) fail(Status::Usage, "decode_layer: layer out of range");
        e.session->decode_layer(layer, x, scores, out, add_input != 0,
                                stream ? static_cast<cudaStream_t>(stream) : e.compute_stream());
    });
}

int moe_decode_record_timeline(moe_engine_t h, int32_t enable) {
    return guarded([&] {
        Engine& e = eng(h);
        if (!e.session) fail(Status::Usage, "record_timeline: no session");
        e.session->record_timeline(enable != 0);
    });
}

int moe_decode_timeline_write(moe_engine_t h, const char* path, int64_t* n_events) {
    return guarded([&] {
        Engine& e = eng(h);
        require(path, "path");
        if (!e.session) fail(Status::Usage, "timeline_write: no session");
        const long long n = e.session->write_timeline(path);
        if (n_events) *n_events = n;
    });
}

int moe_decode_stats_snapshot(moe_engine_t h, moe_decode_stats* stats) {
    return guarded([&] {
        Engine& e = eng(h);
        require(stats, "stats");
        if (!e.session) fail(Status::Usage, "decode_stats: no session");
        export_stats(e.session->snapshot(), stats);
    });
}

int moe_expert_ffn(moe_engine_t h, int32_t layer, int32_t expert, const double* x, float* y) {
    return guarded([&] {
        Engine& e = eng(h);
        require(x, "x");
        require(y, "y");
        if (!e.experts) fail(Status::Usage, "experts not initialised");
        const ModelSpec& s = e.spec();
        if (layer < 0 || layer >= s.num_layers || expert < 0 || expert >= s.experts_per_layer)
            fail(Status::Usage, "ExpertRef out of range");
        e.activate();
        const ExpertStore& st = *e.experts;
        const int D = s.hidden_dim, T = st.tiles, F = st.ffn, Ft = F / T;
        DeviceBuffer w, dx, dh, dy, dout, zero;
        w.reserve(st.expert_bytes);
        dx.reserve(D * sizeof(double));
        dh.reserve(F * sizeof(float));
        dy.reserve(static_cast<size_t>(T) * D * sizeof(float));
        dout.reserve(D * sizeof(float));
        zero.reserve(D * sizeof(double));
        cudaStream_t cs = e.compute_stream();
        upload_expert_tiles(st, layer, expert, 0, st.tiles, w.as<unsigned char>(), e.copy_staging, cs);
        MOE_CUDA(cudaMemcpyAsync(dx.ptr, x, D * sizeof(double), cudaMemcpyHostToDevice, cs));
        MOE_CUDA(cudaMemsetAsync(zero.ptr, 0, D * sizeof(double), cs));
        const size_t gate_up = static_cast<size_t>(2) * Ft * D * 2;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e.device());
        DeviceBuffer partial;
        partial.reserve(static_cast<size_t>(kFfnMaxCtas) * kFfnSlotsPerCta * D * sizeof(float));
        FfnLaunch p;
        p.d = D;
        p.ft = Ft;
        p.x = dx.as<double>();
        p.partial = partial.as<float>();
        for (int t = 0; t < T; ++t) {
            const unsigned char* tile = w.as<unsigned char>() + t * st.tile_bytes;
            FfnSegment s;
            s.gate_up = reinterpret_cast<const std::uint16_t*>(tile);
            s.down_t = reinterpret_cast<const std::uint16_t*>(tile + gate_up);
            p.seg[p.n_seg++] = s;
        }
        MOE_CUDA(launch_ffn(p, sms, cs));
        CombineArgs c;
        c.x = zero.as<double>();
        c.scores = zero.as<double>();  // single rank: weight 1
        c.out = dout.as<float>();
        c.ranks = 1;
        c.d = D;
        c.ft = Ft;
        c.experts[0] = 0;
        c.n_refs = T;
        for (int t = 0; t < T; ++t) {
            c.refs[t] = FfnPartialRef{p.partial, ffn_grid(p, sms), T, t, 0};
            ffn_partial_range(c.refs[t], p.ft);
        }
        MOE_CUDA(launch_combine(c, cs));
        MOE_CUDA(cudaMemcpyAsync(y, dout.ptr, D * sizeof(float), cudaMemcpyDeviceToHost, cs));
        MOE_CUDA(cudaStreamSynchronize(cs));
    });
}

}  // extern "C"

// ---- artifact files -----------------------------------------------------------------------------
struct moe_trace_file {
    adapmoe::TraceData data;
};

namespace {
void copy_hash(char* dst, const std::string& h) {
    if (!dst) return;
    std::memset(dst, 0, 17);
    std::strncpy(dst, h.c_str(), 16);
}
}  // namespace

extern "C" {

int moe_trace_load(const char* path, moe_trace_t* out) {
    return guarded([&] {
        require(path, "path");
        require(out, "out");
        auto t = std::make_unique<moe_trace_file>();
        t->data = load_trace_file(path);
        *out = t.release();
    });
}

int moe_trace_info(moe_trace_t t, moe_model_spec* spec, int32_t* tokens) {
    return guarded([&] {
        require(t, "trace");
        if (spec) *spec = moe_model_spec{t->data.spec.num_layers, t->data.spec.experts_per_layer, t->data.spec.top_k,
                                         t->data.spec.hidden_dim};
        if (tokens) *tokens = t->data.tokens;
    });
}

int moe_trace_read(moe_trace_t t, double* acts, double* scores, int32_t* selected) {
    return guarded([&] {
        require(t, "trace");
        const TraceData& d = t->data;
        if (acts) std::memcpy(acts, d.activations.data(), d.activations.size() * sizeof(double));
        if (scores) std::memcpy(scores, d.scores.data(), d.scores.size() * sizeof(double));
        if (selected)
            for (size_t q = 0; q < d.selected.size(); ++q) selected[q] = d.selected[q];
    });
}

int moe_trace_validate(moe_trace_t t, int64_t* violations, char* msg, int64_t cap) {
    return guarded([&] {
        require(t, "trace");
        const std::vector<std::string> v = validate_trace(t->data);
        if (violations) *violations = static_cast<int64_t>(v.size());
        if (msg && cap > 0) {
            const std::string first = v.empty() ? std::string() : v.front();
            const size_t n = std::min<size_t>(first.size(), static_cast<size_t>(cap - 1));
            std::memcpy(msg, first.data(), n);
            msg[n] = '\0';
        }
    });
}

int moe_trace_free(moe_trace_t t) {
    delete t;
    return MOE_OK;
}

int moe_trace_save(const char* path, const moe_model_spec* spec, int32_t T, const double* acts, const double* scores,
                   const int32_t* selected, int32_t binary) {
    return guarded([&] {
        require(path, "path");
        require(acts, "acts");
        require(scores, "scores");
        TraceData d;
        d.spec = to_spec(spec);
        d.tokens = T;
        const size_t L = d.spec.num_layers, N = d.spec.experts_per_layer, K = d.spec.top_k, D = d.spec.hidden_dim;
        d.activations.assign(acts, acts + T * L * D);
        d.scores.assign(scores, scores + T * L * N);
        d.selected.assign(T * L * K, -1);
        d.selected_count.assign(T * L, 0);
        if (selected)
            for (size_t tl = 0; tl < T * L; ++tl)
                for (size_t k = 0; k < K; ++k) {
                    d.selected[tl * K + k] = selected[tl * K + k];
                    if (selected[tl * K + k] >= 0) ++d.selected_count[tl];
                }
        d.token_index.resize(T);
        for (int q = 0; q < T; ++q) d.token_index[q] = q;
        if (binary)
            save_trace_binary(path, d);
        else
            save_trace_jsonl(path, d);
    });
}

int moe_gates_load(const char* path, moe_model_spec* spec, double* gates, double* first_gate, int32_t* has_first,
                   double* lr, int32_t* steps, uint64_t* seed) {
    return guarded([&] {
        require(path, "path");
        const GatesData g = load_gates_file(path);
        if (spec) *spec = moe_model_spec{g.spec.num_layers, g.spec.experts_per_layer, g.spec.top_k, g.spec.hidden_dim};
        if (gates) std::memcpy(gates, g.gates.data(), g.gates.size() * sizeof(double));
        if (has_first) *has_first = g.first_gate ? 1 : 0;
        if (first_gate && g.first_gate) std::memcpy(first_gate, g.first_gate->data(), g.first_gate->size() * sizeof(double));
        if (lr) *lr = g.learning_rate;
        if (steps) *steps = g.steps;
        if (seed) *seed = g.seed;
    });
}

int moe_gates_save(const char* path, const moe_model_spec* spec, const double* gates, const double* first_gate,
                   double lr, int32_t steps, uint64_t seed) {
    return guarded([&] {
        require(path, "path");
        require(gates, "gates");
        GatesData g;
        g.spec = to_spec(spec);
        const size_t one = static_cast<size_t>(g.spec.hidden_dim) * g.spec.experts_per_layer;
        g.gates.assign(gates, gates + one * g.spec.num_layers);
        if (first_gate) g.first_gate = std::vector<double>(first_gate, first_gate + one);
        g.learning_rate = lr;
        g.steps = steps;
        g.seed = seed;
        save_gates_file(path, g);
    });
}

int moe_profiles_load(const char* path, moe_model_spec* spec, double* alpha, double* beta, double* fisher) {
    return guarded([&] {
        require(path, "path");
        const ProfilesData p = load_profiles_file(path);
        if (spec) *spec = moe_model_spec{p.spec.num_layers, p.spec.experts_per_layer, p.spec.top_k, p.spec.hidden_dim};
        if (static_cast<int>(p.alpha.size()) != p.spec.num_layers)
            fail(Status::Validation, std::string(path) + ": profile count does not match num_layers");
        if (alpha) std::copy(p.alpha.begin(), p.alpha.end(), alpha);
        if (beta) std::copy(p.beta.begin(), p.beta.end(), beta);
        if (fisher) std::copy(p.fisher.begin(), p.fisher.end(), fisher);
    });
}

int moe_profiles_save(const char* path, const moe_model_spec* spec, const double* alpha, const double* beta,
                      const double* fisher, char* hash_out) {
    return guarded([&] {
        require(alpha, "alpha");
        require(beta, "beta");
        require(fisher, "fisher");
        ProfilesData p;
        p.spec = to_spec(spec);
        const int L = p.spec.num_layers;
        p.alpha.assign(alpha, alpha + L);
        p.beta.assign(beta, beta + L);
        p.fisher.assign(fisher, fisher + L);
        if (path) save_profiles_file(path, p);
        copy_hash(hash_out, profile_hash(p));
    });
}

int moe_threshold_load(const char* path, double* tau, double* target, double* realized) {
    return guarded([&] {
        require(path, "path");
        const ThresholdData t = load_threshold_file(path);
        if (tau) *tau = t.tau;
        if (target) *target = t.target_single_ratio;
        if (realized) *realized = t.realized_single_ratio;
    });
}

int moe_threshold_save(const char* path, double tau, double target, double realized) {
    return guarded([&] {
        require(path, "path");
        save_threshold_file(path, ThresholdData{tau, target, realized});
    });
}

int moe_allocation_load(const char* path, int32_t* budget, int32_t* n_layers, int32_t* caps, double* total_cost,
                        char* hash) {
    return guarded([&] {
        require(path, "path");
        const AllocationData a = load_allocation_file(path);
        if (budget) *budget = a.budget;
        if (n_layers) *n_layers = static_cast<int32_t>(a.capacities.size());
        if (caps) std::copy(a.capacities.begin(), a.capacities.end(), caps);
        if (total_cost) *total_cost = a.total_cost;
        copy_hash(hash, a.profile_hash);
    });
}

int moe_allocation_save(const char* path, int32_t budget, int32_t n_layers, const int32_t* caps, double total_cost,
                        const char* hash) {
    return guarded([&] {
        require(path, "path");
        require(caps, "capacities");
        AllocationData a;
        a.budget = budget;
        a.capacities.assign(caps, caps + n_layers);
        a.total_cost = total_cost;
        a.profile_hash = hash ? hash : "";
        save_allocation_file(path, a);
    });
}

int moe_cost_table_load(const char* path, int32_t* n, int32_t* n_layers, double* loads) {
    return guarded([&] {
        require(path, "path");
        const CostTableData c = load_cost_table_file(path);
        if (n) *n = c.experts_per_layer;
        if (n_layers) *n_layers = static_cast<int32_t>(c.loads.size());
        if (loads) {
            size_t o = 0;
            for (const auto& row : c.loads) {
                if (static_cast<int>(row.size()) != c.experts_per_layer + 1)
                    fail(Status::Validation, std::string(path) + ": cost table row length != experts_per_layer + 1");
                for (double v : row) loads[o++] = v;
            }
        }
    });
}

int moe_cost_table_save(const char* path, int32_t n, int32_t n_layers, const double* loads) {
    return guarded([&] {
        require(path, "path");
        require(loads, "loads");
        CostTableData c;
        c.experts_per_layer = n;
        for (int l = 0; l < n_layers; ++l)
            c.loads.emplace_back(loads + static_cast<size_t>(l) * (n + 1), loads + static_cast<size_t>(l + 1) * (n + 1));
        save_cost_table_file(path, c);
    });
}

}  // extern "C"
