// Logical decode engine (see policy_engine.hpp).  Ordering rules that decide the event trace:
//   * channel picks the on-demand FIFO head when it is ready at the would-be start tick,
//     otherwise the prefetch FIFO head (inc/simulator.hpp:276-284);
//   * promotion moves a queued prefetch to the back of the on-demand FIFO; an in-flight tile is
//     never pre-empted (:203-211);
//   * prefetched experts enter the cache (fresh) when their last tile lands, on-demand experts
//     after their tiles were consumed (:297-304, :461);
//   * transfer events are recorded when a tile starts, so the trace is call-ordered (:286-291).
#include "policy_engine.hpp"

#include <algorithm>
#include <limits>

namespace adapmoe {

void LruSet::to_front(int e) {
    auto it = std::find(order_.begin(), order_.end(), e);
    std::rotate(order_.begin(), it, it + 1);
}

void LruSet::touch(int e) {
    if (!contains(e)) fail(Status::Internal, "LruSet::touch: expert not resident");
    to_front(e);
    fresh_ &= ~(1ull << e);
}

std::optional<int> LruSet::insert(int e, bool fresh) {
    if (capacity_ == 0) return e;  // capacity-0 layers hold nothing (inc/simulator.hpp:83)
    if (contains(e)) {
        to_front(e);
        if (!fresh) fresh_ &= ~(1ull << e);
        return std::nullopt;
    }
    std::optional<int> victim;
    if (static_cast<int>(order_.size()) == capacity_) {
        victim = order_.back();
        order_.pop_back();
        members_ &= ~(1ull << *victim);
        fresh_ &= ~(1ull << *victim);
    }
    order_.insert(order_.begin(), e);
    members_ |= 1ull << e;
    if (fresh) fresh_ |= 1ull << e;
    return victim;
}

PolicyEngine::PolicyEngine(const ModelSpec& spec, const SimConfig& cfg, std::span<const int> capacities,
                           std::uint64_t seed, int total_tokens, DecodeListener* listener, bool record_timeline)
    : spec_(spec), cfg_(cfg), total_tokens_(total_tokens), listener_(listener), record_(record_timeline) {
    spec_.validate();
    cfg_.validate();
    if (static_cast<int>(capacities.size()) != spec.num_layers) fail(Status::Usage, "PolicyEngine: capacity count != num_layers");
    prefetch_on_ = cfg.policy.prefetch && cfg.lookahead_depth > 0;
    const int L = spec.num_layers, N = spec.experts_per_layer;
    metrics_.on_demand_loads_per_layer.assign(L, 0);
    pending_.assign(static_cast<std::size_t>(L) * N, -1);
    done_.resize(static_cast<std::size_t>(L) * N);
    // initial residency: one SeededRng(seed) stream, layer by layer, inserted in draw order so
    // the first drawn expert ends up least recently used (inc/simulator.hpp:352-360)
    SeededRng rng(seed);
    caches_.reserve(L);
    for (int l = 0; l < L; ++l) {
        if (capacities[l] < 0 || capacities[l] > N) fail(Status::Usage, "PolicyEngine: capacity out of [0, N]");
        caches_.emplace_back(capacities[l]);
        for (int e : rng.sample_subset(N, capacities[l])) insert(ExpertRef{l, e}, false, -1);
    }
}

void PolicyEngine::record(StreamId s, EventKind k, Tick a, Tick b, int tok, int layer, int expert, int tile) {
    ++events_;
    if (record_) timeline_.push_back(TimelineEvent{s, k, a, b, tok, layer, expert, tile});
}

void PolicyEngine::note_holders() {
    int resident = 0;
    for (const LruSet& c : caches_) resident += c.capacity();  // upper bound once warm
    max_holders_ = std::max(max_holders_, resident + static_cast<int>(live_));
}

void PolicyEngine::insert(ExpertRef ref, bool fresh, int request) {
    std::optional<int> evicted = caches_[ref.layer].insert(ref.expert, fresh);
    if (listener_) listener_->on_insert(ref, request, evicted);
}

void PolicyEngine::enqueue(ExpertRef ref, bool on_demand, Tick ready, int token) {
    int id;
    if (!free_ids_.empty()) {
        id = free_ids_.back();
        free_ids_.pop_back();
    } else {
        id = static_cast<int>(requests_.size());
        requests_.emplace_back();
    }
    Request& r = requests_[id];
    r = Request{ref, 0, on_demand, true, ready, token, {}};
    r.arrivals.reserve(cfg_.tile_count_per_expert);
    pending_[key(ref)] = id;
    (on_demand ? od_ : pf_).push_back(id);
    ++live_;
    note_holders();
    if (listener_) listener_->on_request(id, ref, on_demand);
}

void PolicyEngine::promote(ExpertRef ref) {
    const int id = pending_[key(ref)];
    if (id < 0) fail(Status::Internal, "promote: no pending request");
    Request& r = requests_[id];
    if (r.on_demand) return;
    r.on_demand = true;
    pf_.erase(std::find(pf_.begin(), pf_.end(), id));
    od_.push_back(id);
    if (listener_) listener_->on_promote(id);
}

std::optional<std::pair<int, Tick>> PolicyEngine::next_pick() const {
    Tick earliest = std::numeric_limits<Tick>::max();
    if (!od_.empty()) earliest = std::min(earliest, requests_[od_.front()].ready);
    if (!pf_.empty()) earliest = std::min(earliest, requests_[pf_.front()].ready);
    if (earliest == std::numeric_limits<Tick>::max()) return std::nullopt;
    const Tick start = std::max(cursor_, earliest);
    if (!od_.empty() && requests_[od_.front()].ready <= start) return std::make_pair(od_.front(), start);
    return std::make_pair(pf_.front(), start);
}

void PolicyEngine::start_tile(int id, Tick start) {
    const Request& r = requests_[id];
    in_flight_ = id;
    in_flight_end_ = start + cfg_.tile_transfer_time;
    record(StreamId::Comm, EventKind::TileTransfer, start, in_flight_end_, r.token, r.ref.layer, r.ref.expert, r.tiles_done);
    if (listener_) listener_->on_tile_start(id, r.tiles_done);
}

void PolicyEngine::finish_tile() {
    const int id = *in_flight_;
    Request& r = requests_[id];
    r.arrivals.push_back(in_flight_end_);
    if (++r.tiles_done == cfg_.tile_count_per_expert) {
        std::deque<int>& q = r.on_demand ? od_ : pf_;
        q.erase(std::find(q.begin(), q.end(), id));
        pending_[key(r.ref)] = -1;
        done_[key(r.ref)] = r.arrivals;
        if (!r.on_demand) {
            insert(r.ref, true, id);
            r.live = false;
            free_ids_.push_back(id);
            --live_;
        }
        // on-demand: stays live (its staging copy backs the compute) until the compute-side insert
    }
    cursor_ = in_flight_end_;
    in_flight_.reset();
}

void PolicyEngine::advance_until(Tick t) {
    for (;;) {
        if (in_flight_) {
            if (in_flight_end_ > t) return;
            finish_tile();
            continue;
        }
        auto pick = next_pick();
        if (!pick || pick->second > t) return;
        start_tile(pick->first, pick->second);
    }
}

Tick PolicyEngine::wait_for_tile(ExpertRef ref, int tile) {
    for (;;) {
        const int id = pending_[key(ref)];
        if (id >= 0) {
            if (tile < static_cast<int>(requests_[id].arrivals.size())) return requests_[id].arrivals[tile];
        } else if (tile < static_cast<int>(done_[key(ref)].size())) {
            return done_[key(ref)][tile];
        }
        if (in_flight_) {
            finish_tile();
            continue;
        }
        auto pick = next_pick();
        if (!pick) fail(Status::Internal, "wait_for_tile: tile never transfers");
        start_tile(pick->first, pick->second);
    }
}

void PolicyEngine::step(int tok, int layer, const RouteDecision& d, std::span<const RoutePrediction> predictions,
                        int single_decisions) {
    const int L = spec_.num_layers;
    if (layer == 0) token_start_ = now_;
    record(StreamId::Compute, EventKind::Attention, now_, now_ + cfg_.attention_compute_time, tok, layer, -1, -1);
    now_ += cfg_.attention_compute_time;
    record(StreamId::Compute, EventKind::Gate, now_, now_ + cfg_.gate_compute_time, tok, layer, -1, -1);
    now_ += cfg_.gate_compute_time;
    advance_until(now_);

    metrics_.single_expert_decisions += single_decisions >= 0 ? single_decisions : (d.single ? 1 : 0);
    metrics_.experts_activated_total += d.count;

    // classify the selection (inc/simulator.hpp:400-420)
    std::array<int, kMaxExperts> hit{}, miss{}, miss_req{};
    int n_hit = 0, n_miss = 0;
    LruSet& cache = caches_[layer];
    for (int i = 0; i < d.count; ++i) {
        const int e = d.experts[i];
        if (cache.contains(e)) {
            (cache.fresh(e) ? metrics_.prefetch_hits : metrics_.cache_hits) += 1;
            cache.touch(e);
            hit[n_hit++] = i;
        } else {
            metrics_.on_demand_loads += 1;
            metrics_.on_demand_loads_per_layer[layer] += 1;
            const ExpertRef ref{layer, e};
            if (pending_[key(ref)] >= 0)
                promote(ref);
            else
                enqueue(ref, true, now_, tok);
            miss_req[n_miss] = pending_[key(ref)];
            miss[n_miss++] = i;
        }
    }

    // look-ahead prefetch: nearest target first, deeper only while the nearer one is fully
    // resident; skip what is already in flight (inc/prefetch.hpp:101-119, simulator.hpp:437-443)
    if (prefetch_on_) {
        const int targets = std::min<int>(cfg_.lookahead_depth, static_cast<int>(predictions.size()));
        for (int i = 0; i < targets; ++i) {
            const RoutePrediction& p = predictions[i];
            bool any_missing = false;
            for (int k = 0; k < p.count; ++k) {
                const ExpertRef ref{p.target, p.experts[k]};
                if (caches_[ref.layer].contains(ref.expert)) continue;
                any_missing = true;
                if (pending_[key(ref)] < 0) enqueue(ref, false, now_, tok);
            }
            if (any_missing) break;
        }
    }

    for (int i = 0; i < n_hit; ++i) {
        const int e = d.experts[hit[i]];
        const Tick dur = static_cast<Tick>(cfg_.tile_count_per_expert) * cfg_.tile_compute_time;
        record(StreamId::Compute, EventKind::ExpertCompute, now_, now_ + dur, tok, layer, e, -1);
        now_ += dur;
        if (listener_) listener_->on_resident_compute(tok, ExpertRef{layer, e}, hit[i]);
    }
    for (int i = 0; i < n_miss; ++i) {
        const ExpertRef ref{layer, d.experts[miss[i]]};
        // the request may already have landed (an earlier miss advanced the channel), so use the
        // id captured at classification time
        const int req = miss_req[i];
        for (int tile = 0; tile < cfg_.tile_count_per_expert; ++tile) {
            const Tick arrival = wait_for_tile(ref, tile);
            const Tick start = std::max(now_, arrival);
            metrics_.stall_time += start - now_;
            record(StreamId::Compute, EventKind::TileCompute, start, start + cfg_.tile_compute_time, tok, layer, ref.expert, tile);
            now_ = start + cfg_.tile_compute_time;
            if (listener_) listener_->on_tile_compute(tok, ref, miss[i], tile, req);
        }
        advance_until(now_);
        insert(ref, false, req);
        if (req >= 0 && requests_[req].live) {
            requests_[req].live = false;
            free_ids_.push_back(req);
            --live_;
        }
    }
    if (listener_) listener_->on_layer_done(tok, layer, d);
    if (layer == L - 1) metrics_.latency_per_token.push_back(now_ - token_start_);
    metrics_.total_latency = now_;
}

}  // namespace adapmoe
