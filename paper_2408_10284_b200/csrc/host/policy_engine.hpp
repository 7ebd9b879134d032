// Logical decode engine: the expert-cache / transfer-channel state machine of the reference
// simulator (inc/simulator.hpp:64-107 LruCache, :187-320 CommEngine, :329-468 per-token loop),
// driven by router outputs produced on the GPU.  It is the single source of truth for cache
// residency, request order and the tick-model event trace; the physical executor (runtime/)
// subscribes through DecodeListener and performs the matching HBM slot moves, tile copies and
// FFN launches.  With a null listener this is the host half of simulate_trace.
#pragma once

#include <array>
#include <cstdint>
#include <deque>
#include <optional>
#include <span>
#include <vector>

#include "policy.hpp"

namespace adapmoe {

enum class StreamId : int { Compute = 0, Comm = 1 };
enum class EventKind : int { Attention = 0, Gate = 1, ExpertCompute = 2, TileCompute = 3, TileTransfer = 4 };

struct TimelineEvent {
    StreamId stream;
    EventKind kind;
    Tick start, end;
    int token, layer, expert, tile;
};

struct SimMetrics {
    std::vector<Tick> latency_per_token;
    Tick total_latency = 0;
    Tick stall_time = 0;
    long long on_demand_loads = 0;
    long long cache_hits = 0;
    long long prefetch_hits = 0;
    long long single_expert_decisions = 0;
    long long experts_activated_total = 0;
    std::vector<long long> on_demand_loads_per_layer;
};

constexpr int kMaxExperts = 64;

// Router output for one (token, layer): the actual selection ...
struct RouteDecision {
    int count = 0;
    bool single = false;
    std::array<int, kMaxExperts> experts{};
};
// ... and up to three look-ahead predictions (target layer, predicted experts).
struct RoutePrediction {
    int target = -1;
    int count = 0;
    std::array<int, kMaxExperts> experts{};
};

// Physical mirror hooks.  Request ids are stable for the life of a request.
class DecodeListener {
public:
    virtual ~DecodeListener() = default;
    virtual void on_request(int /*id*/, ExpertRef, bool /*on_demand*/) {}
    virtual void on_promote(int /*id*/) {}
    virtual void on_tile_start(int /*id*/, int /*tile*/) {}
    // cache insert of `ref`; `request` = id whose staging copy now backs it (-1 = initial fill);
    // `evicted` = expert dropped from the layer (== ref.expert when capacity is 0).
    virtual void on_insert(ExpertRef /*ref*/, int /*request*/, std::optional<int> /*evicted*/) {}
    virtual void on_resident_compute(int /*token*/, ExpertRef, int /*rank*/) {}
    virtual void on_tile_compute(int /*token*/, ExpertRef, int /*rank*/, int /*tile*/, int /*request*/) {}
    virtual void on_layer_done(int /*token*/, int /*layer*/, const RouteDecision&) {}
};

class LruSet {
public:
    explicit LruSet(int capacity = 0) : capacity_(capacity) {}
    int capacity() const { return capacity_; }
    bool contains(int e) const { return (members_ >> e) & 1ull; }
    bool fresh(int e) const { return (fresh_ >> e) & 1ull; }
    void touch(int e);
    std::optional<int> insert(int e, bool fresh);

private:
    void to_front(int e);
    int capacity_;
    std::vector<int> order_;  // order_.front() = most recently used
    std::uint64_t members_ = 0, fresh_ = 0;
};

class PolicyEngine {
public:
    PolicyEngine(const ModelSpec& spec, const SimConfig& cfg, std::span<const int> capacities, std::uint64_t seed,
                 int total_tokens, DecodeListener* listener = nullptr, bool record_timeline = true);

    // One (token, layer) of the per-token loop.  predictions: the look-ahead lists evaluated
    // from this layer's activation (empty when prefetch is off or no target exists).
    // single_decisions >= 0 overrides decision.single in the metrics (batched decode: the decision
    // is the union of B streams' selections and each stream's single-expert flag is counted).
    void step(int token, int layer, const RouteDecision& decision, std::span<const RoutePrediction> predictions,
              int single_decisions = -1);

    const SimMetrics& metrics() const { return metrics_; }
    const std::vector<TimelineEvent>& timeline() const { return timeline_; }
    long long events_recorded() const { return events_; }
    int max_slot_holders() const { return max_holders_; }
    int live_requests() const { return static_cast<int>(live_); }
    bool prefetch_on() const { return prefetch_on_; }
    bool resident(ExpertRef r) const { return caches_[r.layer].contains(r.expert); }

private:
    struct Request {
        ExpertRef ref;
        int tiles_done = 0;
        bool on_demand = false;
        bool live = false;
        Tick ready = 0;
        int token = 0;
        std::vector<Tick> arrivals;
    };
    int key(ExpertRef r) const { return r.layer * spec_.experts_per_layer + r.expert; }
    void record(StreamId s, EventKind k, Tick a, Tick b, int tok, int layer, int expert, int tile);
    void enqueue(ExpertRef ref, bool on_demand, Tick ready, int token);
    void promote(ExpertRef ref);
    std::optional<std::pair<int, Tick>> next_pick() const;
    void start_tile(int id, Tick start);
    void finish_tile();
    void advance_until(Tick t);
    Tick wait_for_tile(ExpertRef ref, int tile);
    void insert(ExpertRef ref, bool fresh, int request);
    void note_holders();

    ModelSpec spec_;
    SimConfig cfg_;
    int total_tokens_;
    DecodeListener* listener_;
    bool record_;
    bool prefetch_on_;
    std::vector<LruSet> caches_;
    // transfer channel
    std::vector<Request> requests_;
    std::vector<int> free_ids_;
    std::deque<int> od_, pf_;
    std::vector<int> pending_;              // key -> request id or -1
    std::vector<std::vector<Tick>> done_;   // key -> arrivals of the last completed request
    std::optional<int> in_flight_;
    Tick in_flight_end_ = 0;
    Tick cursor_ = 0;
    // clock + outputs
    Tick now_ = 0;
    Tick token_start_ = 0;
    SimMetrics metrics_;
    std::vector<TimelineEvent> timeline_;
    long long events_ = 0;
    std::size_t live_ = 0;
    int waiting_insert_ = 0;  // on-demand requests finished but not yet inserted
    int max_holders_ = 0;
};

}  // namespace adapmoe
