// Host-side policy layer of the B200 AdapMoE decode path: the value types and the
// offline/online decision rules of the reference moesim API (names kept so C++ callers can
// switch namespaces), re-expressed for this engine.  `inc/` = /root/reference/proj/include/moesim.
//
// What lives here (all host C++, deterministic, bit-exact with the reference):
//   * ModelSpec / LayerProfile / Allocation / GatingThreshold / SimConfig  (inc/core.hpp:22-113,
//     inc/gating.hpp:11-17, inc/simulator.hpp:26-50)
//   * SeededRng: std::mt19937_64 stream + the reference's hand-rolled distributions
//     (inc/core.hpp:118-188) — needed so synthetic inputs are the reference's inputs.
//   * gating: top1 share, perturbation, sensitivity decision, tau calibration (inc/gating.hpp)
//   * cost model + knapsack DP + uniform split (inc/cache_model.hpp:28-74,189-204,
//     inc/allocator.hpp:36-88,140-153)
//   * prefetch planning (inc/prefetch.hpp:101-119)
// The per-token router math (logits/softmax/adaptive top-k/pre-gate) runs on the GPU (router.cu);
// the host versions of those rules below are used by the offline tools and the replay engine.
#pragma once

#include <cstdint>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace adapmoe {

// Error classes map 1:1 onto the C ABI status codes (include/adapmoe.h).
enum class Status : int { Ok = 0, Usage = 1, Io = 2, Format = 3, Validation = 4, Infeasible = 5, Device = 6, Internal = 7 };

struct Error : std::runtime_error {
    Status status;
    Error(Status s, const std::string& what) : std::runtime_error(what), status(s) {}
};

[[noreturn]] inline void fail(Status s, const std::string& what) { throw Error(s, what); }

struct ModelSpec {
    int num_layers = 1;
    int experts_per_layer = 8;
    int top_k = 2;
    int hidden_dim = 1;

    void validate() const;
    bool operator==(const ModelSpec&) const = default;
};

struct ExpertRef {
    int layer = 0;
    int expert = 0;
    bool operator==(const ExpertRef&) const = default;
};

struct LayerProfile {
    double single_expert_prob = 0.0;  // alpha_l
    double prefetch_accuracy = 0.0;   // beta_l
    double fisher_diag_sum = 0.0;     // F_l
    void validate() const;
};

struct Allocation {
    std::vector<int> capacities;
    int budget = 0;
    void validate(const ModelSpec& spec) const;
};

struct GatingThreshold {
    double tau = 0.0;
    void validate() const {
        if (!(tau >= 0.0)) fail(Status::Usage, "GatingThreshold: tau must be >= 0");
    }
};

using Tick = std::int64_t;

struct PolicyFlags {
    bool adaptive_gating = false;
    bool prefetch = false;
    bool adaptive_cache = false;
};

struct SimConfig {
    int tile_count_per_expert = 4;
    Tick tile_transfer_time = 1;
    Tick tile_compute_time = 1;
    Tick attention_compute_time = 1;
    Tick gate_compute_time = 1;
    int lookahead_depth = 2;
    PolicyFlags policy;
    void validate() const;
};

// ---- deterministic random source -----------------------------------------------------------
class SeededRng {
public:
    explicit SeededRng(std::uint64_t seed) : engine_(seed) {}
    std::uint64_t next_u64() { return engine_(); }
    double uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double normal();
    int uniform_int(int n);
    std::vector<int> sample_subset(int n, int t);

private:
    std::mt19937_64 engine_;
    double cached_ = 0.0;
    bool has_cached_ = false;
};

std::uint64_t splitmix64(std::uint64_t x);

// ---- routing rules ---------------------------------------------------------------------------
// Ranking by score descending with the lowest expert index winning ties (inc/core.hpp:192-203).
std::vector<int> top_k_indices(std::span<const double> scores, int k);
std::vector<double> softmax(std::span<const double> logits);
double normalized_top1_share(std::span<const double> scores);
double sensitivity_perturbation(double alpha, double fisher_diag_sum);

struct GatingDecision {
    std::vector<int> selected;
    double perturbation = 0.0;
    bool single = false;
};
GatingDecision gate_decide_sensitivity(std::span<const double> scores, double fisher_diag_sum, double tau, int top_k);

// Smallest observed perturbation whose single-expert ratio reaches the target.
// scores is [T][L][N]; fisher is [L].
double calibrate_threshold(std::span<const double> scores, int tokens, const ModelSpec& spec,
                           std::span<const double> fisher, double target_single_ratio, double* realized = nullptr);

// ---- cache sizing ----------------------------------------------------------------------------
double expected_cost(int t, int n, double alpha, double beta);
// [L][N+1] row-major
std::vector<double> build_cost_table(std::span<const double> alpha, std::span<const double> beta, const ModelSpec& spec);
struct AllocationResult {
    Allocation allocation;
    double total_cost = 0.0;
};
AllocationResult dp_allocate(std::span<const double> table, int budget, const ModelSpec& spec);
Allocation uniform_allocation(int budget, const ModelSpec& spec);
Tick tile_pipeline_latency(int tile_count, Tick transfer, Tick compute);

}  // namespace adapmoe
