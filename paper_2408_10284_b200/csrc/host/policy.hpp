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

#include <algorithm>
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
// MT19937-64 with std::mt19937_64's parameters and seeding (the reference's engine,
// inc/core.hpp:182), plus a bulk fill: the twist runs over the whole 312-word state and the
// tempering over contiguous output, so long streams cost ~1 ns per word.
class Mt64 {
public:
    explicit Mt64(std::uint64_t seed) {
        mt_[0] = seed;
        for (int i = 1; i < kN; ++i) mt_[i] = 6364136223846793005ull * (mt_[i - 1] ^ (mt_[i - 1] >> 62)) + i;
        idx_ = kN;
    }
    std::uint64_t operator()() {
        if (idx_ >= kN) twist();
        return temper(mt_[idx_++]);
    }
    void fill(std::uint64_t* out, size_t n) {
        while (n) {
            if (idx_ >= kN) twist();
            const size_t take = std::min<size_t>(n, kN - idx_);
            for (size_t i = 0; i < take; ++i) out[i] = temper(mt_[idx_ + i]);
            idx_ += static_cast<int>(take);
            out += take;
            n -= take;
        }
    }

private:
    static constexpr int kN = 312, kM = 156;
    static constexpr std::uint64_t kA = 0xb5026f5aa96619e9ull, kUpper = ~0x7fffffffull, kLower = 0x7fffffffull;
    static std::uint64_t temper(std::uint64_t x) {
        x ^= (x >> 29) & 0x5555555555555555ull;
        x ^= (x << 17) & 0x71d67fffeda60000ull;
        x ^= (x << 37) & 0xfff7eee000000000ull;
        return x ^ (x >> 43);
    }
    void twist() {
        auto step = [&](int i, int j, int k) {
            const std::uint64_t y = (mt_[i] & kUpper) | (mt_[j] & kLower);
            mt_[i] = mt_[k] ^ (y >> 1) ^ ((y & 1) ? kA : 0);
        };
        int i = 0;
        for (; i < kN - kM; ++i) step(i, i + 1, i + kM);
        for (; i < kN - 1; ++i) step(i, i + 1, i + kM - kN);
        step(kN - 1, 0, kM - 1);
        idx_ = 0;
    }
    std::uint64_t mt_[kN];
    int idx_;
};

class SeededRng {
public:
    explicit SeededRng(std::uint64_t seed) : engine_(seed) {}
    std::uint64_t next_u64() { return engine_(); }
    double uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double normal();
    // The next `count` normal() values, bit-identical to `count` sequential calls (spare included):
    // the raw mt19937_64 draws stay sequential, the Box-Muller transforms (glibc log / sqrt / sin /
    // cos, the cost) run on host threads.
    void normals(double* out, size_t count);
    int uniform_int(int n);
    std::vector<int> sample_subset(int n, int t);

private:
    Mt64 engine_;
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
