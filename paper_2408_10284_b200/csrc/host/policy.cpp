// Host policy rules; see policy.hpp for the reference mapping.  Arithmetic order mirrors the
// reference expression by expression where it affects rounding (noted inline).
#include "policy.hpp"

#include <algorithm>
#include <cmath>
#include <thread>
#include <limits>
#include <memory>
#include <numeric>

namespace adapmoe {

void ModelSpec::validate() const {
    if (num_layers < 1) fail(Status::Usage, "ModelSpec: num_layers must be >= 1");
    if (experts_per_layer < 2 || experts_per_layer > 64) fail(Status::Usage, "ModelSpec: experts_per_layer must be in [2, 64]");
    if (top_k < 1 || top_k > experts_per_layer) fail(Status::Usage, "ModelSpec: top_k must be in [1, experts_per_layer]");
    if (hidden_dim < 1) fail(Status::Usage, "ModelSpec: hidden_dim must be >= 1");
}

void LayerProfile::validate() const {
    if (!(single_expert_prob >= 0.0 && single_expert_prob <= 1.0)) fail(Status::Usage, "LayerProfile: alpha out of [0,1]");
    if (!(prefetch_accuracy >= 0.0 && prefetch_accuracy <= 1.0)) fail(Status::Usage, "LayerProfile: beta out of [0,1]");
    if (!(fisher_diag_sum >= 0.0)) fail(Status::Usage, "LayerProfile: fisher must be >= 0");
}

void Allocation::validate(const ModelSpec& spec) const {
    if (static_cast<int>(capacities.size()) != spec.num_layers) fail(Status::Usage, "Allocation: capacity count != num_layers");
    long long sum = 0;
    for (int t : capacities) {
        if (t < 0 || t > spec.experts_per_layer) fail(Status::Usage, "Allocation: capacity out of [0, N]");
        sum += t;
    }
    if (sum > budget) fail(Status::Usage, "Allocation: capacities exceed budget");
}

void SimConfig::validate() const {
    if (tile_count_per_expert < 1) fail(Status::Usage, "SimConfig: tile_count_per_expert must be >= 1");
    if (tile_transfer_time < 0 || tile_compute_time < 0 || attention_compute_time < 0 || gate_compute_time < 0)
        fail(Status::Usage, "SimConfig: durations must be >= 0");
    if (lookahead_depth < 0 || lookahead_depth > 3) fail(Status::Usage, "SimConfig: lookahead_depth out of {0,1,2,3}");
}

// Box-Muller with a cached second deviate (inc/core.hpp:130-144).  The expression shapes
// (-2*log(u1), 2pi*u2, r*sin, r*cos) are kept so the doubles match the reference draw for draw.
double SeededRng::normal() {
    if (has_cached_) {
        has_cached_ = false;
        return cached_;
    }
    constexpr double kTwoPi = 6.283185307179586476925286766559;
    double u1 = uniform01();
    const double u2 = uniform01();
    while (u1 <= 0.0) u1 = uniform01();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = kTwoPi * u2;
    cached_ = radius * std::sin(angle);
    has_cached_ = true;
    return radius * std::cos(angle);
}

void SeededRng::normals(double* out, size_t count) {
    size_t i = 0;
    if (count > 0 && has_cached_) {
        has_cached_ = false;
        out[i++] = cached_;
    }
    const size_t pairs = (count - i + 1) / 2;
    if (pairs == 0) return;
    constexpr double kTwoPi = 6.283185307179586476925286766559;
    double spare = 0.0;
    // pair p -> normals i + 2p (cos) and i + 2p + 1 (sin; the cached spare past the end)
    auto emit = [&](size_t p, std::uint64_t w1, std::uint64_t w2) {
        const double u1 = static_cast<double>(w1 >> 11) * 0x1.0p-53;
        const double u2 = static_cast<double>(w2 >> 11) * 0x1.0p-53;
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = kTwoPi * u2;
        out[i + 2 * p] = radius * std::cos(angle);
        if (i + 2 * p + 1 < count)
            out[i + 2 * p + 1] = radius * std::sin(angle);
        else
            spare = radius * std::sin(angle);
    };
    // Raw words in normal()'s draw order (u1, u2 per pair) are drawn sequentially into one of two
    // chunk buffers while host threads transform the other.  A u1 of exactly 0 (probability 2^-53
    // per pair) is redrawn after u2 and shifts the stream: from such a chunk on, the pairs replay
    // sequentially from the buffered words, then the engine.
    constexpr size_t kChunk = size_t{1} << 19;  // pairs per chunk
    const size_t hw = std::max(1u, std::thread::hardware_concurrency());
    std::unique_ptr<std::uint64_t[]> buf[2] = {std::unique_ptr<std::uint64_t[]>(new std::uint64_t[2 * std::min(kChunk, pairs)]),
                                               std::unique_ptr<std::uint64_t[]>(new std::uint64_t[2 * std::min(kChunk, pairs)])};
    size_t done = 0;
    int cur = 0;
    engine_.fill(buf[0].get(), 2 * std::min(kChunk, pairs));
    while (done < pairs) {
        const size_t n = std::min(kChunk, pairs - done);
        const std::uint64_t* w = buf[cur].get();
        bool redraw = false;
        for (size_t p = 0; p < n && !redraw; ++p) redraw = (w[2 * p] >> 11) == 0;
        if (redraw) {
            size_t c = 0;
            auto next = [&]() { return c < 2 * n ? w[c++] : engine_(); };
            for (size_t p = done; p < pairs; ++p) {
                std::uint64_t a = next();
                const std::uint64_t b = next();
                while ((a >> 11) == 0) a = next();
                emit(p, a, b);
            }
            done = pairs;
            break;
        }
        auto transform = [&, w, done](size_t p0, size_t p1) {
            for (size_t p = p0; p < p1; ++p) emit(done + p, w[2 * p], w[2 * p + 1]);
        };
        const size_t n_threads = std::min<size_t>(std::min<size_t>(hw, 16), n / 16384 + 1);
        std::vector<std::thread> pool;
        for (size_t t = 1; t < n_threads; ++t) pool.emplace_back(transform, n * t / n_threads, n * (t + 1) / n_threads);
        const size_t next_n = std::min(kChunk, pairs - done - n);
        if (next_n) engine_.fill(buf[cur ^ 1].get(), 2 * next_n);  // overlaps the workers
        transform(0, n / n_threads);
        for (auto& th : pool) th.join();
        done += n;
        cur ^= 1;
    }
    if ((count - i) % 2 != 0) {
        cached_ = spare;
        has_cached_ = true;
    }
}

int SeededRng::uniform_int(int n) {
    if (n <= 0) fail(Status::Usage, "SeededRng::uniform_int: n must be positive");
    const std::uint64_t span = static_cast<std::uint64_t>(n);
    const std::uint64_t accept_below = (std::numeric_limits<std::uint64_t>::max() / span) * span;
    std::uint64_t draw;
    do draw = next_u64();
    while (draw >= accept_below);
    return static_cast<int>(draw % span);
}

std::vector<int> SeededRng::sample_subset(int n, int t) {
    if (t < 0 || t > n) fail(Status::Usage, "SeededRng::sample_subset: t out of [0, n]");
    std::vector<int> ids(n);
    std::iota(ids.begin(), ids.end(), 0);
    for (int i = 0; i < t; ++i) std::swap(ids[i], ids[i + uniform_int(n - i)]);
    ids.resize(t);
    return ids;
}

std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

std::vector<int> top_k_indices(std::span<const double> scores, int k) {
    const int n = static_cast<int>(scores.size());
    if (k < 0 || k > n) fail(Status::Usage, "top_k_indices: k out of [0, n]");
    std::vector<int> rank(n);
    std::iota(rank.begin(), rank.end(), 0);
    // Deterministic total order: score desc, then index asc.
    std::partial_sort(rank.begin(), rank.begin() + k, rank.end(), [&](int a, int b) {
        return scores[a] > scores[b] || (scores[a] == scores[b] && a < b);
    });
    rank.resize(k);
    return rank;
}

std::vector<double> softmax(std::span<const double> logits) {
    if (logits.empty()) fail(Status::Usage, "softmax: empty input");
    const double peak = *std::max_element(logits.begin(), logits.end());
    std::vector<double> p(logits.size());
    double total = 0.0;  // sequential, index order (inc/core.hpp:210-213)
    for (std::size_t i = 0; i < logits.size(); ++i) total += (p[i] = std::exp(logits[i] - peak));
    for (double& v : p) v /= total;
    return p;
}

double normalized_top1_share(std::span<const double> scores) {
    if (scores.size() < 2) fail(Status::Usage, "normalized_top1_share: needs at least 2 experts");
    double first = -1.0, second = -1.0;
    for (double s : scores) {
        if (s > first) {
            second = first;
            first = s;
        } else if (s > second) {
            second = s;
        }
    }
    const double denom = first + second;
    if (denom <= 0.0) fail(Status::Usage, "normalized_top1_share: all-zero scores");
    return first / denom;
}

double sensitivity_perturbation(double alpha, double fisher) {
    if (!(alpha >= 0.0 && alpha <= 1.0)) fail(Status::Usage, "sensitivity_perturbation: alpha out of [0,1]");
    if (!(fisher >= 0.0)) fail(Status::Usage, "sensitivity_perturbation: fisher must be >= 0");
    const double gap = 1.0 - alpha;
    return gap * gap * fisher;  // (gap*gap)*F, no contraction
}

GatingDecision gate_decide_sensitivity(std::span<const double> scores, double fisher, double tau, int top_k) {
    if (!(tau >= 0.0)) fail(Status::Usage, "GatingThreshold: tau must be >= 0");
    GatingDecision d;
    d.perturbation = sensitivity_perturbation(normalized_top1_share(scores), fisher);
    d.single = d.perturbation <= tau;  // inclusive boundary (inc/gating.hpp:62)
    d.selected = top_k_indices(scores, d.single ? 1 : top_k);
    return d;
}

double calibrate_threshold(std::span<const double> scores, int tokens, const ModelSpec& spec,
                           std::span<const double> fisher, double target, double* realized) {
    spec.validate();
    if (tokens < 1) fail(Status::Usage, "calibrate_threshold: empty trace set");
    if (!(target >= 0.0 && target <= 1.0)) fail(Status::Usage, "calibrate_threshold: target ratio out of [0,1]");
    const int L = spec.num_layers, N = spec.experts_per_layer;
    if (static_cast<int>(fisher.size()) != L) fail(Status::Usage, "calibrate_threshold: fisher vector does not match layers");
    if (scores.size() != static_cast<std::size_t>(tokens) * L * N) fail(Status::Usage, "calibrate_threshold: score array size");
    std::vector<double> observed;
    observed.reserve(static_cast<std::size_t>(tokens) * L);
    for (int t = 0; t < tokens; ++t)
        for (int l = 0; l < L; ++l)
            observed.push_back(sensitivity_perturbation(
                normalized_top1_share(scores.subspan((static_cast<std::size_t>(t) * L + l) * N, N)), fisher[l]));
    std::sort(observed.begin(), observed.end());
    const double m = static_cast<double>(observed.size());
    // fraction of observations <= tau (the realized single ratio at tau)
    auto ratio = [&](double tau) {
        return static_cast<double>(std::upper_bound(observed.begin(), observed.end(), tau) - observed.begin()) / m;
    };
    double tau = 0.0;
    if (ratio(0.0) < target) {
        // first sorted index whose value reaches the target (monotone predicate)
        std::size_t lo = 0, hi = observed.size() - 1;
        while (lo < hi) {
            const std::size_t mid = lo + (hi - lo) / 2;
            if (ratio(observed[mid]) >= target)
                hi = mid;
            else
                lo = mid + 1;
        }
        tau = observed[lo];
    }
    if (realized) *realized = ratio(tau);
    return tau;
}

double expected_cost(int t, int n, double alpha, double beta) {
    if (n < 2) fail(Status::Usage, "cache model: N must be >= 2");
    if (t < 0 || t > n) fail(Status::Usage, "cache model: t out of [0, N]");
    if (!(alpha >= 0.0 && alpha <= 1.0) || !(beta >= 0.0 && beta <= 1.0)) fail(Status::Usage, "cache model: probability out of [0,1]");
    const double dn = n, dt = t;
    const double miss_one = (1.0 - dt / dn) * (1.0 - beta);                    // Eq. 11
    const double both_miss = std::max((dn - dt) * (dn - dt - 1.0) / (dn * (dn - 1.0)), 0.0);
    const double one_hit = 2.0 * (dn - dt) * dt / (dn * (dn - 1.0));
    // Eq. 12-14 summed in the reference's member order
    const double miss_two = 2.0 * both_miss * (1.0 - beta) + both_miss * beta + one_hit * (1.0 - beta);
    return alpha * miss_one + (1.0 - alpha) * miss_two;                       // Eq. 15
}

std::vector<double> build_cost_table(std::span<const double> alpha, std::span<const double> beta, const ModelSpec& spec) {
    spec.validate();
    const int L = spec.num_layers, N = spec.experts_per_layer;
    if (static_cast<int>(alpha.size()) != L || static_cast<int>(beta.size()) != L)
        fail(Status::Usage, "build_cost_table: profile count does not match num_layers");
    std::vector<double> table(static_cast<std::size_t>(L) * (N + 1));
    for (int l = 0; l < L; ++l)
        for (int t = 0; t <= N; ++t) table[static_cast<std::size_t>(l) * (N + 1) + t] = expected_cost(t, N, alpha[l], beta[l]);
    return table;
}

AllocationResult dp_allocate(std::span<const double> table, int budget, const ModelSpec& spec) {
    spec.validate();
    const int L = spec.num_layers, N = spec.experts_per_layer;
    if (table.size() != static_cast<std::size_t>(L) * (N + 1)) fail(Status::Usage, "dp_allocate: cost table does not match model spec");
    if (budget < 0) fail(Status::Infeasible, "dp_allocate: negative budget");
    const int width = static_cast<int>(std::min<long long>(budget, static_cast<long long>(L) * N));
    // best[l][j]: least expected loads over layers < l with <= j slots; pick[l][j]: argmin size
    // for layer l-1 (smallest size wins ties: strict <).
    std::vector<double> best(static_cast<std::size_t>(L + 1) * (width + 1), 0.0);
    std::vector<int> pick(best.size(), 0);
    auto at = [&](int l, int j) { return static_cast<std::size_t>(l) * (width + 1) + j; };
    for (int l = 1; l <= L; ++l) {
        const double* row = table.data() + static_cast<std::size_t>(l - 1) * (N + 1);
        for (int j = 0; j <= width; ++j) {
            double v = std::numeric_limits<double>::infinity();
            int arg = 0;
            for (int k = 0, kmax = std::min(j, N); k <= kmax; ++k) {
                const double c = best[at(l - 1, j - k)] + row[k];
                if (c < v) {
                    v = c;
                    arg = k;
                }
            }
            best[at(l, j)] = v;
            pick[at(l, j)] = arg;
        }
    }
    AllocationResult r;
    r.allocation.budget = budget;
    r.allocation.capacities.assign(L, 0);
    for (int l = L, j = width; l >= 1; --l) {
        r.allocation.capacities[l - 1] = pick[at(l, j)];
        j -= pick[at(l, j)];
    }
    r.total_cost = best[at(L, width)];
    return r;
}

Allocation uniform_allocation(int budget, const ModelSpec& spec) {
    spec.validate();
    if (budget < 0) fail(Status::Infeasible, "uniform_allocation: negative budget");
    Allocation a;
    a.budget = budget;
    a.capacities.resize(spec.num_layers);
    for (int l = 0; l < spec.num_layers; ++l)
        a.capacities[l] = std::min(budget / spec.num_layers + (l < budget % spec.num_layers ? 1 : 0), spec.experts_per_layer);
    return a;
}

Tick tile_pipeline_latency(int tiles, Tick transfer, Tick compute) {
    if (tiles < 1) fail(Status::Usage, "tile_pipeline_latency: tile_count must be >= 1");
    if (transfer < 0 || compute < 0) fail(Status::Usage, "tile_pipeline_latency: negative duration");
    return transfer >= compute ? static_cast<Tick>(tiles) * transfer + compute : transfer + static_cast<Tick>(tiles) * compute;
}

}  // namespace adapmoe
