// Per-GPU engine: owns the device copies of the gate matrices, the router workspace, the pinned
// host expert store and (during a decode session) the HBM slot pool, streams and copy thread.
#pragma once

#include <cuda_runtime_api.h>

#include <functional>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "../host/policy.hpp"
#include "../host/policy_engine.hpp"
#include "../kernels/router.hpp"

namespace adapmoe {

#define MOE_CUDA(expr)                                                                                          \
    do {                                                                                                        \
        cudaError_t _e = (expr);                                                                                \
        if (_e != cudaSuccess)                                                                                  \
            ::adapmoe::fail(::adapmoe::Status::Device, std::string(#expr) + ": " + cudaGetErrorString(_e));     \
    } while (0)

// Grow-only device buffer.
struct DeviceBuffer {
    void* ptr = nullptr;
    size_t bytes = 0;
    void reserve(size_t n);
    ~DeviceBuffer();
    template <typename T>
    T* as() const { return static_cast<T*>(ptr); }
};

struct PinnedBuffer {
    void* ptr = nullptr;
    size_t bytes = 0;
    void reserve(size_t n);
    ~PinnedBuffer();
    template <typename T>
    T* as() const { return static_cast<T*>(ptr); }
};

class DecodeSession;  // runtime/decode.hpp
struct ExpertStore;   // runtime/experts.hpp

// Router outputs of a whole trace, host side.  predictions rows: target, count, experts[K].
struct TraceRoutes {
    std::vector<int> selected;    // [T][L][K]
    std::vector<int> count;       // [T][L]
    std::vector<int> single;      // [T][L]
    std::vector<double> perturbation;
    std::vector<int> predictions;  // [T][L][3][2+K]
};

class Engine {
public:
    Engine(const ModelSpec& spec, int device);
    ~Engine();

    const ModelSpec& spec() const { return spec_; }
    int device() const { return device_; }
    void activate() const;

    void load_gates(const double* gates, const double* first_gate);
    bool has_gates() const { return d_gates_.ptr != nullptr && gates_loaded_; }
    bool has_first_gate() const { return first_gate_loaded_; }
    const double* d_gate(int layer) const { return d_gates_.as<double>() + static_cast<size_t>(layer) * spec_.hidden_dim * spec_.experts_per_layer; }
    const double* d_first_gate() const { return first_gate_loaded_ ? d_first_gate_.as<double>() : nullptr; }
    // fp32 transposed [N][d] copies for K1's fast path
    const float* d_gate32(int layer) const { return d_gates32_.as<float>() + static_cast<size_t>(layer) * spec_.hidden_dim * spec_.experts_per_layer; }
    const float* d_first_gate32() const { return first_gate_loaded_ ? d_first_gate32_.as<float>() : nullptr; }
    // fill a routing item that evaluates gate `layer` (-1 = first-layer predictive gate)
    void gate_item(RouteItem& it, int layer) const {
        it.gate = layer < 0 ? d_first_gate() : d_gate(layer);
        it.gate32 = layer < 0 ? d_first_gate32() : d_gate32(layer);
    }

    // K1 over a whole trace (acts/scores host).  Matches simulate_trace's evaluation points.
    TraceRoutes route_trace(const double* acts, const double* scores, int tokens, std::span<const double> fisher,
                            double tau, const SimConfig& cfg);
    // The same, pipelined: the trace is routed in chunks of `chunk_tokens` (H2D of the chunk's
    // activations, one K1 launch, D2H of its decisions), all enqueued up front; `on_chunk(t0, t1)`
    // runs on the host as soon as tokens [t0, t1) of `out` are filled, while later chunks are still
    // moving / routing on the GPU.
    void route_trace_stream(const double* acts, const double* scores, int tokens, std::span<const double> fisher,
                            double tau, const SimConfig& cfg, int chunk_tokens, TraceRoutes& out,
                            const std::function<void(int, int)>& on_chunk);

    // K1 for one layer on device rows, enqueued on `stream` (moe_router_forward).
    void router_forward(int layer, const double* d_x, int rows, const double* d_scores, double tau,
                        std::span<const double> fisher, int lookahead, bool adaptive, const RouteOutputs& out,
                        cudaStream_t stream);

    // generate_trace with the gate GEMVs on the GPU; returns via the output arrays.
    void generate_trace(const int tokens, double concentration, double drift, std::uint64_t gate_seed,
                        std::uint64_t token_seed, bool shared_gates, const double* fisher_scales,
                        const double* drift_scales, double* gates, double* acts, double* scores, int* selected,
                        double* fisher);

    void generate_profiles(const double* acts, const double* scores, int tokens, std::span<const double> fisher,
                           double tau, double* alpha, double* beta);

    // first_layer_training_pairs + train_predictive_gate (inc/workload.hpp:186-197,
    // inc/prefetch.hpp:194-213) with the logits (K1 exact path) and the gradient steps on the GPU;
    // bit-exact with the reference.  w_out [d][N] row-major.
    void train_first_gate(const double* acts, const double* scores, int tokens, double lr, int steps,
                          std::uint64_t seed, double* w_out);

    // generic: run K1 on device groups with host-visible outputs
    void run_route(const std::vector<RouteGroup>& groups, int rows, int max_gate_items, const RouteParams& p,
                   TraceRoutes* out, std::vector<double>* scores_out, cudaStream_t stream);

    cudaStream_t compute_stream() const { return compute_; }
    cudaStream_t copy_stream() const { return copy_; }

    std::unique_ptr<ExpertStore> experts;
    std::unique_ptr<DecodeSession> session;
    DeviceBuffer ffn_scratch;  // K2 partials of moe_expert_ffn_async (stream-ordered reuse)
    DeviceBuffer copy_staging; // XB12 records of moe_copy_tiles / moe_expert_ffn (stream-ordered reuse)
    int store_format = 0;      // format of the next expert store (moe_experts_set_format)

private:
    ModelSpec spec_;
    int device_;
    cudaStream_t compute_ = nullptr, copy_ = nullptr;
    DeviceBuffer d_gates_, d_first_gate_, d_gates32_, d_first_gate32_;
    bool gates_loaded_ = false, first_gate_loaded_ = false;
    // router workspace
    DeviceBuffer d_groups_, d_x_, d_scores_, d_out_sel_, d_out_cnt_, d_out_single_, d_out_pert_, d_out_scores_;
    // K1 exact-path items decided on the host (kernels/router.hpp RouteOutputs::host_entries)
    DeviceBuffer d_out_exact_, d_host_counter_;
    PinnedBuffer h_host_entries_;
    RouteOutputs host_queue(size_t max_items, cudaStream_t stream);  // outputs with the queue armed (counter zeroed on `stream`)
    PinnedBuffer h_trace_groups_, h_trace_out_;  // route_trace_stream staging
    // router_forward: groups staged in pinned memory, two buffers, each reused only after the
    // copy that read it has completed (event)
    PinnedBuffer h_fwd_groups_[2];
    DeviceBuffer d_fwd_groups_[2];
    cudaEvent_t fwd_done_[2] = {nullptr, nullptr};
    int fwd_next_ = 0;
};

}  // namespace adapmoe
