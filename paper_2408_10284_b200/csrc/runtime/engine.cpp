// Engine: device-resident gates + K1 router drivers (trace routing, synthetic workload
// generation, offline alpha/beta profiling).  inc/ = /root/reference/proj/include/moesim.
#include "engine.hpp"

#include "../kernels/trainer.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <thread>

#include "decode.hpp"
#include "experts.hpp"

namespace adapmoe {

void DeviceBuffer::reserve(size_t n) {
    if (n <= bytes) return;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    MOE_CUDA(cudaMalloc(&ptr, n));
    bytes = n;
}
DeviceBuffer::~DeviceBuffer() {
    if (ptr) cudaFree(ptr);
}
void PinnedBuffer::reserve(size_t n) {
    if (n <= bytes) return;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
    MOE_CUDA(cudaMallocHost(&ptr, n));
    bytes = n;
}
PinnedBuffer::~PinnedBuffer() {
    if (ptr) cudaFreeHost(ptr);
}

Engine::Engine(const ModelSpec& spec, int device) : spec_(spec), device_(device) {
    spec_.validate();
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) fail(Status::Device, "no CUDA device available");
    if (device < 0 || device >= count) fail(Status::Device, "device index out of range");
    MOE_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    MOE_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) fail(Status::Device, std::string("built for sm_100a (B200); found ") + prop.name);
    // the compute stream (router, FFN, combine) outranks background work (the XB12 decode stream)
    // when both want SMs
    int least = 0, greatest = 0;
    MOE_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    MOE_CUDA(cudaStreamCreateWithPriority(&compute_, cudaStreamNonBlocking, greatest));
    MOE_CUDA(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
}

Engine::~Engine() {
    cudaSetDevice(device_);
    session.reset();
    experts.reset();
    for (cudaEvent_t ev : fwd_done_)
        if (ev) cudaEventDestroy(ev);
    if (compute_) cudaStreamDestroy(compute_);
    if (copy_) cudaStreamDestroy(copy_);
}

void Engine::activate() const { MOE_CUDA(cudaSetDevice(device_)); }

void Engine::load_gates(const double* gates, const double* first_gate) {
    activate();
    const size_t one = static_cast<size_t>(spec_.hidden_dim) * spec_.experts_per_layer * sizeof(double);
    d_gates_.reserve(one * spec_.num_layers);
    // stream-ordered with the transposes below: a plain cudaMemcpy from pageable memory may return
    // before its DMA lands, and compute_ does not synchronise with the legacy default stream
    MOE_CUDA(cudaMemcpyAsync(d_gates_.ptr, gates, one * spec_.num_layers, cudaMemcpyHostToDevice, compute_));
    d_gates32_.reserve(one / 2 * spec_.num_layers);
    MOE_CUDA(launch_gate_transpose(d_gates_.as<double>(), d_gates32_.as<float>(), spec_.hidden_dim,
                                   spec_.experts_per_layer, spec_.num_layers, compute_));
    gates_loaded_ = true;
    first_gate_loaded_ = false;
    if (first_gate) {
        d_first_gate_.reserve(one);
        d_first_gate32_.reserve(one / 2);
        MOE_CUDA(cudaMemcpyAsync(d_first_gate_.ptr, first_gate, one, cudaMemcpyHostToDevice, compute_));
        MOE_CUDA(launch_gate_transpose(d_first_gate_.as<double>(), d_first_gate32_.as<float>(), spec_.hidden_dim,
                                       spec_.experts_per_layer, 1, compute_));
        first_gate_loaded_ = true;
    }
    MOE_CUDA(cudaStreamSynchronize(compute_));
}

RouteOutputs Engine::host_queue(size_t max_items, cudaStream_t stream) {
    RouteOutputs o;
    const int cap = static_cast<int>(std::min<size_t>(std::max<size_t>(max_items, 1), 65536));
    h_host_entries_.reserve(static_cast<size_t>(cap) * (2 + spec_.experts_per_layer) * sizeof(double));
    d_host_counter_.reserve(sizeof(unsigned));
    MOE_CUDA(cudaMemsetAsync(d_host_counter_.ptr, 0, sizeof(unsigned), stream));
    o.host_entries = h_host_entries_.as<double>();
    o.host_counter = d_host_counter_.as<unsigned>();
    o.host_cap = cap;
    return o;
}

void Engine::run_route(const std::vector<RouteGroup>& groups, int rows, int max_gate_items, const RouteParams& p,
                       TraceRoutes* out, std::vector<double>* scores_out, cudaStream_t stream) {
    const int K = p.k, N = p.n;
    d_groups_.reserve(groups.size() * sizeof(RouteGroup));
    d_out_sel_.reserve(static_cast<size_t>(rows) * K * sizeof(int));
    d_out_cnt_.reserve(static_cast<size_t>(rows) * sizeof(int));
    d_out_single_.reserve(static_cast<size_t>(rows) * sizeof(int));
    d_out_pert_.reserve(static_cast<size_t>(rows) * sizeof(double));
    if (scores_out) d_out_scores_.reserve(static_cast<size_t>(rows) * N * sizeof(double));
    d_out_exact_.reserve(static_cast<size_t>(rows) * sizeof(int));
    MOE_CUDA(cudaMemcpyAsync(d_groups_.ptr, groups.data(), groups.size() * sizeof(RouteGroup), cudaMemcpyHostToDevice, stream));
    RouteOutputs o = host_queue(static_cast<size_t>(rows), stream);
    o.selected = d_out_sel_.as<int>();
    o.count = d_out_cnt_.as<int>();
    o.single = d_out_single_.as<int>();
    o.perturbation = d_out_pert_.as<double>();
    o.scores = scores_out ? d_out_scores_.as<double>() : nullptr;
    o.exact_used = d_out_exact_.as<int>();
    MOE_CUDA(cudaMemsetAsync(o.exact_used, 0, static_cast<size_t>(rows) * sizeof(int), stream));
    MOE_CUDA(launch_route(d_groups_.as<RouteGroup>(), static_cast<int>(groups.size()), max_gate_items, p, o, stream));
    out->selected.resize(static_cast<size_t>(rows) * K);
    out->count.resize(rows);
    out->single.resize(rows);
    out->perturbation.resize(rows);
    MOE_CUDA(cudaMemcpyAsync(out->selected.data(), o.selected, out->selected.size() * sizeof(int), cudaMemcpyDeviceToHost, stream));
    MOE_CUDA(cudaMemcpyAsync(out->count.data(), o.count, rows * sizeof(int), cudaMemcpyDeviceToHost, stream));
    MOE_CUDA(cudaMemcpyAsync(out->single.data(), o.single, rows * sizeof(int), cudaMemcpyDeviceToHost, stream));
    MOE_CUDA(cudaMemcpyAsync(out->perturbation.data(), o.perturbation, rows * sizeof(double), cudaMemcpyDeviceToHost, stream));
    if (scores_out) {
        scores_out->resize(static_cast<size_t>(rows) * N);
        MOE_CUDA(cudaMemcpyAsync(scores_out->data(), o.scores, scores_out->size() * sizeof(double), cudaMemcpyDeviceToHost, stream));
    }
    std::vector<int> exact(rows);
    MOE_CUDA(cudaMemcpyAsync(exact.data(), o.exact_used, rows * sizeof(int), cudaMemcpyDeviceToHost, stream));
    MOE_CUDA(cudaStreamSynchronize(stream));
    route_host_decide(p, o.host_entries, exact.data(), 0, rows, out->selected.data(), out->count.data(),
                      out->single.data(), out->perturbation.data());
}

// Evaluation points of simulate_trace (inc/simulator.hpp:390-396 decision, :422-436 look-ahead).
TraceRoutes Engine::route_trace(const double* acts, const double* scores, int T, std::span<const double> fisher,
                                double tau, const SimConfig& cfg) {
    TraceRoutes r;
    route_trace_stream(acts, scores, T, fisher, tau, cfg, T, r, [](int, int) {});
    return r;
}

void Engine::route_trace_stream(const double* acts, const double* scores, int T, std::span<const double> fisher,
                                double tau, const SimConfig& cfg, int chunk_tokens, TraceRoutes& r,
                                const std::function<void(int, int)>& on_chunk) {
    activate();
    cfg.validate();
    const int L = spec_.num_layers, N = spec_.experts_per_layer, K = spec_.top_k, D = spec_.hidden_dim;
    if (static_cast<int>(fisher.size()) != L) fail(Status::Usage, "route_trace: fisher count != num_layers");
    const bool prefetch_on = cfg.policy.prefetch && cfg.lookahead_depth > 0;
    if (prefetch_on && !has_gates()) fail(Status::Usage, "simulate_trace: prefetching requires one gate matrix per layer");
    const size_t TL = static_cast<size_t>(T) * L, rows = TL * 4;
    d_x_.reserve(TL * D * sizeof(double));
    d_scores_.reserve(TL * N * sizeof(double));
    d_groups_.reserve(TL * sizeof(RouteGroup));
    d_out_sel_.reserve(rows * K * sizeof(int));
    d_out_cnt_.reserve(rows * sizeof(int));
    d_out_single_.reserve(rows * sizeof(int));
    d_out_pert_.reserve(rows * sizeof(double));
    h_trace_groups_.reserve(TL * sizeof(RouteGroup));
    h_trace_out_.reserve(rows * ((K + 3) * sizeof(int) + sizeof(double)));
    d_out_exact_.reserve(rows * sizeof(int));

    // group (tok, l) writes rows tl*4 + item: decision, then look-ahead depth 1..k (or the first-layer
    // predictive gate at the last layer)
    RouteGroup* groups = h_trace_groups_.as<RouteGroup>();
    int max_gates = 0;
    for (int tok = 0; tok < T; ++tok)
        for (int l = 0; l < L; ++l) {
            const size_t tl = static_cast<size_t>(tok) * L + l;
            RouteGroup& g = groups[tl];
            g = RouteGroup{};
            g.x = d_x_.as<double>() + tl * D;
            RouteItem& dec = g.items[g.n_items++];
            dec.gate = nullptr;
            dec.scores = d_scores_.as<double>() + tl * N;
            dec.fisher = fisher[l];
            dec.flags = cfg.policy.adaptive_gating ? kRouteAdaptive : 0;
            dec.out = static_cast<int>(tl * 4);
            int n_gates = 0;
            if (prefetch_on) {
                const int adaptive = cfg.policy.adaptive_gating ? kRouteAdaptive : 0;
                if (l + 1 < L) {
                    for (int depth = 1; depth <= cfg.lookahead_depth && l + depth < L; ++depth) {
                        RouteItem& it = g.items[g.n_items++];
                        gate_item(it, l + depth);
                        it.fisher = fisher[l + depth];
                        it.flags = adaptive;
                        it.out = static_cast<int>(tl * 4 + depth);
                        ++n_gates;
                    }
                } else if (has_first_gate() && tok + 1 < T) {
                    RouteItem& it = g.items[g.n_items++];
                    gate_item(it, -1);
                    it.fisher = fisher[0];
                    it.flags = adaptive;
                    it.out = static_cast<int>(tl * 4 + 1);
                    ++n_gates;
                }
            }
            max_gates = std::max(max_gates, n_gates);
        }
    MOE_CUDA(cudaMemcpyAsync(d_groups_.ptr, groups, TL * sizeof(RouteGroup), cudaMemcpyHostToDevice, compute_));
    int* h_sel = h_trace_out_.as<int>();
    int* h_cnt = h_sel + rows * K;
    int* h_sgl = h_cnt + rows;
    double* h_pert = reinterpret_cast<double*>(h_sgl + rows);
    int* h_exact = reinterpret_cast<int*>(h_pert + rows);
    RouteParams p{D, N, K, tau, 1.0};
    RouteOutputs o = host_queue(TL * (prefetch_on ? 3 : 0), compute_);
    o.selected = d_out_sel_.as<int>();
    o.count = d_out_cnt_.as<int>();
    o.single = d_out_single_.as<int>();
    o.perturbation = d_out_pert_.as<double>();
    o.exact_used = d_out_exact_.as<int>();
    MOE_CUDA(cudaMemsetAsync(o.exact_used, 0, rows * sizeof(int), compute_));
    const int chunk = std::max(1, std::min(chunk_tokens, T));
    const int n_chunks = (T + chunk - 1) / chunk;
    std::vector<cudaEvent_t> done(n_chunks);
    for (auto& e : done) MOE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct EventGuard {
        std::vector<cudaEvent_t>& v;
        ~EventGuard() {
            for (cudaEvent_t e : v) cudaEventDestroy(e);
        }
    } guard{done};
    // enqueue every chunk: inputs -> K1 -> decisions back, one completion event per chunk
    for (int c = 0; c < n_chunks; ++c) {
        const size_t t0 = static_cast<size_t>(c) * chunk, t1 = std::min<size_t>(T, t0 + chunk);
        const size_t r0 = t0 * L, nr = (t1 - t0) * L;
        MOE_CUDA(cudaMemcpyAsync(d_x_.as<double>() + r0 * D, acts + r0 * D, nr * D * sizeof(double),
                                 cudaMemcpyHostToDevice, compute_));
        MOE_CUDA(cudaMemcpyAsync(d_scores_.as<double>() + r0 * N, scores + r0 * N, nr * N * sizeof(double),
                                 cudaMemcpyHostToDevice, compute_));
        MOE_CUDA(launch_route(d_groups_.as<RouteGroup>() + r0, static_cast<int>(nr), std::max(max_gates, 1), p, o, compute_));
        const size_t q0 = r0 * 4, nq = nr * 4;
        MOE_CUDA(cudaMemcpyAsync(h_sel + q0 * K, o.selected + q0 * K, nq * K * sizeof(int), cudaMemcpyDeviceToHost, compute_));
        MOE_CUDA(cudaMemcpyAsync(h_cnt + q0, o.count + q0, nq * sizeof(int), cudaMemcpyDeviceToHost, compute_));
        MOE_CUDA(cudaMemcpyAsync(h_sgl + q0, o.single + q0, nq * sizeof(int), cudaMemcpyDeviceToHost, compute_));
        MOE_CUDA(cudaMemcpyAsync(h_pert + q0, o.perturbation + q0, nq * sizeof(double), cudaMemcpyDeviceToHost, compute_));
        MOE_CUDA(cudaMemcpyAsync(h_exact + q0, o.exact_used + q0, nq * sizeof(int), cudaMemcpyDeviceToHost, compute_));
        MOE_CUDA(cudaEventRecord(done[c], compute_));
    }
    r.selected.resize(TL * K);
    r.count.resize(TL);
    r.single.resize(TL);
    r.perturbation.resize(TL);
    const int PW = 2 + K;
    r.predictions.assign(TL * 3 * PW, -1);
    for (int c = 0; c < n_chunks; ++c) {
        const int t0 = c * chunk, t1 = std::min(T, t0 + chunk);
        MOE_CUDA(cudaEventSynchronize(done[c]));
        // the chunk's uncertified items: the reference's softmax (libm exp) on their exact logits
        route_host_decide(p, o.host_entries, h_exact, static_cast<long long>(t0) * L * 4,
                          static_cast<long long>(t1) * L * 4, h_sel, h_cnt, h_sgl, h_pert);
        for (size_t tl = static_cast<size_t>(t0) * L; tl < static_cast<size_t>(t1) * L; ++tl) {
            const size_t row = tl * 4;
            for (int k = 0; k < K; ++k) r.selected[tl * K + k] = h_sel[row * K + k];
            r.count[tl] = h_cnt[row];
            r.single[tl] = h_sgl[row];
            r.perturbation[tl] = h_pert[row];
            const RouteGroup& g = groups[tl];
            for (int s = 0; s < 3; ++s) {
                int* dst = &r.predictions[(tl * 3 + s) * PW];
                dst[1] = 0;
                if (s + 1 < g.n_items) {
                    const size_t prow = static_cast<size_t>(g.items[s + 1].out);
                    const int layer = static_cast<int>(tl % L);
                    dst[0] = (g.items[s + 1].gate == d_first_gate() && layer == L - 1) ? 0 : layer + s + 1;
                    dst[1] = h_cnt[prow];
                    for (int k = 0; k < K; ++k) dst[2 + k] = h_sel[prow * K + k];
                }
            }
        }
        on_chunk(t0, t1);
    }
}

void Engine::router_forward(int layer, const double* d_x, int rows, const double* d_scores, double tau,
                            std::span<const double> fisher, int lookahead, bool adaptive, const RouteOutputs& out,
                            cudaStream_t stream) {
    activate();
    const int L = spec_.num_layers, N = spec_.experts_per_layer, K = spec_.top_k, D = spec_.hidden_dim;
    if (layer < 0 || layer >= L) fail(Status::Usage, "router_forward: layer out of range");
    if (rows < 1) fail(Status::Usage, "router_forward: rows must be >= 1");
    if (lookahead < 0 || lookahead > 3) fail(Status::Usage, "router_forward: lookahead out of {0,1,2,3}");
    if (static_cast<int>(fisher.size()) != L) fail(Status::Usage, "router_forward: fisher count != num_layers");
    if (!d_x || !out.selected || !out.count || !out.single) fail(Status::Usage, "router_forward: null device buffer");
    if (!has_gates()) fail(Status::Usage, "router_forward: gates not loaded");
    if (!stream) stream = compute_;
    const int per_row = 1 + lookahead;
    const int b = fwd_next_;
    fwd_next_ ^= 1;
    if (!fwd_done_[b]) MOE_CUDA(cudaEventCreateWithFlags(&fwd_done_[b], cudaEventDisableTiming));
    MOE_CUDA(cudaEventSynchronize(fwd_done_[b]));  // the launch that last used this staging buffer
    h_fwd_groups_[b].reserve(static_cast<size_t>(rows) * sizeof(RouteGroup));
    d_fwd_groups_[b].reserve(static_cast<size_t>(rows) * sizeof(RouteGroup));
    RouteGroup* groups = h_fwd_groups_[b].as<RouteGroup>();
    const int flags = adaptive ? kRouteAdaptive : 0;
    int max_gates = 0;
    for (int r = 0; r < rows; ++r) {
        RouteGroup& g = groups[r];
        g = RouteGroup{};
        g.x = d_x + static_cast<size_t>(r) * D;
        RouteItem& dec = g.items[g.n_items++];
        if (d_scores) {
            dec.scores = d_scores + static_cast<size_t>(r) * N;
        } else {
            gate_item(dec, layer);
        }
        dec.fisher = fisher[layer];
        dec.flags = flags;
        dec.out = r * per_row;
        int n_gates = d_scores ? 0 : 1;
        if (layer + 1 < L) {
            for (int dep = 1; dep <= lookahead && layer + dep < L; ++dep) {
                RouteItem& it = g.items[g.n_items++];
                gate_item(it, layer + dep);
                it.fisher = fisher[layer + dep];
                it.flags = flags;
                it.out = r * per_row + dep;
                ++n_gates;
            }
        } else if (lookahead > 0 && has_first_gate()) {
            RouteItem& it = g.items[g.n_items++];
            gate_item(it, -1);
            it.fisher = fisher[0];
            it.flags = flags;
            it.out = r * per_row + 1;
            ++n_gates;
        }
        max_gates = std::max(max_gates, n_gates);
    }
    // rows without every look-ahead item (near the last layer) keep count 0 in those slots
    MOE_CUDA(cudaMemsetAsync(out.count, 0, static_cast<size_t>(rows) * per_row * sizeof(int), stream));
    MOE_CUDA(cudaMemsetAsync(out.selected, 0xff, static_cast<size_t>(rows) * per_row * K * sizeof(int), stream));
    MOE_CUDA(cudaMemcpyAsync(d_fwd_groups_[b].ptr, groups, static_cast<size_t>(rows) * sizeof(RouteGroup),
                             cudaMemcpyHostToDevice, stream));
    RouteParams p{D, N, K, tau, 1.0};
    MOE_CUDA(launch_route(d_fwd_groups_[b].as<RouteGroup>(), rows, std::max(max_gates, 1), p, out, stream));
    MOE_CUDA(cudaEventRecord(fwd_done_[b], stream));  // staging buffer b (host and device) free after this
}

// inc/workload.hpp:60-112.  The RNG stream is consumed on the host in the reference's order
// (gates, then per token: x draws, per-layer drift draws); the walk never reads the logits, so
// all activations are produced first and the T*L gate GEMVs (+ /conc, softmax, top-K) run as
// one K1 launch.
void Engine::generate_trace(int T, double conc, double drift, std::uint64_t gate_seed, std::uint64_t token_seed,
                            bool shared_gates, const double* fisher_scales, const double* drift_scales, double* gates,
                            double* acts, double* scores, int* selected, double* fisher) {
    activate();
    const int L = spec_.num_layers, N = spec_.experts_per_layer, K = spec_.top_k, D = spec_.hidden_dim;
    if (T < 1) fail(Status::Usage, "SynthConfig: tokens must be >= 1");
    if (!(conc > 0.0)) fail(Status::Usage, "SynthConfig: dirichlet_concentration must be positive");
    if (!(drift >= 0.0)) fail(Status::Usage, "SynthConfig: residual_drift must be >= 0");
    for (int l = 0; l < L; ++l) {
        if (fisher_scales && !(fisher_scales[l] >= 0.0)) fail(Status::Usage, "SynthConfig: fisher scales must be >= 0");
        if (drift_scales && !(drift_scales[l] >= 0.0)) fail(Status::Usage, "SynthConfig: drift scales must be >= 0");
        fisher[l] = fisher_scales ? fisher_scales[l] : 1.0;
    }
    const size_t gsz = static_cast<size_t>(D) * N;
    SeededRng grng(gate_seed);
    const double wscale = 1.0 / std::sqrt(static_cast<double>(D));
    // every normal of both streams is drawn in bulk (SeededRng::normals: sequential raw draws,
    // threaded transforms), then consumed in the reference's order
    // (the two streams are independent: the gate stream is drawn on its own thread)
    const size_t gate_layers = shared_gates ? 1 : static_cast<size_t>(L);
    std::exception_ptr gate_error;
    std::thread gate_thread([&] {
        try {
            grng.normals(gates, gate_layers * gsz);
            for (size_t i = 0; i < gate_layers * gsz; ++i) gates[i] = wscale * gates[i];
            for (int l = 1; shared_gates && l < L; ++l) std::memcpy(gates + l * gsz, gates, gsz * sizeof(double));
        } catch (...) {
            gate_error = std::current_exception();
        }
    });
    int drift_layers = 0;
    for (int l = 0; l < L; ++l) drift_layers += drift * (drift_scales ? drift_scales[l] : 1.0) > 0.0;
    const size_t n_token_normals = static_cast<size_t>(T) * D * (1 + drift_layers);
    std::unique_ptr<double[]> nrm;
    std::exception_ptr token_error;
    try {
        nrm.reset(new double[n_token_normals]);  // no zero fill: every entry is drawn
        SeededRng trng(token_seed);
        trng.normals(nrm.get(), n_token_normals);
    } catch (...) {
        token_error = std::current_exception();
    }
    gate_thread.join();
    if (gate_error) std::rethrow_exception(gate_error);
    if (token_error) std::rethrow_exception(token_error);
    // every token restarts its walk from fresh normals, so given each token's offset in the stream
    // (D * (1 + drift layers) normals per token) the walks run in parallel
    const size_t per_token = static_cast<size_t>(D) * (1 + drift_layers);
    auto walk = [&](int t0, int t1) {
        std::vector<double> x(D);
        for (int tok = t0; tok < t1; ++tok) {
            const double* nv = nrm.get() + static_cast<size_t>(tok) * per_token;
            for (double& v : x) v = *nv++;
            for (int l = 0; l < L; ++l) {
                std::memcpy(acts + (static_cast<size_t>(tok) * L + l) * D, x.data(), D * sizeof(double));
                const double eps = drift * (drift_scales ? drift_scales[l] : 1.0);
                if (eps > 0.0) {
                    double norm_sq = 0.0;
                    for (double v : x) norm_sq += v * v;
                    const double step = eps * std::sqrt(norm_sq / D);
                    for (double& v : x) v += step * *nv++;
                }
            }
        }
    };
    const int n_walkers = static_cast<int>(std::min<size_t>(
        {static_cast<size_t>(std::max(1u, std::thread::hardware_concurrency())), 16, static_cast<size_t>(T),
         n_token_normals / 65536 + 1}));
    if (n_walkers <= 1) {
        walk(0, T);
    } else {
        std::vector<std::thread> pool;
        for (int w = 0; w < n_walkers; ++w) pool.emplace_back(walk, T * w / n_walkers, T * (w + 1) / n_walkers);
        for (auto& th : pool) th.join();
    }
    load_gates(gates, nullptr);
    const size_t TL = static_cast<size_t>(T) * L;
    d_x_.reserve(TL * D * sizeof(double));
    MOE_CUDA(cudaMemcpyAsync(d_x_.ptr, acts, TL * D * sizeof(double), cudaMemcpyHostToDevice, compute_));
    std::vector<RouteGroup> groups(TL);
    for (size_t tl = 0; tl < TL; ++tl) {
        RouteGroup& g = groups[tl];
        g.x = d_x_.as<double>() + tl * D;
        g.n_items = 1;
        g.items[0].gate = d_gate(static_cast<int>(tl % L));
        g.items[0].flags = kRouteEmitLogits;
        g.items[0].out = static_cast<int>(tl);
    }
    RouteParams p{D, N, K, 0.0, conc};
    TraceRoutes raw;
    std::vector<double> logits;
    run_route(groups, static_cast<int>(TL), 1, p, &raw, &logits, compute_);
    // /conc, softmax and top-K on the host with the same libm exp as the reference, so the stored
    // score bits (which tau calibration and every later decision read) are the reference's.
    for (size_t tl = 0; tl < TL; ++tl) {
        double* lg = logits.data() + tl * N;
        for (int j = 0; j < N; ++j) lg[j] /= conc;
        const std::vector<double> sc = softmax(std::span<const double>(lg, N));
        std::memcpy(scores + tl * N, sc.data(), N * sizeof(double));
        const std::vector<int> top = top_k_indices(sc, K);
        std::memcpy(selected + tl * K, top.data(), K * sizeof(int));
    }
}

// inc/workload.hpp:133-181: alpha from the sensitivity rule on stored scores; beta = share of
// tokens whose reuse-predicted top-1 (x_{l-1} . W_l, or the first-layer gate on the previous
// token's last activation) is inside the adaptive selection.
void Engine::generate_profiles(const double* acts, const double* scores, int T, std::span<const double> fisher,
                               double tau, double* alpha, double* beta) {
    activate();
    if (T < 1) fail(Status::Usage, "generate_profiles: empty trace set");
    if (!has_gates()) fail(Status::Usage, "generate_profiles: gates not loaded");
    const int L = spec_.num_layers, N = spec_.experts_per_layer, K = spec_.top_k, D = spec_.hidden_dim;
    if (static_cast<int>(fisher.size()) != L) fail(Status::Usage, "generate_profiles: fisher count does not match num_layers");
    const size_t TL = static_cast<size_t>(T) * L;
    d_x_.reserve(TL * D * sizeof(double));
    d_scores_.reserve(TL * N * sizeof(double));
    MOE_CUDA(cudaMemcpyAsync(d_x_.ptr, acts, TL * D * sizeof(double), cudaMemcpyHostToDevice, compute_));
    MOE_CUDA(cudaMemcpyAsync(d_scores_.ptr, scores, TL * N * sizeof(double), cudaMemcpyHostToDevice, compute_));
    // pass 1: adaptive decisions on the stored scores (K wide)
    std::vector<RouteGroup> dec(TL);
    for (size_t tl = 0; tl < TL; ++tl) {
        dec[tl].x = d_x_.as<double>() + tl * D;
        dec[tl].n_items = 1;
        dec[tl].items[0].scores = d_scores_.as<double>() + tl * N;
        dec[tl].items[0].fisher = fisher[tl % L];
        dec[tl].items[0].flags = kRouteAdaptive;
        dec[tl].items[0].out = static_cast<int>(tl);
    }
    TraceRoutes d;
    run_route(dec, static_cast<int>(TL), 1, RouteParams{D, N, K, tau, 1.0}, &d, nullptr, compute_);
    // pass 2: reuse predictions, top-1
    std::vector<RouteGroup> pre;
    std::vector<int> where;
    for (int tok = 0; tok < T; ++tok)
        for (int l = 0; l < L; ++l) {
            const double* x = nullptr;
            int gate_layer = 0;
            if (l >= 1) {
                x = d_x_.as<double>() + (static_cast<size_t>(tok) * L + (l - 1)) * D;
                gate_layer = l;
            } else if (has_first_gate() && tok >= 1) {
                x = d_x_.as<double>() + (static_cast<size_t>(tok - 1) * L + (L - 1)) * D;
                gate_layer = -1;
            }
            if (!x) continue;
            RouteGroup g;
            g.x = x;
            g.n_items = 1;
            gate_item(g.items[0], gate_layer);
            g.items[0].out = static_cast<int>(pre.size());
            pre.push_back(g);
            where.push_back(tok * L + l);
        }
    TraceRoutes pr;
    if (!pre.empty()) run_route(pre, static_cast<int>(pre.size()), 1, RouteParams{D, N, 1, tau, 1.0}, &pr, nullptr, compute_);
    std::vector<long long> singles(L, 0), hits(L, 0), counted(L, 0);
    for (size_t tl = 0; tl < TL; ++tl) singles[tl % L] += d.single[tl];
    for (size_t i = 0; i < pre.size(); ++i) {
        const int tl = where[i], l = tl % L;
        const int predicted = pr.selected[i];
        ++counted[l];
        for (int k = 0; k < d.count[tl]; ++k)
            if (d.selected[static_cast<size_t>(tl) * K + k] == predicted) {
                ++hits[l];
                break;
            }
    }
    for (int l = 0; l < L; ++l) {
        alpha[l] = static_cast<double>(singles[l]) / static_cast<double>(T);
        beta[l] = counted[l] > 0 ? static_cast<double>(hits[l]) / static_cast<double>(counted[l]) : 0.0;
    }
}

}  // namespace adapmoe

namespace adapmoe {

void Engine::train_first_gate(const double* acts, const double* scores, int T, double lr, int steps,
                              std::uint64_t seed, double* w_out) {
    activate();
    const int L = spec_.num_layers, N = spec_.experts_per_layer, K = spec_.top_k, D = spec_.hidden_dim;
    if (T < 2) fail(Status::Usage, "train_predictive_gate: empty training set (needs >= 2 tokens)");
    const int P = T - 1;
    // pairs (inc/workload.hpp:186-197): input = token p's last-layer activation, target logits =
    // log(max(score, 1e-300)) of token p+1's first layer; their softmax p is fixed for all steps
    std::vector<double> x(static_cast<size_t>(P) * D), target(static_cast<size_t>(P) * N);
    for (int p = 0; p < P; ++p) {
        const double* a = acts + (static_cast<size_t>(p) * L + (L - 1)) * D;
        std::copy(a, a + D, x.begin() + static_cast<size_t>(p) * D);
        std::vector<double> tl(N);
        for (int j = 0; j < N; ++j) tl[j] = std::log(std::max(scores[(static_cast<size_t>(p + 1) * L) * N + j], 1e-300));
        const std::vector<double> ps = softmax(tl);
        std::copy(ps.begin(), ps.end(), target.begin() + static_cast<size_t>(p) * N);
    }
    // initialisation: 0.1 * N(0,1) from SeededRng(seed), row-major (inc/prefetch.hpp:204-205)
    std::vector<double> w(static_cast<size_t>(D) * N);
    SeededRng rng(seed);
    for (double& v : w) v = 0.1 * rng.normal();
    DeviceBuffer d_x, d_w, d_diff, d_groups, d_logits, d_sel, d_cnt, d_sgl;
    d_x.reserve(x.size() * sizeof(double));
    d_w.reserve(w.size() * sizeof(double));
    d_diff.reserve(target.size() * sizeof(double));
    d_logits.reserve(target.size() * sizeof(double));
    d_sel.reserve(static_cast<size_t>(P) * K * sizeof(int));
    d_cnt.reserve(static_cast<size_t>(P) * sizeof(int));
    d_sgl.reserve(static_cast<size_t>(P) * sizeof(int));
    MOE_CUDA(cudaMemcpyAsync(d_x.ptr, x.data(), x.size() * sizeof(double), cudaMemcpyHostToDevice, compute_));
    MOE_CUDA(cudaMemcpyAsync(d_w.ptr, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice, compute_));
    std::vector<RouteGroup> groups(P);
    for (int p = 0; p < P; ++p) {
        RouteGroup& g = groups[p];
        g.x = d_x.as<double>() + static_cast<size_t>(p) * D;
        g.n_items = 1;
        g.items[0].gate = d_w.as<double>();
        g.items[0].flags = kRouteExact | kRouteEmitLogits;  // GateMatrix::logits order, fp64
        g.items[0].out = p;
    }
    d_groups.reserve(groups.size() * sizeof(RouteGroup));
    MOE_CUDA(cudaMemcpyAsync(d_groups.ptr, groups.data(), groups.size() * sizeof(RouteGroup), cudaMemcpyHostToDevice,
                             compute_));
    const RouteParams rp{D, N, K, 0.0, 1.0};
    const RouteOutputs ro{d_sel.as<int>(), d_cnt.as<int>(), d_sgl.as<int>(), nullptr, d_logits.as<double>(), nullptr};
    std::vector<double> logits(target.size()), diff(target.size());
    for (int step = 0; step < steps; ++step) {
        MOE_CUDA(launch_route(d_groups.as<RouteGroup>(), P, 0, rp, ro, compute_));
        MOE_CUDA(cudaMemcpyAsync(logits.data(), d_logits.ptr, logits.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                 compute_));
        MOE_CUDA(cudaStreamSynchronize(compute_));
        // q = softmax(logits) with the host's exp (inc/prefetch.hpp:180), diff = q - p
        for (int p = 0; p < P; ++p) {
            const std::vector<double> q = softmax(std::span<const double>(logits.data() + static_cast<size_t>(p) * N, N));
            for (int j = 0; j < N; ++j) diff[static_cast<size_t>(p) * N + j] = q[j] - target[static_cast<size_t>(p) * N + j];
        }
        MOE_CUDA(cudaMemcpyAsync(d_diff.ptr, diff.data(), diff.size() * sizeof(double), cudaMemcpyHostToDevice, compute_));
        MOE_CUDA(launch_gate_grad_step(d_w.as<double>(), d_x.as<double>(), d_diff.as<double>(), P, D, N, lr, compute_));
    }
    MOE_CUDA(cudaMemcpyAsync(w_out, d_w.ptr, w.size() * sizeof(double), cudaMemcpyDeviceToHost, compute_));
    MOE_CUDA(cudaStreamSynchronize(compute_));
}

}  // namespace adapmoe
