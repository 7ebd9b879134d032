#include "decode.hpp"

#include "nvtx.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <numeric>
#include <thread>

namespace adapmoe {

namespace {
constexpr size_t kSlotAlign = 2u << 20;
}

DecodeSession::DecodeSession(Engine& eng, std::span<const int> capacities, int staging_slots,
                             std::span<const double> fisher, double tau, const SimConfig& cfg, std::uint64_t seed,
                             int total_tokens, int batch, int ep_rank, int ep_world, bool free_running,
                             double concentration, const int* expert_owner)
    : free_running_(free_running),
      concentration_(concentration),
      batch_(batch),
      ep_rank_(ep_rank),
      ep_world_(ep_world),
      eng_(eng),
      spec_(eng.spec()),
      cfg_(cfg),
      caps_(capacities.begin(), capacities.end()),
      fisher_(fisher.begin(), fisher.end()),
      tau_(tau),
      total_tokens_(total_tokens),
      store_(*eng.experts) {
    eng.activate();
    cfg_.validate();
    const int L = spec_.num_layers, N = spec_.experts_per_layer, K = spec_.top_k, D = spec_.hidden_dim;
    if (static_cast<int>(caps_.size()) != L || static_cast<int>(fisher_.size()) != L)
        fail(Status::Usage, "decode_begin: capacities/fisher must have num_layers entries");
    if (store_.tiles != cfg_.tile_count_per_expert)
        fail(Status::Usage, "decode_begin: SimConfig tile count differs from the expert store's tile layout");
    if (total_tokens < 1) fail(Status::Usage, "decode_begin: total_tokens must be >= 1");
    if (K > 8) fail(Status::Usage, "decode: top_k > 8 unsupported by the combine kernel");
    if (K * store_.tiles > kMaxCombineRefs)  // CombineArgs::refs holds one entry per (rank, tile)
        fail(Status::Usage, "decode_begin: top_k * tiles must be <= 128");
    if (free_running_ && !eng.has_gates()) fail(Status::Usage, "free-running decode needs the gate matrices");
    if (!(concentration_ > 0.0)) fail(Status::Usage, "decode_begin: dirichlet concentration must be > 0");
    if (batch_ < 1 || batch_ > 256 || batch_ * K > kGMaxPairs)
        fail(Status::Usage, "decode_begin: batch must be in [1, 256] with batch * top_k <= 512");
    const int Ft = store_.ffn / store_.tiles;
    if (batch_ > 1 && (D % 128 || Ft % 64))
        fail(Status::Usage, "batched decode needs hidden_dim % 128 == 0 and (ffn / tiles) % 64 == 0 (tcgen05 tiles)");
    const bool prefetch_on = cfg_.policy.prefetch && cfg_.lookahead_depth > 0;
    if (prefetch_on && !eng.has_gates()) fail(Status::Usage, "decode: prefetching requires the gate matrices");
    if (ep_world_ < 1 || ep_rank_ < 0 || ep_rank_ >= ep_world_ || ep_world_ > N)
        fail(Status::Usage, "decode_begin: expert-parallel shard must satisfy 0 <= rank < world <= N");
    owner_.resize(static_cast<size_t>(L) * N);
    for (int l = 0; l < L; ++l)
        for (int e = 0; e < N; ++e) {
            const int o = expert_owner ? expert_owner[static_cast<size_t>(l) * N + e] : e % ep_world_;
            if (o < 0 || o >= ep_world_) fail(Status::Usage, "decode_begin: expert_owner entry out of [0, ep_world)");
            owner_[static_cast<size_t>(l) * N + e] = o;
            if (o == ep_rank_ && !store_.has(l, e))
                fail(Status::Usage, "decode_begin: this shard owns expert (" + std::to_string(l) + ", " + std::to_string(e) +
                                        ") but its expert store does not hold it (experts_init with the same owner table)");
        }
    int resident = 0;
    for (int l = 0; l < L; ++l) {
        const int c = caps_[l];
        if (c < 0 || c > N) fail(Status::Usage, "decode_begin: capacity out of [0, N]");
        int owned_here = 0;
        for (int e = 0; e < N; ++e) owned_here += owned(l, e) ? 1 : 0;
        resident += std::min(c, owned_here);  // this shard's resident experts
    }
    resident_slots_ = resident;
    int staging = staging_slots > 0 ? staging_slots : std::min(32, L * N + K);
    n_slots_ = resident + staging;
    stats_.slots_total = n_slots_;
    // slots are 2 MB aligned and a whole number of d-element bf16 rows, so the pool is one 2-D
    // tensor [rows][d] for the TMA maps of the grouped kernels
    const size_t row_bytes = static_cast<size_t>(D) * 2;
    const size_t align = std::lcm(kSlotAlign, row_bytes);
    slot_stride_ = (store_.expert_bytes + align - 1) / align * align;
    pool_.reserve(slot_stride_ * n_slots_);
    slots_.resize(n_slots_);
    for (int s = 0; s < n_slots_; ++s) free_.push_back(s);
    slot_of_.assign(static_cast<size_t>(L) * N, -1);
    MOE_CUDA(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, eng.device()));
    if (const char* v = std::getenv("ADAPMOE_TILE_MERGE")) tile_merge_ = std::clamp(std::atoi(v), 0, 2);  // A/B knob
    d_combine_ticket_.reserve(sizeof(unsigned));
    MOE_CUDA(cudaMemsetAsync(d_combine_ticket_.ptr, 0, sizeof(unsigned), eng.compute_stream()));

    // at most one launch for the resident experts' tiles (split per 32 segments) + one per
    // on-demand tile
    partial_regions_ = (K * store_.tiles + kMaxFfnSegments - 1) / kMaxFfnSegments + K * store_.tiles;
    speculate_ = free_running_ && batch_ == 1 && ep_world_ == 1;
    if (const char* v = std::getenv("ADAPMOE_SPECULATE")) speculate_ = speculate_ && std::atoi(v) != 0;
    // one extra partial region (index partial_regions_) holds the speculative launch
    d_partials_.reserve(static_cast<size_t>(partial_regions_ + 1) * kFfnMaxCtas * kFfnSlotsPerCta * D * sizeof(float));
    if (speculate_) {
        MOE_CUDA(cudaStreamCreateWithFlags(&route_stream_, cudaStreamNonBlocking));
        MOE_CUDA(cudaEventCreateWithFlags(&in_ready_, cudaEventDisableTiming));
    }
    if (batch_ > 1) {
        MOE_CUDA(cudaMemsetAsync(pool_.ptr, 0, slot_stride_ * n_slots_, eng.compute_stream()));  // slot padding read by TMA stays finite
        np_ = (batch_ + 15) / 16 * 16;
        const int F = store_.ffn;
        d_gx_.reserve(static_cast<size_t>(N) * np_ * D * 2);
        d_gh_.reserve(static_cast<size_t>(N) * np_ * F * 2);
        MOE_CUDA(cudaMemsetAsync(d_gx_.ptr, 0, static_cast<size_t>(N) * np_ * D * 2, eng.compute_stream()));
        MOE_CUDA(cudaMemsetAsync(d_gh_.ptr, 0, static_cast<size_t>(N) * np_ * F * 2, eng.compute_stream()));
        const uint64_t pool_rows = slot_stride_ * n_slots_ / row_bytes;
        MOE_CUDA(make_tensor_map_2d(&map_pool_gu_, pool_.ptr, pool_rows, D, 64, 128));
        MOE_CUDA(make_tensor_map_2d(&map_pool_dn_, pool_.ptr, pool_rows, D, 64, 64));
        MOE_CUDA(make_tensor_map_2d(&map_x_, d_gx_.ptr, static_cast<uint64_t>(N) * np_, D, 64, 16));
        MOE_CUDA(make_tensor_map_2d(&map_h_, d_gh_.ptr, static_cast<uint64_t>(N) * np_, F, 64, 16));
        cur_sel_.assign(static_cast<size_t>(batch_) * K, -1);
        cur_cnt_.assign(batch_, 0);
    }
    {
        const size_t fa = static_cast<size_t>(batch_) * kMaxRouteItems * 64 * sizeof(float);
        d_route_scratch_.reserve(2 * fa + static_cast<size_t>(batch_) * sizeof(unsigned));
        MOE_CUDA(cudaMemsetAsync(d_route_scratch_.ptr, 0, 2 * fa + static_cast<size_t>(batch_) * sizeof(unsigned),
                                 eng.compute_stream()));
        unsigned char* base = d_route_scratch_.as<unsigned char>();
        route_scratch_ = RouteScratch{reinterpret_cast<float*>(base), reinterpret_cast<float*>(base + fa),
                                      reinterpret_cast<unsigned*>(base + 2 * fa), batch_};
    }
    // trace replay: one K1 launch routes up to route_window_ tokens (every layer and stream)
    route_window_ = free_running_ ? 1 : std::max(1, std::min(total_tokens, (1 << 20) / (4 * batch_ * L)));
    if (const char* v = std::getenv("ADAPMOE_ROUTE_WINDOW"))  // test knob: force several windows per call
        route_window_ = std::max(1, std::min(route_window_, std::atoi(v)));
    const size_t route_rows = static_cast<size_t>(4) * batch_ * (free_running_ ? 1 : static_cast<size_t>(L) * route_window_);
    MOE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_route_), route_rows * (K + 3) * sizeof(int),
                           cudaHostAllocMapped));
    MOE_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_route_), h_route_, 0));
    route_host_cap_ = static_cast<int>(std::min<size_t>(route_rows, 16384));
    h_route_host_.reserve(static_cast<size_t>(route_host_cap_) * (2 + N) * sizeof(double));
    d_route_counter_.reserve(sizeof(unsigned));
    MOE_CUDA(cudaEventCreateWithFlags(&route_done_, cudaEventDisableTiming));
    MOE_CUDA(cudaEventCreateWithFlags(&user_in_, cudaEventDisableTiming));
    MOE_CUDA(cudaEventCreateWithFlags(&user_out_, cudaEventDisableTiming));
    // per-call buffers sized for the whole announced trace now: growing them inside decode() would put
    // cudaFree / cudaMallocHost (implicit device synchronisation) inside the timed window
    {
        const size_t TL = static_cast<size_t>(total_tokens) * batch_ * L;
        d_in_acts_.reserve(TL * D * sizeof(double));
        d_in_scores_.reserve(TL * N * sizeof(double));
        d_out_.reserve(TL * D * sizeof(float));
        h_groups_.reserve(TL * sizeof(RouteGroup));
        d_groups_.reserve(TL * sizeof(RouteGroup));
        if (free_running_) {
            d_x_free_.reserve(TL * D * sizeof(double));
            d_x_norm_.reserve(TL * D * sizeof(double));
        }
        // gate-decided layers (free-running, moe_decode_layer without scores) emit their scores here
        d_free_scores_.reserve(static_cast<size_t>(4) * batch_ * N * sizeof(double));
    }
    copier_ = std::make_unique<CopyEngine>(eng.copy_stream(), eng.device(),
                                           store_.format != kStoreBf16 ? store_.max_record_bytes() : 0);
    // last: the constructor performs the initial fill through on_insert
    policy_ = std::make_unique<PolicyEngine>(spec_, cfg_, caps_, seed, total_tokens, this, true);
    MOE_CUDA(cudaDeviceSynchronize());
}

DecodeSession::~DecodeSession() {
    copier_.reset();
    for (void* p : ep_ipc_opened_) cudaIpcCloseMemHandle(p);
    if (h_route_) cudaFreeHost(h_route_);
    if (route_done_) cudaEventDestroy(route_done_);
    if (origin_) cudaEventDestroy(origin_);
    if (user_in_) cudaEventDestroy(user_in_);
    if (user_out_) cudaEventDestroy(user_out_);
    if (in_ready_) cudaEventDestroy(in_ready_);
    if (route_stream_) {
        cudaStreamSynchronize(route_stream_);
        cudaStreamDestroy(route_stream_);
    }
    for (auto& p : layer_events_) cudaEventDestroy(p.second);
    for (cudaEvent_t e : layer_event_pool_) cudaEventDestroy(e);
    for (auto& p : pass_events_) {
        cudaEventDestroy(p.e0);
        cudaEventDestroy(p.e1);
    }
    for (auto& p : router_events_) {
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    for (auto& p : stall_events_) {
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    for (cudaEvent_t e : timing_pool_) cudaEventDestroy(e);
}

void DecodeSession::ep_export(int max_tokens_per_call, std::uint64_t* ptr, void* ipc_handle) {
    eng_.activate();
    if (ep_world_ < 2) fail(Status::Usage, "ep_export: the session is not expert-parallel (ep_world < 2)");
    if (ep_world_ > kMaxEpPeers) fail(Status::Usage, "ep_export: at most 8 expert-parallel shards");
    if (max_tokens_per_call < 1) fail(Status::Usage, "ep_export: max_tokens_per_call must be >= 1");
    ep_max_tokens_ = max_tokens_per_call;
    ep_rows_max_ = static_cast<size_t>(max_tokens_per_call) * batch_ * spec_.num_layers;
    const size_t bytes = kEpFlagBytes + 2 * static_cast<size_t>(ep_world_) * ep_rows_max_ * spec_.hidden_dim * sizeof(float);
    d_ep_region_.reserve(bytes);
    MOE_CUDA(cudaMemsetAsync(d_ep_region_.ptr, 0, kEpFlagBytes, eng_.compute_stream()));  // flags + timeout word
    MOE_CUDA(cudaStreamSynchronize(eng_.compute_stream()));
    ep_region_[ep_rank_] = d_ep_region_.as<unsigned char>();
    // Once connected, a shard's reduce kernel waits on its peers; any device-synchronising call
    // (cudaFree / cudaFreeHost when a buffer grows) inside a later decode call would then wait on it
    // while the peer's host thread waits likewise.  Size every per-call buffer for the largest call
    // now, so the exchange never meets an implicit device synchronisation.
    {
        const size_t TL = ep_rows_max_, D = spec_.hidden_dim, N = spec_.experts_per_layer;
        d_in_acts_.reserve(TL * D * sizeof(double));
        d_in_scores_.reserve(TL * N * sizeof(double));
        d_out_.reserve(TL * D * sizeof(float));
        h_groups_.reserve(TL * sizeof(RouteGroup));
        d_groups_.reserve(TL * sizeof(RouteGroup));
        if (batch_ > 1) {  // worst-case grouped down-partial arena of one layer
            const size_t mt = D / 128, T = store_.tiles;
            d_gpart_.reserve((N * mt * 16 + N * T * mt * 16) * np_ * 128 * sizeof(float));
        }
    }
    if (ptr) *ptr = reinterpret_cast<std::uint64_t>(d_ep_region_.ptr);
    if (ipc_handle) {
        cudaIpcMemHandle_t h;
        MOE_CUDA(cudaIpcGetMemHandle(&h, d_ep_region_.ptr));
        std::memcpy(ipc_handle, &h, sizeof h);
    }
}

void DecodeSession::ep_connect(const std::uint64_t* peer_ptrs, const unsigned char* peer_ipc) {
    eng_.activate();
    if (!d_ep_region_.ptr) fail(Status::Usage, "ep_connect: call ep_export first");
    for (int g = 0; g < ep_world_; ++g) {
        if (g == ep_rank_) continue;
        if (peer_ptrs && peer_ptrs[g]) {
            void* p = reinterpret_cast<void*>(peer_ptrs[g]);
            cudaPointerAttributes at{};
            MOE_CUDA(cudaPointerGetAttributes(&at, p));
            if (at.device != eng_.device()) {  // same process, another GPU: peer access over NVLink
                const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) MOE_CUDA(e);
                cudaGetLastError();
            }
            ep_region_[g] = static_cast<unsigned char*>(p);
        } else if (peer_ipc) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, peer_ipc + static_cast<size_t>(g) * 64, sizeof h);
            void* p = nullptr;
            MOE_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            ep_ipc_opened_.push_back(p);
            ep_region_[g] = static_cast<unsigned char*>(p);
        } else {
            fail(Status::Usage, "ep_connect: no pointer or IPC handle for shard " + std::to_string(g));
        }
    }
    ep_connected_ = true;
    sm_count_ = std::max(1, sm_count_ - 1);  // leave an SM for the exchange's 1-warp wait kernel
}

cudaEvent_t DecodeSession::take_timing() {
    if (!timing_pool_.empty()) {
        cudaEvent_t e = timing_pool_.back();
        timing_pool_.pop_back();
        return e;
    }
    cudaEvent_t e;
    MOE_CUDA(cudaEventCreate(&e));
    return e;
}

int DecodeSession::take_slot() {
    if (free_.empty()) release_pending(false);
    while (free_.empty() && !pending_free_.empty() && !layer_events_.empty()) {
        // the host routed ahead of the GPU: wait for the oldest layer still reading a released slot
        MOE_CUDA(cudaEventSynchronize(layer_events_.front().second));
        release_pending(false);
    }
    if (free_.empty())
        fail(Status::Infeasible, "decode: HBM slot pool exhausted (" + std::to_string(n_slots_) +
                                     " slots); pass a larger staging_slots to moe_decode_begin");
    const int s = free_.front();
    free_.pop_front();
    const int in_use = n_slots_ - static_cast<int>(free_.size());
    stats_.staging_high_water = std::max(stats_.staging_high_water, in_use - resident_slots_);
    return s;
}

void DecodeSession::release_slot(int s) { pending_free_.emplace_back(layer_seq_, s); }

// Free the slots released by layers whose FFN + combine have completed on the GPU (all: every
// pending slot; the caller has synchronised the device).
void DecodeSession::release_pending(bool all) {
    while (!layer_events_.empty() && (all || cudaEventQuery(layer_events_.front().second) == cudaSuccess)) {
        layers_complete_ = layer_events_.front().first + 1;
        layer_event_pool_.push_back(layer_events_.front().second);
        layer_events_.pop_front();
    }
    auto it = std::stable_partition(pending_free_.begin(), pending_free_.end(),
                                    [&](const auto& p) { return !(all || p.first < layers_complete_); });
    for (auto jt = it; jt != pending_free_.end(); ++jt) {
        Slot& sl = slots_[jt->second];
        if (sl.fill) {
            copier_->cancel(sl.fill);  // an unused prefetch may still be queued: drop what is not issued
            retiring_.push_back(sl.fill);
        }
        sl.fill.reset();
        sl.fill_done = true;
        free_.push_back(jt->second);
    }
    pending_free_.erase(it, pending_free_.end());
    // recycle copy jobs whose issued tiles have landed
    auto done = std::stable_partition(retiring_.begin(), retiring_.end(),
                                      [&](const std::shared_ptr<CopyJob>& j) { return !copier_->idle(j); });
    for (auto jt = done; jt != retiring_.end(); ++jt) copier_->retire(*jt);
    retiring_.erase(done, retiring_.end());
}

void DecodeSession::on_request(int id, ExpertRef ref, bool on_demand) {
    if (id >= static_cast<int>(req_slot_.size())) {
        req_slot_.resize(id + 1, -1);
        req_job_.resize(id + 1);
    }
    if (!owned(ref.layer, ref.expert)) {  // another shard moves it
        req_slot_[id] = -1;
        req_job_[id].reset();
        return;
    }
    const int s = take_slot();
    req_slot_[id] = s;
    std::vector<TileSource> srcs(store_.tiles);
    for (int t = 0; t < store_.tiles; ++t) {
        srcs[t].src = store_.record(ref.layer, ref.expert, t, &srcs[t].bytes);
        srcs[t].meta = store_.meta(ref.layer, ref.expert, t);
    }
    auto job = copier_->make_job(slot_ptr(s), store_.tile_bytes, std::move(srcs));
    job->serial = job_serial_++;
    job->token = cur_token_;
    job->layer = ref.layer;
    job->expert = ref.expert;
    job->requested_on_demand = on_demand;
    slots_[s].fill = job;
    slots_[s].fill_done = false;
    req_job_[id] = job;
    copier_->submit(job, on_demand);
}

void DecodeSession::on_promote(int id) {
    if (!req_job_[id]) return;
    req_job_[id]->promoted = true;
    req_job_[id]->logical_prefetch = false;  // counted on-demand at decision time (inc/simulator.hpp:410-418)
    copier_->promote(req_job_[id], false);
}

void DecodeSession::on_insert(ExpertRef ref, int request, std::optional<int> evicted) {
    const int N = spec_.experts_per_layer;
    const int key = ref.layer * N + ref.expert;
    if (request < 0) {  // initial residency (session setup, synchronous, untimed)
        if (evicted) fail(Status::Internal, "initial fill evicted an expert");
        if (!owned(ref.layer, ref.expert)) return;
        const int s = take_slot();
        // initial residency (pinned source), ordered before any compute-stream use of the slot
        upload_expert_tiles(store_, ref.layer, ref.expert, 0, store_.tiles, slot_ptr(s), fill_staging_,
                            eng_.compute_stream());
        slots_[s].fill.reset();
        slots_[s].fill_done = true;
        slot_of_[key] = s;
        return;
    }
    const int s = req_slot_[request];  // -1 when another shard owns the expert
    if (evicted && *evicted == ref.expert) {  // capacity-0 layer: the copy was transit only
        if (s >= 0) release_slot(s);
    } else {
        if (s >= 0) {
            if (slot_of_[key] >= 0) fail(Status::Internal, "insert of an expert that already has a slot");
            slot_of_[key] = s;
        }
        if (evicted) {
            if (request >= 0 && req_job_[request]) req_job_[request]->evicts = *evicted;
            const int vkey = ref.layer * N + *evicted;
            if (slot_of_[vkey] >= 0) release_slot(slot_of_[vkey]);  // the victim is ours
            slot_of_[vkey] = -1;
        }
    }
    req_slot_[request] = -1;
}

void DecodeSession::on_resident_compute(int, ExpertRef ref, int rank) {
    if (!owned(ref.layer, ref.expert)) return;
    uses_.push_back(Use{rank, slot_of_[ref.layer * spec_.experts_per_layer + ref.expert], false, {}});
}

void DecodeSession::on_tile_compute(int, ExpertRef ref, int rank, int tile, int request) {
    if (!owned(ref.layer, ref.expert)) return;
    if (uses_.empty() || !uses_.back().missing || uses_.back().rank != rank)
        uses_.push_back(Use{rank, req_slot_[request], true, {}});
    uses_.back().tiles.push_back(tile);
}

void DecodeSession::flush_waits() {
    if (deferred_waits_.empty()) return;
    struct W {
        long long seq;
        int slot, tile;
    };
    std::vector<W> ws;
    for (const auto& [slot, tile] : deferred_waits_) {  // needed now: promote what is still queued
        Slot& sl = slots_[slot];
        if (sl.fill && !sl.fill_done && !copier_->fully_issued(sl.fill)) copier_->promote(sl.fill, true);
    }
    for (const auto& [slot, tile] : deferred_waits_) {
        Slot& sl = slots_[slot];
        if (!sl.fill || sl.fill_done) continue;
        const int t0 = tile < 0 ? 0 : tile, t1 = tile < 0 ? sl.fill->tiles : tile + 1;
        for (int t = t0; t < t1; ++t) {
            copier_->wait_issued(sl.fill, t);
            ws.push_back(W{sl.fill->issue_seq[t], slot, t});
        }
    }
    deferred_waits_.clear();
    std::sort(ws.begin(), ws.end(), [](const W& a, const W& b) { return a.seq < b.seq; });
    defer_waits_ = false;
    for (const W& w : ws) wait_fill(w.slot, w.tile);
    defer_waits_ = true;
}

void DecodeSession::wait_fill(int slot, int tile) {
    if (defer_waits_) {
        deferred_waits_.emplace_back(slot, tile);
        return;
    }
    Slot& sl = slots_[slot];
    if (!sl.fill || sl.fill_done) return;
    const int t0 = tile < 0 ? 0 : tile, t1 = tile < 0 ? sl.fill->tiles : tile + 1;
    cudaStream_t cs = eng_.compute_stream();
    for (int t = t0; t < t1; ++t) {
        if (sl.fill->issued_tiles <= t) copier_->promote(sl.fill, true);
        const bool prefetch = sl.fill->logical_prefetch;
        sl.fill->consumed = true;
        cudaEvent_t ev = copier_->wait_issued(sl.fill, t);
        cudaEvent_t a = take_timing(), b = take_timing();
        MOE_CUDA(cudaEventRecord(a, cs));
        MOE_CUDA(cudaStreamWaitEvent(cs, ev, 0));
        MOE_CUDA(cudaEventRecord(b, cs));
        stall_events_.emplace_back(a, b);
        stall_is_prefetch_.push_back(prefetch);
        if (record_) stall_tags_.push_back(StallTag{cur_token_, sl.fill->layer, sl.fill->expert, t, sl.fill->serial});
    }
    if (tile < 0 || tile == sl.fill->tiles - 1) sl.fill_done = true;
}

// Launch the pending segments of `p` into the next partial region of this layer; `seg_meta`
// gives (rank, tile) per segment so the combine can find each segment's partials.
// One step of the peer-memory exchange (kernels/ep_exchange.hpp), sequence number ep_call_: publish
// this shard's partials of the step (already stored into every shard's slot by the combine), wait
// for every peer's, and sum the G slots of `rows` output rows (row_stride floats apart, at `out`'s
// offset in the call's output) in shard order into `out`.
void DecodeSession::ep_exchange(float* out, long long rows, long long row_stride) {
    cudaStream_t cs = eng_.compute_stream();
    const int D = spec_.hidden_dim;
    EpSignalArgs sa;
    for (int g = 0; g < ep_world_; ++g) sa.peer_flags[g] = reinterpret_cast<unsigned*>(ep_region_[g]);
    sa.world = ep_world_;
    sa.rank = ep_rank_;
    sa.call = ep_call_;
    MOE_CUDA(launch_ep_signal(sa, cs));
    MOE_CUDA(launch_ep_wait(ep_region_[ep_rank_], ep_world_, ep_call_, cs));
    EpReduceArgs ra;
    ra.slots = ep_slot(ep_rank_, 0, ep_call_ & 1) + (out - cur_out_base_);
    ra.slot_stride = static_cast<long long>(ep_rows_max_) * D;
    ra.out = out;
    ra.rows = rows;
    ra.row_stride = row_stride;
    ra.d = D;
    ra.world = ep_world_;
    MOE_CUDA(launch_ep_reduce(ra, cs));
    stats_.kernels += 3;
}

void DecodeSession::timed_ffn(FfnLaunch& p, const std::vector<std::pair<int, int>>& seg_meta,
                              std::vector<std::tuple<int, int, FfnPartialRef>>& refs) {
    cudaStream_t cs = eng_.compute_stream();
    flush_waits();
    const size_t region = static_cast<size_t>(kFfnMaxCtas) * kFfnSlotsPerCta * spec_.hidden_dim;
    if (partial_next_ >= partial_regions_) fail(Status::Internal, "decode: FFN partial pool exhausted");
    p.partial = d_partials_.as<float>() + region * partial_next_++;
    const int grid = ffn_grid(p, sm_count_);
    for (int s = 0; s < p.n_seg; ++s) {
        FfnPartialRef r{p.partial, grid, p.n_seg, s, seg_meta[s].first};
        ffn_partial_range(r, p.ft);
        refs.emplace_back(seg_meta[s].first, seg_meta[s].second, r);
    }
    cudaEvent_t e0 = take_timing(), e1 = take_timing();
    MOE_CUDA(cudaEventRecord(e0, cs));
    MOE_CUDA(launch_ffn(p, sm_count_, cs));
    MOE_CUDA(cudaEventRecord(e1, cs));
    const double gate_up = static_cast<double>(p.n_seg) * 2.0 * p.ft * p.d * 2.0;
    const double down = static_cast<double>(p.n_seg) * p.ft * p.d * 2.0;
    pass_events_.push_back(PassRec{gate_up, down, e0, e1, cur_token_, cur_layer_, launch_serial_++, {}});
    pass_events_.back().segs.swap(seg_info_);
    seg_info_.clear();
    stats_.kernels += 1;
    p.n_seg = 0;
}

void DecodeSession::on_layer_done(int, int, const RouteDecision& d) {
    defer_waits_ = layer_launch();
    if (batch_ > 1)
        layer_ffn_grouped(d);
    else
        layer_ffn_single(d);
    flush_waits();  // (nothing left unless the layer launched nothing)
    defer_waits_ = false;
    uses_.clear();
    cudaEvent_t ev;
    if (layer_event_pool_.empty()) {
        MOE_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    } else {
        ev = layer_event_pool_.back();
        layer_event_pool_.pop_back();
    }
    MOE_CUDA(cudaEventRecord(ev, eng_.compute_stream()));
    layer_events_.emplace_back(layer_seq_, ev);
    ++layer_seq_;
}

// Launch plan for the layer's on-demand (missing) experts, in landing order (ADAPMOE_TILE_MERGE):
//   0 "tiles":  one launch per landed tile (the reference's tile pipeline, inc/simulator.hpp:451-459);
//   1 "groups": an expert that is not the layer's last to land computes all its tiles in one launch
//               once its last tile has landed, the last expert computes tiles 0..n-2 together and its
//               final tile alone, and the resident experts join the first group that is not the final
//               tile (merge_resident()) — the work left after the final tile lands stays one tile's;
//   2 "layer":  the layer's whole FFN (resident experts + every on-demand tile) in ONE launch once its
//               last tile has landed.
// The host link is ~100x slower than HBM: a tile of 88 MB (8x7B) takes 1.6 ms on PCIe Gen5, the
// layer's whole FFN ~0.1 ms, and the link keeps streaming the next layer's copies meanwhile, so
// computing the layer after its last tile costs no link time, while a launch carries ~10 us of fixed
// cost (launch, first bytes, tail: profiles/r2_k2_ring.txt) that a 88 MB single-tile launch cannot
// amortise.  Default (-1): "layer" for tiles >= 8 MiB, "tiles" below.
bool DecodeSession::tile_merge_active() const {
    return tile_merge_ > 0 || (tile_merge_ < 0 && store_.tile_bytes >= (size_t{8} << 20));
}

bool DecodeSession::layer_launch() const {
    return tile_merge_ == 2 || (tile_merge_ < 0 && store_.tile_bytes >= (size_t{8} << 20));
}

bool DecodeSession::merge_resident() const {
    if (!tile_merge_active() || layer_launch()) return false;
    int groups = 0;
    for (const Use& u : uses_)
        if (u.missing && !u.tiles.empty()) groups += u.tiles.size() > 1 ? 2 : 1;
    return groups >= 2;  // some on-demand group lands before the layer's final tile
}

std::vector<std::pair<const DecodeSession::Use*, std::vector<int>>> DecodeSession::tile_groups() const {
    std::vector<std::pair<const Use*, std::vector<int>>> groups;
    std::vector<const Use*> missing;
    for (const Use& u : uses_)
        if (u.missing && !u.tiles.empty()) missing.push_back(&u);
    for (size_t m = 0; m < missing.size(); ++m) {
        const std::vector<int>& tiles = missing[m]->tiles;
        if (!tile_merge_active()) {
            for (int t : tiles) groups.emplace_back(missing[m], std::vector<int>{t});
        } else if (layer_launch() || m + 1 < missing.size() || tiles.size() == 1) {
            groups.emplace_back(missing[m], tiles);
        } else {
            groups.emplace_back(missing[m], std::vector<int>(tiles.begin(), tiles.end() - 1));
            groups.emplace_back(missing[m], std::vector<int>{tiles.back()});
        }
    }
    return groups;
}

// Free-running batch 1: while K1 routes layer `layer` (route_stream_, on the SMs left free), run the
// FFN of the expert the previous layer's look-ahead ranked first for this layer, if it is resident
// (the reference's reuse-based pre-gate, usually right).  layer_ffn_single takes its partials when
// the decision selects it and launches only the rest; otherwise the launch was wasted work.
void DecodeSession::launch_speculative(int layer, const double* x) {
    spec_run_.valid = false;
    const int n_pred = spec_next_n_;
    spec_next_n_ = 0;
    if (n_pred <= 0) return;
    const int N = spec_.experts_per_layer, D = spec_.hidden_dim, T = store_.tiles, Ft = store_.ffn / T;
    cudaStream_t cs = eng_.compute_stream();
    const size_t gate_up_bytes = static_cast<size_t>(2) * Ft * D * 2;
    FfnLaunch p;
    p.d = D;
    p.ft = Ft;
    p.x = x;
    SpecRun run;
    for (int k = 0; k < n_pred && (run.n + 1) * T <= kMaxFfnSegments; ++k) {
        const int slot = slot_of_[static_cast<size_t>(layer) * N + spec_next_[k]];
        if (slot < 0) continue;  // not resident: the decision will load it
        // only an expert whose weights have landed: waiting on an in-flight fill here would promote
        // it ahead of the layer's real on-demand loads and stall compute on a guess
        const Slot& sl = slots_[slot];
        if (sl.fill && !sl.fill_done && !copier_->landed(sl.fill)) continue;
        for (int t = 0; t < T; ++t) {
            const unsigned char* tile = slot_ptr(slot) + t * store_.tile_bytes;
            p.seg[p.n_seg].gate_up = reinterpret_cast<const std::uint16_t*>(tile);
            p.seg[p.n_seg].down_t = reinterpret_cast<const std::uint16_t*>(tile + gate_up_bytes);
            ++p.n_seg;
            note_seg(slot, spec_next_[k], t, true);
        }
        run.slot[run.n++] = slot;
    }
    if (run.n == 0) return;
    const size_t region = static_cast<size_t>(kFfnMaxCtas) * kFfnSlotsPerCta * D;
    p.partial = d_partials_.as<float>() + region * partial_regions_;  // the extra region
    const int sms = std::max(1, sm_count_ - kSpecSpareSms);          // leave SMs for K1
    cudaEvent_t e0 = take_timing(), e1 = take_timing();
    MOE_CUDA(cudaEventRecord(e0, cs));
    MOE_CUDA(launch_ffn(p, sms, cs));
    MOE_CUDA(cudaEventRecord(e1, cs));
    pass_events_.push_back(PassRec{static_cast<double>(p.n_seg) * 2.0 * Ft * D * 2.0,
                                   static_cast<double>(p.n_seg) * Ft * D * 2.0, e0, e1, cur_token_, layer,
                                   launch_serial_++, {}});
    pass_events_.back().segs.swap(seg_info_);
    seg_info_.clear();
    stats_.kernels += 1;
    stats_.spec_launches += 1;
    run.valid = true;
    run.layer_seq = layer_seq_;
    run.n_seg = p.n_seg;
    run.grid = ffn_grid(p, sms);
    run.partial = p.partial;
    spec_run_ = run;
}

void DecodeSession::layer_ffn_single(const RouteDecision& d) {
    const int D = spec_.hidden_dim, T = store_.tiles, F = store_.ffn, Ft = F / T;
    const size_t gate_up_bytes = static_cast<size_t>(2) * Ft * D * 2;
    auto seg = [&](int slot, int t) {
        FfnSegment s;
        const unsigned char* tile = slot_ptr(slot) + t * store_.tile_bytes;
        s.gate_up = reinterpret_cast<const std::uint16_t*>(tile);
        s.down_t = reinterpret_cast<const std::uint16_t*>(tile + gate_up_bytes);
        return s;
    };
    FfnLaunch p;
    p.d = D;
    p.ft = Ft;
    p.x = cur_x_;
    partial_next_ = 0;
    std::vector<std::pair<int, int>> meta;  // (rank, tile) of p's pending segments
    std::vector<std::tuple<int, int, FfnPartialRef>> refs;
    // resident experts: one launch over all their tiles (an expert the speculative launch already
    // computed contributes its partials instead)
    const bool spec_live = spec_run_.valid && spec_run_.layer_seq == layer_seq_;
    spec_run_.valid = false;
    for (const Use& u : uses_) {
        if (u.missing) continue;
        int k_spec = -1;
        for (int k = 0; spec_live && k < spec_run_.n; ++k)
            if (spec_run_.slot[k] == u.slot) k_spec = k;
        if (k_spec >= 0) {
            for (int t = 0; t < T; ++t) {
                FfnPartialRef r{spec_run_.partial, spec_run_.grid, spec_run_.n_seg, k_spec * T + t, u.rank};
                ffn_partial_range(r, Ft);
                refs.emplace_back(u.rank, t, r);
            }
            stats_.ffn_bytes += static_cast<long long>(store_.expert_bytes);
            stats_.spec_hits += 1;
            continue;
        }
        wait_fill(u.slot, -1);
        for (int t = 0; t < T; ++t) {
            if (p.n_seg == kMaxFfnSegments) {
                timed_ffn(p, meta, refs);
                meta.clear();
            }
            p.seg[p.n_seg++] = seg(u.slot, t);
            meta.emplace_back(u.rank, t);
            note_seg(u.slot, d.experts[u.rank], t, true);
        }
        stats_.ffn_bytes += static_cast<long long>(store_.expert_bytes);
    }
    const auto groups = tile_groups();
    // resident segments ride with the first on-demand group when that group is off the critical
    // path and the launch stays within kMaxFfnSegments
    const bool one_launch = layer_launch();
    const bool hold = p.n_seg > 0 && !groups.empty() &&
                      (one_launch || (merge_resident() &&
                                      p.n_seg + static_cast<int>(groups.front().second.size()) <= kMaxFfnSegments));
    if (p.n_seg && !hold) {
        timed_ffn(p, meta, refs);
        meta.clear();
    }
    // on-demand experts, as their tiles land (tile_groups: merged launches off the critical path;
    // "layer" mode: one launch after the layer's last tile)
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        const Use& u = *groups[gi].first;
        for (int t : groups[gi].second) {
            if (p.n_seg == kMaxFfnSegments) {  // launch what has landed so far
                timed_ffn(p, meta, refs);
                meta.clear();
            }
            wait_fill(u.slot, t);
            p.seg[p.n_seg++] = seg(u.slot, t);
            meta.emplace_back(u.rank, t);
            note_seg(u.slot, d.experts[u.rank], t, false);
        }
        if (!one_launch || gi + 1 == groups.size()) {
            timed_ffn(p, meta, refs);
            meta.clear();
        }
        if (groups[gi].second.back() == u.tiles.back()) stats_.ffn_bytes += static_cast<long long>(store_.expert_bytes);
    }
    std::sort(refs.begin(), refs.end(), [](const auto& a, const auto& b) {
        return std::get<0>(a) != std::get<0>(b) ? std::get<0>(a) < std::get<0>(b) : std::get<1>(a) < std::get<1>(b);
    });
    if (refs.size() > static_cast<size_t>(kMaxCombineRefs)) fail(Status::Internal, "combine: too many (rank, tile) segments");
    CombineArgs c;
    c.x = cur_res_;
    c.scores = cur_scores_;
    c.out = cur_out_;
    c.ranks = d.count;
    c.d = D;
    c.ft = Ft;
    c.residual = cur_residual_;
    c.n_refs = static_cast<int>(refs.size());
    for (size_t i = 0; i < refs.size(); ++i) c.refs[i] = std::get<2>(refs[i]);
    for (int r = 0; r < d.count; ++r) c.experts[r] = d.experts[r];
    if (ep_connected_) {  // store the partial into this shard's slot of every shard's region
        c.n_out_peer = ep_world_;
        for (int g = 0; g < ep_world_; ++g) c.out_peer[g] = ep_slot(g, ep_rank_, ep_call_ & 1) + (cur_out_ - cur_out_base_);
    }
    if (fuse_next_res_) {  // free-running batch 1: the combine also forms the next layer's input
        c.next_res = fuse_next_res_;
        c.next_norm = fuse_next_norm_;
        c.ticket = d_combine_ticket_.as<unsigned>();
        c.eps = kFreeRunningNormEps;
    }
    MOE_CUDA(launch_combine(c, eng_.compute_stream()));
    stats_.kernels += 1;
}

void DecodeSession::timed_grouped(GroupedLaunch& p, bool down, const RouteDecision& u) {
    cudaStream_t cs = eng_.compute_stream();
    flush_waits();
    cudaEvent_t e0 = take_timing(), e1 = take_timing();
    MOE_CUDA(cudaEventRecord(e0, cs));
    MOE_CUDA(down ? launch_grouped_down(p, sm_count_, cs) : launch_grouped_gate_up(p, sm_count_, cs));
    MOE_CUDA(cudaEventRecord(e1, cs));
    double tiles = 0;
    for (int s = 0; s < p.n_seg; ++s) tiles += p.seg[s].t1 - p.seg[s].t0;
    const double bytes = tiles * (down ? 1.0 : 2.0) * p.ft * p.d * 2.0;
    pass_events_.push_back(PassRec{down ? 0.0 : bytes, down ? bytes : 0.0, e0, e1, cur_token_, cur_layer_,
                                   launch_serial_++, {}});
    if (record_)
        for (int s = 0; s < p.n_seg; ++s) {
            const int r = p.seg[s].entry;
            int slot = -1;
            bool resident = false;
            for (const Use& us : uses_)
                if (us.rank == r) {
                    slot = us.slot;
                    resident = !us.missing;
                }
            for (int t = p.seg[s].t0; t < p.seg[s].t1; ++t)
                pass_events_.back().segs.push_back(SegInfo{u.experts[r], t, slot >= 0 ? fill_serial(slot) : -1, resident});
        }
    stats_.kernels += 1;
}

// Batched layer: gather the union experts' routed tokens, grouped gate/up + down on tcgen05 for the
// resident experts (one launch pair) and for each on-demand tile as it lands, then the per-stream
// fixed-order weighted combine (see kernels/grouped_ffn.hpp).
void DecodeSession::layer_ffn_grouped(const RouteDecision& u) {
    const int D = spec_.hidden_dim, N = spec_.experts_per_layer, K = spec_.top_k;
    const int T = store_.tiles, F = store_.ffn, Ft = F / T;
    cudaStream_t cs = eng_.compute_stream();
    const size_t row_bytes = static_cast<size_t>(D) * 2;
    // union rank of every expert, and the routed tokens of each rank (stream order)
    int rank_of[kMaxExperts];
    for (int e = 0; e < N; ++e) rank_of[e] = -1;
    for (int r = 0; r < u.count; ++r) rank_of[u.experts[r]] = r;
    GatherArgs g;
    g.acts = cur_x_;
    g.stream_stride = cur_x_stride_;
    g.x = d_gx_.as<std::uint16_t>();
    g.d = D;
    g.np_stride = np_;
    g.n_entries = u.count;
    GCombineArgs c;
    int n_of[kMaxExperts] = {0};
    for (int b = 0; b < batch_; ++b)
        for (int k = 0; k < cur_cnt_[b]; ++k) ++n_of[rank_of[cur_sel_[b * K + k]]];
    g.first[0] = 0;
    for (int r = 0; r < u.count; ++r) g.first[r + 1] = g.first[r] + n_of[r];
    int fill[kMaxExperts] = {0};
    for (int b = 0; b < batch_; ++b)
        for (int k = 0; k < K; ++k) {
            const int pi = b * K + k;
            if (k >= cur_cnt_[b]) {
                c.pair_entry[pi] = c.pair_col[pi] = c.pair_expert[pi] = -1;
                continue;
            }
            const int r = rank_of[cur_sel_[pi]];
            const int col = fill[r]++;
            g.stream[g.first[r] + col] = static_cast<short>(b);
            c.pair_entry[pi] = static_cast<short>(r);
            c.pair_col[pi] = static_cast<short>(col);
            c.pair_expert[pi] = static_cast<short>(cur_sel_[pi]);
        }
    MOE_CUDA(launch_grouped_gather(g, cs));
    stats_.kernels += 1;

    GroupedLaunch base;
    base.d = D;
    base.ft = Ft;
    base.f = F;
    base.np_stride = np_;
    base.h = d_gh_.as<std::uint16_t>();
    for (int r = 0; r < u.count; ++r) {
        base.ent[r].n = n_of[r];
        base.ent[r].np = std::max(16, (n_of[r] + 15) / 16 * 16);
    }
    for (const Use& us : uses_) base.ent[us.rank].slot_row = static_cast<long long>(us.slot) * (slot_stride_ / row_bytes);
    // launch list: resident experts together (all tiles), on-demand experts tile by tile
    struct Job {
        std::vector<GSeg> segs;
        int wait_slot = -1;
        std::vector<int> wait_tiles;
        std::vector<std::pair<int, int>> waits;  // (slot, tile) of a merged job, in landing order
    };
    std::vector<Job> jobs;
    Job res;
    for (const Use& us : uses_)
        if (!us.missing) {
            wait_fill(us.slot, -1);
            res.segs.push_back(GSeg{us.rank, 0, T});
            stats_.ffn_bytes += static_cast<long long>(store_.expert_bytes);
        }
    if (!res.segs.empty()) jobs.push_back(res);
    for (const auto& grp : tile_groups()) {  // on-demand experts, merged off the critical path
        const Use& us = *grp.first;
        Job j;
        j.wait_slot = us.slot;
        j.wait_tiles = grp.second;
        for (size_t q = 0; q < grp.second.size();) {  // contiguous tile runs -> one segment each
            size_t e = q + 1;
            while (e < grp.second.size() && grp.second[e] == grp.second[e - 1] + 1) ++e;
            j.segs.push_back(GSeg{us.rank, grp.second[q], grp.second[e - 1] + 1});
            q = e;
        }
        jobs.push_back(j);
        if (grp.second.back() == us.tiles.back()) stats_.ffn_bytes += static_cast<long long>(store_.expert_bytes);
    }
    if (!res.segs.empty() && jobs.size() >= 3 && merge_resident() &&  // resident + >= 2 on-demand groups
        jobs[0].segs.size() + jobs[1].segs.size() <= static_cast<size_t>(kGMaxSegs)) {
        jobs[1].segs.insert(jobs[1].segs.begin(), jobs[0].segs.begin(), jobs[0].segs.end());
        jobs.erase(jobs.begin());
    }
    if (layer_launch() && jobs.size() > 1) {  // one launch pair once the layer's last tile has landed
        Job all;
        for (size_t i = 0; i < jobs.size(); ++i) {
            if (i > 0 && all.segs.size() + jobs[i].segs.size() > static_cast<size_t>(kGMaxSegs)) break;
            for (int t : jobs[i].wait_tiles) all.waits.emplace_back(jobs[i].wait_slot, t);
            all.segs.insert(all.segs.end(), jobs[i].segs.begin(), jobs[i].segs.end());
            jobs[i].segs.clear();
        }
        std::vector<Job> rest{all};
        for (size_t i = 1; i < jobs.size(); ++i)
            if (!jobs[i].segs.empty()) rest.push_back(jobs[i]);
        jobs.swap(rest);
    }
    // plan every down launch first: the partial arena must hold the whole layer
    std::vector<GroupedLaunch> downs(jobs.size(), base);
    size_t need = 0;
    for (size_t i = 0; i < jobs.size(); ++i) {
        GroupedLaunch& p = downs[i];
        if (jobs[i].segs.size() > static_cast<size_t>(kGMaxSegs)) fail(Status::Internal, "grouped launch: too many segments");
        p.n_seg = static_cast<int>(jobs[i].segs.size());
        for (int s = 0; s < p.n_seg; ++s) p.seg[s] = jobs[i].segs[s];
        grouped_plan_down(p, sm_count_);
        need += static_cast<size_t>(p.units) * np_ * 128;
    }
    if (need * sizeof(float) > d_gpart_.bytes) {
        if (ep_connected_) fail(Status::Internal, "grouped partial arena too small under the EP exchange");
        MOE_CUDA(cudaStreamSynchronize(cs));  // earlier layers may still read the old arena
        d_gpart_.reserve(need * sizeof(float) * 5 / 4);
    }
    size_t off = 0;
    std::vector<std::pair<int, GCombineRef>> refs;  // (rank, ref) in launch order
    for (size_t i = 0; i < jobs.size(); ++i) {
        for (int t : jobs[i].wait_tiles) wait_fill(jobs[i].wait_slot, t);
        for (const auto& w : jobs[i].waits) wait_fill(w.first, w.second);
        GroupedLaunch up = base;
        up.n_seg = downs[i].n_seg;
        for (int s = 0; s < up.n_seg; ++s) up.seg[s] = downs[i].seg[s];
        up.map_a = map_pool_gu_;
        up.map_b = map_x_;
        grouped_plan_gate_up(up);
        timed_grouped(up, false, u);
        GroupedLaunch& dn = downs[i];
        dn.map_a = map_pool_dn_;
        dn.map_b = map_h_;
        dn.partial = d_gpart_.as<float>() + off;
        off += static_cast<size_t>(dn.units) * np_ * 128;
        timed_grouped(dn, true, u);
        for (int s = 0; s < dn.n_seg; ++s) refs.emplace_back(dn.seg[s].entry, GCombineRef{dn.partial, dn.unit_prefix[s], dn.kc});
    }
    std::stable_sort(refs.begin(), refs.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    if (refs.size() > sizeof(c.refs) / sizeof(c.refs[0])) fail(Status::Internal, "grouped combine: too many segments");
    c.ref_first[0] = 0;
    size_t q = 0;
    for (int r = 0; r < u.count; ++r) {
        while (q < refs.size() && refs[q].first == r) {
            c.refs[q] = refs[q].second;
            ++q;
        }
        c.ref_first[r + 1] = static_cast<int>(q);
    }
    c.acts = cur_res_;
    c.scores = cur_scores_;
    c.stream_stride = cur_x_stride_;
    c.score_stride = cur_score_stride_;
    c.out = cur_out_;
    c.out_stride = cur_out_stride_;
    c.d = D;
    c.np_stride = np_;
    c.n_streams = batch_;
    c.top_k = K;
    c.residual = cur_residual_;
    if (ep_connected_) {
        c.n_out_peer = ep_world_;
        for (int g = 0; g < ep_world_; ++g) c.out_peer[g] = ep_slot(g, ep_rank_, ep_call_ & 1) + (cur_out_ - cur_out_base_);
    }
    MOE_CUDA(launch_grouped_combine(c, cs));
    stats_.kernels += 1;
}

double DecodeSession::decode(const double* acts, const double* scores, int count, bool on_device, float* hidden_out) {
    eng_.activate();
    const int L = spec_.num_layers, N = spec_.experts_per_layer, K = spec_.top_k, D = spec_.hidden_dim;
    const int B = batch_;
    if (count < 1) return 0.0;
    NvtxRange call_range("moe_decode_tokens %d..%d", tokens_done_, tokens_done_ + count - 1);
    if (tokens_done_ + count > total_tokens_) fail(Status::Usage, "decode: more tokens than announced in decode_begin");
    if (next_layer_ != 0)
        fail(Status::Usage, "decode: token " + std::to_string(tokens_done_) + " is half done through moe_decode_layer "
                            "(next layer " + std::to_string(next_layer_) + ")");
    cudaStream_t cs = eng_.compute_stream();
    cudaEvent_t t_begin = take_timing(), t_end = take_timing();
    MOE_CUDA(cudaEventRecord(t_begin, cs));
    const size_t TL = static_cast<size_t>(count) * B * L;  // rows of [count][B][L]
    const double* x_all = acts;
    const double* s_all = scores;
    if (!on_device) {
        d_in_acts_.reserve(TL * D * sizeof(double));
        d_in_scores_.reserve(TL * N * sizeof(double));
        MOE_CUDA(cudaMemcpyAsync(d_in_acts_.ptr, acts, TL * D * sizeof(double), cudaMemcpyHostToDevice, cs));
        MOE_CUDA(cudaMemcpyAsync(d_in_scores_.ptr, scores, TL * N * sizeof(double), cudaMemcpyHostToDevice, cs));
        stats_.input_bytes += static_cast<long long>(TL * (D + N) * sizeof(double));
        x_all = d_in_acts_.as<double>();
        s_all = d_in_scores_.as<double>();
    }
    d_out_.reserve(TL * D * sizeof(float));
    float* out_all = (on_device && hidden_out) ? hidden_out : d_out_.as<float>();
    cur_out_base_ = out_all;
    double* x_norm = nullptr;
    if (free_running_) {
        // residual stream: layer 0 = the caller's input, layer l > 0 = layer l-1's output; the router
        // and the experts read its RMSNorm (Mixtral's pre-MoE norm, without gain)
        d_x_free_.reserve(TL * D * sizeof(double));
        d_x_norm_.reserve(TL * D * sizeof(double));
        d_free_scores_.reserve(static_cast<size_t>(4) * B * N * sizeof(double));
        MOE_CUDA(cudaMemcpyAsync(d_x_free_.ptr, x_all, TL * D * sizeof(double), cudaMemcpyDeviceToDevice, cs));
        x_all = d_x_free_.as<double>();
        x_norm = d_x_norm_.as<double>();
    }
    if (free_running_ && ep_world_ > 1 && !ep_connected_)
        fail(Status::Usage, "decode: free-running expert parallelism routes every layer on the summed output: "
                            "connect the shards first (moe_decode_ep_export / moe_decode_ep_connect)");
    if (ep_connected_) {
        if (count > ep_max_tokens_) fail(Status::Usage, "decode: more tokens per call than ep_export allowed");
        if (!free_running_) ++ep_call_;  // one exchange per call (free-running: one per layer, below)
    }

    // router groups for every (token, layer, stream) of this call: they depend only on positions.
    // Free-running: one launch per layer, group (i, l, b) writes rows b*4 + item.  Trace replay: the
    // decisions depend only on the stored trace, so one launch routes a window of tokens ahead of the
    // GPU and group (i, l, b) writes rows ((i % window) * L + l) * B * 4 + b * 4 + item.
    const bool prefetch_on = policy_->prefetch_on();
    h_groups_.reserve(TL * sizeof(RouteGroup));
    d_groups_.reserve(TL * sizeof(RouteGroup));
    RouteGroup* hg = h_groups_.as<RouteGroup>();
    int max_gates = 1;
    const int adaptive = cfg_.policy.adaptive_gating ? kRouteAdaptive : 0;
    for (int i = 0; i < count; ++i)
        for (int l = 0; l < L; ++l)
            for (int b = 0; b < B; ++b) {
                const size_t row = (static_cast<size_t>(i) * B + b) * L + l;  // input row [i][b][l]
                const int tok = tokens_done_ + i;
                const int rb = free_running_ ? b * 4 : (((i % route_window_) * L + l) * B + b) * 4;
                RouteGroup g;
                g.x = (free_running_ ? x_norm : x_all) + row * D;
                g.n_items = 1;
                g.items[0].scores = s_all + row * N;
                g.items[0].fisher = fisher_[l];
                g.items[0].flags = adaptive;
                g.items[0].out = rb;
                if (free_running_) {  // decide from this layer's gate on the evolving hidden state
                    eng_.gate_item(g.items[0], l);
                    g.items[0].flags = adaptive | kRouteDivConc | kRouteEmitScores;
                }
                if (prefetch_on) {
                    if (l + 1 < L) {
                        for (int dep = 1; dep <= cfg_.lookahead_depth && l + dep < L; ++dep) {
                            RouteItem& it = g.items[g.n_items++];
                            eng_.gate_item(it, l + dep);
                            it.fisher = fisher_[l + dep];
                            it.flags = adaptive;
                            it.out = rb + dep;
                        }
                    } else if (eng_.has_first_gate() && tok + 1 < total_tokens_) {
                        RouteItem& it = g.items[g.n_items++];
                        eng_.gate_item(it, -1);
                        it.fisher = fisher_[0];
                        it.flags = adaptive;
                        it.out = rb + 1;
                    }
                }
                max_gates = std::max(max_gates, free_running_ ? g.n_items : g.n_items - 1);
                hg[(static_cast<size_t>(i) * L + l) * B + b] = g;  // launch order [i][l][b]
            }
    MOE_CUDA(cudaMemcpyAsync(d_groups_.ptr, hg, TL * sizeof(RouteGroup), cudaMemcpyHostToDevice, cs));
    RouteParams rp{D, N, K, tau_, concentration_};
    const int rows = 4 * B * (free_running_ ? 1 : L * route_window_);  // output layout stride
    int* d_sel = d_route_;
    int* d_cnt = d_sel + static_cast<size_t>(rows) * K;
    int* d_sgl = d_cnt + rows;
    int* d_exact = d_sgl + rows;
    RouteOutputs ro{d_sel, d_cnt, d_sgl, nullptr, free_running_ ? d_free_scores_.as<double>() : nullptr, d_exact};
    ro.host_entries = h_route_host_.as<double>();
    ro.host_counter = d_route_counter_.as<unsigned>();
    ro.host_cap = route_host_cap_;
    int* sel = h_route_;
    int* cnt = sel + static_cast<size_t>(rows) * K;
    int* sgl = cnt + rows;
    int* exact_used = sgl + rows;

    std::array<RoutePrediction, 3> preds;
    const bool gap_trace = std::getenv("ADAPMOE_GAP_TRACE") != nullptr;
    struct GapRec {
        cudaEvent_t r0, r1, f0, f1;
    };
    std::vector<GapRec> gap_rec;
    cur_x_stride_ = static_cast<long long>(L) * D;
    cur_out_stride_ = static_cast<long long>(L) * D;
    cur_residual_ = ep_rank_ == 0 ? 1 : 0;
    for (int i = 0; i < count; ++i) {
        const int tok = tokens_done_ + i;
        for (int l = 0; l < L; ++l) {
            cur_token_ = tok;
            cur_layer_ = l;
            NvtxRange layer_range("token %d layer %d", tok, l);
            const size_t gl = (static_cast<size_t>(i) * L + l) * B;
            // free-running batch 1 without the EP exchange: layer l > 0's input was formed by layer
            // l-1's combine (CombineArgs::next_res)
            const bool fused_input = free_running_ && B == 1 && ep_world_ == 1;
            if (free_running_ && !(fused_input && l > 0)) {  // residual x_l and its RMSNorm, every stream
                const size_t row_l = (static_cast<size_t>(i) * B) * L + l;
                MOE_CUDA(launch_free_running_input(d_x_free_.as<double>() + row_l * D, x_norm + row_l * D,
                                                   static_cast<long long>(L) * D, l > 0 ? out_all + (row_l - 1) * D : nullptr,
                                                   static_cast<long long>(L) * D, B, D, kFreeRunningNormEps, cs));
                stats_.kernels += 1;
            }
            if (free_running_ || (l == 0 && i % route_window_ == 0)) {
                // free-running: this layer (its input is the previous layer's output); trace replay:
                // every layer of the next window of tokens, once
                const int n_groups = free_running_ ? B : std::min(route_window_, count - i) * L * B;
                cudaStream_t rs = cs;
                if (speculate_) {  // K1 beside the speculative FFN: its input is ready once the layer's input is
                    MOE_CUDA(cudaEventRecord(in_ready_, cs));
                    MOE_CUDA(cudaStreamWaitEvent(route_stream_, in_ready_, 0));
                    rs = route_stream_;
                }
                MOE_CUDA(cudaMemsetAsync(d_route_counter_.ptr, 0, sizeof(unsigned), rs));
                std::memset(exact_used, 0, sizeof(int) * 4 * static_cast<size_t>(n_groups));  // rows without an item stay 0
                cudaEvent_t r0 = take_timing(), r1 = take_timing();
                MOE_CUDA(cudaEventRecord(r0, rs));
                MOE_CUDA(launch_route(d_groups_.as<RouteGroup>() + gl, n_groups, max_gates, rp, ro, rs,
                                      n_groups <= route_scratch_.groups ? &route_scratch_ : nullptr));
                MOE_CUDA(cudaEventRecord(r1, rs));
                router_events_.emplace_back(r0, r1);
                if (record_) router_tokens_.push_back(tok);
                stats_.kernels += 1;
                stats_.router_launches += 1;
                MOE_CUDA(cudaEventRecord(route_done_, rs));
                if (speculate_)
                    launch_speculative(l, x_norm + (static_cast<size_t>(i) * B * L + l) * D);
                const auto h0 = std::chrono::steady_clock::now();
                NvtxRange sync_range("router sync");
                MOE_CUDA(cudaEventSynchronize(route_done_));
                stats_.host_sync_ms +=
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
                // uncertified items: the reference's softmax (libm exp) on their exact logits
                route_host_decide(rp, h_route_host_.as<double>(), exact_used, 0, 4LL * n_groups, sel, cnt, sgl, nullptr);
            }
            const auto h1 = std::chrono::steady_clock::now();
            release_pending(false);
            // actual selection: the union of the streams' selections (B = 1: the stream's own)
            RouteDecision d;
            int singles = 0;
            const int n_items = hg[gl].n_items;
            int np = 0;
            const int base = free_running_ ? 0 : ((i % route_window_) * L + l) * B * 4;
            for (int it = 1; it < n_items; ++it) {
                preds[np].target = (l + 1 < L) ? l + it : 0;
                preds[np].count = 0;
                ++np;
            }
            for (int b = 0; b < B; ++b) {
                const int r0w = base + b * 4;
                singles += sgl[r0w] != 0;
                for (int it = 1; it < n_items; ++it) stats_.router_exact += exact_used[r0w + it] != 0;
                for (int k = 0; k < cnt[r0w]; ++k) {
                    const int e = sel[r0w * K + k];
                    bool seen = false;
                    for (int q = 0; q < d.count; ++q) seen |= d.experts[q] == e;
                    if (!seen) d.experts[d.count++] = e;
                }
                for (int it = 1; it < n_items; ++it) {
                    RoutePrediction& p = preds[it - 1];
                    for (int k = 0; k < cnt[r0w + it]; ++k) {
                        const int e = sel[(r0w + it) * K + k];
                        bool seen = false;
                        for (int q = 0; q < p.count; ++q) seen |= p.experts[q] == e;
                        if (!seen) p.experts[p.count++] = e;
                    }
                }
                if (B > 1) {
                    cur_cnt_[b] = cnt[r0w];
                    for (int k = 0; k < K; ++k) cur_sel_[b * K + k] = k < cnt[r0w] ? sel[r0w * K + k] : -1;
                }
            }
            d.single = B == 1 && sgl[base] != 0;
            const size_t row0 = (static_cast<size_t>(i) * B) * L + l;  // stream 0's input row
            cur_x_ = (free_running_ ? x_norm : x_all) + row0 * D;
            cur_res_ = x_all + row0 * D;
            cur_scores_ = free_running_ ? d_free_scores_.as<double>() : s_all + row0 * N;
            cur_score_stride_ = free_running_ ? 4 * N : static_cast<long long>(L) * N;
            cur_out_ = out_all + row0 * D;
            fuse_next_res_ = (fused_input && l + 1 < L) ? d_x_free_.as<double>() + (row0 + 1) * D : nullptr;
            fuse_next_norm_ = fuse_next_res_ ? x_norm + (row0 + 1) * D : nullptr;
            const size_t npass0 = pass_events_.size();
            if (speculate_) {  // the look-ahead's top-1 for the next layer (item 1): the next speculation
                // (speculating its whole list measured no gain: mispredicted second experts cost what
                // the hits save; top-1 alone: +5 % on the all-resident free-running window)
                spec_next_n_ = (l + 1 < L && np > 0) ? std::min(1, preds[0].count) : 0;
                for (int k = 0; k < spec_next_n_; ++k) spec_next_[k] = preds[0].experts[k];
            }
            if (free_running_ && ep_connected_) ++ep_call_;  // this layer's exchange (its combine's slot parity)
            policy_->step(tok, l, d, std::span<const RoutePrediction>(preds.data(), np), B > 1 ? singles : -1);
            if (free_running_ && ep_connected_)  // the next layer routes on the full output: sum the shards now
                ep_exchange(cur_out_, B, static_cast<long long>(L) * D);
            if (gap_trace && !router_events_.empty() && pass_events_.size() > npass0)
                gap_rec.push_back({router_events_.back().first, router_events_.back().second, pass_events_[npass0].e0,
                                   pass_events_.back().e1});
            stats_.host_step_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h1).count();
        }
    }
    if (ep_connected_ && !free_running_)  // publish this call's partials, then sum every shard's in order
        ep_exchange(out_all, static_cast<long long>(TL), D);
    if (hidden_out && !on_device)
        MOE_CUDA(cudaMemcpyAsync(hidden_out, out_all, TL * D * sizeof(float), cudaMemcpyDeviceToHost, cs));
    MOE_CUDA(cudaEventRecord(t_end, cs));
    if (ep_connected_) {  // a peer that never signals must not hang the caller forever
        const auto t0 = std::chrono::steady_clock::now();
        cudaError_t q;
        while ((q = cudaEventQuery(t_end)) == cudaErrorNotReady) {
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
                fail(Status::Device, "expert-parallel exchange: no signal from a peer shard within 120 s (all shards "
                                     "must decode the same calls concurrently)");
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
        MOE_CUDA(q);
        unsigned timed_out = 0;
        MOE_CUDA(cudaMemcpy(&timed_out, ep_region_[ep_rank_] + 64 * kMaxEpPeers, sizeof timed_out,
                            cudaMemcpyDeviceToHost));
        if (timed_out)
            fail(Status::Device, "expert-parallel exchange: a peer shard did not publish its partials (all shards "
                                 "must decode the same calls concurrently)");
    }
    MOE_CUDA(cudaStreamSynchronize(cs));
    for (size_t q = 0; q < gap_rec.size(); ++q) {  // ADAPMOE_GAP_TRACE (temporary probe)
        float k1 = 0, k1_ffn = 0, ffn = 0, prev = -1;
        cudaEventElapsedTime(&k1, gap_rec[q].r0, gap_rec[q].r1);
        cudaEventElapsedTime(&k1_ffn, gap_rec[q].r1, gap_rec[q].f0);
        cudaEventElapsedTime(&ffn, gap_rec[q].f0, gap_rec[q].f1);
        if (q) cudaEventElapsedTime(&prev, gap_rec[q - 1].f1, gap_rec[q].r0);
        std::fprintf(stderr, "[gap] %zu: K1 %.1f us, K1 end -> FFN start %.1f us, FFN %.1f us, prev FFN end -> K1 start %.1f us\n",
                     q, k1 * 1e3f, k1_ffn * 1e3f, ffn * 1e3f, prev * 1e3f);
    }
    release_pending(true);
    tokens_done_ += count;
    stats_.tokens += static_cast<long long>(count) * B;
    float ms = 0.0f;
    MOE_CUDA(cudaEventElapsedTime(&ms, t_begin, t_end));
    timing_pool_.push_back(t_begin);
    timing_pool_.push_back(t_end);
    return ms;
}

// Fold the (completed) timing events recorded so far into the counters and recycle them.
DecodeStats DecodeSession::snapshot() {
    eng_.activate();
    MOE_CUDA(cudaStreamSynchronize(eng_.compute_stream()));
    auto elapsed = [](cudaEvent_t a, cudaEvent_t b) {
        float ms = 0.0f;
        MOE_CUDA(cudaEventElapsedTime(&ms, a, b));
        return static_cast<double>(ms);
    };
    auto since = [&](cudaEvent_t e) { return origin_ ? elapsed(origin_, e) : 0.0; };
    for (auto& p : pass_events_) {
        const double ms = elapsed(p.e0, p.e1);
        if (record_) {
            const double a = since(p.e0), b = since(p.e1);
            for (const SegInfo& g : p.segs)
                phys_compute_.push_back(PhysCompute{0, a, b, p.token, p.layer, g.expert, g.tile, p.launch, g.fill, g.resident});
        }
        stats_.ffn_ms += ms;
        stats_.gate_up_bytes += p.gate_up_bytes;
        stats_.down_bytes += p.down_bytes;
        stats_.ffn_launches += 1;
        timing_pool_.push_back(p.e0);
        timing_pool_.push_back(p.e1);
    }
    pass_events_.clear();
    for (size_t i = 0; i < router_events_.size(); ++i) {
        const auto& p = router_events_[i];
        stats_.router_ms += elapsed(p.first, p.second);
        if (record_ && i < router_tokens_.size())
            phys_compute_.push_back(PhysCompute{2, since(p.first), since(p.second), router_tokens_[i], -1, -1, -1, -1, -1, false});
        timing_pool_.push_back(p.first);
        timing_pool_.push_back(p.second);
    }
    router_events_.clear();
    router_tokens_.clear();
    for (size_t i = 0; i < stall_events_.size(); ++i) {
        const auto& p = stall_events_[i];
        const double ms = elapsed(p.first, p.second);
        stats_.stall_ms += ms;
        if (stall_is_prefetch_[i]) stats_.prefetch_stall_ms += ms;
        if (record_ && i < stall_tags_.size()) {
            const StallTag& g = stall_tags_[i];
            phys_compute_.push_back(PhysCompute{1, since(p.first), since(p.second), g.token, g.layer, g.expert, g.tile, -1, g.job, false});
        }
        timing_pool_.push_back(p.first);
        timing_pool_.push_back(p.second);
    }
    stall_events_.clear();
    stall_is_prefetch_.clear();
    stall_tags_.clear();
    DecodeStats s = stats_;
    s.tile_copies = copier_->tiles_copied();
    s.copy_bytes = copier_->bytes_copied();
    s.copy_busy_ms = copier_->busy_ms_total(&s.prefetch_copy_ms, &s.prefetch_tiles, &s.prefetch_used_copy_ms);
    long long dec_kernels = 0;
    copier_->decode_totals(&s.decode_ms, &s.decode_launches, &s.decode_bytes, &dec_kernels);
    s.kernels += dec_kernels;  // the coded-tile decode and escape-patch kernels count as ours too
    return s;
}

DecodeStats DecodeSession::finish() {
    eng_.activate();
    copier_->drain();
    MOE_CUDA(cudaDeviceSynchronize());
    release_pending(true);
    for (auto& j : retiring_) copier_->retire(j);
    retiring_.clear();
    return snapshot();
}

// One layer of the current token on caller buffers (moe_decode_layer).  The same policy step and
// FFN / combine launches as decode(), with the routing of one layer per call (its input is the
// caller's, e.g. after the caller's attention) and the caller's stream ordered around the work.
void DecodeSession::decode_layer(int layer, const double* x, const double* scores, float* out, bool add_input,
                                 cudaStream_t user) {
    eng_.activate();
    const int L = spec_.num_layers, N = spec_.experts_per_layer, K = spec_.top_k, D = spec_.hidden_dim, B = batch_;
    if (free_running_ || ep_world_ > 1)
        fail(Status::Usage, "decode_layer: per-layer calls take a session without free_running or expert parallelism");
    if (!x || !out) fail(Status::Usage, "decode_layer: x and out are required");
    if (layer != next_layer_)
        fail(Status::Usage, "decode_layer: layers run in order; expected layer " + std::to_string(next_layer_) +
                                " of token " + std::to_string(tokens_done_) + ", got " + std::to_string(layer));
    if (tokens_done_ >= total_tokens_) fail(Status::Usage, "decode_layer: more tokens than announced in decode_begin");
    if (!scores && !eng_.has_gates()) fail(Status::Usage, "decode_layer: deciding from the gate needs the gate matrices");
    const int tok = tokens_done_;
    cur_token_ = tok;
    cur_layer_ = layer;
    NvtxRange layer_range("moe_decode_layer token %d layer %d", tok, layer);
    cudaStream_t cs = eng_.compute_stream();
    const auto h0 = std::chrono::steady_clock::now();
    if (user != cs) {  // the caller's producer of x (e.g. attention) -> this layer's work
        MOE_CUDA(cudaEventRecord(user_in_, user));
        MOE_CUDA(cudaStreamWaitEvent(cs, user_in_, 0));
    }
    const bool prefetch_on = policy_->prefetch_on();
    RouteGroup* hg = h_groups_.as<RouteGroup>();
    const int adaptive = cfg_.policy.adaptive_gating ? kRouteAdaptive : 0;
    int max_gates = 1;
    for (int b = 0; b < B; ++b) {
        RouteGroup g;
        g.x = x + static_cast<size_t>(b) * D;
        g.n_items = 1;
        g.items[0].fisher = fisher_[layer];
        g.items[0].out = b * 4;
        if (scores) {  // the reference's actual-selection site: stored scores (inc/simulator.hpp:390-396)
            g.items[0].scores = scores + static_cast<size_t>(b) * N;
            g.items[0].flags = adaptive;
        } else {  // the layer's gate on x, softmax(logits / concentration)
            eng_.gate_item(g.items[0], layer);
            g.items[0].flags = adaptive | kRouteDivConc | kRouteEmitScores;
        }
        if (prefetch_on) {
            if (layer + 1 < L) {
                for (int dep = 1; dep <= cfg_.lookahead_depth && layer + dep < L; ++dep) {
                    RouteItem& it = g.items[g.n_items++];
                    eng_.gate_item(it, layer + dep);
                    it.fisher = fisher_[layer + dep];
                    it.flags = adaptive;
                    it.out = b * 4 + dep;
                }
            } else if (eng_.has_first_gate() && tok + 1 < total_tokens_) {
                RouteItem& it = g.items[g.n_items++];
                eng_.gate_item(it, -1);
                it.fisher = fisher_[0];
                it.flags = adaptive;
                it.out = b * 4 + 1;
            }
        }
        max_gates = std::max(max_gates, scores ? g.n_items - 1 : g.n_items);
        hg[b] = g;
    }
    MOE_CUDA(cudaMemcpyAsync(d_groups_.ptr, hg, static_cast<size_t>(B) * sizeof(RouteGroup), cudaMemcpyHostToDevice, cs));
    RouteParams rp{D, N, K, tau_, concentration_};
    const int rows = 4 * B;
    int* d_sel = d_route_;
    int* d_cnt = d_sel + static_cast<size_t>(rows) * K;
    int* d_sgl = d_cnt + rows;
    int* d_exact = d_sgl + rows;
    RouteOutputs ro{d_sel, d_cnt, d_sgl, nullptr, scores ? nullptr : d_free_scores_.as<double>(), d_exact};
    ro.host_entries = h_route_host_.as<double>();
    ro.host_counter = d_route_counter_.as<unsigned>();
    ro.host_cap = route_host_cap_;
    int* sel = h_route_;
    int* cnt = sel + static_cast<size_t>(rows) * K;
    int* sgl = cnt + rows;
    int* exact_used = sgl + rows;
    MOE_CUDA(cudaMemsetAsync(d_route_counter_.ptr, 0, sizeof(unsigned), cs));
    std::memset(exact_used, 0, sizeof(int) * rows);
    cudaEvent_t r0 = take_timing(), r1 = take_timing();
    MOE_CUDA(cudaEventRecord(r0, cs));
    MOE_CUDA(launch_route(d_groups_.as<RouteGroup>(), B, max_gates, rp, ro, cs,
                          B <= route_scratch_.groups ? &route_scratch_ : nullptr));
    MOE_CUDA(cudaEventRecord(r1, cs));
    router_events_.emplace_back(r0, r1);
    if (record_) router_tokens_.push_back(tok);
    stats_.kernels += 1;
    stats_.router_launches += 1;
    MOE_CUDA(cudaEventRecord(route_done_, cs));
    const auto hs = std::chrono::steady_clock::now();
    MOE_CUDA(cudaEventSynchronize(route_done_));
    stats_.host_sync_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hs).count();
    route_host_decide(rp, h_route_host_.as<double>(), exact_used, 0, rows, sel, cnt, sgl, nullptr);
    release_pending(false);
    // decision (union over the streams) and look-ahead predictions, as in decode()
    RouteDecision d;
    std::array<RoutePrediction, 3> preds;
    int singles = 0, np = 0;
    const int n_items = hg[0].n_items;
    for (int it = 1; it < n_items; ++it) {
        preds[np].target = (layer + 1 < L) ? layer + it : 0;
        preds[np].count = 0;
        ++np;
    }
    for (int b = 0; b < B; ++b) {
        const int r0w = b * 4;
        singles += sgl[r0w] != 0;
        for (int it = 1; it < n_items; ++it) stats_.router_exact += exact_used[r0w + it] != 0;
        for (int k = 0; k < cnt[r0w]; ++k) {
            const int e = sel[r0w * K + k];
            bool seen = false;
            for (int q = 0; q < d.count; ++q) seen |= d.experts[q] == e;
            if (!seen) d.experts[d.count++] = e;
        }
        for (int it = 1; it < n_items; ++it) {
            RoutePrediction& pr = preds[it - 1];
            for (int k = 0; k < cnt[r0w + it]; ++k) {
                const int e = sel[(r0w + it) * K + k];
                bool seen = false;
                for (int q = 0; q < pr.count; ++q) seen |= pr.experts[q] == e;
                if (!seen) pr.experts[pr.count++] = e;
            }
        }
        if (B > 1) {
            cur_cnt_[b] = cnt[r0w];
            for (int k = 0; k < K; ++k) cur_sel_[b * K + k] = k < cnt[r0w] ? sel[r0w * K + k] : -1;
        }
    }
    d.single = B == 1 && sgl[0] != 0;
    cur_x_ = x;
    cur_res_ = x;
    cur_scores_ = scores ? scores : d_free_scores_.as<double>();
    cur_score_stride_ = scores ? N : 4 * N;
    cur_out_ = out;
    cur_out_base_ = out;
    cur_x_stride_ = D;
    cur_out_stride_ = D;
    cur_residual_ = add_input ? 1 : 0;
    fuse_next_res_ = fuse_next_norm_ = nullptr;
    policy_->step(tok, layer, d, std::span<const RoutePrediction>(preds.data(), np), B > 1 ? singles : -1);
    if (user != cs) {  // this layer's output -> the caller's consumer
        MOE_CUDA(cudaEventRecord(user_out_, cs));
        MOE_CUDA(cudaStreamWaitEvent(user, user_out_, 0));
    }
    stats_.host_step_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
    if (++next_layer_ == L) {
        next_layer_ = 0;
        ++tokens_done_;
        stats_.tokens += B;
    }
}

void DecodeSession::record_timeline(bool on) {
    eng_.activate();
    if (on == record_) return;
    snapshot();  // fold what ran so far into the counters (untagged)
    if (on) {
        if (!origin_) MOE_CUDA(cudaEventCreate(&origin_));
        MOE_CUDA(cudaEventRecord(origin_, eng_.compute_stream()));
        copier_->record_tiles(origin_, &phys_copies_);
    } else {
        copier_->record_tiles(nullptr, nullptr);
    }
    record_ = on;
}

namespace {
void json_escape_free_line(std::string& o, const char* stream, const char* kind, double start_ms, double end_ms, int expert,
                           int token, int layer, int tile) {
    char buf[256];
    std::snprintf(buf, sizeof buf,
                  "{\"stream\": \"%s\", \"kind\": \"%s\", \"start\": %.3f, \"end\": %.3f, \"expert\": %d, "
                  "\"token\": %d, \"layer\": %d, \"tile\": %d",
                  stream, kind, start_ms * 1e3, end_ms * 1e3, expert, token, layer, tile);
    o += buf;
}
}  // namespace

long long DecodeSession::write_timeline(const std::string& path) {
    eng_.activate();
    if (!origin_) fail(Status::Usage, "timeline_write: recording was never enabled (moe_decode_record_timeline)");
    copier_->drain();
    MOE_CUDA(cudaDeviceSynchronize());
    copier_->collect_landed();  // tiles of jobs still holding slots
    snapshot();
    struct Line {
        double start;
        std::string text;
    };
    std::vector<Line> lines;
    lines.reserve(phys_copies_.size() + phys_compute_.size());
    char buf[256];
    for (const TileCopyRecord& r : phys_copies_) {
        std::string o;
        json_escape_free_line(o, "comm", "tile_transfer", r.start_ms, r.end_ms, r.expert, r.token, r.layer, r.tile);
        std::snprintf(buf, sizeof buf, ", \"request\": \"%s\", \"promoted\": %s, \"evicts\": %d, \"job\": %lld}",
                      r.on_demand ? "on_demand" : "prefetch", r.promoted ? "true" : "false", r.evicts, r.serial);
        o += buf;
        lines.push_back(Line{r.start_ms, std::move(o)});
    }
    for (const PhysCompute& c : phys_compute_) {
        std::string o;
        if (c.kind == 0) {
            json_escape_free_line(o, "compute", c.resident ? "expert_compute" : "tile_compute", c.start_ms, c.end_ms,
                                  c.expert, c.token, c.layer, c.tile);
            std::snprintf(buf, sizeof buf, ", \"launch\": %lld, \"fill\": %lld}", c.launch, c.fill);
        } else if (c.kind == 1) {
            json_escape_free_line(o, "compute", "wait", c.start_ms, c.end_ms, c.expert, c.token, c.layer, c.tile);
            std::snprintf(buf, sizeof buf, ", \"job\": %lld}", c.fill);
        } else {
            json_escape_free_line(o, speculate_ ? "router" : "compute", "gate", c.start_ms, c.end_ms, -1, c.token, -1, -1);
            std::snprintf(buf, sizeof buf, "}");
        }
        o += buf;
        lines.push_back(Line{c.start_ms, std::move(o)});
    }
    std::stable_sort(lines.begin(), lines.end(), [](const Line& a, const Line& b) { return a.start < b.start; });
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) fail(Status::Io, "timeline_write: cannot open " + path);
    for (const Line& l : lines) {
        std::fputs(l.text.c_str(), f);
        std::fputc('\n', f);
    }
    if (std::fclose(f) != 0) fail(Status::Io, "timeline_write: cannot write " + path);
    return static_cast<long long>(lines.size());
}

}  // namespace adapmoe
