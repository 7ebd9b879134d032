// Physical offloaded decode: the HBM expert-slot pool, the copy engine and the per-layer K1 + K2
// launches, driven by the logical PolicyEngine (host/policy_engine.hpp) as its DecodeListener.
//
// Logical -> physical mapping
//   request enqueued      -> take a free HBM slot, queue its tile copies (od or pf priority)
//   request promoted      -> move its remaining tiles to the on-demand queue
//   cache insert          -> the request's slot becomes the expert's resident slot; the evicted
//                            expert's slot is released once the layer that last read it finished
//   resident compute      -> SwiGLU over the slot (waits only if its fill is still in flight)
//   on-demand tile compute-> wait on that tile's copy event, then SwiGLU on that tile
// The logical engine decides every hit/miss/prefetch/eviction with the reference's tick model, so
// the event trace is the reference's; wall-clock only changes when things physically happen.
//
// Batched decode (batch B > 1, BASELINE config 4): B token streams share the cache.  Each layer
// routes all B streams in one K1 launch; the logical engine sees the union of their selections
// and of their look-ahead lists (oracle/moe_oracle.c orc_simulate_batch); the FFN runs as grouped
// tcgen05 GEMMs (kernels/grouped_ffn.hpp) over the union's experts with each expert's routed
// tokens gathered, then a per-stream fixed-order weighted combine.
#pragma once

#include <cuda_runtime_api.h>

#include <array>
#include <string>
#include <memory>
#include <tuple>
#include <utility>
#include <vector>

#include "../host/policy_engine.hpp"
#include "../kernels/expert_ffn.hpp"
#include "../kernels/grouped_ffn.hpp"
#include "../kernels/router.hpp"
#include "copy_engine.hpp"
#include "engine.hpp"
#include "experts.hpp"

namespace adapmoe {

struct DecodeStats {
    long long tokens = 0, kernels = 0, ffn_launches = 0, tile_copies = 0, copy_bytes = 0, input_bytes = 0, ffn_bytes = 0;
    double copy_busy_ms = 0, ffn_ms = 0, gate_up_ms = 0, down_ms = 0, gate_up_bytes = 0, down_bytes = 0;
    double router_ms = 0, stall_ms = 0;
    long long router_launches = 0;
    // logical prefetches (never promoted to on-demand): copy time, tiles, compute-stream wait on them
    double prefetch_copy_ms = 0, prefetch_stall_ms = 0, prefetch_used_copy_ms = 0;
    long long spec_launches = 0, spec_hits = 0;  // speculative next-layer FFN launches / used ones
    long long prefetch_tiles = 0;
    long long router_exact = 0;  // look-ahead items that needed the exact fp64 path
    double host_sync_ms = 0, host_step_ms = 0;  // host wall time: waiting on K1 / policy step + launches
    int slots_total = 0, staging_high_water = 0;
    double decode_ms = 0, decode_bytes = 0;  // coded-tile decode kernels (XB12 / XBH): time, bytes
    long long decode_launches = 0;
};

class DecodeSession : public DecodeListener {
public:
    DecodeSession(Engine& eng, std::span<const int> capacities, int staging_slots, std::span<const double> fisher,
                  double tau, const SimConfig& cfg, std::uint64_t seed, int total_tokens, int batch = 1,
                  int ep_rank = 0, int ep_world = 1, bool free_running = false, double concentration = 1.0,
                  const int* expert_owner = nullptr);
    ~DecodeSession() override;

    // acts [count][B][L][d], scores [count][B][L][N]: host or device pointers
    double decode(const double* acts, const double* scores, int count, bool on_device, float* hidden_out);

    const PolicyEngine& policy() const { return *policy_; }

    // expert-parallel exchange over peer memory (kernels/ep_exchange.hpp): allocate this shard's
    // region for calls of up to max_tokens_per_call tokens; returns its device pointer and (if
    // ipc_handle) a CUDA IPC handle for other processes.
    void ep_export(int max_tokens_per_call, std::uint64_t* ptr, void* ipc_handle);
    // peer_ptrs[g] (same process) or peer_ipc[g] (64-byte IPC handles, other processes) for every
    // shard g != ep_rank; afterwards decode() returns the full (summed) layer outputs.
    void ep_connect(const std::uint64_t* peer_ptrs, const unsigned char* peer_ipc);
    DecodeStats snapshot();  // counters so far (call between decode() calls)
    DecodeStats finish();    // drain the copy engine, then snapshot

    // One MoE layer of the current token on caller device buffers, stream-ordered with `user`
    // (moe_decode_layer): x [B][d] fp64 router/expert input, scores [B][N] fp64 (stored scores:
    // the reference's actual-selection rule) or null (decide from the layer's gate on x, softmax
    // of logits / concentration), out [B][d] fp32 = (add_input ? x : 0) + sum_e w_e E_e(x).
    // Layers must come in order 0..L-1 per token; routing is per layer (K1 + one host sync).
    void decode_layer(int layer, const double* x, const double* scores, float* out, bool add_input,
                      cudaStream_t user);

    // Physical timeline (moe_decode_record_timeline / moe_decode_timeline_write): CUDA-event
    // timestamps of every tile copy (request class, promotion, eviction), FFN launch (its (expert,
    // tile) segments and the copy job each segment's weights came from), compute-stream wait and
    // router launch, relative to an origin event recorded when recording starts.
    void record_timeline(bool on);
    // Drain copies, sync, and write the events recorded so far as JSONL in the reference's
    // timeline schema (inc/io.hpp:402-417; times in microseconds) plus physical fields.
    long long write_timeline(const std::string& path);

    // DecodeListener
    void on_request(int id, ExpertRef ref, bool on_demand) override;
    void on_promote(int id) override;
    void on_insert(ExpertRef ref, int request, std::optional<int> evicted) override;
    void on_resident_compute(int token, ExpertRef ref, int rank) override;
    void on_tile_compute(int token, ExpertRef ref, int rank, int tile, int request) override;
    void on_layer_done(int token, int layer, const RouteDecision& d) override;

private:
    struct Slot {
        std::shared_ptr<CopyJob> fill;  // copy that produced the current contents (null: synchronous)
        bool fill_done = false;         // known complete (no wait needed)
    };
    struct Use {
        int rank, slot;
        bool missing;
        std::vector<int> tiles;  // missing: tiles in compute order
    };
    unsigned char* slot_ptr(int s) const { return pool_.as<unsigned char>() + static_cast<size_t>(s) * slot_stride_; }
    int take_slot();
    void release_slot(int s);
    void release_pending(bool all);
    void wait_fill(int slot, int tile);  // compute stream waits for tile (or all tiles if -1)
    // "layer" launches wait for every tile of the layer before one launch: the waits are collected
    // and enqueued in the order the tiles cross the (serial) link, so each wait's stall is the gap
    // to the next landing and is charged to the tile that really gates the launch
    bool defer_waits_ = false;
    std::vector<std::pair<int, int>> deferred_waits_;
    void flush_waits();
    // launch + time + clear the segment list; records where each (rank, tile) partial lives
    void timed_ffn(FfnLaunch& p, const std::vector<std::pair<int, int>>& seg_meta,
                   std::vector<std::tuple<int, int, FfnPartialRef>>& refs);
    void layer_ffn_single(const RouteDecision& d);   // batch 1: K2 row kernel
    std::vector<std::pair<const Use*, std::vector<int>>> tile_groups() const;
    bool tile_merge_active() const;
    bool layer_launch() const;
    bool merge_resident() const;
    int tile_merge_ = -1;  // -1 auto (tiles >= 8 MiB: 2), 0 per tile, 1 groups, 2 one launch per layer
    void layer_ffn_grouped(const RouteDecision& d);  // batch > 1: K3 grouped tcgen05 kernels
    void timed_grouped(GroupedLaunch& p, bool down, const RouteDecision& u);
    void ep_exchange(float* out, long long rows, long long row_stride);
    // free-running decode: layer l > 0 routes and computes on layer l-1's output (the hidden state
    // flows through the experts); the actual decision comes from the layer's gate (softmax of
    // logits / concentration, like the reference generator) instead of stored scores
    bool free_running_ = false;
    double concentration_ = 1.0;
    DeviceBuffer d_x_free_, d_x_norm_, d_free_scores_;
    double* fuse_next_res_ = nullptr;   // batch 1: next layer's residual / norm rows the combine forms
    double* fuse_next_norm_ = nullptr;
    DeviceBuffer d_combine_ticket_;
    static constexpr double kFreeRunningNormEps = 1e-5;  // Mixtral rms_norm_eps
    long long cur_score_stride_ = 0;
    int batch_ = 1;
    // expert parallelism: shard ep_rank_ of ep_world_ owns experts e % world == rank
    // of every layer.  The logical engine is replicated (same inputs -> same trace on every shard);
    // this shard only holds, copies and computes its own experts, and writes its partial layer
    // output (shard 0 adds the residual); the shards' partials are summed in shard order.
    int ep_rank_ = 0, ep_world_ = 1;
    DeviceBuffer d_ep_region_;
    size_t ep_rows_max_ = 0;
    int ep_max_tokens_ = 0;
    bool ep_connected_ = false;
    unsigned ep_call_ = 0;
    std::array<unsigned char*, kMaxEpPeers> ep_region_{};
    std::vector<void*> ep_ipc_opened_;
    float* ep_slot(int shard, int writer, int parity) const {
        return reinterpret_cast<float*>(ep_region_[shard] + kEpFlagBytes) +
               (static_cast<size_t>(parity) * ep_world_ + writer) * ep_rows_max_ * spec_.hidden_dim;
    }
    // shard of each (layer, expert): the caller's table (e.g. balanced by calibration traffic,
    // ep.balanced_owners) or e % world; the logical trace does not depend on it
    std::vector<int> owner_;
    bool owned(int layer, int expert) const {
        return owner_[static_cast<size_t>(layer) * spec_.experts_per_layer + expert] == ep_rank_;
    }
    int np_ = 16;                       // token rows per expert entry in X / H (B rounded up to 16)
    DeviceBuffer d_gx_, d_gh_, d_gpart_;  // X [N][NP][d], H [N][NP][F] bf16; down partial arena
    size_t gpart_next_ = 0;             // floats used in the arena this layer
    CUtensorMap map_pool_gu_{}, map_pool_dn_{}, map_x_{}, map_h_{};
    // per-stream router results of the current layer
    std::vector<int> cur_sel_, cur_cnt_;
    DeviceBuffer d_partials_;  // per-layer pool of K2 partial regions (reused every layer, stream-ordered)
    int partial_regions_ = 0, partial_next_ = 0;
    // free-running batch 1: speculative FFN of the next layer's predicted top-1 expert (the previous
    // layer's look-ahead), launched on SMs - kSpecSpareSms CTAs while K1 routes on route_stream_
    static constexpr int kSpecSpareSms = 3;
    bool speculate_ = false;
    cudaStream_t route_stream_ = nullptr;
    cudaEvent_t in_ready_ = nullptr;
    struct SpecRun {
        bool valid = false;
        long long layer_seq = -1;
        int n = 0, n_seg = 0, grid = 0;
        int slot[8] = {};            // speculated experts' slots; expert k owns segments k*T .. k*T+T-1
        float* partial = nullptr;
    } spec_run_;
    int spec_next_[8] = {};          // the look-ahead's experts for the next layer (score order)
    int spec_next_n_ = 0;
    void launch_speculative(int layer, const double* x);

    Engine& eng_;
    ModelSpec spec_;
    SimConfig cfg_;
    std::vector<int> caps_;
    std::vector<double> fisher_;
    double tau_;
    int total_tokens_;
    int tokens_done_ = 0;
    std::unique_ptr<PolicyEngine> policy_;
    std::unique_ptr<CopyEngine> copier_;
    ExpertStore& store_;
    int sm_count_ = 148;

    // slots
    DeviceBuffer pool_;
    DeviceBuffer fill_staging_;  // XB12 records of the initial residency (decoded on the compute stream)
    size_t slot_stride_ = 0;
    int n_slots_ = 0;
    int resident_slots_ = 0;
    std::vector<Slot> slots_;
    std::deque<int> free_;
    std::vector<std::pair<long long, int>> pending_free_;  // (layer sequence, slot)
    std::vector<std::shared_ptr<CopyJob>> retiring_;      // released fills awaiting event recycling
    std::vector<int> slot_of_;                             // [L*N] resident expert -> slot
    std::vector<int> req_slot_;
    std::vector<std::shared_ptr<CopyJob>> req_job_;
    long long layer_seq_ = 0;  // global (token, layer) counter of on_layer_done calls
    int in_use_high_ = 0;

    // per-layer work
    std::vector<Use> uses_;
    const double* cur_x_ = nullptr;    // router / expert input of the current layer
    const double* cur_res_ = nullptr;  // residual added by the combine (== cur_x_ in trace replay)
    const double* cur_scores_ = nullptr;
    float* cur_out_ = nullptr;
    float* cur_out_base_ = nullptr;  // out buffer of the current decode call (row offsets for the EP slots)

    // buffers
    DeviceBuffer d_in_acts_, d_in_scores_, d_out_, d_groups_;
    DeviceBuffer d_route_scratch_;  // K1 split launch: F / A per group + tickets
    RouteScratch route_scratch_;
    PinnedBuffer h_groups_;
    // mapped pinned K1 outputs: selected [R][K], count [R], single [R], exact [R] with R = 4 rows per
    // group; free-running routes one layer per launch (R = 4B), trace replay a window of
    // route_window_ tokens per launch (R = 4B * L * window)
    int* h_route_ = nullptr;
    int* d_route_ = nullptr;
    // K1 host-decision queue (kernels/router.hpp RouteOutputs::host_entries): exact logits of the
    // uncertified items, decided on the host with libm exp right after each route sync
    PinnedBuffer h_route_host_;
    DeviceBuffer d_route_counter_;
    int route_host_cap_ = 0;
    int route_window_ = 1;
    cudaEvent_t route_done_ = nullptr;
    cudaEvent_t user_in_ = nullptr, user_out_ = nullptr;  // moe_decode_layer: caller stream <-> compute stream
    // completion of each layer's FFN + combine on the compute stream: a slot released by layer s is
    // reused only after the event of layer s has completed (trace replay routes ahead of the GPU, so
    // there is no per-layer host synchronisation to order slot reuse)
    std::deque<std::pair<long long, cudaEvent_t>> layer_events_;
    std::vector<cudaEvent_t> layer_event_pool_;
    long long layers_complete_ = 0;  // every layer with sequence < this has completed on the GPU
    std::vector<cudaEvent_t> timing_pool_;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> router_events_, stall_events_;
    std::vector<char> stall_is_prefetch_;  // per stall_events_ entry: waited on a logical prefetch
    // physical timeline
    struct SegInfo {
        int expert, tile;
        long long fill;  // copy job serial of the slot's contents (-1: initial residency)
        bool resident;
    };
    struct PhysCompute {
        int kind;  // 0 FFN launch segment, 1 compute-stream wait on a tile copy, 2 router launch
        double start_ms, end_ms;
        int token, layer, expert, tile;
        long long launch, fill;
        bool resident;
    };
    bool record_ = false;
    cudaEvent_t origin_ = nullptr;
    long long job_serial_ = 0, launch_serial_ = 0;
    int cur_token_ = -1, cur_layer_ = -1;
    std::vector<SegInfo> seg_info_;  // segments of the launch being assembled (record_ only)
    std::vector<PhysCompute> phys_compute_;
    std::vector<TileCopyRecord> phys_copies_;
    struct StallTag {
        int token, layer, expert, tile;
        long long job;
    };
    std::vector<StallTag> stall_tags_;
    std::vector<int> router_tokens_;
    long long fill_serial(int slot) const { return slots_[slot].fill ? slots_[slot].fill->serial : -1; }
    void note_seg(int slot, int expert, int tile, bool resident) {
        if (record_) seg_info_.push_back(SegInfo{expert, tile, fill_serial(slot), resident});
    }
    // per-layer entry state
    int next_layer_ = 0;
    long long cur_x_stride_ = 0, cur_out_stride_ = 0;  // stream strides (doubles / floats) of cur_x_ / cur_out_
    int cur_residual_ = 1;
    struct PassRec {
        double gate_up_bytes, down_bytes;
        cudaEvent_t e0, e1;
        int token = -1, layer = -1;
        long long launch = -1;
        std::vector<SegInfo> segs;
    };
    std::vector<PassRec> pass_events_;
    cudaEvent_t take_timing();
    DecodeStats stats_;
};

}  // namespace adapmoe
