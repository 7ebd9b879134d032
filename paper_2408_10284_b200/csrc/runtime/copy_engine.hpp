// Physical transfer channel: host -> HBM expert tile copies on one dedicated copy stream, driven
// by a host thread.  It mirrors the reference CommEngine's rules (inc/simulator.hpp:187-320) in
// real time: on-demand requests go before queued prefetches, a promoted prefetch moves to the
// on-demand queue, and work already handed to the DMA engine is never pre-empted.  Copies are
// issued in <= kChunkBytes pieces with at most kWindow pieces outstanding, so an on-demand
// request waits behind at most ~kWindow*kChunkBytes of prefetch traffic while the link never
// idles.  Each tile's completion is a CUDA event the compute stream waits on.
#pragma once

#include <cuda_runtime_api.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../kernels/xb12.hpp"
#include "../kernels/xbh.hpp"

namespace adapmoe {

// One tile's source in the pinned store: raw bf16 (format 0, copied straight into the slot) or an
// XB12 / XBH record (copied into an HBM staging buffer, then decoded into the slot,
// kernels/xb12.hpp, kernels/xbh.hpp).
struct TileSource {
    const unsigned char* src = nullptr;
    size_t bytes = 0;
    Xb12Tile meta;
};

struct CopyJob {
    unsigned char* dst = nullptr;
    size_t tile_bytes = 0;  // destination stride (decoded bf16 tile)
    int tiles = 0;
    std::vector<TileSource> srcs;  // per tile
    bool on_demand = false;
    bool logical_prefetch = false;  // a prefetch the logical engine never promoted (accounting class)
    bool consumed = false;          // the compute stream waited on (used) its tiles
    // progress (guarded by the engine mutex)
    int next_tile = 0;      // next tile to hand to the DMA engine
    int issued_tiles = 0;   // tiles whose completion event has been recorded
    bool cancelled = false;
    bool queued = false;
    std::vector<cudaEvent_t> done;     // per tile, sync events
    std::vector<cudaEvent_t> t_start;  // per tile, timing
    std::vector<cudaEvent_t> t_end;
    // physical timeline tags (set by the decode session): job serial, the request's expert and the
    // token at which it was made, promotion to on-demand, the expert its insert evicted (-1 none)
    long long serial = -1;
    int token = -1, layer = -1, expert = -1, evicts = -1;
    bool requested_on_demand = false, promoted = false;
    int recorded_tiles = 0;  // tiles already appended to the timeline records
    std::vector<long long> issue_seq;  // per tile: global issue order on the (serial) link, -1 = not issued
};

// One landed tile copy, for the physical timeline (times in ms from the recorder's origin event).
struct TileCopyRecord {
    long long serial;
    int token, layer, expert, tile, evicts;
    bool on_demand, promoted;
    double start_ms, end_ms;
};

class CopyEngine {
public:
    static constexpr size_t kChunkBytes = 32ull << 20;
    static constexpr int kWindow = 2;

    // staging_bytes > 0: XB12 records land in kStaging HBM buffers of that size and a decode stream
    // expands them into the destination (the tile's `done` event follows the decode)
    CopyEngine(cudaStream_t stream, int device, size_t staging_bytes = 0);
    ~CopyEngine();

    std::shared_ptr<CopyJob> make_job(unsigned char* dst, size_t tile_bytes, std::vector<TileSource> srcs);
    void submit(const std::shared_ptr<CopyJob>& job, bool on_demand);
    void promote(const std::shared_ptr<CopyJob>& job, bool to_front);
    // Drop tiles not yet handed to the DMA engine (their data is no longer needed).
    void cancel(const std::shared_ptr<CopyJob>& job);
    // Block until `tile` of `job` has been issued; returns its completion event.
    cudaEvent_t wait_issued(const std::shared_ptr<CopyJob>& job, int tile);
    bool fully_issued(const std::shared_ptr<CopyJob>& job);
    // No tile of `job` is being handed to the DMA engine and every issued tile has landed: its
    // events may be recycled (retire).  Call after cancel(): the copy thread takes no new tile.
    bool idle(const std::shared_ptr<CopyJob>& job);
    // Every tile of `job` has been issued and has landed in HBM (no stream wait needed).
    bool landed(const std::shared_ptr<CopyJob>& job);
    void drain();  // wait for the queues and the stream to empty

    long long tiles_copied() const { return tiles_copied_.load(); }
    long long bytes_copied() const { return bytes_copied_.load(); }
    double busy_ms();        // sum of per-tile copy durations of retired jobs
    // ... plus every completed tile of live jobs; optionally the logical-prefetch share (ms, tiles)
    // and the part of it whose jobs were consumed by the compute stream
    double busy_ms_total(double* prefetch_ms = nullptr, long long* prefetch_tiles = nullptr,
                         double* prefetch_used_ms = nullptr);
    void retire(const std::shared_ptr<CopyJob>& job);  // accumulate timing + recycle events
    // Coded-tile decode kernels so far (CUDA events around each decode on the decode stream):
    // summed duration, launches, and bytes (record read + bf16 tile written).  Waits for none.
    void decode_totals(double* ms, long long* launches, double* bytes, long long* kernels = nullptr);
    // Physical timeline: from now on every retired tile is appended to `out` with its copy interval
    // relative to `origin` (a timed event recorded on the device); nullptr stops recording.
    // Append the landed, not yet recorded tiles of jobs that have not retired (they still hold slots).
    void collect_landed();
    void record_tiles(cudaEvent_t origin, std::vector<TileCopyRecord>* out) {
        std::lock_guard<std::mutex> g(mu_);
        origin_ = origin;
        records_ = out;
    }

private:
    void loop();
    void run();
    void record_tile(CopyJob& job, int t);
    void fail_thread(const std::string& what);
    void throw_if_failed() const;  // caller holds mu_
    cudaEvent_t take_event(bool timing);

    cudaStream_t stream_;
    int device_;
    static constexpr int kStaging = 3;
    cudaStream_t decode_stream_ = nullptr;
    void* staging_[kStaging] = {};
    size_t staging_bytes_ = 0;
    cudaEvent_t staging_landed_[kStaging] = {}, staging_free_[kStaging] = {};
    struct DecodeTiming {
        cudaEvent_t start, end;
        double bytes;
    };
    std::deque<DecodeTiming> dec_pending_;  // guarded by mu_
    double dec_ms_ = 0.0, dec_bytes_ = 0.0;
    long long dec_launches_ = 0;
    std::atomic<long long> dec_kernels_{0};  // decode + escape-patch kernel launches
    void harvest_decodes();  // caller holds mu_: fold completed decode timings into the totals
    int staging_next_ = 0;
    std::mutex mu_;
    std::condition_variable cv_work_, cv_issued_;
    std::deque<std::shared_ptr<CopyJob>> od_, pf_;
    std::deque<cudaEvent_t> inflight_;
    std::vector<cudaEvent_t> free_sync_, free_timing_;
    std::vector<std::shared_ptr<CopyJob>> active_;
    bool stop_ = false;
    bool busy_ = false;
    std::string error_;  // first error of the copy thread (it stops issuing)
    std::atomic<long long> tiles_copied_{0}, bytes_copied_{0};
    long long issue_counter_ = 0;  // guarded by mu_
    double busy_ms_ = 0.0, busy_pf_ms_ = 0.0, busy_pf_used_ms_ = 0.0;
    long long pf_tiles_ = 0;
    cudaEvent_t origin_ = nullptr;
    std::vector<TileCopyRecord>* records_ = nullptr;
    std::thread thread_;
};

}  // namespace adapmoe
