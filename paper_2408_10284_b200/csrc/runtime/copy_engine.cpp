#include "copy_engine.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "../host/policy.hpp"
#include "nvtx.hpp"

namespace adapmoe {

namespace {
void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(Status::Device, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

CopyEngine::CopyEngine(cudaStream_t stream, int device, size_t staging_bytes)
    : stream_(stream), device_(device), staging_bytes_(staging_bytes) {
    if (staging_bytes_) {
        check(cudaStreamCreateWithFlags(&decode_stream_, cudaStreamNonBlocking), "cudaStreamCreate (xb12 decode)");
        for (int k = 0; k < kStaging; ++k) {
            check(cudaMalloc(&staging_[k], staging_bytes_), "cudaMalloc (xb12 staging)");
            check(cudaEventCreateWithFlags(&staging_landed_[k], cudaEventDisableTiming), "cudaEventCreate");
            check(cudaEventCreateWithFlags(&staging_free_[k], cudaEventDisableTiming), "cudaEventCreate");
        }
    }
    thread_ = std::thread([this] { loop(); });
}

CopyEngine::~CopyEngine() {
    {
        std::lock_guard<std::mutex> g(mu_);
        stop_ = true;
    }
    cv_work_.notify_all();
    if (thread_.joinable()) thread_.join();
    cudaSetDevice(device_);
    cudaStreamSynchronize(stream_);
    std::vector<std::shared_ptr<CopyJob>> left;
    left.swap(active_);  // retire() edits active_
    for (auto& j : left) retire(j);
    for (cudaEvent_t e : inflight_) cudaEventDestroy(e);
    if (decode_stream_) cudaStreamSynchronize(decode_stream_);
    for (const DecodeTiming& d : dec_pending_) {  // decode timings never harvested
        cudaEventDestroy(d.start);
        cudaEventDestroy(d.end);
    }
    for (cudaEvent_t e : free_sync_) cudaEventDestroy(e);
    for (cudaEvent_t e : free_timing_) cudaEventDestroy(e);
    if (decode_stream_) {
        for (int k = 0; k < kStaging; ++k) {
            cudaFree(staging_[k]);
            cudaEventDestroy(staging_landed_[k]);
            cudaEventDestroy(staging_free_[k]);
        }
        cudaStreamDestroy(decode_stream_);
    }
}

cudaEvent_t CopyEngine::take_event(bool timing) {
    std::vector<cudaEvent_t>& pool = timing ? free_timing_ : free_sync_;
    if (!pool.empty()) {
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    check(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming), "cudaEventCreate");
    return e;
}

std::shared_ptr<CopyJob> CopyEngine::make_job(unsigned char* dst, size_t tile_bytes, std::vector<TileSource> srcs) {
    auto j = std::make_shared<CopyJob>();
    j->dst = dst;
    j->tile_bytes = tile_bytes;
    j->tiles = static_cast<int>(srcs.size());
    j->srcs = std::move(srcs);
    const int tiles = j->tiles;
    j->issue_seq.assign(tiles, -1);
    for (const TileSource& t : j->srcs)
        if (t.meta.format != 0 && (!staging_bytes_ || t.bytes > staging_bytes_))
            fail(Status::Internal, "copy engine: coded record larger than the staging buffers");
    std::lock_guard<std::mutex> g(mu_);
    for (int t = 0; t < tiles; ++t) {
        j->done.push_back(take_event(false));
        j->t_start.push_back(take_event(true));
        j->t_end.push_back(take_event(true));
    }
    active_.push_back(j);
    return j;
}

void CopyEngine::submit(const std::shared_ptr<CopyJob>& job, bool on_demand) {
    {
        std::lock_guard<std::mutex> g(mu_);
        job->on_demand = on_demand;
        job->logical_prefetch = !on_demand;
        job->queued = true;
        (on_demand ? od_ : pf_).push_back(job);
    }
    cv_work_.notify_one();
}

void CopyEngine::promote(const std::shared_ptr<CopyJob>& job, bool to_front) {
    std::lock_guard<std::mutex> g(mu_);
    if (!job->queued) return;
    auto it = std::find(pf_.begin(), pf_.end(), job);
    if (it != pf_.end()) {
        pf_.erase(it);
    } else {
        if (!to_front) return;
        auto jt = std::find(od_.begin(), od_.end(), job);
        if (jt != od_.end()) od_.erase(jt);
    }
    job->on_demand = true;
    if (to_front)
        od_.push_front(job);
    else
        od_.push_back(job);
}

void CopyEngine::cancel(const std::shared_ptr<CopyJob>& job) {
    std::lock_guard<std::mutex> g(mu_);
    job->cancelled = true;
    if (job->queued) {
        auto& q = job->on_demand ? od_ : pf_;
        auto it = std::find(q.begin(), q.end(), job);
        if (it != q.end()) q.erase(it);
        job->queued = false;
    }
    cv_issued_.notify_all();
}

cudaEvent_t CopyEngine::wait_issued(const std::shared_ptr<CopyJob>& job, int tile) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_issued_.wait(lk, [&] {
        return job->issued_tiles > tile || (job->cancelled && job->next_tile <= tile) || stop_ || !error_.empty();
    });
    throw_if_failed();
    if (job->issued_tiles <= tile) fail(Status::Internal, "copy engine: waited on a tile that will never be copied");
    return job->done[tile];
}

bool CopyEngine::fully_issued(const std::shared_ptr<CopyJob>& job) {
    std::lock_guard<std::mutex> g(mu_);
    return job->issued_tiles == job->tiles;
}

bool CopyEngine::idle(const std::shared_ptr<CopyJob>& job) {
    std::lock_guard<std::mutex> g(mu_);
    if (job->next_tile != job->issued_tiles) return false;  // the copy thread is issuing a tile
    // `done` follows the tile's decode (XB12) and its copy: once it completed, no stream still records
    // or waits on this job's events
    return job->issued_tiles == 0 || (cudaEventQuery(job->t_end[job->issued_tiles - 1]) == cudaSuccess &&
                                      cudaEventQuery(job->done[job->issued_tiles - 1]) == cudaSuccess);
}

bool CopyEngine::landed(const std::shared_ptr<CopyJob>& job) {
    std::lock_guard<std::mutex> g(mu_);
    return job->issued_tiles == job->tiles && cudaEventQuery(job->done[job->tiles - 1]) == cudaSuccess;
}

void CopyEngine::drain() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_issued_.wait(lk, [&] { return (od_.empty() && pf_.empty() && !busy_) || stop_ || !error_.empty(); });
    throw_if_failed();
    lk.unlock();
    check(cudaStreamSynchronize(stream_), "copy stream sync");
    if (decode_stream_) check(cudaStreamSynchronize(decode_stream_), "xb12 decode stream sync");
}

double CopyEngine::busy_ms() {
    std::lock_guard<std::mutex> g(mu_);
    return busy_ms_;
}

double CopyEngine::busy_ms_total(double* prefetch_ms, long long* prefetch_tiles, double* prefetch_used_ms) {
    std::lock_guard<std::mutex> g(mu_);
    double total = busy_ms_, pf = busy_pf_ms_, pf_used = busy_pf_used_ms_;
    long long pft = pf_tiles_;
    for (const auto& job : active_)
        for (int t = 0; t < job->issued_tiles; ++t)
            if (cudaEventQuery(job->t_end[t]) == cudaSuccess) {
                float ms = 0.0f;
                if (cudaEventElapsedTime(&ms, job->t_start[t], job->t_end[t]) == cudaSuccess) {
                    total += ms;
                    if (job->logical_prefetch) {
                        pf += ms;
                        ++pft;
                        if (job->consumed) pf_used += ms;
                    }
                }
            }
    if (prefetch_ms) *prefetch_ms = pf;
    if (prefetch_used_ms) *prefetch_used_ms = pf_used;
    if (prefetch_tiles) *prefetch_tiles = pft;
    return total;
}

void CopyEngine::harvest_decodes() {
    while (!dec_pending_.empty() && cudaEventQuery(dec_pending_.front().end) == cudaSuccess) {
        const DecodeTiming& d = dec_pending_.front();
        float ms = 0.0f;
        if (cudaEventElapsedTime(&ms, d.start, d.end) == cudaSuccess) {
            dec_ms_ += ms;
            dec_bytes_ += d.bytes;
            ++dec_launches_;
        }
        free_timing_.push_back(d.start);
        free_timing_.push_back(d.end);
        dec_pending_.pop_front();
    }
}

void CopyEngine::decode_totals(double* ms, long long* launches, double* bytes, long long* kernels) {
    std::lock_guard<std::mutex> g(mu_);
    harvest_decodes();
    if (kernels) *kernels = dec_kernels_.load();
    if (ms) *ms = dec_ms_;
    if (launches) *launches = dec_launches_;
    if (bytes) *bytes = dec_bytes_;
}

void CopyEngine::retire(const std::shared_ptr<CopyJob>& job) {
    std::lock_guard<std::mutex> g(mu_);
    for (int t = 0; t < job->issued_tiles; ++t) {
        if (cudaEventSynchronize(job->t_end[t]) == cudaSuccess) {
            float ms = 0.0f;
            if (cudaEventElapsedTime(&ms, job->t_start[t], job->t_end[t]) == cudaSuccess) {
                busy_ms_ += ms;
                if (job->logical_prefetch) {
                    busy_pf_ms_ += ms;
                    ++pf_tiles_;
                    if (job->consumed) busy_pf_used_ms_ += ms;
                }
            }
            if (t >= job->recorded_tiles) record_tile(*job, t);
        }
    }
    for (cudaEvent_t e : job->done) free_sync_.push_back(e);
    for (cudaEvent_t e : job->t_start) free_timing_.push_back(e);
    for (cudaEvent_t e : job->t_end) free_timing_.push_back(e);
    job->done.clear();
    job->t_start.clear();
    job->t_end.clear();
    auto it = std::find(active_.begin(), active_.end(), job);
    if (it != active_.end()) active_.erase(it);
}

void CopyEngine::record_tile(CopyJob& job, int t) {  // caller holds mu_; the tile has landed
    float a = 0.0f, b = 0.0f;
    if (records_ && origin_ && cudaEventElapsedTime(&a, origin_, job.t_start[t]) == cudaSuccess &&
        cudaEventElapsedTime(&b, origin_, job.t_end[t]) == cudaSuccess) {
        if (a >= 0.0f)  // copies that started before recording began are not part of the timeline
            records_->push_back(TileCopyRecord{job.serial, job.token, job.layer, job.expert, t, job.evicts,
                                               job.requested_on_demand, job.promoted, a, b});
        job.recorded_tiles = t + 1;
    }
}

void CopyEngine::collect_landed() {
    std::lock_guard<std::mutex> g(mu_);
    for (const auto& job : active_)
        for (int t = job->recorded_tiles; t < job->issued_tiles; ++t)
            if (cudaEventQuery(job->t_end[t]) == cudaSuccess) record_tile(*job, t);
}

// The copy thread never throws: a CUDA error (or any exception) is recorded, every waiter is woken
// and the host thread raises it (MOE_E_DEVICE) from wait_issued / drain.
void CopyEngine::loop() {
    try {
        run();
    } catch (const std::exception& e) {
        fail_thread(e.what());
    } catch (...) {
        fail_thread("copy engine: unknown error");
    }
}

void CopyEngine::fail_thread(const std::string& what) {
    {
        std::lock_guard<std::mutex> g(mu_);
        if (error_.empty()) error_ = what;
    }
    cv_issued_.notify_all();
}

void CopyEngine::throw_if_failed() const {
    if (!error_.empty()) fail(Status::Device, "copy engine: " + error_);
}

void CopyEngine::run() {
    auto ck = [](cudaError_t e, const char* what) {
        if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
    };
    ck(cudaSetDevice(device_), "cudaSetDevice");
    // test knob: fail after this many tiles (exercises the error path end to end)
    const char* fault = std::getenv("ADAPMOE_COPY_FAULT_AFTER");
    const long long fault_after = fault ? std::atoll(fault) : -1;
    for (;;) {
        std::shared_ptr<CopyJob> job;
        int tile = 0;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_work_.wait(lk, [&] { return stop_ || !od_.empty() || !pf_.empty(); });
            if (stop_) return;
            auto& q = !od_.empty() ? od_ : pf_;
            job = q.front();
            tile = job->next_tile++;
            job->issue_seq[tile] = issue_counter_++;
            if (job->next_tile == job->tiles) {
                q.pop_front();
                job->queued = false;
            }
            busy_ = true;
        }
        if (fault_after >= 0 && tiles_copied_.load() >= fault_after) throw std::runtime_error("injected copy fault");
        NvtxRange copy_range("copy L%d E%d tile %d (%s)", job->layer, job->expert, tile, job->on_demand ? "od" : "pf");
        const TileSource& src = job->srcs[tile];
        unsigned char* out = job->dst + static_cast<size_t>(tile) * job->tile_bytes;
        const bool coded = src.meta.format != 0;
        const int k = coded ? staging_next_ : -1;
        if (coded) {  // the staging buffer is free once the decode that last read it has run
            staging_next_ = (staging_next_ + 1) % kStaging;
            ck(cudaStreamWaitEvent(stream_, staging_free_[k], 0), "cudaStreamWaitEvent");
        }
        unsigned char* land = coded ? static_cast<unsigned char*>(staging_[k]) : out;
        ck(cudaEventRecord(job->t_start[tile], stream_), "cudaEventRecord");
        for (size_t off = 0; off < src.bytes; off += kChunkBytes) {
            while (static_cast<int>(inflight_.size()) >= kWindow) {
                ck(cudaEventSynchronize(inflight_.front()), "tile copy");
                std::lock_guard<std::mutex> g(mu_);
                free_sync_.push_back(inflight_.front());
                inflight_.pop_front();
            }
            const size_t n = std::min(kChunkBytes, src.bytes - off);
            ck(cudaMemcpyAsync(land + off, src.src + off, n, cudaMemcpyHostToDevice, stream_),
               "cudaMemcpyAsync (expert tile)");
            cudaEvent_t e;
            {
                std::lock_guard<std::mutex> g(mu_);
                e = take_event(false);
            }
            ck(cudaEventRecord(e, stream_), "cudaEventRecord");
            inflight_.push_back(e);
        }
        ck(cudaEventRecord(job->t_end[tile], stream_), "cudaEventRecord");
        if (coded) {  // decode on its own stream so the link never waits for it
            ck(cudaEventRecord(staging_landed_[k], stream_), "cudaEventRecord");
            ck(cudaStreamWaitEvent(decode_stream_, staging_landed_[k], 0), "cudaStreamWaitEvent");
            const std::uint8_t* rec = static_cast<const std::uint8_t*>(staging_[k]);
            std::uint16_t* dec = reinterpret_cast<std::uint16_t*>(out);
            DecodeTiming dt{};
            {
                std::lock_guard<std::mutex> g(mu_);
                harvest_decodes();
                dt.start = take_event(true);
                dt.end = take_event(true);
            }
            dt.bytes = static_cast<double>(src.bytes) + 2.0 * static_cast<double>(src.meta.n);
            ck(cudaEventRecord(dt.start, decode_stream_), "cudaEventRecord");
            ck(src.meta.format == 2 ? xbh_decode(rec, src.meta, dec, decode_stream_)
                                    : xb12_decode(rec, src.meta, dec, decode_stream_),
               "tile record decode");
            dec_kernels_ += src.meta.n_exc ? 2 : 1;
            ck(cudaEventRecord(dt.end, decode_stream_), "cudaEventRecord");
            {
                std::lock_guard<std::mutex> g(mu_);
                dec_pending_.push_back(dt);
            }
            ck(cudaEventRecord(job->done[tile], decode_stream_), "cudaEventRecord");
            ck(cudaEventRecord(staging_free_[k], decode_stream_), "cudaEventRecord");
        } else {
            ck(cudaEventRecord(job->done[tile], stream_), "cudaEventRecord");
        }
        tiles_copied_ += 1;
        bytes_copied_ += static_cast<long long>(src.bytes);
        {
            std::lock_guard<std::mutex> g(mu_);
            job->issued_tiles = tile + 1;
            busy_ = false;
        }
        cv_issued_.notify_all();
    }
}

}  // namespace adapmoe
