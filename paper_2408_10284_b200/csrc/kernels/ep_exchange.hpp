// Expert-parallel exchange over peer memory (NVLink P2P / same-device peers), replacing a host-side
// all_gather of the shards' partial layer outputs.
//
// Every shard owns one exchange region (exported as a raw pointer for same-process peers or a CUDA
// IPC handle for other processes):
//   [flags: kMaxEpPeers x 64 B]  flag[r] = last decode call whose partials shard r has stored here
//   [slots: 2 (call parity) x G (writer shard) x rows_max x d floats]
// During a decode call the combine kernels of shard r store each layer's partial output straight
// into slot (parity, r) of EVERY shard's region (the P2P stores are the combine's epilogue).  At
// the end of the call shard r publishes flag[r] = call on every region (release, system scope);
// each shard's wait kernel (one warp) acquires until all flags reach the call, then its reduce
// kernel sums the G slots in shard order into its output — the same bits on every shard.  Double-buffering by call
// parity makes slot reuse safe: a shard can only write call c+2 after its reduce of call c+1, which
// needed every peer's call-c+1 flag, which each peer sets after its own reduce of call c.
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>

namespace adapmoe {

constexpr int kMaxEpPeers = 8;
constexpr size_t kEpFlagBytes = 64 * (kMaxEpPeers + 1);  // flags, then the wait-timeout word

struct EpSignalArgs {
    unsigned* peer_flags[kMaxEpPeers];  // flags array of each shard's region
    int world = 0, rank = 0;
    unsigned call = 0;
};
cudaError_t launch_ep_signal(const EpSignalArgs& a, cudaStream_t stream);

// One warp waits (acquire, system scope) until every shard's flag in this region reaches `call`;
// bounded (~20 s): on timeout it sets the region's timeout word and gives up.  A running 1-warp
// kernel never blocks other streams (a stream-level wait-value can stall every stream that shares
// its hardware queue, which deadlocks shards that share a GPU); the big FFN kernels of a connected
// session use SMs - 1 CTAs so the waiter can never starve a peer's grid of an SM.
cudaError_t launch_ep_wait(const unsigned char* region, int world, unsigned call, cudaStream_t stream);

struct EpReduceArgs {
    const float* slots = nullptr;     // writer 0's slot at the rows' offset (this shard's region, parity)
    long long slot_stride = 0;        // floats between writer slots
    float* out = nullptr;             // rows of d floats, row_stride apart (same offsets in the slots)
    long long rows = 0, row_stride = 0;
    int d = 0;
    int world = 0;
};
cudaError_t launch_ep_reduce(const EpReduceArgs& a, cudaStream_t stream);

}  // namespace adapmoe
