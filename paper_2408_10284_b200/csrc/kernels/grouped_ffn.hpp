// K3 — grouped SwiGLU expert FFN for batched decode on the 5th-gen tensor cores (host interface).
//
// Batched decode (BASELINE config 4) routes B tokens per layer; expert e receives the n_e tokens
// whose selection contains it.  Per expert the FFN is two dense contractions,
//   gate/up : G_e [2Ft, n_e] = W13_e [2Ft, d] . X_e^T [d, n_e]   (per tile, rows interleaved W1/W3)
//   down    : Y_e [d, n_e]   = W2_e [d, F]    . H_e^T [F, n_e],  H = silu(G_W1) * G_W3 (bf16)
// both issued "swap-AB": weights are the MMA's M side (128 rows per tcgen05.mma), tokens the N
// side (n_e rounded up to 16), accumulators in TMEM.  Every weight byte is read once per layer, so
// the launch is HBM-bound (~n_e flop/byte); the tensor pipe only has to keep up with the stream.
//
// Operand sources (all TMA, 128-byte swizzle, `cp.async.bulk.tensor.2d`):
//   * weights: the whole HBM slot pool viewed as one 2-D bf16 tensor [rows][d] — the tile-major
//     expert layout (expert_ffn.hpp) makes every gate/up row and every W2^T row a d-element row, so
//     one tensor map covers every slot.  gate/up A tiles are K-major (box 64 x 128 rows); down A
//     tiles are W2^T rows, i.e. MN-major (two 64 x 64 boxes per 128-row M tile).
//   * activations X [entries][NP][d] and H [entries][NP][F] bf16, K-major, box 64 x 16.
// Units (one per CTA iteration, static round-robin over a persistent grid):
//   gate/up: (segment, tile, 128-row M tile), K = d;  epilogue: h = silu(a) * b -> H (bf16)
//   down   : (segment, 128-row M tile of d, K chunk c of kc); epilogue: fp32 partial
//            partial[unit][NP][128] (each unit writes its own; the combine sums them in a fixed
//            order, so results do not depend on the grid or on timing).
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer (one
// elected lane), warps 2-5 = epilogue (TMEM lane quadrant = warp % 4).  Double-buffered TMEM
// accumulators let the epilogue of unit i overlap the MMAs of unit i+1.
#pragma once

#include <cuda.h>
#include <cuda_runtime_api.h>

#include <cstdint>

#include "ep_exchange.hpp"

namespace adapmoe {

constexpr int kGMaxEntries = 64;   // distinct experts of one layer (N <= 64)
constexpr int kGMaxSegs = 64;      // segments per launch
constexpr int kGMaxPairs = 512;    // (stream, rank) pairs per layer: B * K
constexpr int kGMaxStages = 8;
constexpr int kGThreads = 192;

struct GEntry {
    long long slot_row = 0;  // pool row of the expert's first tile (slot byte offset / (2 d))
    int n = 0;               // tokens routed to the entry
    int np = 0;              // MMA N = n rounded up to 16
};

struct GSeg {
    int entry = 0;
    int t0 = 0, t1 = 0;      // expert tiles [t0, t1) covered by the segment
};

struct GroupedLaunch {
    CUtensorMap map_a;       // expert slot pool [rows][d] bf16
    CUtensorMap map_b;       // X [entries*NP][d] (gate/up) or H [entries*NP][F] (down) bf16
    int n_seg = 0, d = 0, ft = 0, f = 0;
    int np_stride = 0;       // NP: row stride (in rows) between entries in X / H; TMEM columns per buffer
    int kc = 1;              // down: K chunks per (segment, M tile)
    int stages = 0;
    int units = 0;
    int unit_prefix[kGMaxSegs + 1];
    GSeg seg[kGMaxSegs];
    GEntry ent[kGMaxEntries];
    std::uint16_t* h = nullptr;   // gate/up output H [entries][NP][F] bf16
    float* partial = nullptr;     // down output [units][NP][128] fp32
};

// Host helpers -------------------------------------------------------------------------------
// 2-D bf16 row-major tensor map [rows][cols] with a box of box_cols x box_rows, 128-byte swizzle.
cudaError_t make_tensor_map_2d(CUtensorMap* map, const void* base, std::uint64_t rows, std::uint64_t cols,
                               std::uint32_t box_cols, std::uint32_t box_rows);

// Fill unit counts / prefix sums / stage count for a launch (segments and entries already set).
void grouped_plan_gate_up(GroupedLaunch& p);
void grouped_plan_down(GroupedLaunch& p, int sm_count);
int grouped_grid(const GroupedLaunch& p, int sm_count);
cudaError_t launch_grouped_gate_up(const GroupedLaunch& p, int sm_count, cudaStream_t stream);
cudaError_t launch_grouped_down(const GroupedLaunch& p, int sm_count, cudaStream_t stream);

// Gather the routed tokens' activations into X [entries][NP][d] bf16 (zero padded rows).
struct GatherArgs {
    const double* acts = nullptr;   // stream b's layer input at acts + b * stream_stride
    long long stream_stride = 0;
    std::uint16_t* x = nullptr;
    int d = 0, np_stride = 0, n_entries = 0;
    int first[kGMaxEntries + 1];    // entry e's streams: stream[first[e] .. first[e+1])
    short stream[kGMaxPairs];
};
cudaError_t launch_grouped_gather(const GatherArgs& a, cudaStream_t stream);

// out[b][j] = x_b[j] + sum_rank w_{b,rank} * y_{entry(b,rank)}[col(b,rank)][j]; y = fixed-order sum
// of the down partials of the entry's segments (tile order) and K chunks.
struct GCombineRef {
    const float* partial = nullptr;  // the launch's partial buffer
    int unit0 = 0;                   // unit index of (segment, M tile 0, chunk 0)
    int kc = 1;
};
struct GCombineArgs {
    const double* acts = nullptr;    // residual x_b at acts + b * stream_stride
    const double* scores = nullptr;  // scores_b at scores + b * score_stride ([N])
    long long stream_stride = 0, score_stride = 0;
    float* out = nullptr;            // out_b at out + b * out_stride
    long long out_stride = 0;
    int d = 0, np_stride = 0, n_streams = 0, top_k = 0;
    int residual = 1;                // add x (expert-parallel: only the first shard adds it)
    int n_out_peer = 0;              // expert-parallel P2P exchange: write out_peer[g] (same layout as out)
    float* out_peer[kMaxEpPeers] = {};
    int ref_first[kGMaxEntries + 1]; // entry e's refs: refs[ref_first[e] .. ref_first[e+1])
    GCombineRef refs[256];
    // per (stream, rank): entry index, token column, expert id (-1 = unused rank)
    short pair_entry[kGMaxPairs];
    short pair_col[kGMaxPairs];
    short pair_expert[kGMaxPairs];
};
cudaError_t launch_grouped_combine(const GCombineArgs& a, cudaStream_t stream);

}  // namespace adapmoe
