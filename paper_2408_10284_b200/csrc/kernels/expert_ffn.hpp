// K2 — SwiGLU expert FFN for batch-1 decode (host launch interface).
//
// Expert memory layout (tile-major, bf16), tile t = ffn rows [t*Ft, (t+1)*Ft), Ft = F / tiles:
//   gate_up_t : [Ft][2][D]  row pair r = (W1[t*Ft + r, :], W3[t*Ft + r, :]) contiguous
//   down_t    : [Ft][D]     row r = W2[:, t*Ft + r]  (W2 transposed)
// so every tile is one contiguous 3*Ft*D*2-byte block: the unit of a host->HBM copy and of a
// tile-granular FFN launch (inc/simulator.hpp:451-459 computes on-demand experts tile by tile),
// and every ffn row r owns three contiguous D-element rows (W1, W3, W2^T).
//
// One launch processes a list of (expert rank, tile) segments; CTA c owns a contiguous range of
// ffn rows of the concatenated segments and, chunk by chunk, forms h_r = silu(W1_r.x) * (W3_r.x)
// and accumulates h_r * W2^T_r into its own fp32 partial of y (no cross-CTA dependency).  The
// combine kernel reduces the partials in a fixed order:
//   out[j] = x[j] + sum_rank w_rank * sum_tiles sum_cta partial[cta][slot][j].
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>

#include "ep_exchange.hpp"

namespace adapmoe {

constexpr int kMaxFfnSegments = 32;
constexpr int kFfnMaxCtas = 160;      // grid cap (>= #SMs of a B200)
constexpr int kFfnSlotsPerCta = 2;    // a CTA's row range touches at most 2 segments (n_seg <= grid)

struct FfnSegment {
    const std::uint16_t* gate_up = nullptr;  // [Ft][2][D] bf16
    const std::uint16_t* down_t = nullptr;   // [Ft][D] bf16 (W2^T rows)
};

struct FfnLaunch {
    int n_seg = 0;
    int d = 0, ft = 0;
    const double* x = nullptr;        // [d] layer input (fp64; converted to fp32 in shared memory)
    float* partial = nullptr;         // [grid][kFfnSlotsPerCta][d] written by the launch
    FfnSegment seg[kMaxFfnSegments];
};

// Grid the launch will use (partial buffer rows = grid * kFfnSlotsPerCta).
int ffn_grid(const FfnLaunch& p, int sm_count);
// Ring = TMA bulk-copy ring (default); Rows = the LDG row-owner kernel (ADAPMOE_K2=rows).  Both
// use the same CTA row split and partial layout.
enum class FfnKernel { Ring, Rows };
FfnKernel ffn_kernel_variant();
cudaError_t launch_ffn(const FfnLaunch& p, int sm_count, cudaStream_t stream);

// One (rank, tile) segment's location among the launches of a layer.
struct FfnPartialRef {
    const float* partial = nullptr;  // that launch's partial buffer
    int grid = 0;                    // that launch's grid
    int n_seg = 0;                   // that launch's segment count
    int seg = 0;                     // index of the segment in that launch
    int rank = 0;                    // expert rank in the selection
    // CTAs of that launch whose row ranges intersect the segment, and the partial slot of the
    // first one (later ones start inside the segment: slot 0); filled by ffn_partial_range()
    int c_lo = 0, c_hi = -1, slot_lo = 0;
};

// Host: fill r.c_lo / c_hi / slot_lo from (grid, n_seg, seg) for row-tile ft (same integer
// arithmetic as the kernel's row split).
void ffn_partial_range(FfnPartialRef& r, int ft);

constexpr int kMaxCombineRefs = 128;

struct CombineArgs {
    const double* x = nullptr;       // [D] layer input (residual; all-zero for a bare FFN)
    const double* scores = nullptr;  // [N] post-softmax scores of this (token, layer)
    float* out = nullptr;            // [D]
    int experts[8] = {0};            // selected experts in rank order
    int ranks = 0, d = 0, ft = 0;
    int residual = 1;                // add x (expert-parallel: only the first shard adds it)
    // expert-parallel P2P exchange: when n_out_peer > 0 the result goes to out_peer[g] (this shard's
    // slot in every shard's exchange region, same row offset as out) instead of out
    int n_out_peer = 0;
    float* out_peer[kMaxEpPeers] = {};
    int n_refs = 0;                  // refs sorted by (rank, tile)
    // free-running batch 1: the block that finishes last (ticket) also forms the next layer's input
    // from `out` — next_res = (double) out, next_norm = RMSNorm(next_res) in the fixed order of
    // launch_free_running_input — so that launch disappears.  next_res == nullptr: off.
    double* next_res = nullptr;
    double* next_norm = nullptr;
    unsigned* ticket = nullptr;      // zero before the launch; the last block re-arms it
    double eps = 0.0;
    float scale = 1.0f;              // extra factor on every rank's weight (moe_expert_ffn_async)
    int accumulate = 0;              // out[j] += ... instead of out[j] = ... (n_out_peer == 0 only)
    FfnPartialRef refs[kMaxCombineRefs];
};
cudaError_t launch_combine(const CombineArgs& a, cudaStream_t stream);

// Free-running decode, per layer and stream row r (stride `stride` doubles between rows):
//   res[r] = src ? (double) src[r] (previous layer's fp32 output) : res[r] (unchanged, layer 0)
//   norm[r] = res[r] / sqrt(sum_i res[r][i]^2 / d + eps)     (RMSNorm without gain, Mixtral's
// pre-MoE norm).  One warp per row: lane j sums res[i]^2 for i = j, j+32, ... in order (separately
// rounded fp64 ops), then a fixed xor butterfly — reproducible bit for bit on the host.
cudaError_t launch_free_running_input(double* res, double* norm, long long stride, const float* src,
                                      long long src_stride, int rows, int d, double eps, cudaStream_t stream);

// Deterministic counter-based bf16 init of one expert in the tile-major layout (same values as
// oracle/moe_oracle.c orc_expert_init): value = bf16_rne(float(sum of 4 x 16-bit lanes of
// splitmix64(base_m + index) - 131070) * scale_m), index = logical row-major index in W1/W3 [F][D]
// or W2 [D][F].
cudaError_t launch_expert_init(std::uint16_t* dst, int d, int f, int tiles, const std::uint64_t base[3],
                               const float scale[3], cudaStream_t stream);

}  // namespace adapmoe
