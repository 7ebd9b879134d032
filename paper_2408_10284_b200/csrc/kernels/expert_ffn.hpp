// K2 — SwiGLU expert FFN for batch-1 decode (host launch interface).
//
// Expert memory layout (tile-major, bf16), tile t = ffn rows [t*Ft, (t+1)*Ft), Ft = F / tiles:
//   gate_up_t : [Ft][2][D]  row pair r = (W1[t*Ft + r, :], W3[t*Ft + r, :]) contiguous
//   down_t    : [D][Ft]     W2[:, t*Ft : (t+1)*Ft]
// so every tile is one contiguous 3*Ft*D*2-byte block: the unit of a host->HBM copy and of a
// tile-granular FFN launch (inc/simulator.hpp:451-459 computes on-demand experts tile by tile).
//
// One launch processes a list of (expert rank, tile) segments in a single persistent kernel:
//   phase A (gate/up): h_t[r] = silu(W1[r] . x) * (W3[r] . x)
//   phase B (down)   : y_t[j] = W2_t[j, :] . h_t
// phase-B work of a segment starts when that segment's phase-A units are all done (device-side
// counters), so weight streaming never pauses between the two projections.
// Combine: out[j] = x[j] + sum_rank w_rank * sum_t y_t[j] (fixed order, deterministic).
// Partial results are kept per (rank, tile) so a resident expert computed in one launch and an
// on-demand expert computed tile by tile give bit-identical outputs.
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>

namespace adapmoe {

constexpr int kMaxFfnSegments = 32;

struct FfnSegment {
    const std::uint16_t* gate_up = nullptr;  // [Ft][2][D] bf16
    const std::uint16_t* down = nullptr;     // [D][Ft] bf16
    float* h = nullptr;                      // [Ft] phase-A output (phase-B input)
    float* y = nullptr;                      // [D] phase-B output
};

struct FfnLaunch {
    int n_seg = 0;
    int d = 0, ft = 0;
    const double* x = nullptr;       // [d] layer input (fp64; converted to fp32 in shared memory)
    unsigned int* counters = nullptr;  // [n_seg] zero on entry: phase-A units finished per segment
    FfnSegment seg[kMaxFfnSegments];
};

// Streams every segment's weights once (TMA bulk copies into a shared-memory ring).
cudaError_t launch_ffn(const FfnLaunch& p, int sm_count, cudaStream_t stream);

struct CombineArgs {
    const double* x = nullptr;       // [D] layer input (residual)
    const double* scores = nullptr;  // [N] post-softmax scores of this (token, layer)
    const float* y = nullptr;        // [ranks][tiles][D] partial outputs
    float* out = nullptr;            // [D]
    int experts[8] = {0};            // selected experts in rank order
    int ranks = 0, tiles = 0, d = 0;
};
cudaError_t launch_combine(const CombineArgs& a, cudaStream_t stream);

// Deterministic counter-based bf16 init of one expert in the tile-major layout (same values as
// oracle/moe_oracle.c orc_expert_init): value = bf16_rne(float(sum of 4 x 16-bit lanes of
// splitmix64(base_m + index) - 131070) * scale_m).
cudaError_t launch_expert_init(std::uint16_t* dst, int d, int f, int tiles, const std::uint64_t base[3],
                               const float scale[3], cudaStream_t stream);

}  // namespace adapmoe
