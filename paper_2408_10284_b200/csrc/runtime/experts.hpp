// Pinned host expert store: every (layer, expert) SwiGLU weight block, tile-major bf16
// (kernels/expert_ffn.hpp), page-locked so tile copies run at host-link speed.
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>
#include <vector>

#include "../kernels/xb12.hpp"
#include "../kernels/xbh.hpp"

namespace adapmoe {

class Engine;
struct DeviceBuffer;

enum StoreFormat : int { kStoreBf16 = 0, kStoreXb12 = 1, kStoreXbh = 2 };

struct ExpertStore {
    int layers = 0, experts = 0, d = 0, ffn = 0, tiles = 0, alias = 0;
    std::uint64_t seed = 0;
    size_t expert_bytes = 0;  // 3 * F * d * 2
    size_t tile_bytes = 0;    // expert_bytes / tiles
    std::vector<unsigned char*> blocks;  // registered host memory, one per stored expert
    std::vector<size_t> pinned;          // [block] bytes registered (expert_bytes, or a coded block's records)
    // [L*N] block of each (layer, expert); -1 = not held by this store (an expert-parallel shard
    // pins only the experts it owns)
    std::vector<int> index;
    int numa_node = -1;  // host NUMA node the blocks were placed on (-1: no binding)
    double pin_seconds = 0.0, fill_seconds = 0.0;
    // kStoreXb12 / kStoreXbh: every tile is an XB12 (kernels/xb12.hpp) / XBH (kernels/xbh.hpp)
    // record or, if it would not shrink, raw bf16; records are packed in tile order (tile_off)
    // inside the expert's block
    int format = kStoreBf16;
    std::vector<Xb12Tile> tile_meta;   // [stored block][tile]
    std::vector<size_t> tile_off;      // [stored block][tile] byte offset of the record in the block
    size_t link_bytes = 0;             // sum of the stored records (bytes a full copy of the store moves)

    const Xb12Tile& meta(int layer, int expert, int tile) const {
        return tile_meta[static_cast<size_t>(stored_index(layer, expert)) * tiles + tile];
    }
    // host address + bytes of one tile's record (raw tile for kStoreBf16)
    const unsigned char* record(int layer, int expert, int tile, size_t* bytes) const;
    size_t max_record_bytes() const;

    bool has(int layer, int expert) const { return index[static_cast<size_t>(layer) * experts + expert] >= 0; }
    int stored_index(int layer, int expert) const;  // fails (Usage) for an expert the store does not hold
    const unsigned char* expert(int layer, int expert) const { return blocks[stored_index(layer, expert)]; }
    size_t pinned_bytes() const {
        size_t b = 0;
        for (size_t p : pinned) b += p;
        return b;
    }
    ~ExpertStore();
};

// Allocate + pin (parallel first touch on the GPU's NUMA node + cudaHostRegister) and, with
// `init_values`, fill with the deterministic init (GPU init kernel, D2H into the pinned blocks);
// without, the store is zero and the caller provides the weights through set_expert_weights.
// owner [L*N] (may be null): hold only the experts with owner[l*N + e] == rank (expert-parallel
// shard); alias > 0 maps the held experts onto that many distinct blocks.
void build_expert_store(Engine& engine, ExpertStore& store, int ffn, int tiles, std::uint64_t seed, int alias,
                        bool init_values = true, const int* owner = nullptr, int rank = 0, int format = kStoreBf16);

// Pack one expert's weights, given in the usual checkpoint layout (bf16 bits, row-major:
// w1 = gate_proj [ffn][d], w3 = up_proj [ffn][d], w2 = down_proj [d][ffn]), into the store's
// tile-major layout (W1/W3 row pairs + W2 transposed, kernels/expert_ffn.hpp).  Host threads.
void set_expert_weights(Engine& engine, ExpertStore& store, int layer, int expert, const std::uint16_t* w1,
                        const std::uint16_t* w3, const std::uint16_t* w2);

// Copy tiles [t0, t1) of (layer, expert) into device memory laid out like the store (dst + t *
// tile_bytes) on `stream`; XB12 records are staged in `staging` (reserved here, >= max_record_bytes,
// reused in stream order) and decoded on the same stream.  tile_done (may be null): an event per
// tile recorded after that tile is usable.
void upload_expert_tiles(const ExpertStore& store, int layer, int expert, int t0, int t1, unsigned char* dst,
                         DeviceBuffer& staging, cudaStream_t stream, cudaEvent_t const* tile_done = nullptr);

// Decode (or copy) one expert's tiles into host bf16 (tile-major, expert_bytes).
void read_expert_host(const ExpertStore& store, int layer, int expert, std::uint16_t* out);

// Per-matrix init constants shared with the CUDA init kernel and the oracle.
void expert_init_constants(std::uint64_t seed, int layer, int expert, int d, int ffn, std::uint64_t base[3], float scale[3]);

}  // namespace adapmoe
