#include "experts.hpp"

#include <cuda_runtime.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>

#include "../kernels/expert_ffn.hpp"
#include "../kernels/xb12.hpp"
#include "../kernels/xbh.hpp"
#include "engine.hpp"

namespace adapmoe {

const unsigned char* ExpertStore::record(int layer, int expert, int tile, size_t* bytes) const {
    const int b = stored_index(layer, expert);
    const size_t k = static_cast<size_t>(b) * tiles + tile;
    if (bytes) *bytes = tile_meta[k].format != 0 ? tile_meta[k].bytes : tile_bytes;
    return blocks[b] + tile_off[k];
}

size_t ExpertStore::max_record_bytes() const {
    size_t m = 0;
    for (const Xb12Tile& t : tile_meta) m = std::max(m, t.format != 0 ? static_cast<size_t>(t.bytes) : tile_bytes);
    return m;
}

int ExpertStore::stored_index(int layer, int expert) const {
    const int b = index[static_cast<size_t>(layer) * experts + expert];
    if (b < 0)
        fail(Status::Usage, "expert (" + std::to_string(layer) + ", " + std::to_string(expert) +
                                ") is owned by another expert-parallel shard: this store does not hold it");
    return b;
}

namespace {

// NUMA node of the engine's GPU (sysfs), -1 if unknown or single-node.  ADAPMOE_NUMA=0 disables the
// placement, ADAPMOE_NUMA=<n+1> forces node n.
int gpu_numa_node(int device) {
    if (const char* v = std::getenv("ADAPMOE_NUMA")) {
        const int n = std::atoi(v);
        return n <= 0 ? -1 : n - 1;
    }
    char bus[32] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) return -1;
    for (char* c = bus; *c; ++c) *c = static_cast<char>(std::tolower(*c));
    std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
    FILE* f = std::fopen(path.c_str(), "r");
    if (!f) {  // sysfs uses a 4-digit domain; CUDA may print 8
        std::string b(bus);
        if (b.size() > 12) path = "/sys/bus/pci/devices/" + b.substr(b.size() - 12) + "/numa_node";
        f = std::fopen(path.c_str(), "r");
    }
    if (!f) return -1;
    int node = -1;
    if (std::fscanf(f, "%d", &node) != 1) node = -1;
    std::fclose(f);
    return node;
}

// Prefer `node` for the pages of [p, p + bytes) (falls back to other nodes when it is full).
void prefer_node(void* p, size_t bytes, int node) {
    if (node < 0 || node >= 64) return;
    unsigned long mask = 1ul << node;
    constexpr int kMpolPreferred = 1;
    syscall(SYS_mbind, p, bytes, kMpolPreferred, &mask, 64ul, 0u);  // best effort: errors keep the default policy
}

}  // namespace

ExpertStore::~ExpertStore() {
    for (size_t i = 0; i < blocks.size(); ++i) {
        if (!blocks[i]) continue;
        if (i < pinned.size() && pinned[i]) cudaHostUnregister(blocks[i]);
        std::free(blocks[i]);
    }
}

void expert_init_constants(std::uint64_t seed, int layer, int expert, int d, int ffn, std::uint64_t base[3], float scale[3]) {
    for (int m = 0; m < 3; ++m)
        base[m] = splitmix64(splitmix64(seed) ^ (static_cast<std::uint64_t>(static_cast<std::uint32_t>(layer)) << 24) ^
                             (static_cast<std::uint64_t>(static_cast<std::uint32_t>(expert)) << 4) ^
                             static_cast<std::uint64_t>(m));
    // weight std ~ 1/sqrt(fan_in): a sum of four uniform 16-bit lanes has std 37837.22
    scale[0] = scale[1] = static_cast<float>(1.0 / (37837.22 * std::sqrt(static_cast<double>(d))));
    scale[2] = static_cast<float>(1.0 / (37837.22 * std::sqrt(static_cast<double>(ffn))));
}

namespace {

// The raw layout: tile t of every block at t * tile_bytes (kStoreBf16, and an XB12 store before
// its experts are encoded).
void raw_tile_layout(ExpertStore& st) {
    const size_t nb = st.blocks.size();
    st.tile_meta.assign(nb * st.tiles, Xb12Tile{});
    st.tile_off.assign(nb * st.tiles, 0);
    for (size_t b = 0; b < nb; ++b)
        for (int t = 0; t < st.tiles; ++t) {
            Xb12Tile& m = st.tile_meta[b * st.tiles + t];
            m.format = 0;
            m.n = st.tile_bytes / 2;
            m.bytes = st.tile_bytes;
            st.tile_off[b * st.tiles + t] = static_cast<size_t>(t) * st.tile_bytes;
        }
    st.link_bytes = nb * st.expert_bytes;
}

// Encode one expert (raw tile-major bf16 in device memory) into stored block b as XB12 records;
// a tile whose escapes exceed n / 64 stays raw.  Synchronous on `s`.
struct Xb12Scratch {
    DeviceBuffer rec, work;
};
void encode_block(ExpertStore& st, int b, const std::uint16_t* d_raw, Xb12Scratch& x, cudaStream_t s) {
    const std::uint64_t n = st.tile_bytes / 2, cap = n / 64;
    const size_t lo_nib = xb12_align(xb12_align(n) + n / 2);
    const size_t region = lo_nib + cap * 8;
    x.rec.reserve(region * st.tiles);
    x.work.reserve(static_cast<size_t>(kXb12WorkWords) * st.tiles * sizeof(std::uint32_t));
    for (int t = 0; t < st.tiles; ++t) {
        unsigned char* r = x.rec.as<unsigned char>() + region * t;
        MOE_CUDA(xb12_encode(d_raw + n * t, n, r, r + xb12_align(n), reinterpret_cast<std::uint64_t*>(r + lo_nib), cap,
                             x.work.as<std::uint32_t>() + static_cast<size_t>(kXb12WorkWords) * t, s));
    }
    std::vector<std::uint32_t> work(static_cast<size_t>(kXb12WorkWords) * st.tiles);
    MOE_CUDA(cudaMemcpyAsync(work.data(), x.work.ptr, work.size() * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, s));
    MOE_CUDA(cudaStreamSynchronize(s));
    size_t off = 0;
    std::vector<std::uint64_t> exc;
    for (int t = 0; t < st.tiles; ++t) {
        Xb12Tile& m = st.tile_meta[static_cast<size_t>(b) * st.tiles + t];
        const std::uint32_t* w = work.data() + static_cast<size_t>(kXb12WorkWords) * t;
        m = Xb12Tile{};
        m.n = n;
        m.base = w[256];
        m.n_exc = w[257];
        unsigned char* dst = st.blocks[b] + off;
        st.tile_off[static_cast<size_t>(b) * st.tiles + t] = off;
        if (m.n_exc > cap) {  // does not pay: keep the raw tile
            m.format = 0;
            m.bytes = st.tile_bytes;
            MOE_CUDA(cudaMemcpyAsync(dst, d_raw + n * t, st.tile_bytes, cudaMemcpyDeviceToHost, s));
        } else {
            m.format = 1;
            xb12_layout(m);
            const unsigned char* r = x.rec.as<unsigned char>() + region * t;
            // the alignment padding after the escapes is zero (a record is a pure function of the tile,
            // whatever the block held before)
            std::memset(dst + m.exc_off, 0, m.bytes - m.exc_off);
            MOE_CUDA(cudaMemcpyAsync(dst, r, m.exc_off, cudaMemcpyDeviceToHost, s));
            exc.resize(m.n_exc);
            if (m.n_exc) {
                MOE_CUDA(cudaMemcpyAsync(exc.data(), r + lo_nib, m.n_exc * 8, cudaMemcpyDeviceToHost, s));
                MOE_CUDA(cudaStreamSynchronize(s));
                std::sort(exc.begin(), exc.end());  // ascending index (the escapes arrive unordered)
                std::memcpy(dst + m.exc_off, exc.data(), m.n_exc * 8);
            }
        }
        off += m.format == 1 ? m.bytes : st.tile_bytes;
        if (off > st.expert_bytes) fail(Status::Internal, "xb12: records exceed the expert block");
    }
    MOE_CUDA(cudaStreamSynchronize(s));
}

// The same for XBH records: exponent histograms -> per-tile Huffman codes (host) -> device encode
// -> records D2H; a tile whose escapes exceed n / 64 or whose record would not shrink stays raw.
struct XbhScratch {
    DeviceBuffer rec, gaps, bases, exc, seglen, work, code;
};
void encode_block_xbh(ExpertStore& st, int b, const std::uint16_t* d_raw, XbhScratch& x, cudaStream_t s) {
    const std::uint64_t n = st.tile_bytes / 2, cap = n / 64, nseg = xbh_enc_segments(n);
    const std::uint64_t max_bits = n * kXbhMaxLen;
    const size_t region = xbh_region_bytes(n), gw = xbh_gap_words(max_bits), bw = xbh_blocks(max_bits) + 1;
    const int T = st.tiles;
    x.rec.reserve(region * T);
    x.gaps.reserve(4 * gw * T);
    x.bases.reserve(4 * bw * T);
    x.exc.reserve(cap * 8 * T);
    x.seglen.reserve(4 * (nseg + 1) * T);
    x.work.reserve(sizeof(std::uint32_t) * (256 + kXbhWorkWords) * T);
    x.code.reserve(sizeof(XbhCode) * T);
    std::uint32_t* hist = x.work.as<std::uint32_t>();
    std::uint32_t* work = hist + 256 * T;
    for (int t = 0; t < T; ++t) MOE_CUDA(xb12_histogram(d_raw + n * t, n, hist + 256 * t, s));
    std::vector<std::uint32_t> h(256 * static_cast<size_t>(T));
    MOE_CUDA(cudaMemcpyAsync(h.data(), hist, h.size() * 4, cudaMemcpyDeviceToHost, s));
    MOE_CUDA(cudaStreamSynchronize(s));
    std::vector<XbhCode> codes(T);
    for (int t = 0; t < T; ++t) xbh_build_code(h.data() + 256 * t, codes[t]);
    MOE_CUDA(cudaMemcpyAsync(x.code.ptr, codes.data(), sizeof(XbhCode) * T, cudaMemcpyHostToDevice, s));
    XbhCode* dcode = x.code.as<XbhCode>();
    for (int t = 0; t < T; ++t)
        MOE_CUDA(xbh_encode(d_raw + n * t, n, dcode + t, x.rec.as<std::uint8_t>() + region * t,
                            x.gaps.as<std::uint32_t>() + gw * t, x.bases.as<std::uint32_t>() + bw * t,
                            x.exc.as<std::uint64_t>() + cap * t, cap, x.seglen.as<std::uint32_t>() + (nseg + 1) * t,
                            work + kXbhWorkWords * t, s));
    std::vector<std::uint32_t> wk(kXbhWorkWords * static_cast<size_t>(T));
    MOE_CUDA(cudaMemcpyAsync(wk.data(), work, wk.size() * 4, cudaMemcpyDeviceToHost, s));
    MOE_CUDA(cudaStreamSynchronize(s));
    size_t off = 0;
    std::vector<std::uint64_t> exc;
    for (int t = 0; t < T; ++t) {
        Xb12Tile& m = st.tile_meta[static_cast<size_t>(b) * T + t];
        m = Xb12Tile{};
        m.n = n;
        m.base = codes[t].base;
        m.n_exc = wk[kXbhWorkWords * t];
        const std::uint64_t bits = wk[kXbhWorkWords * t + 1];
        if (m.n_exc <= cap) xbh_layout(m, bits);
        unsigned char* dst = st.blocks[b] + off;
        st.tile_off[static_cast<size_t>(b) * T + t] = off;
        if (m.n_exc > cap || m.bytes >= st.tile_bytes) {  // does not pay: keep the raw tile
            m = Xb12Tile{};
            m.format = 0;
            m.n = n;
            m.bytes = st.tile_bytes;
            MOE_CUDA(cudaMemcpyAsync(dst, d_raw + n * t, st.tile_bytes, cudaMemcpyDeviceToHost, s));
        } else {
            m.format = 2;
            // every byte of the record is written (alignment gaps zero): a pure function of the tile
            std::memset(dst, 0, m.bytes);
            const unsigned char* r = x.rec.as<unsigned char>() + region * t;
            const size_t hdr = xbh_hdr_off(n), bo = xbh_bits_off(n), go = xbh_gap_off(n, bits), so = xbh_base_off(n, bits);
            const std::uint64_t blocks = xbh_blocks(bits);
            MOE_CUDA(cudaMemcpyAsync(dst, r, hdr, cudaMemcpyDeviceToHost, s));
            MOE_CUDA(cudaMemcpyAsync(dst + bo, r + bo, 4 * xbh_words(bits), cudaMemcpyDeviceToHost, s));
            MOE_CUDA(cudaMemcpyAsync(dst + go, x.gaps.as<std::uint32_t>() + gw * t, 4 * xbh_gap_words(bits),
                                     cudaMemcpyDeviceToHost, s));
            MOE_CUDA(cudaMemcpyAsync(dst + so, x.bases.as<std::uint32_t>() + bw * t, 4 * blocks, cudaMemcpyDeviceToHost, s));
            const std::uint64_t hv[2] = {bits, m.n_exc};
            std::memcpy(dst + hdr, hv, sizeof hv);
            const std::uint32_t last = static_cast<std::uint32_t>(n);
            std::memcpy(dst + so + 4 * blocks, &last, 4);
            exc.resize(m.n_exc);
            if (m.n_exc)
                MOE_CUDA(cudaMemcpyAsync(exc.data(), x.exc.as<std::uint64_t>() + cap * t, m.n_exc * 8,
                                         cudaMemcpyDeviceToHost, s));
            MOE_CUDA(cudaStreamSynchronize(s));
            std::sort(exc.begin(), exc.end());  // ascending index (the escapes arrive unordered)
            if (m.n_exc) std::memcpy(dst + m.exc_off, exc.data(), m.n_exc * 8);
        }
        off += m.bytes;
        if (off > st.expert_bytes) fail(Status::Internal, "xbh: records exceed the expert block");
    }
    MOE_CUDA(cudaStreamSynchronize(s));
}

// the store's encoder for one block
struct StoreScratch {
    Xb12Scratch xb12;
    XbhScratch xbh;
};
void encode_store_block(ExpertStore& st, int b, const std::uint16_t* d_raw, StoreScratch& x, cudaStream_t s) {
    if (st.format == kStoreXbh)
        encode_block_xbh(st, b, d_raw, x.xbh, s);
    else
        encode_block(st, b, d_raw, x.xb12, s);
}

void recount_link_bytes(ExpertStore& st) {
    st.link_bytes = 0;
    for (const Xb12Tile& m : st.tile_meta) st.link_bytes += m.format != 0 ? m.bytes : st.tile_bytes;
}

// Pin every block of a coded store over its records only (host threads, after the encoder wrote them
// into the unpinned blocks; the pages past the records were never touched).
void pin_coded_blocks(ExpertStore& st) {
    const size_t page = 2u << 20;
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    std::vector<std::string> errors(hw);
    for (unsigned w = 0; w < hw; ++w)
        pool.emplace_back([&, w] {
            for (size_t b = w; b < st.blocks.size(); b += hw) {
                const size_t k = b * st.tiles + st.tiles - 1;  // the last record ends the block's content
                const size_t used = st.tile_off[k] + (st.tile_meta[k].format ? st.tile_meta[k].bytes : st.tile_bytes);
                const size_t keep = std::min(st.expert_bytes, (used + page - 1) / page * page);
                const cudaError_t e = cudaHostRegister(st.blocks[b], keep, cudaHostRegisterDefault);
                if (e != cudaSuccess) {
                    errors[w] = std::string("cudaHostRegister: ") + cudaGetErrorString(e);
                    return;
                }
                st.pinned[b] = keep;
            }
        });
    for (auto& t : pool) t.join();
    for (auto& e : errors)
        if (!e.empty()) fail(Status::Device, "experts_init: " + e);
}

}  // namespace

void upload_expert_tiles(const ExpertStore& st, int layer, int expert, int t0, int t1, unsigned char* dst,
                         DeviceBuffer& staging, cudaStream_t stream, cudaEvent_t const* tile_done) {
    for (int t = t0; t < t1; ++t) {
        size_t bytes = 0;
        const unsigned char* rec = st.record(layer, expert, t, &bytes);
        unsigned char* out = dst + static_cast<size_t>(t) * st.tile_bytes;
        const Xb12Tile& m = st.meta(layer, expert, t);
        if (m.format == 0) {
            MOE_CUDA(cudaMemcpyAsync(out, rec, bytes, cudaMemcpyHostToDevice, stream));
        } else {
            staging.reserve(st.max_record_bytes());
            MOE_CUDA(cudaMemcpyAsync(staging.ptr, rec, bytes, cudaMemcpyHostToDevice, stream));
            if (m.format == 2)
                MOE_CUDA(xbh_decode(staging.as<std::uint8_t>(), m, reinterpret_cast<std::uint16_t*>(out), stream));
            else
                MOE_CUDA(xb12_decode(staging.as<std::uint8_t>(), m, reinterpret_cast<std::uint16_t*>(out), stream));
        }
        if (tile_done && tile_done[t - t0]) MOE_CUDA(cudaEventRecord(tile_done[t - t0], stream));
    }
}

void read_expert_host(const ExpertStore& st, int layer, int expert, std::uint16_t* out) {
    for (int t = 0; t < st.tiles; ++t) {
        size_t bytes = 0;
        const unsigned char* rec = st.record(layer, expert, t, &bytes);
        std::uint16_t* o = out + st.tile_bytes / 2 * t;
        const Xb12Tile& m = st.meta(layer, expert, t);
        if (m.format == 0)
            std::memcpy(o, rec, st.tile_bytes);
        else if (m.format == 2)
            xbh_decode_host(rec, m, o, 0, m.n);
        else
            xb12_decode_host(rec, m, o, 0, m.n);
    }
}

void build_expert_store(Engine& eng, ExpertStore& st, int ffn, int tiles, std::uint64_t seed, int alias,
                        bool init_values, const int* owner, int rank, int format) {
    const ModelSpec& spec = eng.spec();
    if (ffn <= 0 || tiles < 1 || ffn % tiles) fail(Status::Usage, "experts_init: ffn must be a positive multiple of tiles");
    const int ft = ffn / tiles;
    if (spec.hidden_dim % 32 || ft % 32) fail(Status::Usage, "experts_init: hidden_dim and ffn/tiles must be multiples of 32");
    if (spec.hidden_dim > 16384 || ft > 16384) fail(Status::Usage, "experts_init: rows longer than 16384 elements unsupported");
    // one K2 launch covers a whole expert (FfnLaunch::seg) and a layer's combine every (rank, tile)
    if (tiles > kMaxFfnSegments) fail(Status::Usage, "experts_init: at most 32 tiles per expert");
    if (alias < 0) fail(Status::Usage, "experts_init: host_alias must be >= 0");
    eng.activate();
    st.layers = spec.num_layers;
    st.experts = spec.experts_per_layer;
    st.d = spec.hidden_dim;
    st.ffn = ffn;
    st.tiles = tiles;
    st.seed = seed;
    const int total = spec.num_layers * spec.experts_per_layer;
    // experts this store holds (all, or one expert-parallel shard's)
    std::vector<int> held;
    for (int id = 0; id < total; ++id) {
        if (owner && (owner[id] < 0)) fail(Status::Usage, "experts_init: negative expert owner");
        if (!owner || owner[id] == rank) held.push_back(id);
    }
    if (held.empty()) fail(Status::Usage, "experts_init: this shard owns no expert");
    const int n_held = static_cast<int>(held.size());
    st.alias = (alias > 0 && alias < n_held) ? alias : 0;
    st.expert_bytes = static_cast<size_t>(3) * ffn * spec.hidden_dim * 2;
    st.tile_bytes = st.expert_bytes / tiles;
    const int stored = st.alias > 0 ? st.alias : n_held;
    st.index.assign(total, -1);
    for (int i = 0; i < n_held; ++i) st.index[held[i]] = st.alias > 0 ? i % st.alias : i;
    std::vector<int> first_id(stored, -1);  // the (layer, expert) whose init values fill each block
    for (int i = 0; i < n_held; ++i)
        if (first_id[st.index[held[i]]] < 0) first_id[st.index[held[i]]] = held[i];
    st.blocks.assign(stored, nullptr);
    st.pinned.assign(stored, 0);
    st.numa_node = gpu_numa_node(eng.device());

    // a coded store built from the synthetic init is encoded straight into unpinned blocks (D2H through
    // pageable memory, touching only the records' pages) and pinned afterwards, records only
    const bool defer_pin = format != kStoreBf16 && init_values;
    // allocate + first-touch + pin in parallel: page faulting and locking dominate at 90+ GB
    auto t0 = std::chrono::steady_clock::now();
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    std::vector<std::string> errors(hw);
    for (unsigned w = 0; w < hw; ++w)
        pool.emplace_back([&, w] {
            for (int i = static_cast<int>(w); i < stored; i += static_cast<int>(hw)) {
                void* p = nullptr;
                if (posix_memalign(&p, 2u << 20, st.expert_bytes) != 0) {
                    errors[w] = "host allocation failed";
                    return;
                }
                madvise(p, st.expert_bytes, MADV_HUGEPAGE);
                prefer_node(p, st.expert_bytes, st.numa_node);  // before first touch
                st.blocks[i] = static_cast<unsigned char*>(p);
                if (defer_pin) continue;  // coded synthetic store: pinned after encoding, records only
                std::memset(p, 0, st.expert_bytes);
                cudaError_t e = cudaHostRegister(p, st.expert_bytes, cudaHostRegisterDefault);
                if (e != cudaSuccess) {
                    st.blocks[i] = nullptr;
                    std::free(p);
                    errors[w] = std::string("cudaHostRegister: ") + cudaGetErrorString(e);
                    return;
                }
                st.pinned[i] = st.expert_bytes;
            }
        });
    for (auto& t : pool) t.join();
    for (auto& e : errors)
        if (!e.empty()) fail(Status::Device, "experts_init: " + e);
    auto t1 = std::chrono::steady_clock::now();
    st.pin_seconds = std::chrono::duration<double>(t1 - t0).count();
    if (format != kStoreBf16 && format != kStoreXb12 && format != kStoreXbh)
        fail(Status::Usage, "experts_init: unknown store format");
    if (format != kStoreBf16 && (st.tile_bytes / 2) % 16) fail(Status::Usage, "coded store: tile values must be a multiple of 16");
    if (format == kStoreXbh && st.tile_bytes / 2 * kXbhMaxLen >= (1ull << 32))
        fail(Status::Usage, "xbh store: tiles of at most 357M values (use more tiles)");
    st.format = format;
    raw_tile_layout(st);
    if (!init_values) return;
    if (format != kStoreBf16) {  // GPU init kernel -> XB12 / XBH encode on the device -> D2H records
        DeviceBuffer raw;
        raw.reserve(st.expert_bytes);
        StoreScratch x;
        cudaStream_t s;
        MOE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        for (int i = 0; i < stored; ++i) {
            const int layer = first_id[i] / spec.experts_per_layer, expert = first_id[i] % spec.experts_per_layer;
            std::uint64_t base[3];
            float scale[3];
            expert_init_constants(seed, layer, expert, spec.hidden_dim, ffn, base, scale);
            MOE_CUDA(launch_expert_init(raw.as<std::uint16_t>(), spec.hidden_dim, ffn, tiles, base, scale, s));
            encode_store_block(st, i, raw.as<std::uint16_t>(), x, s);
        }
        cudaStreamDestroy(s);
        recount_link_bytes(st);
        pin_coded_blocks(st);
        st.fill_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
        return;
    }
    // fill: GPU init kernel into two device scratch blocks, D2H into the pinned store
    DeviceBuffer scratch[2];
    cudaStream_t s[2];
    cudaEvent_t copied[2];
    for (int k = 0; k < 2; ++k) {
        scratch[k].reserve(st.expert_bytes);
        MOE_CUDA(cudaStreamCreateWithFlags(&s[k], cudaStreamNonBlocking));
        MOE_CUDA(cudaEventCreateWithFlags(&copied[k], cudaEventDisableTiming));
    }
    for (int i = 0; i < stored; ++i) {
        const int k = i & 1;
        const int layer = first_id[i] / spec.experts_per_layer, expert = first_id[i] % spec.experts_per_layer;
        std::uint64_t base[3];
        float scale[3];
        expert_init_constants(seed, layer, expert, spec.hidden_dim, ffn, base, scale);
        MOE_CUDA(launch_expert_init(scratch[k].as<std::uint16_t>(), spec.hidden_dim, ffn, tiles, base, scale, s[k]));
        MOE_CUDA(cudaMemcpyAsync(st.blocks[i], scratch[k].ptr, st.expert_bytes, cudaMemcpyDeviceToHost, s[k]));
    }
    for (int k = 0; k < 2; ++k) {
        MOE_CUDA(cudaStreamSynchronize(s[k]));
        cudaStreamDestroy(s[k]);
        cudaEventDestroy(copied[k]);
    }
    st.fill_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
}

void set_expert_weights(Engine& eng, ExpertStore& st, int layer, int expert, const std::uint16_t* w1,
                        const std::uint16_t* w3, const std::uint16_t* w2) {
    if (layer < 0 || layer >= st.layers || expert < 0 || expert >= st.experts) fail(Status::Usage, "ExpertRef out of range");
    if (st.alias > 0) fail(Status::Usage, "expert_set: the store aliases experts (host_alias); allocate it without");
    if (!st.has(layer, expert)) fail(Status::Usage, "expert_set: this store (an expert-parallel shard) does not hold the expert");
    const size_t D = st.d, F = st.ffn, Ft = F / st.tiles;
    const int b = st.stored_index(layer, expert);
    if (st.pinned[b] < st.expert_bytes) {  // a coded block pinned over its records only: pin all of it
        if (st.pinned[b]) MOE_CUDA(cudaHostUnregister(st.blocks[b]));
        st.pinned[b] = 0;
        MOE_CUDA(cudaHostRegister(st.blocks[b], st.expert_bytes, cudaHostRegisterDefault));
        st.pinned[b] = st.expert_bytes;
    }
    std::vector<std::uint16_t> packed;  // coded stores: pack here, then encode into the block
    if (st.format != kStoreBf16) packed.resize(st.expert_bytes / 2);
    std::uint16_t* dst = st.format != kStoreBf16 ? packed.data() : reinterpret_cast<std::uint16_t*>(st.blocks[b]);
    const size_t tile_elems = 3 * Ft * D;
    auto pack_rows = [&](size_t f0, size_t f1) {
        constexpr size_t kB = 64;  // W2 transposed in kB x kB blocks (both sides cache friendly)
        for (size_t f = f0; f < f1; ++f) {
            const size_t t = f / Ft, r = f % Ft;
            std::uint16_t* gu = dst + t * tile_elems + r * 2 * D;
            std::memcpy(gu, w1 + f * D, D * 2);
            std::memcpy(gu + D, w3 + f * D, D * 2);
        }
        for (size_t fb = f0; fb < f1; fb += kB)
            for (size_t jb = 0; jb < D; jb += kB)
                for (size_t f = fb; f < std::min(f1, fb + kB); ++f) {
                    std::uint16_t* row = dst + (f / Ft) * tile_elems + 2 * Ft * D + (f % Ft) * D;
                    for (size_t j = jb; j < std::min(D, jb + kB); ++j) row[j] = w2[j * F + f];
                }
    };
    const size_t hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const size_t n = std::min(hw, F / 64 + 1);
    std::vector<std::thread> pool;
    for (size_t k = 1; k < n; ++k) pool.emplace_back(pack_rows, F * k / n, F * (k + 1) / n);
    pack_rows(0, F / n);
    for (auto& th : pool) th.join();
    if (st.format != kStoreBf16) {
        eng.activate();
        DeviceBuffer raw;
        raw.reserve(st.expert_bytes);
        StoreScratch x;
        cudaStream_t s = eng.copy_stream();
        MOE_CUDA(cudaMemcpyAsync(raw.ptr, packed.data(), st.expert_bytes, cudaMemcpyHostToDevice, s));
        encode_store_block(st, b, raw.as<std::uint16_t>(), x, s);
        recount_link_bytes(st);
    }
}

}  // namespace adapmoe
