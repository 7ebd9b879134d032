#include "experts.hpp"

#include <cuda_runtime.h>
#include <sys/mman.h>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "../kernels/expert_ffn.hpp"
#include "engine.hpp"

namespace adapmoe {

int ExpertStore::stored_index(int layer, int expert) const {
    const int id = layer * experts + expert;
    return alias > 0 ? id % alias : id;
}

ExpertStore::~ExpertStore() {
    for (unsigned char* b : blocks) {
        if (!b) continue;
        cudaHostUnregister(b);
        std::free(b);
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

void build_expert_store(Engine& eng, ExpertStore& st, int ffn, int tiles, std::uint64_t seed, int alias) {
    const ModelSpec& spec = eng.spec();
    if (ffn <= 0 || tiles < 1 || ffn % tiles) fail(Status::Usage, "experts_init: ffn must be a positive multiple of tiles");
    const int ft = ffn / tiles;
    if (spec.hidden_dim % 32 || ft % 32) fail(Status::Usage, "experts_init: hidden_dim and ffn/tiles must be multiples of 32");
    if (spec.hidden_dim > 16384 || ft > 16384) fail(Status::Usage, "experts_init: rows longer than 16384 elements unsupported");
    if (alias < 0) fail(Status::Usage, "experts_init: host_alias must be >= 0");
    eng.activate();
    st.layers = spec.num_layers;
    st.experts = spec.experts_per_layer;
    st.d = spec.hidden_dim;
    st.ffn = ffn;
    st.tiles = tiles;
    st.seed = seed;
    const int total = spec.num_layers * spec.experts_per_layer;
    st.alias = (alias > 0 && alias < total) ? alias : 0;
    st.expert_bytes = static_cast<size_t>(3) * ffn * spec.hidden_dim * 2;
    st.tile_bytes = st.expert_bytes / tiles;
    const int stored = st.alias > 0 ? st.alias : total;
    st.blocks.assign(stored, nullptr);

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
                std::memset(p, 0, st.expert_bytes);
                cudaError_t e = cudaHostRegister(p, st.expert_bytes, cudaHostRegisterDefault);
                if (e != cudaSuccess) {
                    std::free(p);
                    errors[w] = std::string("cudaHostRegister: ") + cudaGetErrorString(e);
                    return;
                }
                st.blocks[i] = static_cast<unsigned char*>(p);
            }
        });
    for (auto& t : pool) t.join();
    for (auto& e : errors)
        if (!e.empty()) fail(Status::Device, "experts_init: " + e);
    auto t1 = std::chrono::steady_clock::now();
    st.pin_seconds = std::chrono::duration<double>(t1 - t0).count();

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
        const int layer = i / spec.experts_per_layer, expert = i % spec.experts_per_layer;
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

}  // namespace adapmoe
