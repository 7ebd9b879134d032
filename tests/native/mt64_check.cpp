// CPU check (tests/test_host_rng.py): the engine's bulk MT19937-64 (csrc/host/policy.hpp) emits
// std::mt19937_64's sequence, word for word, through single draws and bulk fills of any length.
#include <cstdio>
#include <random>
#include <vector>

#include "host/policy.hpp"

int main() {
    for (std::uint64_t seed : {0ull, 1ull, 5ull, 99ull, 5000ull, 0xffffffffffffffffull, 1234567890123ull}) {
        std::mt19937_64 ref(seed);
        adapmoe::Mt64 ours(seed);
        std::vector<std::uint64_t> buf;
        size_t n = 0;
        for (size_t chunk : {1ul, 7ul, 311ul, 312ul, 313ul, 1000ul, 100000ul, 3ul, 624ul}) {
            buf.resize(chunk);
            if (chunk % 2) {
                ours.fill(buf.data(), chunk);
            } else {
                for (auto& v : buf) v = ours();
            }
            for (size_t i = 0; i < chunk; ++i, ++n) {
                const std::uint64_t r = ref();
                if (buf[i] != r) {
                    std::printf("MISMATCH seed %llu word %zu\n", static_cast<unsigned long long>(seed), n);
                    return 1;
                }
            }
        }
    }
    std::printf("OK\n");
    return 0;
}
