// CPU check (tests/test_host_rng.py): SeededRng::normals (bulk raw draws + threaded Box-Muller)
// returns exactly the values of sequential normal() calls, across odd / even counts, a cached
// spare carried in and out, and lengths above the threading threshold.
#include <cstdio>
#include <cstring>
#include <vector>

#include "host/policy.hpp"

int main() {
    using adapmoe::SeededRng;
    for (std::uint64_t seed : {0ull, 99ull, 5000ull, 77ull}) {
        SeededRng a(seed), b(seed);
        for (size_t n : {1ul, 2ul, 5ul, 4096ul, 37ul, 1ul, 300001ul, 64ul, 2000000ul, 3ul}) {
            std::vector<double> bulk(n), seq(n);
            a.normals(bulk.data(), n);
            for (auto& v : seq) v = b.normal();
            if (std::memcmp(bulk.data(), seq.data(), n * sizeof(double)) != 0) {
                std::printf("MISMATCH seed %llu n %zu\n", static_cast<unsigned long long>(seed), n);
                return 1;
            }
        }
        if (a.next_u64() != b.next_u64()) {
            std::printf("STREAM POSITION seed %llu\n", static_cast<unsigned long long>(seed));
            return 1;
        }
    }
    std::printf("OK\n");
    return 0;
}
