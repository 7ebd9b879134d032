// Standalone check + microbenchmark of the K3 grouped tcgen05 kernels (tools/, not product).
// Builds a small slot pool of random bf16 experts in the tile-major layout, runs gate/up and down
// over a few segments, and compares H and the down partial sums with a CPU reference.  Then times
// the Mixtral-8x7B shape (8 experts x 352 MB, n tokens each).
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/grouped_check tools/grouped_check.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2408_10284_b200/csrc/kernels/grouped_ffn.cu"

using namespace adapmoe;

static float bf2f(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}
static uint16_t f2bf(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                     \
        }                                                                                \
    } while (0)

static int check(int D, int F, int tiles, std::vector<int> ns, std::vector<GSeg> segs) {
    const int Ft = F / tiles, E = (int)ns.size(), NP = 32;
    const size_t expert_elems = (size_t)3 * F * D;
    const size_t slot_elems = expert_elems + (size_t)64 * D;  // padding rows
    std::vector<uint16_t> pool(slot_elems * E);
    uint64_t s = 12345;
    for (auto& v : pool) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        v = f2bf(((float)((s >> 33) % 2001) - 1000.0f) / 1000.0f * 0.05f);
    }
    std::vector<uint16_t> X((size_t)E * NP * D, 0);
    for (int e = 0; e < E; ++e)
        for (int i = 0; i < ns[e]; ++i)
            for (int c = 0; c < D; ++c) {
                s = s * 6364136223846793005ull + 1442695040888963407ull;
                X[((size_t)e * NP + i) * D + c] = f2bf(((float)((s >> 33) % 2001) - 1000.0f) / 1000.0f);
            }
    uint16_t *d_pool, *d_x, *d_h;
    float* d_part;
    CK(cudaMalloc(&d_pool, pool.size() * 2));
    CK(cudaMalloc(&d_x, X.size() * 2));
    CK(cudaMalloc(&d_h, (size_t)E * NP * F * 2));
    CK(cudaMemset(d_h, 0, (size_t)E * NP * F * 2));
    CK(cudaMalloc(&d_part, (size_t)64 << 20));
    CK(cudaMemcpy(d_pool, pool.data(), pool.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_x, X.data(), X.size() * 2, cudaMemcpyHostToDevice));
    GroupedLaunch p;
    p.d = D; p.ft = Ft; p.f = F; p.np_stride = NP; p.h = d_h; p.partial = d_part;
    for (int e = 0; e < E; ++e) {
        p.ent[e].slot_row = (long long)e * (slot_elems / D);
        p.ent[e].n = ns[e];
        p.ent[e].np = std::max(16, (ns[e] + 15) / 16 * 16);
    }
    p.n_seg = (int)segs.size();
    for (int i = 0; i < p.n_seg; ++i) p.seg[i] = segs[i];
    const uint64_t rows = pool.size() / D;
    GroupedLaunch up = p, dn = p;
    CK(make_tensor_map_2d(&up.map_a, d_pool, rows, D, 64, 128));
    CK(make_tensor_map_2d(&up.map_b, d_x, (uint64_t)E * NP, D, 64, 16));
    CK(make_tensor_map_2d(&dn.map_a, d_pool, rows, D, 64, 64));
    CK(make_tensor_map_2d(&dn.map_b, d_h, (uint64_t)E * NP, F, 64, 16));
    grouped_plan_gate_up(up);
    grouped_plan_down(dn, 148);
    CK(launch_grouped_gate_up(up, 148, 0));
    CK(launch_grouped_down(dn, 148, 0));
    CK(cudaDeviceSynchronize());
    std::vector<uint16_t> H((size_t)E * NP * F);
    std::vector<float> part((size_t)dn.units * NP * 128);
    CK(cudaMemcpy(H.data(), d_h, H.size() * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(part.data(), d_part, part.size() * 4, cudaMemcpyDeviceToHost));
    // CPU reference
    double max_h_err = 0, max_h = 0, max_y_err = 0, max_y = 0;
    int bad_h = 0;
    std::vector<float> Href((size_t)E * NP * F, 0.f);
    for (const GSeg& sg : segs) {
        const int e = sg.entry;
        const uint16_t* W = pool.data() + (size_t)e * slot_elems;
        for (int t = sg.t0; t < sg.t1; ++t)
            for (int r = 0; r < Ft; ++r) {
                const uint16_t* w1 = W + ((size_t)t * 3 * Ft + 2 * r) * D;
                const uint16_t* w3 = w1 + D;
                for (int i = 0; i < ns[e]; ++i) {
                    const uint16_t* x = X.data() + ((size_t)e * NP + i) * D;
                    double a = 0, b = 0;
                    for (int c = 0; c < D; ++c) {
                        a += (double)bf2f(w1[c]) * bf2f(x[c]);
                        b += (double)bf2f(w3[c]) * bf2f(x[c]);
                    }
                    const double h = a / (1 + exp(-a)) * b;
                    const size_t idx = ((size_t)e * NP + i) * F + t * Ft + r;
                    Href[idx] = bf2f(f2bf((float)h));
                    const double g = bf2f(H[idx]);
                    const double err = fabs(g - h);
                    if (err > 0.02 * fabs(h) + 1e-3) {
                        if (bad_h < 5) printf("  H mismatch e%d i%d t%d r%d: got %g ref %g\n", e, i, t, r, g, h);
                        ++bad_h;
                    }
                    max_h_err = std::max(max_h_err, err);
                    max_h = std::max(max_h, fabs(h));
                }
            }
    }
    for (int sgi = 0; sgi < (int)segs.size(); ++sgi) {
        const GSeg& sg = segs[sgi];
        const int e = sg.entry;
        const uint16_t* W = pool.data() + (size_t)e * slot_elems;
        for (int j = 0; j < D; ++j)
            for (int i = 0; i < ns[e]; ++i) {
                double y = 0;
                for (int t = sg.t0; t < sg.t1; ++t)
                    for (int r = 0; r < Ft; ++r)
                        y += (double)bf2f(W[((size_t)t * 3 * Ft + 2 * Ft + r) * D + j]) *
                             Href[((size_t)e * NP + i) * F + t * Ft + r];
                double g = 0;
                const int m = j / 128;
                for (int c = 0; c < dn.kc; ++c)
                    g += part[((size_t)(dn.unit_prefix[sgi] + m * dn.kc + c) * NP + i) * 128 + (j % 128)];
                max_y_err = std::max(max_y_err, fabs(g - y));
                max_y = std::max(max_y, fabs(y));
            }
    }
    printf("check D=%d F=%d tiles=%d segs=%zu: H max err %.3g (max |h| %.3g, %d bad)  Y max err %.3g (max |y| %.3g) rel %.3g  kc=%d units=%d/%d\n",
           D, F, tiles, segs.size(), max_h_err, max_h, bad_h, max_y_err, max_y, max_y_err / max_y, dn.kc, up.units,
           dn.units);
    cudaFree(d_pool); cudaFree(d_x); cudaFree(d_h); cudaFree(d_part);
    return (bad_h == 0 && max_y_err / max_y < 2e-2) ? 0 : 1;
}

static void bench(int D, int F, int tiles, int experts, int n) {
    const int Ft = F / tiles, NP = (n + 15) / 16 * 16;
    const size_t expert_bytes = (size_t)3 * F * D * 2;
    uint16_t *d_pool, *d_x, *d_h;
    float* d_part;
    CK(cudaMalloc(&d_pool, expert_bytes * experts));
    CK(cudaMemset(d_pool, 0x11, expert_bytes * experts));
    CK(cudaMalloc(&d_x, (size_t)experts * NP * D * 2));
    CK(cudaMemset(d_x, 0x22, (size_t)experts * NP * D * 2));
    CK(cudaMalloc(&d_h, (size_t)experts * NP * F * 2));
    CK(cudaMalloc(&d_part, (size_t)256 << 20));
    GroupedLaunch p;
    p.d = D; p.ft = Ft; p.f = F; p.np_stride = NP; p.h = d_h; p.partial = d_part;
    p.n_seg = experts;
    for (int e = 0; e < experts; ++e) {
        p.ent[e].slot_row = (long long)e * (expert_bytes / (2 * D));
        p.ent[e].n = n;
        p.ent[e].np = NP;
        p.seg[e] = GSeg{e, 0, tiles};
    }
    const uint64_t rows = expert_bytes * experts / (2 * D);
    GroupedLaunch up = p, dn = p;
    CK(make_tensor_map_2d(&up.map_a, d_pool, rows, D, 64, 128));
    CK(make_tensor_map_2d(&up.map_b, d_x, (uint64_t)experts * NP, D, 64, 16));
    CK(make_tensor_map_2d(&dn.map_a, d_pool, rows, D, 64, 64));
    CK(make_tensor_map_2d(&dn.map_b, d_h, (uint64_t)experts * NP, F, 64, 16));
    grouped_plan_gate_up(up);
    grouped_plan_down(dn, 148);
    cudaEvent_t a, b, c;
    cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c);
    float best_up = 1e9, best_dn = 1e9;
    for (int r = 0; r < 8; ++r) {
        cudaEventRecord(a);
        CK(launch_grouped_gate_up(up, 148, 0));
        cudaEventRecord(b);
        CK(launch_grouped_down(dn, 148, 0));
        cudaEventRecord(c);
        CK(cudaEventSynchronize(c));
        float m1, m2;
        cudaEventElapsedTime(&m1, a, b);
        cudaEventElapsedTime(&m2, b, c);
        if (r >= 2) { best_up = std::min(best_up, m1); best_dn = std::min(best_dn, m2); }
    }
    const double gu = (double)experts * 2 * F * D * 2, dw = (double)experts * F * D * 2;
    const double flops_up = 2.0 * experts * 2 * F * D * n, flops_dn = 2.0 * experts * F * D * n;
    printf("bench D=%d F=%d experts=%d n=%d: gate/up %.1f us = %.0f GB/s %.1f TF/s (units %d) | down %.1f us = %.0f GB/s %.1f TF/s (units %d kc %d) | total %.0f GB/s\n",
           D, F, experts, n, best_up * 1e3, gu / (best_up * 1e-3) / 1e9, flops_up / (best_up * 1e-3) / 1e12, up.units,
           best_dn * 1e3, dw / (best_dn * 1e-3) / 1e9, flops_dn / (best_dn * 1e-3) / 1e12, dn.units, dn.kc,
           (gu + dw) / ((best_up + best_dn) * 1e-3) / 1e9);
    cudaFree(d_pool); cudaFree(d_x); cudaFree(d_h); cudaFree(d_part);
}

int main(int argc, char** argv) {
    if (argc > 1 && !strcmp(argv[1], "bench-only")) {  // ncu target: one 8-expert n=16 launch pair
        bench(4096, 14336, 4, 8, 16);
        return 0;
    }
    int fails = 0;
    const bool small = argc > 1 && !strcmp(argv[1], "check-small");  // compute-sanitizer target
    fails += check(256, 1024, 4, {5, 17}, {GSeg{0, 0, 4}, GSeg{1, 2, 3}});
    if (small) {
        fails += check(512, 2048, 2, {16, 3, 9}, {GSeg{0, 0, 2}, GSeg{1, 0, 2}, GSeg{2, 1, 2}});
        printf("%s (%d failing checks)\n", fails ? "FAIL" : "PASS", fails);
        return fails;
    }
    fails += check(256, 1024, 4, {1, 32}, {GSeg{1, 0, 4}, GSeg{0, 1, 2}, GSeg{0, 3, 4}});
    fails += check(512, 2048, 2, {16, 3, 9}, {GSeg{0, 0, 2}, GSeg{1, 0, 2}, GSeg{2, 1, 2}});
    fails += check(4096, 14336, 4, {7, 30}, {GSeg{0, 0, 4}, GSeg{1, 3, 4}});
    printf("%s (%d failing checks)\n", fails ? "FAIL" : "PASS", fails);
    if (argc > 1 || fails == 0) {
        for (int n : {1, 4, 8, 16, 32, 64}) bench(4096, 14336, 4, 8, n);
        bench(4096, 14336, 4, 2, 16);
        bench(6144, 16384, 4, 8, 16);
    }
    return fails;
}
