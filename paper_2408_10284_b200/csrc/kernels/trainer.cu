// First-layer predictive gate trainer: the gradient + update half of one full-batch gradient-descent
// step of train_predictive_gate (inc/prefetch.hpp:194-213), bit-exact with the reference.
//
// The reference accumulates dW[i][j] over the training pairs in pair order, skipping pairs whose
// input x_i is zero, as separately rounded fp64 multiply / add (no FMA contraction in its build),
// then scales by 1/P and applies W -= lr * dW (kl_training_grad, inc/prefetch.hpp:171-192).  Every
// (i, j) is an independent sequential chain, so one thread per weight reproduces the order exactly.
// The logits (GateMatrix::logits) come from K1's exact fp64 path and the softmaxes from the host's
// glibc exp (see runtime/engine.cpp Engine::train_first_gate).
#include <cuda_runtime.h>

#include "trainer.hpp"

namespace adapmoe {

namespace {

__global__ void gate_grad_step_kernel(double* __restrict__ w, const double* __restrict__ x,
                                      const double* __restrict__ diff, int pairs, int d, int n, double inv,
                                      double lr) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= d * n) return;
    const int i = k / n, j = k % n;
    double g = 0.0;
    for (int p = 0; p < pairs; ++p) {
        const double xi = x[static_cast<size_t>(p) * d + i];
        if (xi == 0.0) continue;
        g = __dadd_rn(g, __dmul_rn(xi, diff[static_cast<size_t>(p) * n + j]));
    }
    g = __dmul_rn(g, inv);
    w[k] = __dsub_rn(w[k], __dmul_rn(lr, g));
}

}  // namespace

cudaError_t launch_gate_grad_step(double* w, const double* x, const double* diff, int pairs, int d, int n,
                                  double lr, cudaStream_t stream) {
    if (pairs < 1 || d < 1 || n < 1) return cudaErrorInvalidValue;
    const int total = d * n;
    gate_grad_step_kernel<<<(total + 255) / 256, 256, 0, stream>>>(w, x, diff, pairs, d, n,
                                                                   1.0 / static_cast<double>(pairs), lr);
    return cudaGetLastError();
}

}  // namespace adapmoe
