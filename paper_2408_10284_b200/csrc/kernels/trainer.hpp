// First-layer predictive gate trainer kernel (host launch interface), see trainer.cu.
#pragma once

#include <cuda_runtime_api.h>

namespace adapmoe {

// W[d][n] -= lr * (1/P) * sum_p x_p (outer) diff_p, reference order.  x [P][d], diff [P][n] = q - p.
cudaError_t launch_gate_grad_step(double* w, const double* x, const double* diff, int pairs, int d, int n,
                                  double lr, cudaStream_t stream);

}  // namespace adapmoe
