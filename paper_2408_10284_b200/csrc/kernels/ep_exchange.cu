// Expert-parallel exchange kernels (see ep_exchange.hpp).
#include <cuda_runtime.h>

#include "ep_exchange.hpp"

namespace adapmoe {

namespace {

__global__ void ep_signal_kernel(const __grid_constant__ EpSignalArgs a) {
    // every partial store of this call precedes this kernel on the stream; make them visible to the
    // peers before the flag (system scope: peers may be other GPUs)
    __threadfence_system();
    const int g = threadIdx.x;
    if (g < a.world) {
        unsigned* f = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(a.peer_flags[g]) + 64 * a.rank);
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(a.call) : "memory");
    }
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void ep_wait_kernel(const unsigned char* region, int world, unsigned call) {
    const int g = threadIdx.x;
    if (g < world) {
        const unsigned* f = reinterpret_cast<const unsigned*>(region + 64 * g);
        long long budget = 80ll * 1000 * 1000;  // ~20 s of 256 ns sleeps
        while (static_cast<int>(ld_acquire_sys(f) - call) < 0) {
            if (--budget < 0) {
                atomicExch(reinterpret_cast<unsigned*>(const_cast<unsigned char*>(region) + 64 * kMaxEpPeers), 1u);
                break;
            }
            __nanosleep(256);
        }
    }
    __syncwarp();
    __threadfence();  // later kernels on this stream read the slots the peers published
}

__global__ void ep_reduce_kernel(const __grid_constant__ EpReduceArgs a) {
    const long long elems = a.rows * a.d;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < elems;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long o = (i / a.d) * a.row_stride + i % a.d;
        float s = a.slots[o];
        for (int g = 1; g < a.world; ++g) s = __fadd_rn(s, a.slots[g * a.slot_stride + o]);
        a.out[o] = s;
    }
}

}  // namespace

cudaError_t launch_ep_signal(const EpSignalArgs& a, cudaStream_t stream) {
    if (a.world < 1 || a.world > kMaxEpPeers) return cudaErrorInvalidValue;
    ep_signal_kernel<<<1, 32, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_ep_wait(const unsigned char* region, int world, unsigned call, cudaStream_t stream) {
    if (world < 1 || world > kMaxEpPeers) return cudaErrorInvalidValue;
    ep_wait_kernel<<<1, 32, 0, stream>>>(region, world, call);
    return cudaGetLastError();
}

cudaError_t launch_ep_reduce(const EpReduceArgs& a, cudaStream_t stream) {
    if (a.rows <= 0 || a.d <= 0) return cudaSuccess;
    const long long blocks = (a.rows * a.d + 255) / 256;
    ep_reduce_kernel<<<static_cast<int>(blocks < 296 ? blocks : 296), 256, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace adapmoe
