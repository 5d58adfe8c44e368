// copy_probe.cu -- a stand-in for NCCL's collective kernels (a fixed number of CTAs streaming
// a buffer) to measure on ONE GPU how well the DCDS search overlaps with a concurrent
// communication-like kernel on a high-priority stream (tools/overlap_probe.py).  Not part of
// libme.so.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

extern "C" int probe_copy(const void* src, void* dst, size_t bytes, int nctas, void* stream) {
    copy_kernel<<<nctas, 512, 0, (cudaStream_t)stream>>>((const uint4*)src, (uint4*)dst, bytes / 16);
    return (int)cudaGetLastError();
}
