// tex_probe.cu -- does the texture path add gather bandwidth beside shared memory on B200?
// Random 32-bit gathers: (A) LDS from a 12 KB shared buffer, (B) tex1Dfetch from a 12 KB
// texture (L1-resident), (C) both interleaved 2:1.  Prints gathers/s for each.  Not part of libme.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int NW = 3072;  // 12 KB of words

template <int MODE>
__global__ void __launch_bounds__(128) probe(cudaTextureObject_t tex, const uint32_t* g, uint32_t* out, int iters) {
    __shared__ uint32_t sh[NW];
    for (int i = threadIdx.x; i < NW; i += blockDim.x) sh[i] = g[i];
    __syncthreads();
    uint32_t x = threadIdx.x * 2654435761u + blockIdx.x * 97u, acc = 0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 6; u++) {
            x = x * 1664525u + 1013904223u;
            const int a = (x >> 8) % NW;
            if (MODE == 0) acc += sh[a];
            if (MODE == 1) acc += tex1Dfetch<uint32_t>(tex, a);
            if (MODE == 2) acc += (u % 3 == 2) ? tex1Dfetch<uint32_t>(tex, a) : sh[a];
        }
    }
    if (acc == 0x12345u) out[0] = acc;
}

template <int MODE>
double run(cudaTextureObject_t tex, const uint32_t* g, uint32_t* out, int sms) {
    const int iters = 4000;
    dim3 grid(sms * 12);
    probe<MODE><<<grid, 128>>>(tex, g, out, 10);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<MODE><<<grid, 128>>>(tex, g, out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return (double)grid.x * 128 * iters * 6 / (ms * 1e-3);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *g, *out;
    cudaMalloc(&g, NW * 4); cudaMalloc(&out, 4);
    cudaMemset(g, 1, NW * 4);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = g;
    rd.res.linear.desc = cudaCreateChannelDesc<uint32_t>();
    rd.res.linear.sizeInBytes = NW * 4;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex; cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    printf("LDS gathers/s %.3e\n", run<0>(tex, g, out, sms));
    printf("TEX gathers/s %.3e\n", run<1>(tex, g, out, sms));
    printf("mix 2:1 gathers/s %.3e\n", run<2>(tex, g, out, sms));
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
