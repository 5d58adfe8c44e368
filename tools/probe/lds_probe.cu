// lds_probe.cu -- random shared-memory gathers by width on B200: LDS.32 / LDS.64 / LDS.128,
// lanes partly active (12 of 32, as in the DCDS kernel) or all.  Prints loads/s and bytes/s.
// Not part of libme.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int NW = 3072;  // 12 KB

template <int WIDTH, bool PARTIAL>
__global__ void __launch_bounds__(128) probe(const uint32_t* g, uint32_t* out, int iters) {
    __shared__ __align__(16) uint32_t sh[NW];
    for (int i = threadIdx.x; i < NW; i += blockDim.x) sh[i] = g[i];
    __syncthreads();
    uint32_t x = threadIdx.x * 2654435761u + blockIdx.x * 97u, acc = 0;
    const bool on = !PARTIAL || (threadIdx.x & 31) < 12;
    if (on) {
        for (int it = 0; it < iters; it++) {
#pragma unroll
            for (int u = 0; u < 6; u++) {
                x = x * 1664525u + 1013904223u;
                const int a = ((x >> 8) % (NW / 4)) * 4;  // 16-byte aligned word index
                if (WIDTH == 4) acc += sh[a + (x & 3)];
                if (WIDTH == 8) { const uint2 v = *reinterpret_cast<const uint2*>(&sh[a + (x & 2)]); acc += v.x ^ v.y; }
                if (WIDTH == 16) { const uint4 v = *reinterpret_cast<const uint4*>(&sh[a]); acc += v.x ^ v.y ^ v.z ^ v.w; }
            }
        }
    }
    if (acc == 0x12345u) out[0] = acc;
}

template <int WIDTH, bool PARTIAL>
void run(const uint32_t* g, uint32_t* out, int sms) {
    const int iters = 4000;
    dim3 grid(sms * 12);
    probe<WIDTH, PARTIAL><<<grid, 128>>>(g, out, 10);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<WIDTH, PARTIAL><<<grid, 128>>>(g, out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double lanes = (double)grid.x * 128 * (PARTIAL ? 12.0 / 32 : 1.0) * iters * 6;
    printf("LDS.%d %s: %.3e loads/s, %.3e bytes/s, %.2f lane-loads/clk/SM\n", WIDTH * 8,
           PARTIAL ? "12 lanes" : "32 lanes", lanes / (ms * 1e-3), lanes * WIDTH / (ms * 1e-3),
           lanes / (ms * 1e-3) / (sms * 1.965e9));
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *g, *out;
    cudaMalloc(&g, NW * 4); cudaMalloc(&out, 4);
    cudaMemset(g, 1, NW * 4);
    run<4, false>(g, out, sms); run<8, false>(g, out, sms); run<16, false>(g, out, sms);
    run<4, true>(g, out, sms); run<8, true>(g, out, sms); run<16, true>(g, out, sms);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
