// int_peaks.cu -- microbenchmark of the integer SIMD instructions the DCDS path issues, on
// the GPU it runs on (B200 / sm_100a).  Not part of libme.so; its JSON output (committed under
// profiles/) supplies the "alu" roofline denominator the paper's hardware guide does not
// document (SURVEY.md finding 9: the VABSDIFF4 issue rate is unknown).
//
// Each thread runs NCHAIN independent accumulate chains; the grid fills every SM at full
// occupancy; the loop runs long enough (>= ~0.5 s) for clocks to settle.  Rates are reported
// as lane-ops per SM per clock using the measured SM clock (clock64 over the same kernel).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/int_peaks tools/int_peaks.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int NCHAIN = 8;

__device__ __forceinline__ uint32_t vsad4(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int OP>
__global__ void kern(uint32_t* out, int iters, uint32_t seed, long long* cycles) {
    uint32_t acc[NCHAIN];
    uint32_t a = seed ^ threadIdx.x, b = seed * 2654435761u + blockIdx.x;
#pragma unroll
    for (int k = 0; k < NCHAIN; k++) acc[k] = a + k;
    long long t0 = clock64();
    unsigned long long g0 = gtimer();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < NCHAIN; k++) {
            if (OP == 0) acc[k] = vsad4(a + k, b, acc[k]);               // VABSDIFF4.U8.ACC
            if (OP == 1) acc[k] = __dp4a(a + k, b, acc[k]);              // IDP.4A
            if (OP == 2) acc[k] = acc[k] + (a ^ k) + b;                  // IADD3
            if (OP == 3) acc[k] = __funnelshift_r(acc[k], b, a + k);     // SHF
            if (OP == 4) acc[k] = __byte_perm(acc[k], b, a + k);         // PRMT
            if (OP == 5) acc[k] = k < NCHAIN / 2 ? vsad4(a + k, b, acc[k])    // half VABSDIFF4,
                                                 : __byte_perm(acc[k], b, a + k);  // half PRMT
            if (OP == 6) acc[k] = k < NCHAIN / 2 ? vsad4(a + k, b, acc[k])    // half VABSDIFF4,
                                                 : __funnelshift_r(acc[k], b, a + k);  // half SHF
            if (OP == 7) acc[k] = k < NCHAIN / 2 ? vsad4(a + k, b, acc[k])    // half VABSDIFF4,
                                                 : acc[k] + (a ^ k) + b;   // half IADD3/LOP3
        }
    }
    long long t1 = clock64();
    unsigned long long g1 = gtimer();
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < NCHAIN; k++) s ^= acc[k];
    if (s == 0x12345678u) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) { cycles[0] = t1 - t0; cycles[1] = (long long)(g1 - g0); }
}

template <int OP>
double run(const char* name, int sms, int blocks_per_sm, int threads, int iters, double* ops_per_sm_clk) {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 4);
    cudaMalloc(&cyc, 16);
    dim3 grid(sms * blocks_per_sm);
    kern<OP><<<grid, threads>>>(out, iters / 10, 1u, cyc);  // warm-up
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<OP><<<grid, threads>>>(out, iters, 1u, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c[2] = {0, 1};
    cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
    const double lane_ops = (double)grid.x * threads * iters * NCHAIN;
    const double per_s = lane_ops / (ms * 1e-3);
    const double clk_hz = (double)c[0] / ((double)c[1] * 1e-9);  // block 0: cycles / ns
    *ops_per_sm_clk = per_s / (clk_hz * sms);
    printf("  \"%s\": {\"lane_ops_per_s\": %.6e, \"ms\": %.3f, \"sm_clock_mhz_est\": %.1f, "
           "\"lane_ops_per_sm_per_clk\": %.3f},\n",
           name, per_s, ms, clk_hz / 1e6, *ops_per_sm_clk);
    cudaFree(out);
    cudaFree(cyc);
    return per_s;
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const int sms = prop.multiProcessorCount;
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("{\n  \"gpu\": \"%s\", \"sms\": %d, \"sm_max_mhz\": %.1f,\n", prop.name, sms, clk_khz / 1e3);
    double r;
    run<0>("vabsdiff4_add", sms, 8, 256, 200000, &r);
    run<1>("dp4a", sms, 8, 256, 200000, &r);
    run<2>("iadd3", sms, 8, 256, 200000, &r);
    run<3>("shf", sms, 8, 256, 200000, &r);
    run<4>("prmt", sms, 8, 256, 200000, &r);
    run<5>("vabsdiff4_prmt_mix", sms, 8, 256, 200000, &r);
    run<6>("vabsdiff4_shf_mix", sms, 8, 256, 200000, &r);
    run<7>("vabsdiff4_iadd_mix", sms, 8, 256, 200000, &r);
    printf("  \"nchain\": %d, \"threads_per_sm\": %d\n}\n", NCHAIN, 8 * 256);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
