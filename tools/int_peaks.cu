// int_peaks.cu -- microbenchmark of the integer instructions the DCDS path issues, on the GPU
// it runs on (B200 / sm_100a).  Not part of libme.so; its JSON output (committed under
// profiles/) supplies the "alu" roofline denominator the hardware guide does not document
// (SURVEY.md finding 9: the VABSDIFF4 issue rate is unknown) and the pipe-sharing facts the
// kernel design uses (which instruction pairs co-issue).
//
// Every operation is one `asm volatile` PTX instruction on a loop-carried accumulator (acc[k]
// feeds the next iteration's instruction of chain k), so nothing can be folded, hoisted or
// merged by the compiler (round 1's IADD3 leg was loop-invariant and got folded).
// Each thread runs NCHAIN independent chains; the grid fills every SM at full occupancy.
// Rates are lane-ops per SM per clock at the clock measured over the same kernel (clock64 /
// globaltimer of block 0).  The SASS of each variant is checked by tests/test_int_peaks_sass.py.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/int_peaks tools/int_peaks.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int NCHAIN = 8;

#define OP3(name, ptx)                                                                   \
    __device__ __forceinline__ uint32_t name(uint32_t a, uint32_t b, uint32_t c) {       \
        uint32_t d;                                                                      \
        asm volatile(ptx : "=r"(d) : "r"(a), "r"(b), "r"(c));                            \
        return d;                                                                        \
    }
OP3(op_vabsdiff4, "vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;")  // VABSDIFF4.U8.ACC
OP3(op_dp4a, "dp4a.u32.u32 %0, %1, %2, %3;")                    // IDP.4A
OP3(op_shf, "shf.r.wrap.b32 %0, %1, %2, %3;")                   // SHF.R.W
OP3(op_prmt, "prmt.b32 %0, %1, %2, %3;")                        // PRMT
OP3(op_lop3, "lop3.b32 %0, %1, %2, %3, 0x96;")                  // LOP3 (xor3)
OP3(op_imad, "mad.lo.u32 %0, %1, %2, %3;")                      // IMAD
OP3(op_imadhi, "mad.hi.u32 %0, %1, %2, %3;")                    // IMAD.HI
OP3(op_iadd3, "{.reg .u32 t; add.u32 t, %1, %2; add.u32 %0, t, %3;}")  // IADD3 (or IMAD.IADD)

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// OP < 10: one instruction kind on all chains; OP >= 10: chains alternate between
// VABSDIFF4 and a second kind (does the pair co-issue on different pipes?)
template <int OP>
__device__ __forceinline__ uint32_t step(int k, uint32_t acc, uint32_t a, uint32_t b) {
    const int op = OP < 10 ? OP : ((k & 1) ? OP - 10 : 0);
    switch (op) {
        case 0: return op_vabsdiff4(a, b, acc);
        case 1: return op_dp4a(a, b, acc);
        case 2: return op_shf(acc, b, a);
        case 3: return op_prmt(acc, b, a);
        case 4: return op_lop3(acc, b, a);
        case 5: return op_imad(acc, b, a);
        case 6: return op_imadhi(acc, b, a);
        default: return op_iadd3(acc, b, a);
    }
}

template <int OP>
__global__ void kern(uint32_t* out, int iters, uint32_t seed, long long* cycles) {
    uint32_t acc[NCHAIN];
    const uint32_t a = seed ^ threadIdx.x, b = seed * 2654435761u + blockIdx.x;
#pragma unroll
    for (int k = 0; k < NCHAIN; k++) acc[k] = a + k;
    long long t0 = clock64();
    unsigned long long g0 = gtimer();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < NCHAIN; k++) acc[k] = step<OP>(k, acc[k], a + k, b);
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
void run(const char* name, int sms, int blocks_per_sm, int threads, int iters, bool last = false) {
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
    const double r = per_s / (clk_hz * sms);
    printf("  \"%s\": {\"lane_ops_per_s\": %.6e, \"ms\": %.3f, \"sm_clock_mhz_est\": %.1f, "
           "\"lane_ops_per_sm_per_clk\": %.3f, \"warp_instr_per_sm_per_clk\": %.3f}%s\n",
           name, per_s, ms, clk_hz / 1e6, r, r / 32.0, last ? "" : ",");
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const int sms = prop.multiProcessorCount;
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("{\n  \"gpu\": \"%s\", \"sms\": %d, \"sm_max_mhz\": %.1f, \"nchain\": %d, \"threads_per_sm\": %d,\n",
           prop.name, sms, clk_khz / 1e3, NCHAIN, 8 * 256);
    const int it = 200000;
    run<0>("vabsdiff4_add", sms, 8, 256, it);
    run<1>("dp4a", sms, 8, 256, it);
    run<2>("shf", sms, 8, 256, it);
    run<3>("prmt", sms, 8, 256, it);
    run<4>("lop3", sms, 8, 256, it);
    run<5>("imad", sms, 8, 256, it);
    run<6>("imad_hi", sms, 8, 256, it);
    run<7>("iadd3", sms, 8, 256, it);
    run<11>("mix_vabsdiff4_dp4a", sms, 8, 256, it);
    run<12>("mix_vabsdiff4_shf", sms, 8, 256, it);
    run<13>("mix_vabsdiff4_prmt", sms, 8, 256, it);
    run<14>("mix_vabsdiff4_lop3", sms, 8, 256, it);
    run<15>("mix_vabsdiff4_imad", sms, 8, 256, it);
    run<16>("mix_vabsdiff4_imad_hi", sms, 8, 256, it);
    run<17>("mix_vabsdiff4_iadd3", sms, 8, 256, it, true);
    printf("}\n");
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
