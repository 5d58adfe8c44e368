// fs_kernel.cuh -- Full search and motion-compensated SSE (P:342 aspect 4) on sm_100a.
//
// Full search evaluates every candidate of the +-p window (reading C9: all (2p+1)^2 are
// scorable over the edge-replicated reference; P:355 prints NSP 225 for +-7).  Tie rule
// (reading C13): (0,0) first, then raster order (dy outer, dx inner), strict minimum -- the
// argmin of the packed key (SAD << 13) | rank with rank(0,0) = 0 and
// rank(dx,dy) = 1 + (dy+p)(2p+1) + (dx+p) otherwise (SAD <= 65280 and rank <= 4225 keep it in
// 32 bits for B <= 16, p <= 32).
//
// One CTA per block.  The CTA stages the (B+2p) x (B+2p) edge-replicated window as four
// byte-phase copies (copy k holds the window shifted left by k bytes), so any candidate row
// is read as aligned 32-bit words; the current block sits in shared memory and is read by
// broadcast.  Each thread owns a strided subset of the candidates; the CTA argmin is a
// REDUX/CREDUX min over packed keys.
#pragma once
#include <stdint.h>

#include "dcds_kernel.cuh"

namespace me {

struct FsArgs {
    const uint8_t* cur0;
    const uint8_t* ref0;
    long long stride;
    int W, H, p;
    int nbx, nb;
    int lw;  // words per phase-copy row
    uint32_t* mv;
    uint32_t* sad;
    uint16_t* pts;
    unsigned long long* stats;
};

template <int B>
__global__ void __launch_bounds__(256) fs_kernel(const FsArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int pair = blockIdx.y;
    const int bi = blockIdx.x;
    const int bx = (bi % a.nbx) * B, by = (bi / a.nbx) * B;
    const uint8_t* cur = a.cur0 + (long long)pair * a.stride;
    const uint8_t* ref = a.ref0 + (long long)pair * a.stride;
    const int p = a.p, side = 2 * p + 1, nr = B + 2 * p, lw = a.lw;
    uint32_t* win = reinterpret_cast<uint32_t*>(smem);  // [4][nr][lw]
    uint32_t* cw = win + 4 * nr * lw;                   // [B][B/4]
    __shared__ uint32_t red[8];

    // stage the four phase copies: word (k, r, w) = bytes R(bx-p+4w+k+j, by-p+r), j = 0..3
    for (int e = threadIdx.x; e < 4 * nr * lw; e += blockDim.x) {
        const int k = e / (nr * lw);
        const int rem = e - k * nr * lw;
        const int r = rem / lw, w = rem - r * lw;
        const int y = min(max(by - p + r, 0), a.H - 1);
        const uint8_t* row = ref + (long long)y * a.W;
        uint32_t v = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int x = min(max(bx - p + 4 * w + k + j, 0), a.W - 1);
            v |= (uint32_t)row[x] << (8 * j);
        }
        win[e] = v;
    }
    for (int e = threadIdx.x; e < B * B / 4; e += blockDim.x) {
        const int r = e / (B / 4), w = e - r * (B / 4);
        cw[e] = *reinterpret_cast<const uint32_t*>(cur + (long long)(by + r) * a.W + bx + 4 * w);
    }
    __syncthreads();

    uint32_t key = 0xffffffffu;
    for (int c = threadIdx.x; c < side * side; c += blockDim.x) {
        const int dyp = c / side, dxp = c - dyp * side;  // dy+p, dx+p
        const uint32_t* rw = win + (dxp & 3) * nr * lw + dyp * lw + (dxp >> 2);
        uint32_t acc = 0;
#pragma unroll
        for (int i = 0; i < B; i++) {
#pragma unroll
            for (int w = 0; w < B / 4; w++) acc = vsad4(cw[i * (B / 4) + w], rw[i * lw + w], acc);
        }
        const uint32_t rank = (dxp == p && dyp == p) ? 0u : (uint32_t)(1 + c);
        key = min(key, (acc << 13) | rank);
    }
    key = __reduce_min_sync(FULL, key);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = key;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t k2 = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0xffffffffu;
        k2 = __reduce_min_sync(FULL, k2);
        const uint32_t rank = k2 & 0x1fffu;
        const int cidx = rank == 0 ? p * side + p : (int)rank - 1;
        const int mdy = cidx / side - p, mdx = cidx % side - p;
        // SSE of the block at the FS MV (for the per-pair statistics)
        uint32_t sse = 0;
        const int dxp = mdx + p, dyp = mdy + p;
        const uint32_t* rw = win + (dxp & 3) * nr * lw + dyp * lw + (dxp >> 2);
        for (int e = threadIdx.x; e < B * B / 4; e += 32) {
            const int r = e / (B / 4), w = e - r * (B / 4);
            sse = ssd4(cw[e], rw[r * lw + w], sse);
        }
        sse = __reduce_add_sync(FULL, sse);
        if (threadIdx.x == 0) {
            const long long g = (long long)pair * a.nb + bi;
            a.mv[g] = (uint32_t)(mdx & 0xffff) | ((uint32_t)mdy << 16);
            a.sad[g] = k2 >> 13;
            a.pts[g] = (uint16_t)(side * side);
            if (a.stats) {
                atomicAdd(&a.stats[pair * 3 + 0], (unsigned long long)(side * side));
                atomicAdd(&a.stats[pair * 3 + 1], (unsigned long long)(k2 >> 13));
                atomicAdd(&a.stats[pair * 3 + 2], (unsigned long long)sse);
            }
        }
    }
}

// Motion-compensated SSE: one warp per block, clamped reference reads (reading C9).
struct McArgs {
    const uint8_t* cur0;
    const uint8_t* ref0;
    long long stride;
    int W, H, B;
    int nbx, nb;
    const uint32_t* mv;  // packed (dx, dy) int16 pairs
    unsigned long long* sse;
};

__global__ void __launch_bounds__(256) mc_sse_kernel(const McArgs a) {
    const int lane = threadIdx.x & 31;
    const int bi = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int pair = blockIdx.y;
    if (bi >= a.nb) return;
    const uint8_t* cur = a.cur0 + (long long)pair * a.stride;
    const uint8_t* ref = a.ref0 + (long long)pair * a.stride;
    const int B = a.B;
    const int bx = (bi % a.nbx) * B, by = (bi / a.nbx) * B;
    const uint32_t m = a.mv[(long long)pair * a.nb + bi];
    const int dx = (int)(int16_t)(m & 0xffff), dy = (int)(int16_t)(m >> 16);
    uint32_t s = 0;
    for (int e = lane; e < B * B; e += 32) {
        const int i = e / B, j = e - i * B;
        const int c = cur[(long long)(by + i) * a.W + bx + j];
        const int y = min(max(by + i + dy, 0), a.H - 1), x = min(max(bx + j + dx, 0), a.W - 1);
        const int d = c - (int)ref[(long long)y * a.W + x];
        s += (uint32_t)(d * d);
    }
    s = __reduce_add_sync(FULL, s);
    if (lane == 0) atomicAdd(&a.sse[pair], (unsigned long long)s);
}

}  // namespace me
