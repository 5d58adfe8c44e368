// fs_kernel.cuh -- Full search and motion-compensated SSE (P:342 aspect 4) on sm_100a.
//
// Full search evaluates every candidate of the +-p window (reading C9: all (2p+1)^2 are
// scorable over the edge-replicated reference; P:355 prints NSP 225 for +-7).  Tie rule
// (reading C13): (0,0) first, then raster order (dy outer, dx inner), strict minimum.  The
// kernel takes the argmin of the packed key (SAD << 13) + rank, rank(dx,dy) = 1 + (dy+p)(2p+1)
// + (dx+p) for every candidate (SAD <= 65280 and rank <= 4225 keep it in 32 bits for B <= 16,
// p <= 32) -- the raster-first minimum -- and then applies centre-first once per block: (0,0)
// is the MV iff its SAD is <= that minimum's.
//
// One CTA per tile of blocks: the tile's edge-replicated reference region is staged by TMA
// (as for DCDS) and expanded into four byte-phase copies; see fs_kernel below.
#pragma once
#include <stdint.h>

#include "dcds_kernel.cuh"

namespace me {

struct FsArgs {
    int W, H, p;
    int tbx, tby, ntx;      // tile of blocks per CTA, tiles per row
    int pitch, rh;          // staged region (TMA box) width / rows
    int rh_pad;             // rows of each byte-phase copy (>= rh; rows past rh are padding)
    int cstride;            // bytes between byte-phase copies (cstride/4 = 8 mod 32 words)
    int cur_off;            // byte offset of the current tile in shared memory
    int nbx, nb;
    int nch;                // dy chunks of B candidates: ceil((2p+1) / B)
    int nsplit;             // a (block, dx) item's chunks are split over nsplit thread items
    uint32_t* mv;
    uint32_t* sad;
    uint16_t* pts;
    unsigned long long* stats;
};

// One CTA per tile of blocks.  Thread items are (block, dx, chunk of B consecutive dy); a
// thread keeps the current block in registers and streams the 2B-1 reference rows of its
// chunk once, accumulating the SADs of all B candidates of the chunk (each reference row is
// loaded once and reused by up to B candidates: W4 loads feed B*W4 VABSDIFF4).  Rows come
// from the byte-phase copy (dx & 3) so they are aligned words; consecutive lanes take
// consecutive dx, which the copy stride spreads over all 32 banks.  Per-block argmin:
// shared-memory atomicMin on (SAD << 13 | rank) keys (reading C13).
// SIDE > 0 (with the region pitch PITCH): a build for one window size (2p + 1 = SIDE) whose
// thread items sweep all SIDE + B - 1 rows of their dx column once -- every row loaded once
// for up to B candidates, at immediate offsets from one base, each candidate's key formed as
// its last row passes (at most B accumulators live).
template <int B, int SIDE = 0, int PITCH = 0>
__global__ void __launch_bounds__(512)
    fs_kernel(const __grid_constant__ CUtensorMap tm_cur, const __grid_constant__ CUtensorMap tm_ref,
              const FsArgs a) {
    constexpr int W4 = B / 4;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ uint32_t s_key[64];
    __shared__ unsigned long long s_stat[16][2];  // per-warp sums of SAD, SSE (one pair per CTA)
    uint8_t* smem = smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127);
    const int pair = blockIdx.y;
    const int tx = blockIdx.x % a.ntx, ty = blockIdx.x / a.ntx;
    const int TW = a.tbx * B, TH = a.tby * B;
    const int x0 = tx * TW, y0 = ty * TH;
    const int xs = (x0 - a.p) & ~15, ys = y0 - a.p;
    const int pitch = a.pitch, p = a.p, side = 2 * p + 1;
    uint8_t* sref = smem;
    uint8_t* scur = smem + a.cur_off;
    const int nby = a.nb / a.nbx;
    const int tbx_e = min(a.tbx, a.nbx - tx * a.tbx), tby_e = min(a.tby, nby - ty * a.tby);
    const int nbt = tbx_e * tby_e;

    if (threadIdx.x == 0) {  // init and issue at once: the barrier publishes the init meanwhile
        mbar_init(&s_bar, 1);
        mbar_expect_tx(&s_bar, (uint32_t)(pitch * a.rh + TW * TH));
        tma_load_3d(sref, &tm_ref, xs, ys, pair, &s_bar);
        tma_load_3d(scur, &tm_cur, x0, y0, pair, &s_bar);
    }
    if (threadIdx.x < 64) s_key[threadIdx.x] = 0xffffffffu;
    __syncthreads();
    mbar_wait(&s_bar, 0);
    if (xs < 0 || ys < 0 || xs + pitch > a.W || ys + a.rh > a.H)
        fixup_edges(sref, pitch, a.rh, xs, ys, a.W, a.H);
    __syncthreads();
    // byte-phase copies 1..3 of the region (copy k word q = region bytes 4q+k .. 4q+k+3)
    {
        const uint32_t* c0 = reinterpret_cast<const uint32_t*>(sref);
        const int nw = pitch * a.rh_pad / 4;
        for (int q = threadIdx.x; q < nw; q += blockDim.x) {
            const uint32_t lo = c0[q], hi = (q + 1 < nw) ? c0[q + 1] : 0u;
#pragma unroll
            for (int k = 1; k < 4; k++)
                reinterpret_cast<uint32_t*>(sref + k * a.cstride)[q] = __funnelshift_r(lo, hi, 8 * k);
        }
    }
    __syncthreads();

    // Thread items are (block, dx, split); each loops over its share of the ceil((2p+1)/B)
    // chunks of B consecutive dy with the current block held in registers.  Staged rows are padded (rh_pad) so the
    // row loop needs no bounds check: rows past the window only feed candidates dy > p, which
    // are masked out of the key.
    const int nsplit = a.nsplit, cps = (a.nch + nsplit - 1) / nsplit;  // chunks per item
    const int nitem = nbt * side * nsplit;
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(sref);
    const int cwords = a.cstride >> 2, pw = pitch >> 2;
    // x / d as floor((x + 1/2) * rcp(d)): exact here (x < 2^14, d <= 65: the product stays
    // >= 0.5/d from an integer, far above the float rounding error)
    const float r_side = __frcp_rn((float)side), r_split = __frcp_rn((float)nsplit),
                r_tbx = __frcp_rn((float)tbx_e);
    auto fdiv = [](int x, float r) { return (int)(((float)x + 0.5f) * r); };
    for (int it = threadIdx.x; it < nitem; it += blockDim.x) {
        const int bs = fdiv(it, r_side);
        const int dxp = it - bs * side;  // dx + p
        const int b = fdiv(bs, r_split), sp = bs - b * nsplit;
        const int lby = fdiv(b, r_tbx), lbx = b - lby * tbx_e;
        uint32_t cw[B][W4];
#pragma unroll
        for (int i = 0; i < B; i++)
#pragma unroll
            for (int w = 0; w < W4; w++)
                cw[i][w] = reinterpret_cast<const uint32_t*>(scur + (lby * B + i) * TW + lbx * B)[w];
        // candidate (dx, dy) block row i sits at region row lby*B + dy + p + i, column
        // (x0 + lbx*B - p - xs) + dx + p
        const int col = (x0 + lbx * B - p - xs) + dxp;
        const uint32_t* base = sw + (col & 3) * cwords + (col >> 2) + (lby * B) * pw;
        uint32_t key = 0xffffffffu;
        if constexpr (SIDE > 0) {
            // candidate (dx, dy = d - p) block row i is region row y = d + i (from base); its
            // key (SAD << 13) + rank, rank = 1 + d*SIDE + (dx + p): the d*SIDE part is added
            // per candidate, 1 + dx + p once for the column
            constexpr int PW = PITCH / 4;
            uint32_t acc[SIDE];
#pragma unroll
            for (int y = 0; y < SIDE + B - 1; y++) {
                uint32_t rw[W4];
#pragma unroll
                for (int w = 0; w < W4; w++) rw[w] = base[y * PW + w];
#pragma unroll
                for (int d = 0; d < SIDE; d++) {
                    const int i = y - d;
                    if (i >= 0 && i < B) {
#pragma unroll
                        for (int w = 0; w < W4; w++) acc[d] = vsad4(cw[i][w], rw[w], (i == 0 && w == 0) ? 0u : acc[d]);
                        if (i == B - 1) key = min(key, (acc[d] << 13) + (uint32_t)(d * SIDE));
                    }
                }
            }
            atomicMin(&s_key[b], key + (uint32_t)(1 + dxp));
            continue;
        }
        const int c1 = min(a.nch, (sp + 1) * cps);
        for (int c = sp * cps; c < c1; c++) {
            const uint32_t* rb = base + (c * B) * pw;  // region row of (dy = c*B - p, i = 0)
            const uint32_t r0 = (uint32_t)(1 + c * B * side + dxp);
            if ((c + 1) * B > side && 2 * (side - c * B) <= B) {
                // the last chunk holds side - c*B <= B/2 candidates: score them one by one (a
                // full chunk would spend B*B*W4 VABSDIFF4 on rows past dy = p); a fuller last
                // chunk runs as a full one over padded rows, its extra candidates masked below
                const int nd = side - c * B;
                for (int d = 0; d < nd; d++) {
                    uint32_t acc = 0;
#pragma unroll
                    for (int i = 0; i < B; i++)
#pragma unroll
                        for (int w = 0; w < W4; w++) acc = vsad4(cw[i][w], rb[(d + i) * pw + w], acc);
                    key = min(key, (acc << 13) + (r0 + (uint32_t)(d * side)));
                }
                continue;
            }
            uint32_t acc[B];
#pragma unroll
            for (int d = 0; d < B; d++) acc[d] = 0;
#pragma unroll
            for (int y = 0; y < 2 * B - 1; y++) {
                uint32_t rw[W4];
#pragma unroll
                for (int w = 0; w < W4; w++) rw[w] = rb[y * pw + w];
#pragma unroll
                for (int d = 0; d < B; d++) {
                    const int i = y - d;
                    if (i >= 0 && i < B) {
#pragma unroll
                        for (int w = 0; w < W4; w++) acc[d] = vsad4(cw[i][w], rw[w], acc[d]);
                    }
                }
            }
            // raster ranks 1 + (dy+p)(2p+1) + (dx+p) for every candidate, (0,0) included; the
            // centre-first rule (reading C13) is applied once per block in the output phase
            if ((c + 1) * B <= side) {
#pragma unroll
                for (int d = 0; d < B; d++) key = min(key, (acc[d] << 13) + (r0 + (uint32_t)(d * side)));
            } else {  // a fuller last chunk: rows past dy = p are padding
                const int nd = side - c * B;
#pragma unroll
                for (int d = 0; d < B; d++)
                    if (d < nd) key = min(key, (acc[d] << 13) + (r0 + (uint32_t)(d * side)));
            }
        }
        atomicMin(&s_key[b], key);
    }
    __syncthreads();
    // outputs + SSE at the FS MV (per-pair statistics), one warp per block
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned long long w_sad = 0, w_sse = 0;  // this warp's blocks (lane 0)
    for (int b = warp; b < nbt; b += nw) {
        const int lby = fdiv(b, r_tbx), lbx = b - lby * tbx_e;
        // centre first (reading C13): (0,0) is the MV unless another candidate is strictly
        // cheaper; the raster-first minimum of the others is the key's candidate
        const int col0 = x0 + lbx * B - xs;
        const uint32_t* base0 = sw + (col0 & 3) * cwords + (col0 >> 2);
        uint32_t s0 = 0;
        for (int e = lane; e < B * W4; e += 32) {
            const int i = e / W4, w = e - i * W4;
            const uint32_t cv = reinterpret_cast<const uint32_t*>(scur + (lby * B + i) * TW + lbx * B)[w];
            s0 = vsad4(cv, base0[(lby * B + p + i) * pw + w], s0);
        }
        s0 = __reduce_add_sync(FULL, s0);
        uint32_t k2 = s_key[b];
        if ((k2 >> 13) >= s0) k2 = s0 << 13;  // rank 0 = the centre
        const uint32_t rank = k2 & 0x1fffu;
        const int cidx = rank == 0 ? p * side + p : (int)rank - 1;
        const int cq = fdiv(cidx, r_side);
        const int mdy = cq - p, mdx = cidx - cq * side - p;
        uint32_t sse = 0;
        const int col = (x0 + lbx * B - p - xs) + mdx + p;
        const uint32_t* base = sw + (col & 3) * cwords + (col >> 2);
        for (int e = lane; e < B * W4; e += 32) {
            const int i = e / W4, w = e - i * W4;
            const uint32_t cv = reinterpret_cast<const uint32_t*>(scur + (lby * B + i) * TW + lbx * B)[w];
            sse = ssd4(cv, base[(lby * B + mdy + p + i) * pw + w], sse);
        }
        sse = __reduce_add_sync(FULL, sse);
        if (lane == 0) {
            const int bxg = x0 + lbx * B, byg = y0 + lby * B;
            const long long g = (long long)pair * a.nb + (byg / B) * a.nbx + (bxg / B);
            a.mv[g] = (uint32_t)(mdx & 0xffff) | ((uint32_t)mdy << 16);
            a.sad[g] = k2 >> 13;
            a.pts[g] = (uint16_t)(side * side);
            w_sad += k2 >> 13;
            w_sse += sse;
        }
    }
    if (a.stats) {  // the CTA's sums first: 3 global atomics per CTA, not per block
        if (lane == 0) {
            s_stat[warp][0] = w_sad;
            s_stat[warp][1] = w_sse;
        }
        __syncthreads();
        if (threadIdx.x < 3) {
            unsigned long long t = (unsigned long long)nbt * (unsigned long long)(side * side);
            if (threadIdx.x > 0) {
                t = 0;
                for (int w = 0; w < nw; w++) t += s_stat[w][threadIdx.x - 1];
            }
            atomicAdd(&a.stats[pair * 3 + threadIdx.x], t);
        }
    }
}

// Motion-compensated SSE (P:342 aspect 4; reading C18): SSE = sum over the frame of
// (cur - R(x + mvx, y + mvy))^2 with R the edge-replicated reference (reading C9).
// HBM-bound: every frame byte is read once.  One lane per block row (B lanes per block, 32/B
// blocks per warp): the current row is one aligned vector load (8 / 16 bytes: bx is a
// multiple of B and W of 16), the reference row at the MV is B/4 + 1 aligned words funnel-
// shifted to the row's byte offset, squared differences by VABSDIFF4 + IDP.4A.  Blocks whose
// displaced block leaves the frame take the clamped byte path (border blocks only).  Per-CTA
// sums (32-bit: at most 8 warps x 32 / B blocks x 65025 B^2 = 133 M (B = 8) / 266 M (B = 16)) are added to the
// pair's u64 with one atomic per CTA.
struct McArgs {
    const uint8_t* cur0;
    const uint8_t* ref0;
    long long stride;
    int W, H, B;
    int nbx, nb;
    const uint32_t* mv;  // packed (dx, dy) int16 pairs
    unsigned long long* sse;
};

template <int B>
__global__ void __launch_bounds__(256) mc_sse_kernel(const McArgs a) {
    constexpr int BPW = 32 / B;            // blocks per warp
    constexpr int W4 = B / 4;              // words per row
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int row = lane % B;
    const int bi = (blockIdx.x * 8 + warp) * BPW + lane / B;
    const int pair = blockIdx.y;
    const uint8_t* cur = a.cur0 + (long long)pair * a.stride;
    const uint8_t* ref = a.ref0 + (long long)pair * a.stride;
    uint32_t s = 0;
    if (bi < a.nb) {
        const int bx = (bi % a.nbx) * B, by = (bi / a.nbx) * B;
        const uint32_t m = a.mv[(long long)pair * a.nb + bi];
        const int dx = (int)(int16_t)(m & 0xffff), dy = (int)(int16_t)(m >> 16);
        const int y = by + row, x = bx;
        uint32_t c[W4];
        if (B == 8) {
            const uint2 v = *reinterpret_cast<const uint2*>(cur + (long long)y * a.W + x);
            c[0] = v.x; c[W4 - 1] = v.y;
        } else {
            const uint4 v = *reinterpret_cast<const uint4*>(cur + (long long)y * a.W + x);
            c[0] = v.x; c[1] = v.y; c[2] = v.z; c[W4 - 1] = v.w;
        }
        const int rx = x + dx, ry = y + dy;
        const bool inside = bx + dx >= 0 && bx + dx + B <= a.W && by + dy >= 0 && by + dy + B <= a.H;
        uint32_t r[W4];
        if (inside) {  // interior: aligned words, funnel-shifted (rows never cross the frame)
            const uint8_t* rp = ref + (long long)ry * a.W + rx;
            const uint32_t* w = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(rp) & ~(uintptr_t)3);
            const int sh = (int)(reinterpret_cast<uintptr_t>(rp) & 3) * 8;
            uint32_t wv[W4 + 1];
#pragma unroll
            for (int k = 0; k < W4; k++) wv[k] = __ldg(w + k);
            // the last word only when the row is unaligned (never read past the frame)
            wv[W4] = sh ? __ldg(w + W4) : 0u;
#pragma unroll
            for (int k = 0; k < W4; k++) r[k] = __funnelshift_r(wv[k], wv[k + 1], sh);
        } else {  // border: clamped bytes (reading C9)
            const int yy = min(max(ry, 0), a.H - 1);
#pragma unroll
            for (int k = 0; k < W4; k++) {
                uint32_t v = 0;
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int xx = min(max(rx + 4 * k + q, 0), a.W - 1);
                    v |= (uint32_t)ref[(long long)yy * a.W + xx] << (8 * q);
                }
                r[k] = v;
            }
        }
#pragma unroll
        for (int k = 0; k < W4; k++) {
            const uint32_t d = __vabsdiffu4(c[k], r[k]);
            s = __dp4a(d, d, s);
        }
    }
    s = __reduce_add_sync(FULL, s);
    __shared__ uint32_t ws[8];
    if (lane == 0) ws[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
#pragma unroll
        for (int w = 0; w < 8; w++) t += ws[w];
        if (t) atomicAdd(&a.sse[pair], (unsigned long long)t);
    }
}

// Standalone MC-SSE with TMA staging (me_mc_sse_batch / me_mc_psnr on frames at least one
// tile large): the DCDS kernels' tile geometry (SearchArgs from plan_dcds with a fixed halo
// hp: 16 for 8x8, 32 for 16x16 blocks) -- the tile's reference region and current tile are
// staged by TMA (each frame byte read from HBM once; the halo re-reads hit L2) and edge-fixed
// (reading C9).  One lane per block row (B lanes per block): the current row from the staged
// tile, the reference row at the block's MV from the region (B/4 + 1 words, funnel-shifted),
// squared differences by VABSDIFF4 + IDP.4A.  A block whose displaced block leaves the staged
// region (|mv| > hp) reads the clamped reference from global memory instead (exact, rare).
template <int B>
__global__ void __launch_bounds__(256)
    mc_sse_tma_kernel(const __grid_constant__ CUtensorMap tm_cur, const __grid_constant__ CUtensorMap tm_ref,
                      const SearchArgs a, const uint32_t* __restrict__ mvf) {
    constexpr int W4 = B / 4;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pair = blockIdx.z, tx = blockIdx.x, ty = blockIdx.y;
    const int TW = a.tbx * B, TH = a.tby * B;
    const int x0 = tx * TW, y0 = ty * TH;
    const int xs = (x0 - a.p) & ~15, ys = y0 - a.p;
    const int pitch = a.pitch;
    uint8_t* sref = smem;
    uint8_t* scur = smem + a.cur_off;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + ((a.cur_off + TW * TH + 7) & ~7));
    __shared__ unsigned long long ssum[8];
    if (threadIdx.x == 0) {  // init and issue at once: the barrier publishes the init meanwhile
        mbar_init(bar, 1);
        mbar_expect_tx(bar, (uint32_t)(pitch * a.rh + TW * TH));
        tma_load_3d(sref, &tm_ref, xs, ys, pair, bar);
        tma_load_3d(scur, &tm_cur, x0, y0, pair, bar);
    }
    __syncthreads();
    mbar_wait(bar, 0);
    if (xs < 0 || ys < 0 || xs + pitch > a.W || ys + a.rh > a.H)
        fixup_edges(sref, pitch, a.rh, xs, ys, a.W, a.H);
    __syncthreads();
    const int tbx_e = min(a.tbx, a.nbx - tx * a.tbx), tby_e = min(a.tby, a.nby - ty * a.tby);
    const int nbt = tbx_e * tby_e;
    const uint8_t* gref = a.ref0 + (long long)pair * a.stride;
    uint32_t s = 0;
    // (block, row) items: 256 threads = 256 / B blocks per round
    for (int e = threadIdx.x; e < nbt * B; e += blockDim.x) {
        const int lb = e / B, r = e - lb * B;
        const int lby = lb / tbx_e, lbx = lb - lby * tbx_e;
        const int bxg = x0 + lbx * B, byg = y0 + lby * B;
        const uint32_t m = mvf[(long long)pair * a.nb + (byg / B) * a.nbx + bxg / B];
        const int dx = (int)(int16_t)(m & 0xffff), dy = (int)(int16_t)(m >> 16);
        const uint32_t* crow = reinterpret_cast<const uint32_t*>(scur + (lby * B + r) * TW + lbx * B);
        uint32_t rw[W4];
        if (dx >= -a.p && dx <= a.p && dy >= -a.p && dy <= a.p) {
            const int o = (byg + r + dy - ys) * pitch + (bxg + dx - xs);  // inside the staged region
            const uint32_t* b = reinterpret_cast<const uint32_t*>(sref) + (o >> 2);
            uint32_t wv[W4 + 1];
#pragma unroll
            for (int w = 0; w <= W4; w++) wv[w] = b[w];
#pragma unroll
            for (int w = 0; w < W4; w++) rw[w] = __funnelshift_r(wv[w], wv[w + 1], o << 3);
        } else {  // beyond the staged halo: clamped global reads (reading C9)
            const int yy = min(max(byg + r + dy, 0), a.H - 1);
#pragma unroll
            for (int w = 0; w < W4; w++) {
                uint32_t v = 0;
#pragma unroll
                for (int q = 0; q < 4; q++)
                    v |= (uint32_t)gref[(long long)yy * a.W + min(max(bxg + dx + 4 * w + q, 0), a.W - 1)] << (8 * q);
                rw[w] = v;
            }
        }
#pragma unroll
        for (int w = 0; w < W4; w++) {
            const uint32_t d = __vabsdiffu4(crow[w], rw[w]);
            s = __dp4a(d, d, s);
        }
    }
    // a lane's sum <= a few rows x 65025 x B: 32 bits; warp and CTA sums in 64
    const unsigned long long sw = __reduce_add_sync(FULL, s);  // <= 32 x 2 x 65025 x 16 < 2^32
    if (lane == 0) ssum[warp] = sw;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += ssum[w];
        if (t) atomicAdd(&a.stats[pair], t);
    }
}

// Table-IX-style quality of a motion field against the FS field (P:342 aspects 5 and 6):
// per pair, the number of blocks whose MV equals the FS MV and the sum of the Euclidean
// distances |mv - mv_fs| (double).  One CTA per pair; each thread sums a fixed strided subset
// of the blocks and the CTA reduces in a fixed order, so the result is deterministic.
__global__ void __launch_bounds__(256) quality_kernel(const uint32_t* mv, const uint32_t* mv_fs,
                                                      int nb, double* out) {
    const int pair = blockIdx.x;
    const uint32_t* m = mv + (long long)pair * nb;
    const uint32_t* f = mv_fs + (long long)pair * nb;
    double dsum = 0.0;
    unsigned hits = 0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        const uint32_t a = m[i], b = f[i];
        const int dx = (int)(int16_t)(a & 0xffff) - (int)(int16_t)(b & 0xffff);
        const int dy = (int)(int16_t)(a >> 16) - (int)(int16_t)(b >> 16);
        hits += (a == b);
        dsum += sqrt((double)(dx * dx + dy * dy));
    }
    __shared__ double sd[8];
    __shared__ unsigned sh[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dsum += __shfl_xor_sync(FULL, dsum, o);
        hits += __shfl_xor_sync(FULL, hits, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sd[threadIdx.x >> 5] = dsum;
        sh[threadIdx.x >> 5] = hits;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double d = 0.0;
        unsigned h = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            d += sd[w];
            h += sh[w];
        }
        out[2 * pair] = (double)h;
        out[2 * pair + 1] = d;
    }
}

}  // namespace me
