// bma_kernel.cuh -- the paper's comparison block-matching algorithms on sm_100a (SURVEY 8(f)
// row 3): CDS (ref. [13]), DS (ref. [10]), h-HEXBS (ref. [12], Fig. 2a) and v-HEXBS (Fig. 2b,
// P:43), on the same engine as the DCDS kernel (dcds_kernel.cuh): TMA-staged tile, lane groups
// of G lanes with one block each, per-group bordered visited bitmap (reading C5; window-only
// feasibility, C8) over the edge-replicated reference (C9), strict compare (C6), fused
// motion-compensated SSE and per-pair statistics.
//
// Readings (C23-C26, pinned by Table VII's CDS and DS blocks):
//   DS     large diamond (9 points at the origin, then 8 recentred on the BMP) until the BMP is
//          the centre, then the small diamond once.
//   CDS    the 5x5 cross (9 points), stop if the centre is the BMP; the two unchecked central
//          3x3 points beside the arm of the BMP m (a tie moves the BMP there); stop if m is a
//          distance-1 point that stayed the BMP; then DS from the BMP.
//   HEXBS  the large hexagon (7 points at the origin, 6 recentred) until centred, then the 4
//          distance-1 points.
//   Point order (C26): ascending distance from the pattern centre, ties by (|dy|,|dx|,dy,dx).
//
// A search is a chain of passes over ROWS of a table (<= 4 slots each, offsets relative to
// the pattern centre); patterns longer than 4 points are consecutive rows scanned against the
// same incumbent, which is exactly the oracle's scan().  Row ids below; the transition after
// each row is bma_next().
#pragma once
#include "dcds_kernel.cuh"

namespace me {

enum : int {
    ALG_CDS = 2, ALG_DS = 3, ALG_HEXBS_H = 4, ALG_HEXBS_V = 5  // ids shared with me.h / the oracle
};

enum : int {
    R_L0A = 0, R_L0B, R_L0C,            // large diamond at the origin incl. the centre (DS)
    R_L1A, R_L1B,                       // large diamond recentred (8 points)
    R_SD,                               // small diamond (4 points)
    R_C0A, R_C0B, R_C0C,                // 5x5 cross incl. the centre (CDS step 1)
    R_PX1, R_PX2P, R_PX2N,              // CDS step 2, arm along x: m = (+-1,0) / (2,0) / (-2,0)
    R_PY1, R_PY2P, R_PY2N,              //                 along y: m = (0,+-1) / (0,2) / (0,-2)
    R_HH0A, R_HH0B, R_HH1A, R_HH1B,     // horizontal hexagon: at the origin (7), recentred (6)
    R_HV0A, R_HV0B, R_HV1A, R_HV1B,     // vertical hexagon
    NROW
};

struct RowTable {
    int n[NROW];
    int d[NROW][4][2];
};
constexpr RowTable kRows = {
    {4, 4, 1, 4, 4, 4, 4, 4, 1, 2, 2, 2, 2, 2, 2, 4, 3, 4, 2, 4, 3, 4, 2},
    {
        {{0, 0}, {-1, -1}, {1, -1}, {-1, 1}},  {{1, 1}, {-2, 0}, {2, 0}, {0, -2}},  {{0, 2}},
        {{-1, -1}, {1, -1}, {-1, 1}, {1, 1}},  {{-2, 0}, {2, 0}, {0, -2}, {0, 2}},
        {{-1, 0}, {1, 0}, {0, -1}, {0, 1}},
        {{0, 0}, {-1, 0}, {1, 0}, {0, -1}},    {{0, 1}, {-2, 0}, {2, 0}, {0, -2}},  {{0, 2}},
        {{0, -1}, {0, 1}},  {{-1, -1}, {-1, 1}},  {{1, -1}, {1, 1}},
        {{-1, 0}, {1, 0}},  {{-1, -1}, {1, -1}},  {{-1, 1}, {1, 1}},
        {{0, 0}, {-2, 0}, {2, 0}, {-1, -2}},   {{1, -2}, {-1, 2}, {1, 2}},
        {{-2, 0}, {2, 0}, {-1, -2}, {1, -2}},  {{-1, 2}, {1, 2}},
        {{0, 0}, {0, -2}, {0, 2}, {-2, -1}},   {{2, -1}, {-2, 1}, {2, 1}},
        {{0, -2}, {0, 2}, {-2, -1}, {2, -1}},  {{-2, 1}, {2, 1}},
    }};

// Row code word (kernel argument): bits 6k..6k+5 = (dx+2) | (dy+2) << 3, bits 24..27 = slots.
inline constexpr uint32_t row_code(int r) {
    uint32_t w = (uint32_t)((1 << kRows.n[r]) - 1) << 24;
    for (int k = 0; k < kRows.n[r]; k++)
        w |= (uint32_t)((kRows.d[r][k][0] + 2) | ((kRows.d[r][k][1] + 2) << 3)) << (6 * k);
    return w;
}
__host__ __device__ __forceinline__ int rc_dx(uint32_t w, int k) { return (int)((w >> (6 * k)) & 7u) - 2; }
__host__ __device__ __forceinline__ int rc_dy(uint32_t w, int k) { return (int)((w >> (6 * k + 3)) & 7u) - 2; }

struct BmaArgs {
    const uint8_t* cur0;
    const uint8_t* ref0;
    long long stride;
    int W, H, p;
    int tbx, tby;
    int pitch, rh;
    int cur_off;            // current tile (TMA destination); the group bitmaps overlay it
    int init_off;           // bitmap template, row tables, mbarrier
    int bm_words;
    int nbx, nby, nb;
    uint32_t* mv;
    uint32_t* sad;
    uint16_t* pts;
    unsigned long long* stats;
    uint32_t rcode[NROW];
};

// First row of each algorithm (the pattern at the window origin, incl. the centre).
__host__ __device__ constexpr int bma_first_row(int alg) {
    return alg == ALG_CDS ? R_C0A : alg == ALG_DS ? R_L0A : alg == ALG_HEXBS_H ? R_HH0A : R_HV0A;
}

// Transition after row r (the scan of r is done): next row, new centre, or the end.  c = the
// pattern centre the row was scanned at, b = the incumbent BMP after it.  Returns -1 = done.
__device__ __forceinline__ int bma_next(int alg, int r, int& cx, int& cy, int bx, int by) {
    const bool centred = (bx == cx && by == cy);
    switch (r) {
        case R_L0A: return R_L0B;
        case R_L0B: return R_L0C;
        case R_L0C:
        case R_L1B:  // large diamond done: recentre, or the small diamond (DS [10])
            if (centred) return R_SD;
            cx = bx; cy = by;
            return R_L1A;
        case R_L1A: return R_L1B;
        case R_SD: return -1;
        case R_C0A: return R_C0B;
        case R_C0B: return R_C0C;
        case R_C0C:  // CDS step 1: first-step stop, else step 2 at the arm point m = BMP
            if (bx == 0 && by == 0) return -1;
            cx = bx; cy = by;
            if (by == 0) return bx == 2 ? R_PX2P : bx == -2 ? R_PX2N : R_PX1;
            return by == 2 ? R_PY2P : by == -2 ? R_PY2N : R_PY1;
        case R_PX1: case R_PX2P: case R_PX2N: case R_PY1: case R_PY2P: case R_PY2N:
            // second-step stop when m is a distance-1 point that stayed the BMP
            if (centred && abs(cx) + abs(cy) == 1) return -1;
            cx = bx; cy = by;
            return R_L1A;
        case R_HH0A: return R_HH0B;
        case R_HH1A: return R_HH1B;
        case R_HV0A: return R_HV0B;
        case R_HV1A: return R_HV1B;
        case R_HH0B: case R_HH1B:
            if (centred) return R_SD;
            cx = bx; cy = by;
            return R_HH1A;
        default:  // R_HV0B, R_HV1B
            if (centred) return R_SD;
            cx = bx; cy = by;
            return R_HV1A;
    }
}

// One CTA per tile of TBX x TBY blocks, exactly one block per lane group (the geometry of the
// DCDS kernels' ONE path, dcds_kernel.cuh): every group reads its current rows into registers,
// the CTA overwrites the current tile with the groups' visited bitmaps (interleaved, bordered:
// a point outside the window reads as visited, reading C8), the groups run their searches,
// and one dense phase after the last search of a warp computes the SSEs and outputs.
template <int B, int G, int NWARP, int ALG>
__global__ void __launch_bounds__(NWARP * 32)
    bma_kernel(const __grid_constant__ CUtensorMap tm_cur, const __grid_constant__ CUtensorMap tm_ref,
               const BmaArgs a) {
    constexpr int R = B / G;      // rows per lane (lane j of a group: rows j, j+G, ...)
    constexpr int W4 = B / 4;     // 32-bit words per block row
    constexpr int NG = 32 / G;    // groups per warp
    constexpr int NH = G >= 4 ? 1 : 4 / G;
    constexpr int BST = NWARP * NG + 4;  // interleaved bitmap word stride
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 127) != 0) __trap();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = lane % G, g = lane / G, leader = g * G;
    const int pair = blockIdx.z;
    const int tx = blockIdx.x, ty = blockIdx.y;
    const int TW = a.tbx * B, TH = a.tby * B;
    const int x0 = tx * TW, y0 = ty * TH;
    const int xs = (x0 - a.p) & ~15;
    const int ys = y0 - a.p;
    const int pitch = a.pitch, p = a.p;
    const int bw = bm_row(p), c0 = (p + 2) * bw + p + 2;  // bitmap row length, bit of (0,0)
    uint8_t* sref = smem;
    uint8_t* scur = smem + a.cur_off;
    uint32_t* bms = reinterpret_cast<uint32_t*>(scur);
    uint32_t* bm = bms + (warp * NG + g);
    uint32_t* bm_init = reinterpret_cast<uint32_t*>(smem + a.init_off);
    int4* s_off = reinterpret_cast<int4*>(smem + ((a.init_off + 4 * a.bm_words + 15) & ~15));
    uint32_t* s_code = reinterpret_cast<uint32_t*>(s_off + NROW);
    uint64_t* bar = reinterpret_cast<uint64_t*>(s_code + NROW + (NROW & 1));

    if (threadIdx.x == 0) {  // init and issue at once: the barrier publishes the init meanwhile
        mbar_init(bar, 1);
        mbar_expect_tx(bar, (uint32_t)(pitch * a.rh + TW * TH));
        tma_load_3d(sref, &tm_ref, xs, ys, pair, bar);
        tma_load_3d(scur, &tm_cur, x0, y0, pair, bar);
    }
    __syncthreads();
    for (int r = threadIdx.x; r < NROW; r += NWARP * 32) {
        const uint32_t w = a.rcode[r];
        s_code[r] = w;
        s_off[r] = make_int4(rc_dy(w, 0) * pitch + rc_dx(w, 0), rc_dy(w, 1) * pitch + rc_dx(w, 1),
                             rc_dy(w, 2) * pitch + rc_dx(w, 2), rc_dy(w, 3) * pitch + rc_dx(w, 3));
    }
    // bitmap template: border bits set (rows < 2 or >= 2p+3, columns < 2 of the row length)
    for (int t = threadIdx.x; t < a.bm_words; t += NWARP * 32) {
        const int lo = 32 * t;
        auto span = [lo](int b0, int b1) -> uint32_t {
            b0 = max(b0, lo); b1 = min(b1, lo + 32);
            return b1 > b0 ? (uint32_t)(((1ull << (b1 - b0)) - 1ull) << (b0 - lo)) : 0u;
        };
        uint32_t w = span(0, 2 * bw) | span((2 * p + 3) * bw, lo + 32);
        for (int rs = (lo / bw) * bw; rs < lo + 32; rs += bw) w |= span(rs, rs + 2);
        bm_init[t] = w;
    }
    mbar_wait(bar, 0);
    if (xs < 0 || ys < 0 || xs + pitch > a.W || ys + a.rh > a.H)
        fixup_edges(sref, pitch, a.rh, xs, ys, a.W, a.H);
    __syncthreads();

    const uint32_t* s = reinterpret_cast<const uint32_t*>(sref);
    const int rstride = G * pitch, jrow = j * pitch;
    const int tbx_e = min(a.tbx, a.nbx - tx * a.tbx), tby_e = min(a.tby, a.nby - ty * a.tby);
    const int nbt = tbx_e * tby_e;

    // group state (identical in the G lanes of a group)
    const int idx = warp * NG + g;
    bool act = idx < nbt;
    const bool have = act;
    int row = bma_first_row(ALG), cx = 0, cy = 0, bx = 0, by = 0, pts = 0, bofs = 0;
    uint32_t best = 0xffffffffu;
    long long gblk = 0;
    uint32_t cw[R][W4];
    if (have) {
        const int lby = idx / tbx_e, lbx = idx - lby * tbx_e;
        const int bxg = x0 + lbx * B, byg = y0 + lby * B;
        gblk = (long long)pair * a.nb + (byg / B) * a.nbx + (bxg / B);
        bofs = (byg - ys) * pitch + (bxg - xs);
#pragma unroll
        for (int r = 0; r < R; r++) {
            const uint32_t* crow = reinterpret_cast<const uint32_t*>(scur + (lby * B + j + G * r) * TW + lbx * B);
#pragma unroll
            for (int w = 0; w < W4; w++) cw[r][w] = crow[w];
        }
    } else {
#pragma unroll
        for (int r = 0; r < R; r++)
#pragma unroll
            for (int w = 0; w < W4; w++) cw[r][w] = 0;
    }
    __syncthreads();  // every current row is in registers: the bitmaps may overwrite them
    for (int e = threadIdx.x; e < a.bm_words * (BST / 4); e += NWARP * 32) {
        const uint32_t v = bm_init[e / (BST / 4)];
        reinterpret_cast<uint4*>(bms)[e] = make_uint4(v, v, v, v);
    }
    __syncthreads();

    while (__any_sync(FULL, act)) {
        // ---- one row: visited test-and-set, SADs, first strict minimum (C5, C6, C26)
        const uint32_t pw = s_code[row];
        const int4 po = s_off[row];
        const uint32_t used = act ? ((pw >> 24) & 0xfu) : 0u;
        unsigned m4 = 0;
#pragma unroll
        for (int h = 0; h < NH; h++) {
            const int k = j + h * G;
            bool nw = false;
            if (k < 4 && ((used >> k) & 1)) {
                // the border bits make points outside the window read as visited (C8)
                const int bi = c0 + (cy + rc_dy(pw, k)) * bw + (cx + rc_dx(pw, k));
                const uint32_t bit = 1u << (bi & 31);
                nw = (atomicOr(&bm[(bi >> 5) * BST], bit) & bit) == 0;
            }
            const unsigned bb = __ballot_sync(FULL, nw) >> leader;
            m4 |= (G >= 4 ? (bb & 0xfu) : ((bb & ((1u << G) - 1u)) << (h * G)));
        }
        const int cpos = bofs + cy * pitch + cx + jrow;
        const int ok[4] = {po.x, po.y, po.z, po.w};
        uint32_t sadk[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            uint32_t acc = 0;
            if ((m4 >> k) & 1) {
                uint32_t rw[R][W4];
                ref_rows<R, W4>(s, cpos + ok[k], rstride, rw);
#pragma unroll
                for (int r = 0; r < R; r++)
#pragma unroll
                    for (int w = 0; w < W4; w++) acc = vsad4(cw[r][w], rw[r][w], acc);
            }
            sadk[k] = acc;
        }
        uint32_t v01 = sadk[0] | (sadk[1] << 16), v23 = sadk[2] | (sadk[3] << 16);
#pragma unroll
        for (int o = 1; o < G; o <<= 1) {
            v01 += __shfl_xor_sync(FULL, v01, o);
            v23 += __shfl_xor_sync(FULL, v23, o);
        }
        sadk[0] = v01 & 0xffffu; sadk[1] = v01 >> 16;
        sadk[2] = v23 & 0xffffu; sadk[3] = v23 >> 16;
        uint32_t key = 0xffffffffu;
#pragma unroll
        for (int k = 0; k < 4; k++)
            if ((m4 >> k) & 1) key = min(key, (sadk[k] << 2) | k);
        if (act) {
            pts += __popc(m4);
            // CDS step 2 prefers the central 3x3 square: a tie with m moves the BMP (C23)
            const bool pair_row = row >= R_PX1 && row <= R_PY2N;
            if (key != 0xffffffffu && ((key >> 2) < best || (pair_row && (key >> 2) == best))) {
                best = key >> 2;
                bx = cx + rc_dx(pw, key & 3);
                by = cy + rc_dy(pw, key & 3);
            }
            const int nr = bma_next(ALG, row, cx, cy, bx, by);
            if (nr < 0) act = false;
            else row = nr;
        }
    }

    // ---- every search of the warp ended: SSE at the MV (P:342 aspect 4), outputs, stats
    uint32_t ss = 0;
    if (have) {
        uint32_t rw[R][W4];
        ref_rows<R, W4>(s, bofs + by * pitch + bx + jrow, rstride, rw);
#pragma unroll
        for (int r = 0; r < R; r++)
#pragma unroll
            for (int w = 0; w < W4; w++) ss = ssd4(cw[r][w], rw[r][w], ss);
    }
#pragma unroll
    for (int o2 = 1; o2 < G; o2 <<= 1) ss += __shfl_xor_sync(FULL, ss, o2);
    unsigned long long acc_pts = 0, acc_sad = 0, acc_sse = 0;
    if (have && j == 0) {
        a.mv[gblk] = (uint32_t)(bx & 0xffff) | ((uint32_t)by << 16);
        a.sad[gblk] = best;
        a.pts[gblk] = (uint16_t)pts;
        acc_pts = (unsigned)pts;
        acc_sad = best;
        acc_sse = ss;
    }
    if (a.stats) {  // warp sums, then the CTA's: 3 global atomics per CTA (as dcds_kernel)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            acc_pts += __shfl_xor_sync(FULL, acc_pts, o);
            acc_sad += __shfl_xor_sync(FULL, acc_sad, o);
            acc_sse += __shfl_xor_sync(FULL, acc_sse, o);
        }
        unsigned long long* cs = reinterpret_cast<unsigned long long*>(bar + 1);  // [NWARP][3]
        if (lane == 0) {
            cs[3 * warp + 0] = acc_pts;
            cs[3 * warp + 1] = acc_sad;
            cs[3 * warp + 2] = acc_sse;
        }
        __syncthreads();  // (every warp of the CTA gets here)
        if (threadIdx.x < 3) {
            unsigned long long t = 0;
#pragma unroll
            for (int w = 0; w < NWARP; w++) t += cs[3 * w + threadIdx.x];
            if (t) atomicAdd(&a.stats[pair * 3 + threadIdx.x], t);
        }
    }
}

}  // namespace me
