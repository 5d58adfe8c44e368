// ideal_kernel.cuh -- the analytical side of the paper on sm_100a:
//   * the ideal-condition simulator of P:299-301 -- "the block-matching distortion of other
//     reference block P is defined as its Euclid distance to the best-matched block" -- run
//     for every true-MV placement t of the window at once (one thread per placement), for
//     DCDS, DCDS^S and the comparison BMAs (Table VII; ANSP of Table VIII);
//   * the MV histogram of a motion field (the MVP distribution of P:71-98, Tables II-III,
//     Fig. 3) -- the data-parallel reduction behind the MVP statistics.
//
// The simulator uses the cost |q - t|^2 (an integer): it orders every pair of candidates
// exactly as the Euclidean distance |q - t| does, ties included, so the strict-compare search
// takes the same path.  Each thread keeps its visited set (reading C5) in a local bitmap.
#pragma once
#include "bma_kernel.cuh"

namespace me {

// DCDS rows of the scalar engine (readings C1-C7, C10; slot order C7) -- ids after NROW.
enum : int {
    R_D1A = NROW, R_D1B,       // HCSP (0,0) (-1,0) (1,0) (-2,0) | (2,0) (0,-1) (0,1)
    R_DH, R_DV,                // HDSP / VDSP
    R_MH, R_MV,                // middle points of HDSP / VDSP
    R_MHN, R_MHP, R_MVN, R_MVP,  // a single middle point (DCDS^S, reading C22)
    NROW_ALL
};
struct DcdsRows {
    int n[NROW_ALL - NROW];
    int d[NROW_ALL - NROW][4][2];
};
constexpr DcdsRows kDRows = {
    {4, 3, 4, 4, 2, 2, 1, 1, 1, 1},
    {{{0, 0}, {-1, 0}, {1, 0}, {-2, 0}}, {{2, 0}, {0, -1}, {0, 1}},
     {{-2, 0}, {2, 0}, {0, -1}, {0, 1}}, {{-1, 0}, {1, 0}, {0, -2}, {0, 2}},
     {{-1, 0}, {1, 0}}, {{0, -1}, {0, 1}},
     {{-1, 0}}, {{1, 0}}, {{0, -1}}, {{0, 1}}}};

inline constexpr uint32_t any_row_code(int r) {
    if (r < NROW) return row_code(r);
    const int i = r - NROW;
    uint32_t w = (uint32_t)((1 << kDRows.n[i]) - 1) << 24;
    for (int k = 0; k < kDRows.n[i]; k++)
        w |= (uint32_t)((kDRows.d[i][k][0] + 2) | ((kDRows.d[i][k][1] + 2) << 3)) << (6 * k);
    return w;
}

struct IdealArgs {
    int alg, p;
    int* nsp;       // [(2p+1)^2], row-major over (ty, tx)
    int* mvx;
    int* mvy;
    uint32_t rcode[NROW_ALL];
};

__device__ __forceinline__ int isq(int x) { return x * x; }

// One search of algorithm alg on the ideal surface with true MV (tx, ty).
__device__ void ideal_search(const IdealArgs& a, const uint32_t* code, int tx, int ty,
                             uint32_t* seen, int& mvx, int& mvy, int& pts) {
    const int p = a.p, side = 2 * p + 1, alg = a.alg;
    for (int w = 0; w < (side * side + 31) / 32; w++) seen[w] = 0;
    int row = alg == 0 || alg == 1 ? R_D1A : bma_first_row(alg);
    int cx = 0, cy = 0, bx = 0, by = 0;
    int best = 0x7fffffff;
    pts = 0;
    for (;;) {
        const uint32_t w = code[row];
        const int n = __popc((w >> 24) & 0xfu);
        int kb = -1, kc = 0x7fffffff;
        for (int k = 0; k < n; k++) {  // scan: first strict minimum among new points (C6, C7)
            const int qx = cx + rc_dx(w, k), qy = cy + rc_dy(w, k);
            if (qx < -p || qx > p || qy < -p || qy > p) continue;  // window only (C8)
            const int idx = (qy + p) * side + (qx + p);
            if (seen[idx >> 5] & (1u << (idx & 31))) continue;     // scored before (C5)
            seen[idx >> 5] |= 1u << (idx & 31);
            pts++;
            const int c = isq(qx - tx) + isq(qy - ty);
            if (c < kc) { kc = c; kb = k; }
        }
        const bool pair_row = row >= R_PX1 && row <= R_PY2N;
        if (kb >= 0 && (kc < best || (pair_row && kc == best))) {
            best = kc;
            bx = cx + rc_dx(w, kb);
            by = cy + rc_dy(w, kb);
        }
        int nr;
        if (row < NROW) {
            nr = bma_next(alg, row, cx, cy, bx, by);
        } else if (row == R_D1A) {
            nr = R_D1B;
        } else if (row == R_D1B) {  // halfway stop, switching strategy one
            if (bx == 0 && by == 0) { nr = -1; }
            else { cx = bx; cy = by; nr = by == 0 ? R_DH : R_DV; }
        } else if (row == R_DH || row == R_DV) {
            if (bx == cx && by == cy) {  // Step 4
                const bool h = row == R_DH;
                if (alg == 0) {
                    nr = h ? R_MH : R_MV;
                } else {
                    // DCDS^S: the middle point beside the cheaper distant point; an
                    // infeasible distant point costs +inf, a tie picks the negative side (C22)
                    const int ax = h ? 2 : 0, ay = h ? 0 : 2;
                    const bool fn = abs(cx - ax) <= p && abs(cy - ay) <= p;
                    const bool fp = abs(cx + ax) <= p && abs(cy + ay) <= p;
                    const long long dn = fn ? isq(cx - ax - tx) + isq(cy - ay - ty) : (1ll << 40);
                    const long long dp = fp ? isq(cx + ax - tx) + isq(cy + ay - ty) : (1ll << 40);
                    nr = dp < dn ? (h ? R_MHP : R_MVP) : (h ? R_MHN : R_MVN);
                }
            } else {  // switching strategy two
                const bool nearp = abs(bx - cx) + abs(by - cy) == 1;
                nr = nearp ? (row == R_DH ? R_DV : R_DH) : row;
                cx = bx; cy = by;
            }
        } else {
            nr = -1;  // Step 4 done
        }
        if (nr < 0) break;
        row = nr;
    }
    mvx = bx;
    mvy = by;
}

__global__ void __launch_bounds__(128) ideal_kernel(const IdealArgs a) {
    __shared__ uint32_t code[NROW_ALL];
    for (int r = threadIdx.x; r < NROW_ALL; r += blockDim.x) code[r] = a.rcode[r];
    __syncthreads();
    const int side = 2 * a.p + 1;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= side * side) return;
    uint32_t seen[(65 * 65 + 31) / 32];  // p <= 32
    int mx, my, pts;
    ideal_search(a, code, i % side - a.p, i / side - a.p, seen, mx, my, pts);
    a.nsp[i] = pts;
    if (a.mvx) a.mvx[i] = mx;
    if (a.mvy) a.mvy[i] = my;
}

// Histogram of a motion field over the +-p window ("MVPs accumulated at the
// corresponding positions"): hist[(dy+p)*(2p+1) + dx+p] += 1 per block.  Shared-memory
// sub-histograms per CTA, one global atomic per non-empty bin and CTA.
__global__ void __launch_bounds__(256) mv_hist_kernel(const uint32_t* mv, long long n, int p,
                                                      unsigned long long* hist) {
    extern __shared__ unsigned int sh[];
    const int side = 2 * p + 1, nbin = side * side;
    for (int b = threadIdx.x; b < nbin; b += blockDim.x) sh[b] = 0;
    __syncthreads();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const uint32_t m = mv[i];
        const int dx = (int)(int16_t)(m & 0xffff), dy = (int)(int16_t)(m >> 16);
        if (dx >= -p && dx <= p && dy >= -p && dy <= p) atomicAdd(&sh[(dy + p) * side + dx + p], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nbin; b += blockDim.x)
        if (sh[b]) atomicAdd(&hist[b], (unsigned long long)sh[b]);
}

}  // namespace me
