// dcds_kernel.cuh -- DCDS block motion estimation on sm_100a (B200).
//
// Paper: Jia & Zhang, DCDS (arxiv 0806.0689).  P:n = PAPER.md line n.
//   Step 1: HCSP {(0,0),(+-1,0),(+-2,0),(0,+-1)} at the window
//                   origin; halfway stop when the centre stays the BMP.
//   Step 2: switching strategy one: BMP with dy == 0 -> HDSP else VDSP.
//   Step 3: switching strategy two: BMP on a near point (L1 = 1) -> the
//                   other DDSP, on a distant point (L1 = 2) -> keep; repeat until the BMP is
//                   the centre.
//   Step 4: the two middle points of the final pattern.
// Readings: strict improvement, incumbent wins ties, fixed pattern order (C6,
// C7); each position scored once per block (C5); window-only feasibility with an
// edge-replicated reference (C8, C9); integer SAD (C12).
//
// Design: one CTA per tile of TBX x TBY blocks of one pair; the tile's
// reference region (tile + the whole +-p window, edge-replicated) and current tile are staged
// once into shared memory; each warp then runs DCDS for one block at a time (blocks handed
// out by a shared counter).  Inside a warp, lanes split the block's rows (and, for 8x8
// blocks, four candidate slots); SADs use VABSDIFF4 (inline PTX vabsdiff4.add), warp sums
// use REDUX.SUM, argmins are packed integer keys, and the visited set is a per-warp bitmap in
// shared memory.  The data-dependent step count runs inside the warp with no block/grid sync.
#pragma once
#include <stdint.h>

namespace me {

constexpr unsigned FULL = 0xffffffffu;

struct SearchArgs {
    const uint8_t* cur0;
    const uint8_t* ref0;
    long long stride;       // bytes between consecutive pairs
    int W, H, p;
    int tbx, tby, ntx;      // tile size in blocks; tiles per row
    int pitch, rh;          // staged reference region: row pitch (bytes, 16*odd) and rows
    int bm_words;           // visited-bitmap words per warp (multiple of 4)
    int nbx, nb;            // blocks per row, blocks per pair
    uint32_t* mv;           // [npairs][nb] packed (dx & 0xffff) | (dy << 16)
    uint32_t* sad;          // [npairs][nb]
    uint16_t* pts;          // [npairs][nb]
    unsigned long long* stats;  // [npairs][3] or null
};

__device__ __forceinline__ uint32_t vsad4(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ uint32_t ssd4(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d = __vabsdiffu4(a, b);
    return __dp4a(d, d, c);
}

// 4 bytes starting at byte offset o of a 4-byte aligned shared buffer.
__device__ __forceinline__ uint32_t lds_u8x4(const uint32_t* s, int o) {
    const uint32_t lo = s[o >> 2], hi = s[(o >> 2) + 1];
    return __funnelshift_r(lo, hi, (o & 3) << 3);
}

// Stage the reference region [ys, ys+rh) x [xs, xs+pitch) with edge replication, and the
// current tile [y0, y0+TH) x [x0, x0+TW) (in-frame part), 16 bytes per thread-iteration.
__device__ __forceinline__ void stage_tile(const SearchArgs& a, const uint8_t* cur,
                                           const uint8_t* ref, int xs, int ys, int x0, int y0,
                                           int TW, int TH, uint8_t* sref, uint8_t* scur) {
    const int cpr = a.pitch >> 4;
    for (int c = threadIdx.x; c < cpr * a.rh; c += blockDim.x) {
        const int i = c / cpr, j = c - i * cpr;
        const int y = min(max(ys + i, 0), a.H - 1);
        const int x = xs + 16 * j;
        const uint8_t* row = ref + (long long)y * a.W;
        uint4 v;
        if (x >= 0 && x < a.W) {
            v = __ldg(reinterpret_cast<const uint4*>(row + x));
        } else {
            uint32_t b = (x < 0) ? row[0] : row[a.W - 1];
            b *= 0x01010101u;
            v = make_uint4(b, b, b, b);
        }
        *reinterpret_cast<uint4*>(sref + i * a.pitch + 16 * j) = v;
    }
    const int ccr = TW >> 4;
    for (int c = threadIdx.x; c < ccr * TH; c += blockDim.x) {
        const int i = c / ccr, j = c - i * ccr;
        const int y = y0 + i, x = x0 + 16 * j;
        if (y < a.H && x < a.W)
            *reinterpret_cast<uint4*>(scur + i * TW + 16 * j) =
                __ldg(reinterpret_cast<const uint4*>(cur + (long long)y * a.W + x));
    }
}

// Offsets of the DDSP points in the fixed order (reading C7), candidate k = 0..3.
//   HDSP: (-2,0) (2,0) (0,-1) (0,1)      VDSP: (-1,0) (1,0) (0,-2) (0,2)
__device__ __forceinline__ int ddsp_dx(int kind, int k) {
    return kind == 0 ? (k < 2 ? 4 * k - 2 : 0) : (k < 2 ? 2 * k - 1 : 0);
}
__device__ __forceinline__ int ddsp_dy(int kind, int k) {
    return kind == 0 ? (k < 2 ? 0 : 2 * k - 5) : (k < 2 ? 0 : 4 * k - 10);
}
// near point of the pattern (L1 distance 1): HDSP k >= 2, VDSP k < 2.
__device__ __forceinline__ bool ddsp_near(int kind, int k) { return kind == 0 ? k >= 2 : k < 2; }
// HCSP order: (0,0) (-1,0) (1,0) (-2,0) (2,0) (0,-1) (0,1), k = 0..6
__device__ __forceinline__ int hcsp_dx(int k) {
    return k == 0 ? 0 : (k <= 4 ? ((k & 1) ? -((k + 1) >> 1) : (k >> 1)) : 0);
}
__device__ __forceinline__ int hcsp_dy(int k) { return k < 5 ? 0 : (k == 5 ? -1 : 1); }

// Warp-level bitmap test-and-set of the candidate handled by this lane.  Returns true when the
// candidate is feasible (|q| <= p) and was not visited before.
__device__ __forceinline__ bool visit(uint32_t* bm, int qx, int qy, int p, bool active) {
    if (!active || qx < -p || qx > p || qy < -p || qy > p) return false;
    const int side = 2 * p + 1;
    const int idx = (qy + p) * side + (qx + p);
    const uint32_t bit = 1u << (idx & 31);
    const uint32_t old = atomicOr(&bm[idx >> 5], bit);
    return (old & bit) == 0;
}

// ----------------------------------------------------------------------------------------
// Per-block SAD engines.
//   B = 16: lane = (r = lane>>2, w = lane&3) covers rows r and r+8, bytes 4w..4w+3: one
//           candidate per warp pass, sum by REDUX.SUM.  Conflict-free LDS when the region
//           pitch is 16*odd bytes.
//   B = 8:  lane = (slot = lane>>3, r = lane&7) covers row r, 8 bytes, of candidate `slot`:
//           four candidates per warp pass; slot sums (<= 16320) are packed two per 32-bit
//           word so two REDUX.SUM give all four.
// ----------------------------------------------------------------------------------------
template <int B>
struct Engine;

template <>
struct Engine<16> {
    uint32_t c0, c1;  // current-block words held in registers
    int lb0, lb1;     // lane byte offsets inside the candidate window

    __device__ __forceinline__ void load(const uint8_t* scur, int TW, int lbx, int lby,
                                         int pitch, int lane) {
        const int r = lane >> 2, w = lane & 3;
        const uint8_t* base = scur + (lby * 16 + r) * TW + lbx * 16 + 4 * w;
        c0 = *reinterpret_cast<const uint32_t*>(base);
        c1 = *reinterpret_cast<const uint32_t*>(base + 8 * TW);
        lb0 = r * pitch + 4 * w;
        lb1 = lb0 + 8 * pitch;
    }
    // SAD of one candidate at byte offset o (block origin + dy*pitch + dx) -- warp-uniform.
    __device__ __forceinline__ uint32_t sad(const uint32_t* s, int o) const {
        const uint32_t r0 = lds_u8x4(s, o + lb0);
        const uint32_t r1 = lds_u8x4(s, o + lb1);
        return __reduce_add_sync(FULL, vsad4(c1, r1, vsad4(c0, r0, 0u)));
    }
    __device__ __forceinline__ uint32_t sse(const uint32_t* s, int o) const {
        const uint32_t r0 = lds_u8x4(s, o + lb0);
        const uint32_t r1 = lds_u8x4(s, o + lb1);
        return __reduce_add_sync(FULL, ssd4(c1, r1, ssd4(c0, r0, 0u)));
    }
};

template <>
struct Engine<8> {
    uint32_t c0, c1;
    int lb;
    int slot;

    __device__ __forceinline__ void load(const uint8_t* scur, int TW, int lbx, int lby,
                                         int pitch, int lane) {
        const int r = lane & 7;
        slot = lane >> 3;
        const uint8_t* base = scur + (lby * 8 + r) * TW + lbx * 8;
        c0 = *reinterpret_cast<const uint32_t*>(base);
        c1 = *reinterpret_cast<const uint32_t*>(base + 4);
        lb = r * pitch;
    }
    // Four candidates: this lane evaluates the one of its slot at byte offset o.
    // Returns packed sums: lo = {slot0 | slot1 << 16}, hi = {slot2 | slot3 << 16}.
    __device__ __forceinline__ void sad4(const uint32_t* s, int o, uint32_t& s01,
                                         uint32_t& s23) const {
        const int a = o + lb;
        const uint32_t w0 = s[a >> 2], w1 = s[(a >> 2) + 1], w2 = s[(a >> 2) + 2];
        const int sh = (a & 3) << 3;
        const uint32_t r0 = __funnelshift_r(w0, w1, sh), r1 = __funnelshift_r(w1, w2, sh);
        uint32_t v = vsad4(c1, r1, vsad4(c0, r0, 0u));
        v <<= (slot & 1) << 4;
        s01 = __reduce_add_sync(FULL, slot < 2 ? v : 0u);
        s23 = __reduce_add_sync(FULL, slot < 2 ? 0u : v);
    }
    // SSE at byte offset o using slot-0 lanes only.
    __device__ __forceinline__ uint32_t sse(const uint32_t* s, int o) const {
        const int a = o + lb;
        const uint32_t w0 = s[a >> 2], w1 = s[(a >> 2) + 1], w2 = s[(a >> 2) + 2];
        const int sh = (a & 3) << 3;
        const uint32_t r0 = __funnelshift_r(w0, w1, sh), r1 = __funnelshift_r(w1, w2, sh);
        const uint32_t v = ssd4(c1, r1, ssd4(c0, r0, 0u));
        return __reduce_add_sync(FULL, slot == 0 ? v : 0u);
    }
};

__device__ __forceinline__ uint32_t unpack4(uint32_t s01, uint32_t s23, int k) {
    const uint32_t w = (k < 2) ? s01 : s23;
    return (k & 1) ? (w >> 16) : (w & 0xffffu);
}

// SAD of a single candidate at byte offset o (warp-uniform) for either engine.
template <int B>
__device__ __forceinline__ uint32_t sad1(const Engine<B>& E, const uint32_t* s, int o) {
    if constexpr (B == 8) {
        uint32_t a01, a23;
        E.sad4(s, o, a01, a23);
        return a01 & 0xffffu;
    } else {
        return E.sad(s, o);
    }
}

// ----------------------------------------------------------------------------------------
// The search of one block by one warp.  Returns (mx, my, sad, points); all warp-uniform.
// VARIANT 0 = DCDS, 1 = DCDS^S.
// ----------------------------------------------------------------------------------------
template <int B, int VARIANT>
__device__ __forceinline__ void dcds_block(const Engine<B>& E, const uint32_t* s, int base,
                                           int pitch, int p, uint32_t* bm, int bm_words,
                                           int lane, int& mx, int& my, uint32_t& best,
                                           int& points) {
    // fresh visited set (reading C5)
    for (int i = lane * 4; i < bm_words; i += 128)
        *reinterpret_cast<uint4*>(bm + i) = make_uint4(0, 0, 0, 0);
    __syncwarp();

    // ---- Step 1: HCSP at the origin, 7 points, k = 0 is the centre.
    const int k1 = lane & 7;
    const bool f1 = visit(bm, hcsp_dx(k1), hcsp_dy(k1), p, lane < 7);
    const uint32_t m1 = __ballot_sync(FULL, f1) & 0x7f;
    points = __popc(m1);
    uint32_t s0;
    uint32_t key = 0xffffffffu;  // (sad << 3) | k of the best new point
    if constexpr (B == 8) {
        // pass A: slots = HCSP k 0..3; pass B: k 4..6 (slot 3 idle -> centre)
        const int slot = lane >> 3;
        {
            const int o = base + hcsp_dy(slot) * pitch + hcsp_dx(slot);
            uint32_t a01, a23;
            E.sad4(s, ((m1 >> slot) & 1) ? o : base, a01, a23);
            s0 = unpack4(a01, a23, 0);
#pragma unroll
            for (int k = 1; k < 4; k++)
                if ((m1 >> k) & 1) key = min(key, (unpack4(a01, a23, k) << 3) | k);
        }
        {
            const int k = 4 + slot;
            const bool ok = slot < 3 && ((m1 >> k) & 1);
            const int o = base + hcsp_dy(k) * pitch + hcsp_dx(k);
            uint32_t a01, a23;
            E.sad4(s, ok ? o : base, a01, a23);
#pragma unroll
            for (int j = 0; j < 3; j++)
                if ((m1 >> (4 + j)) & 1) key = min(key, (unpack4(a01, a23, j) << 3) | (4 + j));
        }
    } else {
        s0 = E.sad(s, base);
#pragma unroll
        for (int k = 1; k < 7; k++)
            if ((m1 >> k) & 1) key = min(key, (E.sad(s, base + hcsp_dy(k) * pitch + hcsp_dx(k)) << 3) | k);
    }
    best = s0;
    int cx = 0, cy = 0;
    if ((key >> 3) >= s0) {  // halfway stop
        mx = 0; my = 0;
        return;
    }
    best = key >> 3;
    cx = hcsp_dx(key & 7);
    cy = hcsp_dy(key & 7);
    int kind = (cy == 0) ? 0 : 1;  // switching strategy one: 0 = HDSP, 1 = VDSP

    // ---- Steps 2 and 3
    uint32_t last_s01 = 0, last_s23 = 0;   // DCDS^S: SADs of the final pattern
    uint32_t last_m = 0;
    for (;;) {
        const int kk = lane & 3;
        const bool fk = visit(bm, cx + ddsp_dx(kind, kk), cy + ddsp_dy(kind, kk), p, lane < 4);
        const uint32_t m = __ballot_sync(FULL, fk) & 0xf;
        points += __popc(m);
        key = 0xffffffffu;
        const int cbase = base + cy * pitch + cx;
        if constexpr (B == 8) {
            const int slot = lane >> 3;
            const int o = cbase + ddsp_dy(kind, slot) * pitch + ddsp_dx(kind, slot);
            uint32_t a01, a23;
            E.sad4(s, ((m >> slot) & 1) ? o : cbase, a01, a23);
#pragma unroll
            for (int k = 0; k < 4; k++)
                if ((m >> k) & 1) key = min(key, (unpack4(a01, a23, k) << 2) | k);
            last_s01 = a01; last_s23 = a23;
        } else {
            uint32_t mm = m;
            last_s01 = 0; last_s23 = 0;
            while (mm) {
                const int k = __ffs(mm) - 1;
                mm &= mm - 1;
                const uint32_t v = E.sad(s, cbase + ddsp_dy(kind, k) * pitch + ddsp_dx(kind, k));
                key = min(key, (v << 2) | k);
                if (k < 2) last_s01 |= v << ((k & 1) << 4);
                else last_s23 |= v << ((k & 1) << 4);
            }
        }
        last_m = m;
        if ((key >> 2) >= best) break;  // BMP at the centre -> Step 4
        const int k = key & 3;
        best = key >> 2;
        cx += ddsp_dx(kind, k);
        cy += ddsp_dy(kind, k);
        if (ddsp_near(kind, k)) kind ^= 1;  // switching strategy two
    }

    // ---- Step 4: middle points of the final pattern, (-1,0),(1,0) or (0,-1),(0,1).
    const int mdx0 = kind == 0 ? -1 : 0, mdy0 = kind == 0 ? 0 : -1;
    bool want0 = true, want1 = true;
    if constexpr (VARIANT == 1) {
        // DCDS^S: only the side of the cheaper distant point (reading C22).
        // Distant points of the final pattern: HDSP k = 0,1; VDSP k = 2,3.
        const int kd = kind == 0 ? 0 : 2;
        uint32_t dn = 0xffffffffu, dp = 0xffffffffu;
        const int ax = kind == 0 ? 2 : 0, ay = kind == 0 ? 0 : 2;
        const int cbase = base + cy * pitch + cx;
        const bool fn = (cx - ax >= -p) && (cy - ay >= -p);
        const bool fp = (cx + ax <= p) && (cy + ay <= p);
        // a distant point scored in the final pass has its SAD at hand; one visited earlier
        // is re-evaluated (same value as when it was scored; not counted again).
        if (fn) {
            dn = ((last_m >> kd) & 1) ? unpack4(last_s01, last_s23, kd) : 0xffffffffu;
            if (dn == 0xffffffffu) dn = sad1<B>(E, s, cbase - ay * pitch - ax);
        }
        if (fp) {
            dp = ((last_m >> (kd + 1)) & 1) ? unpack4(last_s01, last_s23, kd + 1) : 0xffffffffu;
            if (dp == 0xffffffffu) dp = sad1<B>(E, s, cbase + ay * pitch + ax);
        }
        // infeasible distant point = +inf; choose the positive side only if strictly cheaper
        const bool pos = (fp ? dp : 0xffffffffu) < (fn ? dn : 0xffffffffu) ||
                         (fp && !fn);
        want0 = !pos;
        want1 = pos;
    }
    const int kk = lane & 1;
    const bool fm = visit(bm, cx + (kk ? -mdx0 : mdx0), cy + (kk ? -mdy0 : mdy0), p,
                          lane < 2 && (kk ? want1 : want0));
    const uint32_t m4 = __ballot_sync(FULL, fm) & 0x3;
    points += __popc(m4);
    if (m4) {
        const int cbase = base + cy * pitch + cx;
        key = 0xffffffffu;
        if constexpr (B == 8) {
            const int slot = lane >> 3;
            const int sg = (slot & 1) ? 1 : -1;
            const int o = cbase + sg * (mdy0 * -1) * pitch + sg * (mdx0 * -1);
            uint32_t a01, a23;
            E.sad4(s, (slot < 2 && ((m4 >> slot) & 1)) ? o : cbase, a01, a23);
#pragma unroll
            for (int k = 0; k < 2; k++)
                if ((m4 >> k) & 1) key = min(key, (unpack4(a01, a23, k) << 1) | k);
        } else {
            uint32_t mm = m4;
            while (mm) {
                const int k = __ffs(mm) - 1;
                mm &= mm - 1;
                const int sg = k ? 1 : -1;
                key = min(key, (E.sad(s, cbase + sg * (-mdy0) * pitch + sg * (-mdx0)) << 1) | k);
            }
        }
        if ((key >> 1) < best) {
            const int k = key & 1;
            const int sg = k ? 1 : -1;
            best = key >> 1;
            cx += sg * (-mdx0);
            cy += sg * (-mdy0);
        }
    }
    mx = cx;
    my = cy;
}

template <int B, int NWARP, int VARIANT>
__global__ void __launch_bounds__(NWARP * 32) dcds_kernel(const SearchArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pair = blockIdx.y;
    const int tx = blockIdx.x % a.ntx, ty = blockIdx.x / a.ntx;
    const int TW = a.tbx * B, TH = a.tby * B;
    const int x0 = tx * TW, y0 = ty * TH;
    const int xs = (x0 - a.p) & ~15;  // floor to 16 (two's complement)
    const int ys = y0 - a.p;
    const uint8_t* cur = a.cur0 + (long long)pair * a.stride;
    const uint8_t* ref = a.ref0 + (long long)pair * a.stride;

    uint8_t* sref = smem;
    uint8_t* scur = smem + a.pitch * a.rh + 16;
    uint32_t* bms = reinterpret_cast<uint32_t*>(scur + TW * TH);
    uint32_t* bm = bms + warp * a.bm_words;
    unsigned long long* cst = reinterpret_cast<unsigned long long*>(bms + NWARP * a.bm_words);
    int* ctr = reinterpret_cast<int*>(cst + 3);

    if (threadIdx.x < 3) cst[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) *ctr = 0;
    stage_tile(a, cur, ref, xs, ys, x0, y0, TW, TH, sref, scur);
    __syncthreads();

    const uint32_t* s = reinterpret_cast<const uint32_t*>(sref);
    const int nbt = a.tbx * a.tby;
    unsigned long long acc_pts = 0, acc_sad = 0, acc_sse = 0;
    for (;;) {
        int i = 0;
        if (lane == 0) i = atomicAdd(ctr, 1);
        i = __shfl_sync(FULL, i, 0);
        if (i >= nbt) break;
        const int lbx = i % a.tbx, lby = i / a.tbx;
        const int bxg = x0 + lbx * B, byg = y0 + lby * B;
        if (bxg >= a.W || byg >= a.H) continue;
        Engine<B> E;
        E.load(scur, TW, lbx, lby, a.pitch, lane);
        const int base = (byg - ys) * a.pitch + (bxg - xs);
        int mx, my, points;
        uint32_t best;
        dcds_block<B, VARIANT>(E, s, base, a.pitch, a.p, bm, a.bm_words, lane, mx, my, best,
                               points);
        const uint32_t sse = E.sse(s, base + my * a.pitch + mx);
        if (lane == 0) {
            const long long g = (long long)pair * a.nb + (byg / B) * a.nbx + (bxg / B);
            a.mv[g] = (uint32_t)(mx & 0xffff) | ((uint32_t)my << 16);
            a.sad[g] = best;
            a.pts[g] = (uint16_t)points;
            acc_pts += (unsigned)points;
            acc_sad += best;
            acc_sse += sse;
        }
    }
    if (a.stats) {
        if (lane == 0) {
            atomicAdd(&cst[0], acc_pts);
            atomicAdd(&cst[1], acc_sad);
            atomicAdd(&cst[2], acc_sse);
        }
        __syncthreads();
        if (threadIdx.x < 3) atomicAdd(&a.stats[pair * 3 + threadIdx.x], cst[threadIdx.x]);
    }
}

}  // namespace me
