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
// once into shared memory by TMA.  Each warp is split into 32/G lane groups (G lanes split a
// block's rows).  In the default geometry (ONE) every group owns exactly one block of the
// tile: it reads its current rows into registers, Step 1 runs as one straight-line step, and
// Steps 2-4 are a per-group state machine (S3 = the 4 DDSP points, S4 = the middle points,
// PRE = the DCDS^S look-up) advanced one pass per warp iteration, so groups at different
// steps share one instruction stream and the data-dependent step count never needs a block
// or grid sync; one dense phase after the warp's last search writes SSEs and outputs.  Other
// tile shapes hand blocks out from a shared counter.  SADs use VABSDIFF4 (inline PTX
// vabsdiff4.add) on funnel-shifted unaligned rows; the 4 slot sums are packed two per word
// (each <= 255*B*B < 2^16) and reduced across the group with xor shuffles; argmins are
// packed (SAD, order) keys; the visited set is a bordered per-group bitmap in shared memory.
#pragma once
#include <cuda.h>  // CUtensorMap
#include <stdint.h>

namespace me {

constexpr unsigned FULL = 0xffffffffu;

// ME_DEBUG builds (libme_debug.so, paper_0806_0689_b200/build.py): bounds checks of every
// staged-region load and visited-bitmap access, trapping with a message (compute-sanitizer is
// not available on the GPU pool).  Release builds compile them out.
#ifdef ME_DEBUG
#define ME_CHECK(cond)                                                                      \
    do {                                                                                    \
        if (!(cond)) {                                                                      \
            printf("ME_DEBUG check failed %s:%d: %s (block %d,%d,%d thread %d)\n", __FILE__, \
                   __LINE__, #cond, blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x);      \
            __trap();                                                                       \
        }                                                                                   \
    } while (0)
#else
#define ME_CHECK(cond) \
    do {               \
    } while (0)
#endif

struct SearchArgs {
    const uint8_t* cur0;
    const uint8_t* ref0;
    long long stride;       // bytes between consecutive pairs
    int W, H, p;
    int tbx, tby, ntx;      // tile size in blocks; tiles per row
    int pitch, rh;          // staged reference region: row pitch (bytes, 16*odd) and rows
    int cur_off;            // byte offset of the current tile in shared memory (128-aligned)
    int bm_off, init_off;   // byte offsets of the group bitmaps and of the bitmap template
    int bm_words;           // visited-bitmap words per group (bm_nwords(p))
    int nbx, nby, nb;       // blocks per row, block rows, blocks per pair
    uint32_t* mv;           // [npairs][nb] packed (dx & 0xffff) | (dy << 16)
    uint32_t* sad;          // [npairs][nb]
    uint16_t* pts;          // [npairs][nb]
    int packed;             // mv as int8 pairs [npairs][nb][2], sad as uint16 (me_dcds_batch_packed)
    unsigned long long* stats;  // [npairs][3] or null
    uint64_t* trace;            // TRACE builds: [npairs][nb][tcap] pass records
    uint16_t* tlen;             // TRACE builds: [npairs][nb] passes of each block
    int tcap;
    // visited-bitmap geometry (half-widths; = p unless compact) and the compact visited set of
    // the B=16 ONE kernels (DESIGN.md §7 "Compact visited set"): a search whose centre leaves
    // the compact window is abandoned and its block index (pair * nb + block) appended to ovf:
    // [0] / [1] counts of interior / border blocks, [2] / [3] claim counters of the overflow
    // passes, interior blocks at [4 + i], border blocks at [4 + ovf_cap - 1 - i]
    int bmx, bmy;
    int compact;
    uint32_t* ovf;
    uint32_t ovf_cap;  // npairs * nb
    // warm-start records of the first rec_cap interior entries: the abandoned search's state
    // (centre, kind, SAD, points) and its compact bitmap, [rec_cap][2 + bm_words]
    uint32_t* rec;
    int rec_cap;
};

__device__ __forceinline__ uint32_t vsad4(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// Shared-memory word load executed only when `p` (predicated: a lane with p false makes no
// shared-memory access and keeps `v`) -- slot loads without a branch per slot.
__device__ __forceinline__ uint32_t lds_if(uint32_t saddr, bool p, uint32_t v) {
    asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.u32 %0, [%1];\n}"
        : "+r"(v) : "r"(saddr), "r"((int)p));
    return v;
}

__device__ __forceinline__ uint32_t ssd4(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d = __vabsdiffu4(a, b);
    return __dp4a(d, d, c);
}


// ---- TMA / mbarrier helpers (sm_90+ PTX; SASS: UTMALDG, SYNCS.*) ---------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(phase)
        : "memory");
}
// 3-D tiled TMA load (x, y, pair) -> shared; out-of-bounds elements are zero-filled.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int x, int y, int z,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}


// Edge replication (reading C9) of a TMA-staged region whose box reached outside the frame
// (TMA zero-fills there).  Region rows i <-> frame row ys+i, columns c <-> frame column xs+c.
// Phase A replicates the edge column into out-of-frame columns of every in-frame row; phase B
// copies the nearest in-frame row into out-of-frame rows.  Border tiles only.
__device__ __forceinline__ void fixup_edges(uint8_t* sref, int pitch, int rh, int xs, int ys,
                                            int W, int H) {
    const int i0 = max(0, -ys), i1 = min(rh, H - ys);      // in-frame rows [i0, i1)
    const int cl = max(0, -xs), cr = min(pitch, W - xs);    // in-frame cols [cl, cr)
    if (cl > 0 || cr < pitch) {
        // xs, W and pitch are multiples of 16: the out-of-frame column spans are whole uint4s
        const int nl = cl >> 4, nr = (pitch - cr) >> 4;
#pragma unroll 1
        for (int e = threadIdx.x; e < (i1 - i0) * (nl + nr); e += blockDim.x) {
            const int i = i0 + e / (nl + nr), q = e % (nl + nr);
            uint8_t* row = sref + i * pitch;
            const uint32_t v = (q < nl ? row[cl] : row[cr - 1]) * 0x01010101u;
            reinterpret_cast<uint4*>(row)[q < nl ? q : (cr >> 4) + (q - nl)] = make_uint4(v, v, v, v);
        }
    }
    __syncthreads();
    if (i0 > 0 || i1 < rh) {
        const int n16 = pitch >> 4;
#pragma unroll 1
        for (int e = threadIdx.x; e < rh * n16; e += blockDim.x) {
            const int i = e / n16, q = e - i * n16;
            if (i >= i0 && i < i1) continue;
            const int src = i < i0 ? i0 : i1 - 1;
            reinterpret_cast<uint4*>(sref + i * pitch)[q] = reinterpret_cast<const uint4*>(sref + src * pitch)[q];
        }
    }
}

// R rows x W4 words of the reference at byte offset o of the staged region (funnel-shifted
// from W4 + 1 aligned words per row); rstride = bytes between the rows.
template <int R, int W4>
__device__ __forceinline__ void ref_rows(const uint32_t* s, int o, int rstride,
                                         uint32_t (&out)[R][W4]) {
    const int sh = o << 3;  // funnel shifts use the low 5 bits: (o & 3) * 8
    const uint32_t* b = s + (o >> 2);
#pragma unroll
    for (int r = 0; r < R; r++) {
        uint32_t wv[W4 + 1];
#pragma unroll
        for (int w = 0; w <= W4; w++) wv[w] = b[r * (rstride >> 2) + w];
#pragma unroll
        for (int w = 0; w < W4; w++) out[r][w] = __funnelshift_r(wv[w], wv[w + 1], sh);
    }
}

// ref_rows from GLOBAL memory (the overflow pass's interior blocks, rows W bytes apart, W a
// multiple of 16): per row two 16-byte loads from the aligned chunk holding byte o, the W4 + 1
// words at word offset (o >> 2) & 3 picked by two select levels, then the funnel shifts --
// 2 vector loads per row where ref_rows issues W4 + 1 scalar ones (each scalar global load of a
// warp touches one line per lane: the L1 tag rate bounds that pass).  Reads [o & ~15, +32).
template <int R, int W4>
__device__ __forceinline__ void ref_rows_gld(const uint32_t* s, int o, int rstride,
                                             uint32_t (&out)[R][W4]) {
    static_assert(W4 + 1 <= 6, "two 16-byte chunks cover W4 + 1 words at any word offset");
    const int sh = o << 3, k = (o >> 2) & 3;
    const uint4* b = reinterpret_cast<const uint4*>(s + ((o >> 2) & ~3));
#pragma unroll
    for (int r = 0; r < R; r++) {
        const uint4 v0 = b[r * (rstride >> 4)], v1 = b[r * (rstride >> 4) + 1];
        const uint32_t v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
        uint32_t u[6], wv[W4 + 1];
#pragma unroll
        for (int i = 0; i < 6; i++) u[i] = (k & 2) ? v[i + 2] : v[i];
#pragma unroll
        for (int w = 0; w <= W4; w++) wv[w] = (k & 1) ? u[w + 1] : u[w];
#pragma unroll
        for (int w = 0; w < W4; w++) out[r][w] = __funnelshift_r(wv[w], wv[w + 1], sh);
    }
}
template <int R, int W4, bool GLD>
__device__ __forceinline__ void ref_rows_any(const uint32_t* s, int o, int rstride, uint32_t (&out)[R][W4]) {
    if constexpr (GLD) ref_rows_gld<R, W4>(s, o, rstride, out);
    else ref_rows<R, W4>(s, o, rstride, out);
}

// W4+2 words around an ALIGNED row start a (a multiple of 4*W4 bytes: one vector load of
// the row): w[0] = the word before, w[1..W4] = the row, w[W4+1] = the word after.
template <int W4>
__device__ __forceinline__ void aligned_row(const uint32_t* s, int a, uint32_t (&w)[W4 + 2]) {
    const uint32_t* b = s + (a >> 2);
    w[0] = b[-1];
    if (W4 == 2) {
        const uint2 v = *reinterpret_cast<const uint2*>(b);
        w[1] = v.x; w[2] = v.y;
    } else {
#pragma unroll
        for (int q = 0; q < W4; q += 4) {
            const uint4 v = *reinterpret_cast<const uint4*>(b + q);
            w[1 + q] = v.x; w[2 + q] = v.y; w[3 + q] = v.z; w[4 + q] = v.w;
        }
    }
    w[W4 + 1] = b[W4];
}
// SAD of one row against the reference shifted by t bytes (t in [-3, 3]) from an aligned_row.
template <int W4>
__device__ __forceinline__ uint32_t sad_shift(const uint32_t (&c)[W4], const uint32_t (&w)[W4 + 2],
                                              int t, uint32_t acc) {
#pragma unroll
    for (int i = 0; i < W4; i++) {
        const uint32_t r = t == 0 ? w[i + 1]
                          : t > 0 ? __funnelshift_r(w[i + 1], w[i + 2], 8 * t)
                                  : __funnelshift_r(w[i], w[i + 1], 8 * (4 + t));
        acc = vsad4(c[i], r, acc);
    }
    return acc;
}

// HCSP order: (0,0) (-1,0) (1,0) (-2,0) (2,0) (0,-1) (0,1), k = 0..6
__device__ __forceinline__ int hcsp_dx(int k) {
    return k == 0 ? 0 : (k <= 4 ? ((k & 1) ? -((k + 1) >> 1) : (k >> 1)) : 0);
}
__device__ __forceinline__ int hcsp_dy(int k) { return k < 5 ? 0 : (k == 5 ? -1 : 1); }

// ----------------------------------------------------------------------------------------
// Lane-group state machine.
//
// Each pass evaluates the (up to) 4 candidate slots of one search pattern, given by a
// pattern id:  2 S3H  HDSP (-2,0) (2,0) (0,-1) (0,1)               [Steps 2-3, P:257]
//              3 S3V  VDSP (-1,0) (1,0) (0,-2) (0,2)
//              4 S4H  middle points (-1,0) (1,0)                    [Step 4]
//              5 S4V  middle points (0,-1) (0,1)
//              6 PREH distant points (-2,0) (2,0)   (DCDS^S look-up, not counted)
//              7 PREV distant points (0,-2) (0,2)
// (ids 0 / 1 name the two halves of the HCSP in the trace format; Step 1 itself runs as one
// straight-line step, GroupState::step1.)  Slot order is the fixed pattern order of reading
// C7: every pattern is -d0, +d0, -d1, +d1, so a group keeps d0 and d1 in registers, as byte
// offsets in the staged region (dy*pitch + dx) and as offsets in the visited bitmap (dy*BW + dx,
// below), and updates them when its pattern changes.
//
// Visited bitmap (reading C5) of a group: one bit per candidate of the +-p window plus a
// 2-wide border, row length BW = 2p+3 (the 2 border columns between consecutive rows serve
// as the right border of one row and the left border of the next): bit of (dx, dy) =
// (dy+p+2)*BW + (dx+p+2).  The border bits start set, so a pattern point outside the window
// (reading C8; pattern offsets are at most 2) reads as "already visited" and is neither
// scored nor counted -- the test-and-set is the whole feasibility test.
// ----------------------------------------------------------------------------------------
enum : int { ST_DONE = 0, ST_S1A = 1, ST_S3 = 3, ST_S4 = 4, ST_S4PRE = 5, ST_IDLE = 6, ST_ESC = 7 };
// (searching: ST_S1A <= st <= ST_S4PRE; ST_ESC: left the compact visited window)

// Visited-bitmap geometry for window +-p: row length, words.  The bitmaps of a CTA's groups
// are interleaved: word w of group gi at bms[w * (groups + 4) + gi], so the groups' test-and-
// sets spread over the banks and the CTA initialises all bitmaps with dense stores.
__host__ __device__ constexpr int bm_row(int p) { return 2 * p + 3; }
__host__ __device__ constexpr int bm_nwords(int p) { return ((2 * p + 5) * bm_row(p) + 2 + 31) / 32; }
// Compact visited set (the B=16 ONE kernels): the same layout over half-widths
// bmx x bmy < p, no border (every bit is a point inside the +-p window), bit of (dx, dy) =
// (dy+bmy+2)*(2bmx+3) + (dx+bmx+2).  A search may test points while its centre stays in
// cx in [-bmx, bmx-2], cy in [-bmy, bmy] (pattern offsets are at most 2; the columns past
// dx = bmx alias the next row); a centre moving out of that range ends the search (ST_ESC)
// and the overflow pass (dcds_redo_kernel) searches the block again with the full bitmap.
__host__ __device__ constexpr int bm_nwords_xy(int bmx, int bmy) {
    return ((2 * bmy + 5) * (2 * bmx + 3) + 2 + 31) / 32;
}


// The two bitmap templates of window +-p (word t of the bordered bitmap): border bits set
// (rows < 2 or >= 2p+3, the 2 border columns between rows), and with_hcsp the 7 HCSP points of
// Step 1 at the window origin as well.  me_init evaluates them once for every p in
// [1, 32] into constant memory (c_bm_tmpl); the kernels copy them instead of rebuilding them
// per CTA.
__host__ __device__ inline uint32_t bm_template_word(int p, int t, bool with_hcsp) {
    const int bw = bm_row(p), lo = 32 * t;
    auto span = [lo](int b0, int b1) -> uint32_t {  // bits [b0, b1) of [lo, lo + 32)
        b0 = b0 > lo ? b0 : lo;
        b1 = b1 < lo + 32 ? b1 : lo + 32;
        return b1 > b0 ? (uint32_t)(((1ull << (b1 - b0)) - 1ull) << (b0 - lo)) : 0u;
    };
    uint32_t w = span(0, 2 * bw) | span((2 * p + 3) * bw, lo + 32);
    for (int rs = (lo / bw) * bw; rs < lo + 32; rs += bw) w |= span(rs, rs + 2);
    if (with_hcsp) {
        const int c = (p + 2) * bw + p + 2;
        const int hc[7] = {c, c - 1, c + 1, c - 2, c + 2, c - bw, c + bw};
        for (int k = 0; k < 7; k++)
            if (hc[k] >= lo && hc[k] < lo + 32) w |= 1u << (hc[k] - lo);
    }
    return w;
}
__host__ __device__ constexpr int bm_tmpl_off(int p) {  // words before p's two templates
    int o = 0;
    for (int q = 1; q < p; q++) o += 2 * bm_nwords(q);
    return o;
}
constexpr int BM_TMPL_WORDS = bm_tmpl_off(33);
__constant__ uint32_t c_bm_tmpl[BM_TMPL_WORDS];

// GLD: the reference rows are read from global memory (ref_rows_gld), not shared memory.
template <int B, int G, bool TRACE = false, bool GLD = false>
struct GroupState {
    static constexpr int R = B / G;   // rows per lane (lane j of a group: rows j, j+G, ...)
    static constexpr int W4 = B / 4;  // 32-bit words per block row
    // 8x8 blocks: a slot with no new point gets the sum SENT (> any SAD, 255*64 = 16320) so
    // the argmin needs no mask; 16x16 SADs (<= 65280) leave no room in the 16-bit fields.
    static constexpr bool SENTINEL = (B == 8);
#ifdef ME_V14
    static constexpr uint32_t SENT_LANE = 16384u / G;
#else
    // 16376 = 8 * 2047: the group sum of a slot with no new point; as a packed key
    // 16376 * 4 + slot >= 65504 > any SAD key (16320 * 4 + 3) and < 2^16
    static constexpr uint32_t SENT_LANE = 16376u / G;
#endif
    // TRACE builds only (me_dcds_trace_batch): one record per scoring pass of the block,
    // bits 0-7 pass (0 = Step 1), 8-11 pattern row (15 = HCSP), 12-19 slots scored,
    // 20-27 / 28-35 pattern centre dx / dy (int8), 36-51 incumbent SAD after the pass
    uint64_t* tr = nullptr;
    int tcap = 0, npass = 0;
    __device__ __forceinline__ void trace(int j, int row, unsigned mask, int ccx, int ccy) {
        if (TRACE && j == 0 && npass < tcap)
            tr[npass] = (uint64_t)(npass & 0xff) | ((uint64_t)row << 8) | ((uint64_t)(mask & 0xff) << 12) |
                        ((uint64_t)(ccx & 0xff) << 20) | ((uint64_t)(ccy & 0xff) << 28) |
                        ((uint64_t)(best & 0xffff) << 36);
        if (TRACE) npass++;
    }
    int st = ST_DONE, pid = 0, kind = 0, pts = 0;
    int want = 0;  // slot mask of the next pass (0 when done / idle)
    int bofs = 0, cpos = 0;  // staged byte offset of the (0,0) candidate / of the centre
    int cidx = 0;            // visited-bitmap bit of the centre
    // the pattern's slots are -d0, +d0, -d1, +d1 (reading C7 order): d0 / d1 as byte offsets in
    // the staged region (db0, db1) and as bitmap offsets (de0, de1), set on state changes
    int db0 = 0, db1 = 0, de0 = 0, de1 = 0;
    int dbg_region = 0, dbg_bits = 0;  // ME_DEBUG: staged-region bytes, bitmap bits
    uint32_t best = 0;
    uint32_t cw[R][W4];

    // move the centre to slot kb of the current pattern
    __device__ __forceinline__ void move(int kb) {
        const int db = (kb & 2) ? db1 : db0, de = (kb & 2) ? de1 : de0;
        cpos += (kb & 1) ? db : -db;
        cidx += (kb & 1) ? de : -de;
    }

    // centre (dx, dy) from its bitmap bit (bitmap half-widths bmx, bmy; row length 2bmx + 3)
    __device__ __forceinline__ void centre(int bmx, int bmy, int& cx, int& cy) const {
        const int bw = 2 * bmx + 3;
        // cidx / bw by a float quotient: cidx < 2^13 and the quotient stays >= 0.5/bw from an
        // integer, far above the error of the approximate division
        const int row = (int)__fdividef((float)cidx + 0.5f, (float)bw);
        cy = row - bmy - 2;
        cx = cidx - row * bw - bmx - 2;
    }

    // Pattern steps of pid (ids above): HDSP d0 (2,0) d1 (0,1); VDSP (1,0) (0,2); middle points
    // (1,0) / (0,1); DCDS^S distant points (2,0) / (0,2).
    // (kind 0 = horizontal, 1 = vertical; each setter is a few selects)
    __device__ __forceinline__ void set_ddsp(int k, int pitch, int bw) {  // HDSP / VDSP
        pid = 2 + k;
        db0 = k ? 1 : 2;
        de0 = db0;
        db1 = k ? 2 * pitch : pitch;
        de1 = k ? 2 * bw : bw;
    }
    __device__ __forceinline__ void set_middle(int k, int pitch, int bw) {  // Step 4
        pid = 4 + k;
        db0 = k ? pitch : 1;
        de0 = k ? bw : 1;
    }
    __device__ __forceinline__ void set_distant(int k, int pitch, int bw) {  // DCDS^S look-up
        pid = 6 + k;
        db0 = k ? 2 * pitch : 2;
        de0 = k ? 2 * bw : 2;
    }

    // Load the lane's current rows of the block at `crow0` (row stride `cpitch`).
    __device__ __forceinline__ void load_cur(int origin, const uint8_t* crow0, int cpitch, int j) {
        bofs = origin;
        cpos = origin;
#pragma unroll
        for (int r = 0; r < R; r++) {
            const uint32_t* crow = reinterpret_cast<const uint32_t*>(crow0 + (j + G * r) * cpitch);
#pragma unroll
            for (int w = 0; w < W4; w++) cw[r][w] = crow[w];
        }
    }
    // Reset the group's visited bitmap (interleaved, word stride bst) to the border template
    // (skipped when the CTA initialised every bitmap) and enter Step 1.
    __device__ __forceinline__ void init_search(int j, uint32_t* bm, int bst, const uint32_t* bm_init,
                                                int bm_words, int bmx, int bmy, bool reset) {
        if (reset)
            for (int w = j; w < bm_words; w += G) bm[w * bst] = bm_init[w];
        const int bw = 2 * bmx + 3;
        cidx = (bmy + 2) * bw + bmx + 2;
        st = ST_S1A; pid = 0; kind = 0; pts = 0; want = 0xf;
    }

    // Step 1 of a block that starts it now (st == ST_S1A), in one straight-line
    // pass: the HCSP points (0,0) (-1,0) (1,0) (-2,0) (2,0) (0,-1) (0,1) (reading C7 order)
    // come from aligned vector row loads with static shifts -- the pattern centre is the
    // window origin, whose staged address is a multiple of 4*W4 bytes for every block.  Ends
    // in Step 3 (switching strategy one) or, on the halfway stop, in a Step-4
    // state with no slots, which the next pass finishes.  All lanes of the warp call it (and
    // __syncwarp after it).
    __device__ __forceinline__ void step1(const uint32_t* s, int j, int p, int bw, int pitch, int rstride,
                                          int jrow) {
        const bool live = (st == ST_S1A);
        uint32_t sk[7] = {0u, 0u, 0u, 0u, 0u, 0u, 0u};
        if (live) {
#pragma unroll
            for (int r = 0; r < R; r++) {
                const int a = bofs + jrow + r * rstride;
                ME_CHECK(a - pitch - 4 >= 0 && a + pitch + 4 * W4 + 4 <= dbg_region);
                uint32_t w[W4 + 2], u[W4 + 2], d[W4 + 2];
                aligned_row<W4>(s, a, w);
                aligned_row<W4>(s, a - pitch, u);
                aligned_row<W4>(s, a + pitch, d);
                sk[0] = sad_shift<W4>(cw[r], w, 0, sk[0]);
                sk[1] = sad_shift<W4>(cw[r], w, -1, sk[1]);
                sk[2] = sad_shift<W4>(cw[r], w, 1, sk[2]);
                sk[3] = sad_shift<W4>(cw[r], w, -2, sk[3]);
                sk[4] = sad_shift<W4>(cw[r], w, 2, sk[4]);
                sk[5] = sad_shift<W4>(cw[r], u, 0, sk[5]);
                sk[6] = sad_shift<W4>(cw[r], d, 0, sk[6]);
            }
        }
        uint32_t v[4] = {sk[0] | (sk[1] << 16), sk[2] | (sk[3] << 16), sk[4] | (sk[5] << 16), sk[6]};
#pragma unroll
        for (int o = 1; o < G; o <<= 1)
#pragma unroll
            for (int q = 0; q < 4; q++) v[q] += __shfl_xor_sync(FULL, v[q], o);
        if (!live) return;
        // feasibility (reading C8): only (+-2,0) can leave the window (p = 1)
        const unsigned feas = p >= 2 ? 0x7fu : 0x67u;
        uint32_t key = 0xffffffffu;
#pragma unroll
        for (int k = 0; k < 7; k++) {
            const uint32_t sad = (v[k >> 1] >> (16 * (k & 1))) & 0xffffu;
            if ((feas >> k) & 1) key = min(key, (sad << 3) | k);
        }
        // visited set (reading C5): the HCSP points are already set in every group's initial
        // bitmap (the pattern sits at the window origin for every block)
        pts = __popc(feas);
        best = key >> 3;
        trace(j, 15, feas, 0, 0);
        const int kb = key & 7;
        if (kb == 0) {  // halfway stop: finish with no further slots
            st = ST_S4; pid = 4; want = 0;
        } else {
            const int cx = hcsp_dx(kb), cy = hcsp_dy(kb);
            cpos = bofs + cy * pitch + cx;
            cidx += cy * bw + cx;
            kind = (cy == 0) ? 0 : 1;  // switching strategy one
            st = ST_S3; want = 0xf;
            set_ddsp(kind, pitch, bw);
        }
    }

    // SSE (P:342 aspect 4) of this lane's rows at the current centre.
    __device__ __forceinline__ uint32_t sse_rows(const uint32_t* s, int jrow, int rstride) const {
        uint32_t rw[R][W4];
        ME_CHECK(cpos + jrow >= 0 && cpos + jrow + (R - 1) * rstride + 4 * W4 + 4 <= dbg_region);
        ref_rows_any<R, W4, GLD>(s, cpos + jrow, rstride, rw);
        uint32_t ss = 0;
#pragma unroll
        for (int r = 0; r < R; r++)
#pragma unroll
            for (int w = 0; w < W4; w++) ss = ssd4(cw[r][w], rw[r][w], ss);
        return ss;
    }

    // One pass of the group's state machine; returns true when the block's search ended.
    // bm_win: the border-only template (the DCDS^S look-up's window test).
    // bmx, bmy: bitmap half-widths; cpt: compact visited set (a centre leaving its range ends
    // the search in ST_ESC).
    template <int VARIANT>
    __device__ __forceinline__ bool pass(const uint32_t* s, uint32_t* bm, int bst, const uint32_t* bm_win,
                                         int j, int leader, int bmx, int bmy, bool cpt, int pitch, int jrow,
                                         int rstride) {
        const int bw = 2 * bmx + 3;
#ifdef ME_DEBUG
        if (cpt && want) {  // compact set: the pattern's points stay inside the window
            int dcx, dcy;
            centre(bmx, bmy, dcx, dcy);
            ME_CHECK(dcx >= -bmx && dcx <= bmx - 2 && dcy >= -bmy && dcy <= bmy);
        }
#endif
        // ---- visited-set test-and-set (reading C5): lane j of a group owns slots j, j+G, ...
        unsigned m4 = 0;
#pragma unroll
        for (int h = 0; h < (G >= 4 ? 1 : 4 / G); h++) {
            const int k = j + h * G;
            bool nw = false;
            if (k < 4 && ((want >> k) & 1)) {
                const int de = (k & 2) ? de1 : de0;
                const int idx = cidx + ((k & 1) ? de : -de);
                const uint32_t bit = 1u << (idx & 31);
                ME_CHECK(idx >= 0 && idx < dbg_bits);
                if (VARIANT && st == ST_S4PRE)
                    nw = (bm_win[idx >> 5] & bit) == 0;  // DCDS^S look-up: in the window
                else
                    nw = (atomicOr(&bm[(idx >> 5) * bst], bit) & bit) == 0;
            }
            const unsigned bb = __ballot_sync(FULL, nw) >> leader;
            m4 |= (G >= 4 ? (bb & 0xfu) : ((bb & ((1u << G) - 1u)) << (h * G)));
        }

        // ---- SADs of the 4 slots over this lane's rows, packed and reduced over the group
        const int o = cpos + jrow;
        uint32_t sadk[4];
#ifndef ME_PRED_SLOTS
#pragma unroll
        for (int k = 0; k < 4; k++) {
            uint32_t acc = SENTINEL ? SENT_LANE : 0u;
            if ((m4 >> k) & 1) {  // slots not scored this pass issue no shared-memory loads
                const int db = (k & 2) ? db1 : db0;
                uint32_t rw[R][W4];
                ME_CHECK(((k & 1) ? o + db : o - db) >= 0 &&
                         ((k & 1) ? o + db : o - db) + (R - 1) * rstride + 4 * W4 + 4 <= dbg_region);
                ref_rows_any<R, W4, GLD>(s, (k & 1) ? o + db : o - db, rstride, rw);
                acc = 0;
#pragma unroll
                for (int r = 0; r < R; r++)
#pragma unroll
                    for (int w = 0; w < W4; w++) acc = vsad4(cw[r][w], rw[r][w], acc);
            }
            sadk[k] = acc;
        }
#else
        // (experiment, measured slower on B200: c3 1.578 vs 1.465 ms, c4 18.7 vs 16.9 ms)
        // no branch per slot: every slot's row words are loaded under the slot's predicate (a
        // lane whose slot is not new makes no shared-memory access), its SAD is computed
        // regardless and replaced by the sentinel / masked out of the argmin below
        const uint32_t sbase = smem_u32(s);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const bool nk = (m4 >> k) & 1;
            const int db = (k & 2) ? db1 : db0;
            const int ok = (k & 1) ? o + db : o - db;
            ME_CHECK(!nk || (ok >= 0 && ok + (R - 1) * rstride + 4 * W4 + 4 <= dbg_region));
            const uint32_t a0 = sbase + (uint32_t)(ok & ~3);
            const uint32_t sh = (uint32_t)ok << 3;  // funnel shifts use the low 5 bits
            uint32_t acc = 0;
#pragma unroll
            for (int r = 0; r < R; r++) {
                uint32_t wv[W4 + 1];
#pragma unroll
                for (int w = 0; w <= W4; w++) wv[w] = lds_if(a0 + r * rstride + 4 * w, nk, 0u);
#pragma unroll
                for (int w = 0; w < W4; w++) acc = vsad4(cw[r][w], __funnelshift_r(wv[w], wv[w + 1], sh), acc);
            }
            sadk[k] = SENTINEL ? (nk ? acc : SENT_LANE) : acc;
        }
#endif
        uint32_t v01 = sadk[0] | (sadk[1] << 16), v23 = sadk[2] | (sadk[3] << 16);
#pragma unroll
        for (int q = 1; q < G; q <<= 1) {
            v01 += __shfl_xor_sync(FULL, v01, q);
            v23 += __shfl_xor_sync(FULL, v23, q);
        }

        // ---- argmin over the new points of this pass, (SAD, slot) keys (reading C6/C7)
        uint32_t key;
        if constexpr (SENTINEL) {
#ifdef ME_V14
            key = min(min(((v01 & 0xffffu) << 2) | 0u, ((v01 >> 16) << 2) | 1u),
                      min(((v23 & 0xffffu) << 2) | 2u, ((v23 >> 16) << 2) | 3u));
#else
            // packed 16-bit keys SAD * 4 + slot (SAD <= 16376: no carry between the halves),
            // min of the two halves of each, then of the two
            const uint32_t m = __vminu2((v01 << 2) + 0x00010000u, (v23 << 2) + 0x00030002u);
            key = min(m & 0xffffu, m >> 16);
#endif
        } else {
            key = 0xffffffffu;
            const uint32_t sv[4] = {v01 & 0xffffu, v01 >> 16, v23 & 0xffffu, v23 >> 16};
#pragma unroll
            for (int k = 0; k < 4; k++)
                if ((m4 >> k) & 1) key = min(key, (sv[k] << 2) | k);
        }
        const int kb = key & 3;

        // ---- advance the state machine (group-uniform)
        bool fin = false;
        int ccx = 0, ccy = 0;
        const int cpid = pid;
        const bool scoring = (st == ST_S3 || st == ST_S4);
        if (TRACE) centre(bmx, bmy, ccx, ccy);
        if (st != ST_S4PRE) pts += __popc(m4);
        if (st == ST_S3) {
            // Step 2 / Step 3
            if ((key >> 2) < best) {
                best = key >> 2;
                move(kb);
                if ((kb >= 2) != (kind == 1)) { kind ^= 1; set_ddsp(kind, pitch, bw); }  // near point
                if (cpt) {  // compact visited set: the next pattern must stay inside it
                    int cx, cy;
                    centre(bmx, bmy, cx, cy);
                    if (cx < -bmx || cx > bmx - 2 || cy < -bmy || cy > bmy) { st = ST_ESC; want = 0; }
                }
            } else {
                st = VARIANT ? ST_S4PRE : ST_S4;  // BMP at the centre -> Step 4
                if (VARIANT) set_distant(kind, pitch, bw);
                else set_middle(kind, pitch, bw);
                want = 3;
            }
        } else if (VARIANT && st == ST_S4PRE) {
            // DCDS^S: keep only the middle point beside the cheaper distant point;
            // an infeasible distant point costs +inf, ties go to the negative side (C22)
            const uint32_t dn = (m4 & 1) ? (v01 & 0xffffu) : 0xffffffffu;
            const uint32_t dp = (m4 & 2) ? (v01 >> 16) : 0xffffffffu;
            want = (dp < dn) ? 2 : 1;
            st = ST_S4;
            set_middle(kind, pitch, bw);
        } else if (st == ST_S4) {
            // Step 4: strict minimum of the middle points against the centre
            if ((key >> 2) < best) {
                best = key >> 2;
                move(kb);
            }
            fin = true;
        }
        if (TRACE && scoring) trace(j, cpid, m4, ccx, ccy);

        return fin;
    }
};

// The outputs of block gblk (index pair * nb + block): MV, SAD, NSP.
__device__ __forceinline__ void store_block(const SearchArgs& a, long long gblk, int cx, int cy,
                                            uint32_t best, int pts) {
    if (a.packed) {  // 6-byte records: int8 (dx, dy), 16-bit SAD (<= 255*256), NSP
        reinterpret_cast<uint16_t*>(a.mv)[gblk] = (uint16_t)((cx & 0xff) | ((cy & 0xff) << 8));
        reinterpret_cast<uint16_t*>(a.sad)[gblk] = (uint16_t)best;
    } else {
        a.mv[gblk] = (uint32_t)(cx & 0xffff) | ((uint32_t)cy << 16);
        a.sad[gblk] = best;
    }
    a.pts[gblk] = (uint16_t)pts;
}

// Overflow pass (below): an interior block's +-p window and the row loads' over-read lie inside
// the frame's rows, so it reads the reference frame directly.
__device__ __forceinline__ bool redo_interior(const SearchArgs& a, long long gblk) {
    const int blk = (int)(gblk % a.nb), by = blk / a.nbx, bx = blk - by * a.nbx;
    const int B = a.W / a.nbx, x0 = bx * B, y0 = by * B;
    // (ref_rows_gld reads [o & ~15, +32) for a candidate at column o: x0 - p - 15 >= 0 and
    // x0 + p + 32 <= W keep every read inside the window's own rows)
    return x0 >= a.p + 15 && x0 + a.p + 32 <= a.W && y0 >= a.p && y0 + B + a.p <= a.H;
}

// ONE: the tile holds at most one block per lane group (the default geometries: 16x4 blocks
// for 64 groups at B=8, 8x4 for 32 groups at B=16) -- every group takes its block at the
// start, keeps the finished search in registers, and the SSE and outputs of all blocks are
// produced in one dense phase after the last search ends.  Otherwise blocks are handed out
// from a tile counter as groups finish.
// CPT: the compact-visited-set build of the 16x16 ONE kernel (5 CTAs per SM: <= 48 registers).
template <int B, int G, int NWARP, int VARIANT, bool TRACE = false, bool ONE = false, int PITCH = 0,
          bool CPT = false>
__global__ void __launch_bounds__(NWARP * 32, ONE ? (B == 8 ? 36 / NWARP : (CPT ? 5 : 1)) : 1)
    dcds_kernel(const __grid_constant__ CUtensorMap tm_cur, const __grid_constant__ CUtensorMap tm_ref,
                const SearchArgs a) {
    static_assert(G == 1 || G == 2 || G == 4 || G == 8 || G == 16, "lane-group size");
    constexpr int NG = 32 / G;    // groups per warp (rows per lane and words per row: GroupState)
    // all shared memory is dynamic, from a 1024-aligned base (TMA destinations are 128-byte
    // aligned; the launch fails loudly otherwise)
    extern __shared__ __align__(1024) uint8_t smem[];
    if ((smem_u32(smem) & 127) != 0) __trap();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = lane % G, g = lane / G, leader = g * G;
    const int pair = blockIdx.z;
    const int tx = blockIdx.x, ty = blockIdx.y;
    const int TW = a.tbx * B, TH = a.tby * B;
    const int x0 = tx * TW, y0 = ty * TH;
    const int xs = (x0 - a.p) & ~15;  // floor to 16 (two's complement)
    const int ys = y0 - a.p;
    const int pitch = PITCH ? PITCH : a.pitch, p = a.p;
    // compact visited set: the B=16 ONE kernels (4-8x8 tiles at +-32 need 5 CTAs/SM)
    constexpr bool CPT_OK = CPT && ONE && B == 16 && !TRACE;
    const bool cpt = CPT_OK && a.compact;
    // GCUR: the 8x8 ONE kernels load each group's current rows from global memory during the
    // region's TMA load and initialise the bitmaps before waiting for it (c3 1.407 -> 1.401 ms;
    // for 16x16 blocks the TMA-staged current tile measured faster: 14.78 vs 15.16 ms at c4)
    constexpr bool GCUR = ONE && B == 8;
    const int bmx = CPT_OK ? a.bmx : p, bmy = CPT_OK ? a.bmy : p;

    // shared layout: reference region (pitch x rh) | current tile (TW x TH) | group bitmaps |
    // bitmap template | tile counter | mbarrier | per-warp statistics sums (NWARP x 3 u64).  ONE
    // kernels overlay the bitmaps on the current tile (read into registers first; GCUR kernels
    // read the current rows from global memory and use the space for the bitmaps only).
    uint8_t* sref = smem;
    uint8_t* scur = smem + a.cur_off;
    uint32_t* bms = reinterpret_cast<uint32_t*>(smem + a.bm_off);
    // interleaved bitmap word stride: groups + 4 keeps the rows 16-byte aligned (one uint4
    // store initialises 4 groups' words) and a warp's 32/G groups on distinct banks
    constexpr int BST = NWARP * NG + 4;
    uint32_t* bm = bms + (warp * NG + g);
    uint32_t* bm_init = reinterpret_cast<uint32_t*>(smem + a.init_off);  // border + HCSP
    uint32_t* bm_win = bm_init + a.bm_words;                               // border only
    int* ctr = reinterpret_cast<int*>(bm_win + a.bm_words);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + ((a.init_off + 8 * a.bm_words + 4 + 7) & ~7));

    // ---- stage the tile with TMA: reference region + current tile, one mbarrier
    if (threadIdx.x == 0) {
        // the thread that initialises the mbarrier issues the loads right away (the init is
        // made visible to the async proxy first); the barrier below publishes the init to the
        // other threads while the loads are in flight (measured: c4 15.19 -> 14.78 ms against
        // issuing after the barrier)
        // (GCUR kernels read their current rows from global memory: only the region is staged)
        mbar_init(bar, 1);  // (with fence.mbarrier_init)
        mbar_expect_tx(bar, (uint32_t)(pitch * a.rh + (GCUR ? 0 : TW * TH)));
        tma_load_3d(sref, &tm_ref, xs, ys, pair, bar);
        if (!GCUR) tma_load_3d(scur, &tm_cur, x0, y0, pair, bar);
        *ctr = 0;
    }
    __syncthreads();
    const int bw = 2 * bmx + 3;
    // bitmap templates (border only / border + HCSP), precomputed in constant memory; the
    // compact set has no border (no bits / the 7 HCSP bits)
    for (int t = threadIdx.x; t < a.bm_words; t += NWARP * 32) {
        if (cpt) {
            const int c = (bmy + 2) * bw + bmx + 2;
            const int hc[7] = {c, c - 1, c + 1, c - 2, c + 2, c - bw, c + bw};
            uint32_t w = 0;
#pragma unroll
            for (int k = 0; k < 7; k++)
                if ((hc[k] >> 5) == t) w |= 1u << (hc[k] & 31);
            bm_win[t] = 0;
            bm_init[t] = w;
        } else {
            bm_win[t] = c_bm_tmpl[bm_tmpl_off(p) + t];
            bm_init[t] = c_bm_tmpl[bm_tmpl_off(p) + a.bm_words + t];
        }
    }
    const bool border = xs < 0 || ys < 0 || xs + pitch > a.W || ys + a.rh > a.H;
    if constexpr (!GCUR) {
        mbar_wait(bar, 0);
        if (border) fixup_edges(sref, pitch, a.rh, xs, ys, a.W, a.H);
        __syncthreads();
    }

    const uint32_t* s = reinterpret_cast<const uint32_t*>(sref);
    const int rstride = G * pitch;  // bytes between a lane's rows
    const int jrow = j * pitch;     // byte offset of the lane's first row
    const int tbx_e = min(a.tbx, a.nbx - tx * a.tbx), tby_e = min(a.tby, a.nby - ty * a.tby);
    const int nbt = tbx_e * tby_e;

    GroupState<B, G, TRACE> gs;  // group state (every lane of a group holds the same values)
    long long gblk = 0;
    unsigned long long acc_pts = 0, acc_sad = 0, acc_sse = 0;

    // block idx of the tile (row-major over tbx_e columns): its output index and current rows
    auto take = [&](int idx) {
        const int lby = (int)__fdividef((float)idx + 0.5f, (float)tbx_e);  // idx < 2^12: exact
        const int lbx = idx - lby * tbx_e;
        const int bxg = x0 + lbx * B, byg = y0 + lby * B;
        gblk = (long long)pair * a.nb + (byg / B) * a.nbx + (bxg / B);
        if (TRACE) { gs.tr = a.trace + gblk * a.tcap; gs.tcap = a.tcap; gs.npass = 0; }
        if constexpr (GCUR)  // the current block's rows straight from the frame (L2 / HBM)
            gs.load_cur((byg - ys) * pitch + (bxg - xs), a.cur0 + (long long)pair * a.stride + (long long)byg * a.W + bxg,
                        a.W, j);
        else
            gs.load_cur((byg - ys) * pitch + (bxg - xs), scur + (lby * B) * TW + lbx * B, TW, j);
#ifdef ME_DEBUG
        gs.dbg_region = pitch * a.rh;
        gs.dbg_bits = 32 * a.bm_words;
#endif
    };
    auto output = [&](uint32_t ss) {
        int cx, cy;
        gs.centre(bmx, bmy, cx, cy);
        store_block(a, gblk, cx, cy, gs.best, gs.pts);
        if (TRACE) a.tlen[gblk] = (uint16_t)gs.npass;
        acc_pts += (unsigned)gs.pts;
        acc_sad += gs.best;
        acc_sse += ss;
    };

    if constexpr (ONE) {
        const int idx = warp * NG + g;
        const bool have = idx < nbt;
        if (have) take(idx);  // (GCUR: global loads, in flight with the region's TMA load)
        __syncthreads();  // the templates are written; every current row is in registers
        // all bitmaps of the CTA at once: word w of every group, dense 16-byte stores (over the
        // current tile, which is in registers by now)
        for (int e = threadIdx.x; e < a.bm_words * (BST / 4); e += NWARP * 32) {
            const uint32_t v = bm_init[e / (BST / 4)];  // constant divisor
            reinterpret_cast<uint4*>(bms)[e] = make_uint4(v, v, v, v);
        }
        if constexpr (GCUR) {
            mbar_wait(bar, 0);
            if (border) fixup_edges(sref, pitch, a.rh, xs, ys, a.W, a.H);
        }
        __syncthreads();  // the bitmaps (and an edge-fixed region) are visible
        if (have) gs.init_search(j, bm, BST, bm_init, a.bm_words, bmx, bmy, false);
        else { gs.st = ST_IDLE; gs.want = 0; }
        if (__any_sync(FULL, have)) {
            gs.step1(s, j, p, bw, pitch, rstride, jrow);
            __syncwarp();  // the visited bits are set before the pass tests them
            while (__any_sync(FULL, gs.st != ST_DONE && gs.st < ST_IDLE))
                if (gs.template pass<VARIANT>(s, bm, BST, bm_win, j, leader, bmx, bmy, cpt, pitch, jrow,
                                              rstride)) {
                    gs.st = ST_DONE; gs.want = 0;
                }
            // every search of the warp ended: SSE of the compensated blocks (P:342 aspect 4)
            // and the outputs, in one dense phase (a search that left the compact visited set
            // hands its block to the overflow pass instead)
            const bool live = have && (!CPT_OK || gs.st != ST_ESC);
            uint32_t ss = live ? gs.sse_rows(s, jrow, rstride) : 0u;
#pragma unroll
            for (int o2 = 1; o2 < G; o2 <<= 1) ss += __shfl_xor_sync(FULL, ss, o2);
            if (live && j == 0) output(ss);
            if (CPT_OK && have && !live && j == 0) {
                // hand the abandoned search to the overflow passes: interior blocks to the
                // front of the list with a warm-start record (centre, kind, SAD, points, the
                // compact bitmap) while records last, border blocks to the back
                if (redo_interior(a, gblk)) {
                    const uint32_t e = atomicAdd(&a.ovf[0], 1u);
                    a.ovf[4 + e] = (uint32_t)gblk;
                    if (e < (uint32_t)a.rec_cap) {
                        uint32_t* rc = a.rec + (size_t)e * (2 + a.bm_words);
#pragma unroll 1
                        for (int w = 0; w < a.bm_words; w++) rc[2 + w] = bm[w * BST];
                        int cx, cy;
                        gs.centre(bmx, bmy, cx, cy);
                        rc[0] = (uint32_t)(cx & 0xff) | ((uint32_t)(cy & 0xff) << 8) | ((uint32_t)gs.kind << 16);
                        rc[1] = gs.best | ((uint32_t)gs.pts << 16);
                    }
                } else {
                    a.ovf[4 + a.ovf_cap - 1 - atomicAdd(&a.ovf[1], 1u)] = (uint32_t)gblk;
                }
            }
        }
    } else for (;;) {
        // ---- groups that are done take the next block of the tile
        const bool need = (gs.st == ST_DONE);
        const unsigned ball = __ballot_sync(FULL, need && j == 0);
        if (ball) {
            if (*reinterpret_cast<volatile int*>(ctr) >= nbt) {
                // the tile's blocks are all taken (one shared load, warp-uniform)
                if (need) { gs.st = ST_IDLE; gs.want = 0; }
            } else {
                int base = 0;
                if (lane == 0) base = atomicAdd(ctr, __popc(ball));
                base = __shfl_sync(FULL, base, 0);
                int idx = base + __popc(ball & ((1u << lane) - 1u));
                idx = __shfl_sync(FULL, idx, leader);
                if (need) {
                    if (idx < nbt) {
                        take(idx);
                        gs.init_search(j, bm, BST, bm_init, a.bm_words, bmx, bmy, true);
                    } else {
                        gs.st = ST_IDLE; gs.want = 0;
                    }
                }
            }
            __syncwarp();
        }
        if (__all_sync(FULL, gs.st == ST_IDLE)) break;
        // ---- groups that just took a block run Step 1 in one straight-line step
        if (__any_sync(FULL, gs.st == ST_S1A)) {
            gs.step1(s, j, p, bw, pitch, rstride, jrow);
            __syncwarp();  // the visited bits are set before the pass tests them
        }

        const bool fin = gs.template pass<VARIANT>(s, bm, BST, bm_win, j, leader, bmx, bmy, false, pitch,
                                                   jrow, rstride);

        // ---- finished blocks: SSE of the compensated block (P:342 aspect 4), outputs
        if (__any_sync(FULL, fin)) {
            uint32_t ss = fin ? gs.sse_rows(s, jrow, rstride) : 0u;  // finishing groups only
#pragma unroll
            for (int o2 = 1; o2 < G; o2 <<= 1) ss += __shfl_xor_sync(FULL, ss, o2);
            if (fin) {
                if (j == 0) output(ss);
                gs.st = ST_DONE; gs.want = 0;
            }
        }
    }
    if (a.stats) {
        // per-pair statistics: warp sums of the group leaders, then the CTA's sums, 3 global
        // atomics per CTA (one address triple per pair: atomics from every warp cost 3.5 % of
        // the kernel at c3, 7 % at c4; a fence-ordered last-warp hand-off measured slower)
        unsigned long long sp, sd, se;
        if constexpr (ONE) {
            // one block per group: a warp's sums fit 32 bits (<= 32 blocks x 255^2 x 256)
            sp = __reduce_add_sync(FULL, (uint32_t)acc_pts);
            sd = __reduce_add_sync(FULL, (uint32_t)acc_sad);
            se = __reduce_add_sync(FULL, (uint32_t)acc_sse);
        } else {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                acc_pts += __shfl_xor_sync(FULL, acc_pts, o);
                acc_sad += __shfl_xor_sync(FULL, acc_sad, o);
                acc_sse += __shfl_xor_sync(FULL, acc_sse, o);
            }
            sp = acc_pts; sd = acc_sad; se = acc_sse;
        }
        unsigned long long* cs = reinterpret_cast<unsigned long long*>(bar + 1);  // [NWARP][3]
        if (lane == 0) {
            cs[3 * warp + 0] = sp;
            cs[3 * warp + 1] = sd;
            cs[3 * warp + 2] = se;
        }
        __syncthreads();  // (every warp of the CTA gets here)
        if (threadIdx.x < 3) {
            unsigned long long t = 0;
#pragma unroll
            for (int w = 0; w < NWARP; w++) t += cs[3 * w + threadIdx.x];
            atomicAdd(&a.stats[pair * 3 + threadIdx.x], t);
        }
    }
}

// ---- overflow passes of the compact visited set (DESIGN.md §7 "Compact visited set") ----
// Every block whose search left the compact window (SearchArgs::ovf) is searched again from
// the start by the same GroupState code with the full +-p bitmap (border template), so its
// outputs are those of the full-bitmap kernels.  One block per lane group, groups claiming
// blocks from the list.  GLOBAL: the interior blocks, reading the reference frame directly
// (region base = the frame row y0 - p, pitch W; no shared staging, so 32 warps per SM);
// otherwise the border blocks, one warp per CTA, each group staging its block's (B + 2p) x
// redo_pitch window by cp.async with edge replication (reading C9, as fixup_edges).
__host__ __device__ constexpr int redo_pitch(int B, int p) {
    // the main kernel's bound for a one-block tile (TW + 2p + 31 bytes), 16 * odd bytes
    const int w = (B + 2 * p + 31 + 15) & ~15;
    return ((w >> 4) & 1) ? w : w + 16;
}
__host__ __device__ constexpr int redo_smem(int B, int G, int p, bool global, int nwarps) {
    return (global ? 0 : nwarps * (32 / G) * redo_pitch(B, p) * (B + 2 * p)) +
           (2 + nwarps * (32 / G)) * bm_nwords(p) * 4;
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int B, int G, int VARIANT, bool GLOBAL>
__global__ void __launch_bounds__(GLOBAL ? 128 : 32, GLOBAL ? 8 : 1) dcds_redo_kernel(const SearchArgs a) {
    constexpr int NG = 32 / G;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = lane % G, g = lane / G, leader = g * G, slot = warp * NG + g;
    const int nslots = (blockDim.x >> 5) * NG;
    const int p = a.p, W = a.W, H = a.H;
    const int rp = GLOBAL ? W : redo_pitch(B, p), rr = B + 2 * p;
    const int words = bm_nwords(p);
    // shared: staged windows (border pass) | templates (border + HCSP, border only) | bitmaps
    uint8_t* region = smem + (GLOBAL ? 0 : slot * rp * rr);
    uint32_t* bm_init = reinterpret_cast<uint32_t*>(smem + (GLOBAL ? 0 : nslots * rp * rr));
    uint32_t* bm_win = bm_init + words;
    uint32_t* bm = bm_win + words + slot * words;
    for (int t = threadIdx.x; t < words; t += blockDim.x) {
        bm_win[t] = c_bm_tmpl[bm_tmpl_off(p) + t];
        bm_init[t] = c_bm_tmpl[bm_tmpl_off(p) + words + t];
    }
    __syncthreads();
    const uint32_t count = a.ovf[GLOBAL ? 0 : 1];
    uint32_t* claim = &a.ovf[GLOBAL ? 2 : 3];
    const int rstride = G * rp, jrow = j * rp;
    GroupState<B, G, false, GLOBAL> gs;
    for (;;) {
        uint32_t e = 0xffffffffu;
        if (j == 0) e = atomicAdd(claim, 1u);
        e = __shfl_sync(FULL, e, leader);
        const bool have = e < count;
        if (!__any_sync(FULL, have)) break;
        long long gblk = 0;
        int pair = 0, x0 = 0, y0 = 0, xs = 0;
        const uint32_t* s = reinterpret_cast<const uint32_t*>(region);
        const uint8_t* ref = a.ref0;
        if (have) {
            gblk = a.ovf[GLOBAL ? 4 + e : 4 + a.ovf_cap - 1 - e];
            pair = (int)(gblk / a.nb);
            const int blk = (int)(gblk - (long long)pair * a.nb);
            const int by = blk / a.nbx, bx = blk - by * a.nbx;
            x0 = bx * B;
            y0 = by * B;
            ref += (long long)pair * a.stride;
            xs = (x0 - p) & ~15;
            if constexpr (GLOBAL) {
                s = reinterpret_cast<const uint32_t*>(ref + (long long)(y0 - p) * W);
            } else {
                // xs and W are multiples of 16: a 16-byte chunk is wholly inside or outside the
                // frame; rows clamp to the frame, in-frame chunks by cp.async, then (below) the
                // out-of-frame chunks replicate the row's edge byte
                for (int q = j; q < rr * (rp >> 4); q += G) {
                    const int i = q / (rp >> 4), x = xs + 16 * (q - i * (rp >> 4));
                    if (x >= 0 && x + 16 <= W)
                        cp_async16(region + i * rp + (x - xs), ref + (long long)min(max(y0 - p + i, 0), H - 1) * W + x);
                }
            }
        }
        if constexpr (!GLOBAL) {
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncwarp();  // every lane of the warp: the copies of the whole group are visible
            if (have)
                for (int q = j; q < rr * (rp >> 4); q += G) {
                    const int i = q / (rp >> 4), x = xs + 16 * (q - i * (rp >> 4));
                    if (x < 0 || x + 16 > W) {
                        const uint32_t e4 = region[i * rp + (x < 0 ? -xs : W - 1 - xs)] * 0x01010101u;
                        *reinterpret_cast<uint4*>(region + i * rp + (x - xs)) = make_uint4(e4, e4, e4, e4);
                    }
                }
        }
        if (have) {
            const int origin = GLOBAL ? p * W + x0 : p * rp + (x0 - xs);
            gs.load_cur(origin, a.cur0 + (long long)pair * a.stride + (long long)y0 * W + x0, W, j);
#ifdef ME_DEBUG
            gs.dbg_region = rp * rr;
            gs.dbg_bits = 32 * words;
#endif
            gs.init_search(j, bm, 1, bm_init, words, p, p, true);
        } else {
            gs.st = ST_IDLE; gs.want = 0;
        }
        if constexpr (GLOBAL) {
            // warm start: continue the abandoned search from its record -- its compact visited
            // bits remapped into the full bitmap, its Step-3 state restored (Step 1 is skipped)
            __syncwarp();  // the group's template words are written before the remap ORs in
            if (have && e < (uint32_t)a.rec_cap) {
                const uint32_t* rc = a.rec + (size_t)e * (2 + a.bm_words);
                const int bwc = 2 * a.bmx + 3, bwf = bm_row(p);
                for (int w = j; w < a.bm_words; w += G) {
                    uint32_t v = rc[2 + w];
                    while (v) {
                        const int ci = 32 * w + __ffs(v) - 1;
                        v &= v - 1;
                        const int row = ci / bwc, dx = ci - row * bwc - (a.bmx + 2), dy = row - (a.bmy + 2);
                        const int fi = (dy + p + 2) * bwf + (dx + p + 2);
                        atomicOr(&bm[fi >> 5], 1u << (fi & 31));
                    }
                }
                const uint32_t s0 = rc[0], s1 = rc[1];
                const int cx = (int)(int8_t)(s0 & 0xff), cy = (int)(int8_t)((s0 >> 8) & 0xff);
                gs.kind = (int)((s0 >> 16) & 1u);
                gs.best = s1 & 0xffffu;
                gs.pts = (int)(s1 >> 16);
                gs.cidx = (cy + p + 2) * bwf + (cx + p + 2);
                gs.cpos = gs.bofs + cy * rp + cx;
                gs.st = ST_S3;
                gs.want = 0xf;
                gs.set_ddsp(gs.kind, rp, bwf);
            }
        }
        __syncwarp();  // the staged windows and bitmaps are visible to the group
        gs.step1(s, j, p, bm_row(p), rp, rstride, jrow);
        __syncwarp();
        while (__any_sync(FULL, gs.st != ST_DONE && gs.st < ST_IDLE))
            if (gs.template pass<VARIANT>(s, bm, 1, bm_win, j, leader, p, p, false, rp, jrow, rstride)) {
                gs.st = ST_DONE; gs.want = 0;
            }
        uint32_t ss = have ? gs.sse_rows(s, jrow, rstride) : 0u;
#pragma unroll
        for (int o2 = 1; o2 < G; o2 <<= 1) ss += __shfl_xor_sync(FULL, ss, o2);
        if (have && j == 0) {
            int cx, cy;
            gs.centre(p, p, cx, cy);
            store_block(a, gblk, cx, cy, gs.best, gs.pts);
            if (a.stats) {
                atomicAdd(&a.stats[pair * 3 + 0], (unsigned long long)gs.pts);
                atomicAdd(&a.stats[pair * 3 + 1], (unsigned long long)gs.best);
                atomicAdd(&a.stats[pair * 3 + 2], (unsigned long long)ss);
            }
        }
        __syncwarp();  // every lane is done with the windows before the next blocks replace them
    }
}

}  // namespace me
