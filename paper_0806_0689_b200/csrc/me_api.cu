// me_api.cu -- C ABI of libme.so (include/me.h): validation, launch configuration, streams.
//
// Every entry point validates its arguments before any device work and launches the
// sm_100a kernels of dcds_kernel.cuh / fs_kernel.cuh on the library stream.  There is no
// CPU fallback: without a working sm_100 device every call fails with ME_ENOTINIT/ME_ECUDA.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>

#include "../../include/me.h"
#include "bma_kernel.cuh"
#include "ideal_kernel.cuh"
#include "dcds_kernel.cuh"
#include "fs_kernel.cuh"

namespace {

int g_dev = -1;
cudaStream_t g_stream = nullptr;
cudaStream_t g_copy_streams[2] = {nullptr, nullptr};
unsigned long long* g_scratch = nullptr;  // device u64 scratch (me_mc_psnr)
char g_err[512] = "";
long long g_launches = 0;
int g_smem_optin = 0;
int g_smem_sm = 233472;  // shared memory per SM (bytes)
int g_sms = 148;
// overflow list of the compact visited set (SearchArgs::ovf; grow-only, 4 bytes per block)
uint8_t* g_ovf = nullptr;
size_t g_ovf_cap = 0;
uint8_t* g_rec = nullptr;  // warm-start records of the overflow pass (grow-only)
size_t g_rec_cap = 0;
bool g_ovf_used = false;  // the last DCDS batch call used the compact set
// the list is one buffer: a compact call on another stream than the previous one waits for it
cudaEvent_t g_ovf_ev = nullptr;
cudaStream_t g_ovf_stream = nullptr;
int grow(uint8_t** p, size_t* cap, size_t need);
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;  // driver entry point (no -lcuda)

// grow-only staging buffers of me_dcds_batch_host (two sets for double buffering)
struct HostStage {
    uint8_t* frames = nullptr;
    size_t frames_cap = 0;
    uint8_t* out = nullptr;
    size_t out_cap = 0;
};
HostStage g_stage[2];
// frames per staging buffer of me_dcds_batch_host (allocated by me_init; a call whose single
// pair exceeds it grows the buffers once)
constexpr long long kStageFrames = 128ll << 20;
cudaEvent_t g_order_ev = nullptr;  // orders the host-path copies after the library stream

int set_cuda_err(cudaError_t e, const char* where) {
    snprintf(g_err, sizeof g_err, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
    return ME_ECUDA;
}

int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

#define CK(call)                                               \
    do {                                                       \
        cudaError_t _e = (call);                               \
        if (_e != cudaSuccess) return set_cuda_err(_e, #call); \
    } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
bool aligned(const void* p, unsigned a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

int validate_frames(const uint8_t* cur, const uint8_t* ref, long long stride, int npairs, int W,
                    int H, int block) {
    if (!cur || !ref) return fail(ME_EINVAL, "NULL frame pointer");
    if (W <= 0 || H <= 0) return fail(ME_EINVAL, "W and H must be positive");
    if (block != 8 && block != 16) return fail(ME_EINVAL, "block must be 8 or 16");
    if (W % block || H % block) return fail(ME_EINVAL, "W and H must be multiples of block");
    if (npairs < 1) return fail(ME_EINVAL, "npairs must be >= 1");
    if (W > 32768 || H > 32768) return fail(ME_EINVAL, "frame larger than 32768");
    if ((long long)(W / block) * (H / block) > (1ll << 31) / 4) return fail(ME_EINVAL, "too many blocks");
    if (npairs > 65535) return fail(ME_EINVAL, "npairs must be <= 65535");
    if (W % 16) return fail(ME_EALIGN, "W must be a multiple of 16");
    if (!aligned16(cur) || !aligned16(ref)) return fail(ME_EALIGN, "frame pointers must be 16-byte aligned");
    if (npairs > 1 && (stride % 16)) return fail(ME_EALIGN, "pair_stride must be a multiple of 16");
    if (npairs > 1 && stride < (long long)W * H) return fail(ME_EINVAL, "pair_stride smaller than a frame");
    return ME_OK;
}

int validate_search(const uint8_t* cur, const uint8_t* ref, long long stride, int npairs, int W,
                    int H, int block, int p, const void* mv, const void* sad, const void* pts) {
    int rc = validate_frames(cur, ref, stride, npairs, W, H, block);
    if (rc) return rc;
    if (p < 1 || p > 32) return fail(ME_EINVAL, "p must be in [1, 32]");
    if (!mv || !sad || !pts) return fail(ME_EINVAL, "NULL output pointer");
    if (!aligned(mv, 4) || !aligned(sad, 4) || !aligned(pts, 2))
        return fail(ME_EALIGN, "output pointers must be naturally aligned (mv 4 B)");
    return ME_OK;
}

struct DcdsLaunch {
    me::SearchArgs a;
    dim3 grid;
    size_t smem;
    int G;
    int NW;  // warps per CTA
    int TW, TH;
    bool one;  // at most one block per lane group: the ONE kernels (default geometry)
};

// Launch geometry: lane-group size G, tile of tbx x tby blocks.
// ME_G / ME_TILE=tbx,tby override the defaults (tuning only).
DcdsLaunch plan_dcds(int W, int H, int B, int p, int npairs, bool allow_compact = false) {
    DcdsLaunch L;
    me::SearchArgs& a = L.a;
    const int nbx = W / B, nby = H / B;
    L.G = (B == 16) ? 8 : 2;
    L.NW = (B == 16) ? 8 : 4;
    if (const char* e = getenv("ME_NW")) {
        const int nw = atoi(e);
        if (nw == 2 || nw == 4 || nw == 8) L.NW = nw;
    }

    // measured on B200 (profiles/r1/SUMMARY.md): B=8: G=2, 4 warps, 16x4 blocks;
    // B=16: G=8, 8 warps, 4x8 blocks (profiles/r1c/SUMMARY.md)
    int tbx = (B == 16) ? 4 : 16;
    int tby = (B == 16) ? 8 : 4;
    if (const char* e = getenv("ME_G")) {
        const int g = atoi(e);
        // G = 1 (thread per block) is instantiated for 8x8 blocks only
        if (g == 2 || g == 4 || g == 8 || (g == 1 && B == 8)) L.G = g;
    }
    if (const char* e = getenv("ME_TILE")) {
        int tx = 0, ty = 0;
        if (sscanf(e, "%d,%d", &tx, &ty) == 2 && tx > 0 && ty > 0 && (tx * B) % 16 == 0) {
            tbx = tx;
            tby = ty;
        }
    }
    tbx = std::min(tbx, nbx);
    tby = std::min(tby, nby);
    const int TW = tbx * B, TH = tby * B;
    a.W = W; a.H = H; a.p = p;
    a.tbx = tbx; a.tby = tby;
    a.ntx = (nbx + tbx - 1) / tbx;
    const int nty = (nby + tby - 1) / tby;
    // region width: x0 - xs <= p + 15, plus TW + p, plus 16 bytes of over-read slack
    int pitch = ((TW + 2 * p + 31) + 15) & ~15;
    // 8x8 blocks: 64 (mod 128) bytes, so the two lanes of a group (rows one pitch apart) read
    // banks 16 apart -- measured by replaying real search traces through the warp's loads
    // (tools/sim_banks.py: 1.54 wavefronts per candidate-row load vs 1.77 at 208 bytes);
    // otherwise (or past the 256-byte TMA box) 16 * odd bytes
    int p64 = pitch;
    while ((p64 & 127) != 64) p64 += 16;
    if (B == 8 && p64 <= 256) pitch = p64;
    else if (((pitch >> 4) & 1) == 0) pitch += 16;
    a.pitch = pitch;
    a.rh = TH + 2 * p;
    a.bm_words = me::bm_nwords(p);
    a.nbx = nbx;
    a.nby = nby;
    a.nb = nbx * nby;
    L.grid = dim3(a.ntx, nty, npairs);
    const int groups = L.NW * 32 / L.G;
    // TMA destinations are 128-byte aligned; the 3-word row loads never pass the region's
    // last row (pitch >= TW + 2p + 16 + 15), so nothing needs slack after it
    a.cur_off = (pitch * a.rh + 127) & ~127;
    L.TW = TW; L.TH = TH;
    // the ONE kernels (one block per lane group) exist for the default geometry
    L.one = tbx * tby <= groups && L.G == (B == 16 ? 8 : 2) && (L.NW == (B == 16 ? 8 : 4) || (B == 8 && L.NW == 8));
    auto layout = [&](int words) {  // bitmaps, templates, counter, mbarrier; returns the bytes
        const int bm_bytes = (groups + 4) * words * 4;  // interleaved, word stride groups + 4
        if (L.one) {  // bitmaps overlay the current tile (read into registers first)
            a.bm_off = a.cur_off;
            a.init_off = a.cur_off + ((std::max(TW * TH, bm_bytes) + 15) & ~15);
        } else {
            a.bm_off = a.cur_off + TW * TH;
            a.init_off = a.bm_off + ((bm_bytes + 15) & ~15);
        }
        // template words (initial bitmap, window border), tile counter, mbarrier (8-aligned),
        // the warps' statistics sums (NW x 3 x 8 bytes)
        return (size_t)((a.init_off + 8 * words + 4 + 7) & ~7) + 8 + 24 * L.NW;  // 2 templates
    };
    a.bmx = a.bmy = p;
    a.compact = 0;
    a.ovf = nullptr;
    a.rec = nullptr;
    a.rec_cap = 0;
    L.smem = layout(a.bm_words);
    // Compact visited set (B=16 ONE kernels): at +-32 the bitmaps (145 words per
    // group) hold the CTA to 4 per SM; a 51 x 45 window (bmx 24, bmy 20: 72 words) fits 5, and
    // 0.14 % of c4's searches leave it (tools/excursion.py, profiles/r2/excursion.json) -- the
    // overflow pass searches those again.  Used where it raises the CTAs per SM (the ONE
    // kernels' launch bound is 5); ME_COMPACT=0 disables it, ME_COMPACT=bmx,bmy forces a
    // window (tests: 4 <= bmx, 2 <= bmy, both <= p - 2).
    if (allow_compact && L.one && B == 16) {
        int cx = 0, cy = 0;
        const char* e = getenv("ME_COMPACT");
        if (e && sscanf(e, "%d,%d", &cx, &cy) == 2) {
            if (cx < 4 || cy < 2 || cx > p - 2 || cy > p - 2) cx = cy = 0;
        } else if (!(e && atoi(e) == 0) && p >= 26) {
            cx = std::min(24, p - 2);
            cy = std::min(20, p - 2);
            auto ctas = [](size_t b) { return std::min(5, g_smem_sm / ((int)b + 1024)); };
            if (ctas(layout(me::bm_nwords_xy(cx, cy))) <= ctas(L.smem)) cx = cy = 0;
        }
        if (cx > 0) {
            a.bmx = cx;
            a.bmy = cy;
            a.compact = 1;
            a.bm_words = me::bm_nwords_xy(cx, cy);
        }
        L.smem = layout(a.bm_words);
    }
    if (const char* e = getenv("ME_SMEM_PAD")) L.smem += (size_t)std::max(0, atoi(e));  // tuning only
    return L;
}

template <int B, int G, int VARIANT>
void launch_dcds_t(const DcdsLaunch& L, const CUtensorMap& tc, const CUtensorMap& tr, cudaStream_t s) {
    constexpr int DG = B == 16 ? 8 : 2, DNW = B == 16 ? 8 : 4;  // default geometry
    if constexpr (G == DG && B == 8) {
        if (L.one && L.NW == 8) {  // 8x8 blocks, 16x8 tiles of 8 warps (tuning: ME_NW=8 ME_TILE=16,8)
            me::dcds_kernel<8, 2, 8, VARIANT, false, true><<<L.grid, 256, L.smem, s>>>(tc, tr, L.a);
            return;
        }
    }
    if constexpr (G == DG) {
        if (L.one) {
            // the bench geometries (B=8: 16x4 tiles, +-16; B=16: 4x8 tiles, +-32) also exist
            // with the region pitch as a constant (immediate row offsets in the loads)
            constexpr int PC = B == 16 ? 176 : 192;
            if constexpr (B == 16) {
                if (L.a.compact) {  // the compact-visited-set builds (5 CTAs per SM)
                    if (L.a.pitch == PC)
                        me::dcds_kernel<B, G, DNW, VARIANT, false, true, PC, true><<<L.grid, DNW * 32, L.smem, s>>>(tc, tr, L.a);
                    else
                        me::dcds_kernel<B, G, DNW, VARIANT, false, true, 0, true><<<L.grid, DNW * 32, L.smem, s>>>(tc, tr, L.a);
                    return;
                }
            }
            if (L.a.pitch == PC)
                me::dcds_kernel<B, G, DNW, VARIANT, false, true, PC><<<L.grid, DNW * 32, L.smem, s>>>(tc, tr, L.a);
            else
                me::dcds_kernel<B, G, DNW, VARIANT, false, true><<<L.grid, DNW * 32, L.smem, s>>>(tc, tr, L.a);
            return;
        }
    }
    if (L.NW == 2) me::dcds_kernel<B, G, 2, VARIANT><<<L.grid, 64, L.smem, s>>>(tc, tr, L.a);
    else if (L.NW == 8) me::dcds_kernel<B, G, 8, VARIANT><<<L.grid, 256, L.smem, s>>>(tc, tr, L.a);
    else me::dcds_kernel<B, G, 4, VARIANT><<<L.grid, 128, L.smem, s>>>(tc, tr, L.a);
}

template <int B, int VARIANT>
void launch_dcds_b(const DcdsLaunch& L, const CUtensorMap& tc, const CUtensorMap& tr, cudaStream_t s) {
    if (L.G == 8) launch_dcds_t<B, 8, VARIANT>(L, tc, tr, s);
    else if (L.G == 2) launch_dcds_t<B, 2, VARIANT>(L, tc, tr, s);
    else if (B == 8 && L.G == 1) launch_dcds_t<8, 1, VARIANT>(L, tc, tr, s);
    else launch_dcds_t<B, 4, VARIANT>(L, tc, tr, s);
}

#define ME_DCDS_KERNELS(X) \
    X(16, 8, 0) X(16, 8, 1) X(16, 4, 0) X(16, 4, 1) X(16, 2, 0) X(16, 2, 1) X(8, 8, 0) X(8, 8, 1) \
    X(8, 4, 0) X(8, 4, 1) X(8, 2, 0) X(8, 2, 1) X(8, 1, 0) X(8, 1, 1)

// 3-D tiled tensor map over npairs frames (x = column, y = row, z = pair) for TMA.
int make_tmap(CUtensorMap* tm, const uint8_t* base, int W, int H, int npairs, long long stride,
              int box_w, int box_h) {
    if (!g_encode) return fail(ME_ECUDA, "cuTensorMapEncodeTiled unavailable");
    if (box_w > 256 || box_h > 256 || (box_w & 15)) return fail(ME_EINVAL, "TMA box too large");
    cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)npairs};
    cuuint64_t strides[2] = {(cuuint64_t)W, (cuuint64_t)(npairs > 1 ? stride : (long long)W * H)};
    cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(base), dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        snprintf(g_err, sizeof g_err, "cuTensorMapEncodeTiled failed (%d)", (int)r);
        return ME_ECUDA;
    }
    return ME_OK;
}

// Trace builds (me_dcds_trace_batch) exist for the default geometry only.
template <int B, int G, int NW>
void launch_dcds_trace(const DcdsLaunch& L, int variant, const CUtensorMap& tc, const CUtensorMap& tr,
                       cudaStream_t s) {
    if (L.one) {
        if (variant) me::dcds_kernel<B, G, NW, 1, true, true><<<L.grid, NW * 32, L.smem, s>>>(tc, tr, L.a);
        else me::dcds_kernel<B, G, NW, 0, true, true><<<L.grid, NW * 32, L.smem, s>>>(tc, tr, L.a);
    } else {
        if (variant) me::dcds_kernel<B, G, NW, 1, true><<<L.grid, NW * 32, L.smem, s>>>(tc, tr, L.a);
        else me::dcds_kernel<B, G, NW, 0, true><<<L.grid, NW * 32, L.smem, s>>>(tc, tr, L.a);
    }
}

int run_dcds(const uint8_t* cur0, const uint8_t* ref0, long long stride, int npairs, int W, int H,
             int block, int p, int16_t* mv, uint32_t* sad, uint16_t* pts, uint64_t* stats,
             int variant, cudaStream_t s, uint64_t* trace = nullptr, uint16_t* tlen = nullptr,
             int tcap = 0, bool packed = false) {
    // the compact visited set's overflow list holds 32-bit block indices
    const bool compact_ok = !trace && (long long)npairs * (W / block) * (H / block) < (1ll << 31);
    DcdsLaunch L = plan_dcds(W, H, block, p, npairs, compact_ok);
    if ((int)L.smem > g_smem_optin) return fail(ME_EINVAL, "tile does not fit in shared memory");
    // a call captured into a CUDA graph neither waits for nor records the ordering event (its
    // replays are ordered by the caller; an event recorded during capture cannot be waited on)
    bool capturing = false;
    if (L.a.compact) {
        L.a.ovf_cap = (uint32_t)((long long)npairs * L.a.nb);
        int rc = grow(&g_ovf, &g_ovf_cap, 4 * (4 + (size_t)L.a.ovf_cap));
        if (rc) return rc;
        L.a.ovf = reinterpret_cast<uint32_t*>(g_ovf);
        // warm-start records for the first 1/32 of the blocks (at least 64k) that reach the
        // interior overflow pass; later ones restart there from the window origin
        L.a.rec_cap = (int)std::min<long long>(L.a.ovf_cap, std::max<long long>(1 << 16, L.a.ovf_cap / 32));
        if (const char* e = getenv("ME_REC_CAP")) L.a.rec_cap = std::max(0, std::min(L.a.rec_cap, atoi(e)));  // tests
        if ((rc = grow(&g_rec, &g_rec_cap, 4 * (size_t)L.a.rec_cap * (2 + L.a.bm_words)))) return rc;
        L.a.rec = reinterpret_cast<uint32_t*>(g_rec);
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CK(cudaStreamIsCapturing(s, &cs));
        capturing = cs != cudaStreamCaptureStatusNone;
        if (!capturing && g_ovf_stream && g_ovf_stream != s) CK(cudaStreamWaitEvent(s, g_ovf_ev, 0));
        CK(cudaMemsetAsync(g_ovf, 0, 16, s));
    }
    g_ovf_used = L.a.compact != 0;
    if (trace && !(L.G == (block == 16 ? 8 : 2) && L.NW == (block == 16 ? 8 : 4)))
        return fail(ME_EINVAL, "trace builds exist for the default lane-group geometry only (unset ME_G/ME_NW)");
    L.a.trace = trace; L.a.tlen = tlen; L.a.tcap = tcap;
    L.a.packed = packed ? 1 : 0;
    L.a.cur0 = cur0; L.a.ref0 = ref0; L.a.stride = stride;
    L.a.mv = reinterpret_cast<uint32_t*>(mv);
    L.a.sad = sad;
    L.a.pts = pts;
    L.a.stats = reinterpret_cast<unsigned long long*>(stats);
    CUtensorMap tc, tr;
    int rc = make_tmap(&tc, cur0, W, H, npairs, stride, L.TW, L.TH);
    if (rc) return rc;
    rc = make_tmap(&tr, ref0, W, H, npairs, stride, L.a.pitch, L.a.rh);
    if (rc) return rc;
    if (stats) CK(cudaMemsetAsync(stats, 0, sizeof(uint64_t) * 3 * (size_t)npairs, s));
    if (trace) {
        if (block == 16) launch_dcds_trace<16, 8, 8>(L, variant, tc, tr, s);
        else launch_dcds_trace<8, 2, 4>(L, variant, tc, tr, s);
    } else if (block == 16) {
        if (variant) launch_dcds_b<16, 1>(L, tc, tr, s); else launch_dcds_b<16, 0>(L, tc, tr, s);
        if (L.a.compact) {
            // overflow passes (persistent grids): interior blocks from global memory (4 warps
            // per CTA, 8 CTAs per SM), border blocks staged (one warp per CTA)
            CK(cudaGetLastError());
            g_launches += 2;
            const int gs_ = me::redo_smem(16, 8, p, true, 4), bs_ = me::redo_smem(16, 8, p, false, 1);
            const dim3 gg(g_sms * 8), bg(g_sms * std::max(1, std::min(32, g_smem_sm / (bs_ + 1024))));
            if (variant) {
                me::dcds_redo_kernel<16, 8, 1, true><<<gg, 128, gs_, s>>>(L.a);
                me::dcds_redo_kernel<16, 8, 1, false><<<bg, 32, bs_, s>>>(L.a);
            } else {
                me::dcds_redo_kernel<16, 8, 0, true><<<gg, 128, gs_, s>>>(L.a);
                me::dcds_redo_kernel<16, 8, 0, false><<<bg, 32, bs_, s>>>(L.a);
            }
            CK(cudaGetLastError());
            if (!capturing) {
                CK(cudaEventRecord(g_ovf_ev, s));
                g_ovf_stream = s;
            }
        }
    } else {
        if (variant) launch_dcds_b<8, 1>(L, tc, tr, s); else launch_dcds_b<8, 0>(L, tc, tr, s);
    }
    g_launches++;
    CK(cudaGetLastError());
    return ME_OK;
}

// The comparison BMAs on the DCDS engine's default geometry.
template <int B, int G, int NW>
void launch_bma_b(int alg, dim3 grid, size_t smem, const CUtensorMap& tc, const CUtensorMap& tr,
                  const me::BmaArgs& a, cudaStream_t s) {
    switch (alg) {
        case me::ALG_CDS: me::bma_kernel<B, G, NW, me::ALG_CDS><<<grid, NW * 32, smem, s>>>(tc, tr, a); break;
        case me::ALG_DS: me::bma_kernel<B, G, NW, me::ALG_DS><<<grid, NW * 32, smem, s>>>(tc, tr, a); break;
        case me::ALG_HEXBS_H: me::bma_kernel<B, G, NW, me::ALG_HEXBS_H><<<grid, NW * 32, smem, s>>>(tc, tr, a); break;
        default: me::bma_kernel<B, G, NW, me::ALG_HEXBS_V><<<grid, NW * 32, smem, s>>>(tc, tr, a); break;
    }
}

int run_bma(int alg, const uint8_t* cur0, const uint8_t* ref0, long long stride, int npairs, int W,
            int H, int block, int p, int16_t* mv, uint32_t* sad, uint16_t* pts, uint64_t* stats,
            cudaStream_t s) {
    // the DCDS default geometry (B=8: G=2, 4 warps, 16x4 tiles; B=16: G=8, 8 warps, 4x8):
    // one block per lane group
    const int B = block, nbx = W / B, nby = H / B;
    const int G = B == 16 ? 8 : 2, NW = B == 16 ? 8 : 4;
    int tbx = std::min(B == 16 ? 4 : 16, nbx), tby = std::min(B == 16 ? 8 : 4, nby);
    while ((tbx * B) % 16) tbx++;
    me::BmaArgs a;
    a.cur0 = cur0; a.ref0 = ref0; a.stride = stride;
    a.W = W; a.H = H; a.p = p;
    a.tbx = tbx; a.tby = tby;
    const int ntx = (nbx + tbx - 1) / tbx, nty = (nby + tby - 1) / tby;
    const int TW = tbx * B, TH = tby * B;
    int pitch = ((TW + 2 * p + 31) + 15) & ~15;
    int p64 = pitch;  // the DCDS kernels' bank rule (plan_dcds)
    while ((p64 & 127) != 64) p64 += 16;
    if (B == 8 && p64 <= 256) pitch = p64;
    else if (((pitch >> 4) & 1) == 0) pitch += 16;
    a.pitch = pitch;
    a.rh = TH + 2 * p;
    a.bm_words = me::bm_nwords(p);
    a.nbx = nbx; a.nby = nby; a.nb = nbx * nby;
    a.mv = reinterpret_cast<uint32_t*>(mv); a.sad = sad; a.pts = pts;
    a.stats = reinterpret_cast<unsigned long long*>(stats);
    for (int r = 0; r < me::NROW; r++) a.rcode[r] = me::row_code(r);
    const int groups = NW * 32 / G;
    a.cur_off = (pitch * a.rh + 127) & ~127;  // no slack needed (see plan_dcds)
    a.init_off = a.cur_off + ((std::max(TW * TH, (groups + 4) * a.bm_words * 4) + 15) & ~15);
    // template words | row offsets (int4, 16-aligned) | row codes | mbarrier (8-aligned) |
    // the warps' statistics sums (NW x 3 x 8 bytes)
    const size_t tables = (size_t)((a.init_off + 4 * a.bm_words + 15) & ~15) + 16 * me::NROW + 4 * (me::NROW + (me::NROW & 1));
    const size_t smem = tables + 8 + 24 * NW;
    if ((int)smem > g_smem_optin) return fail(ME_EINVAL, "tile does not fit in shared memory");
    CUtensorMap tc, tr;
    int rc = make_tmap(&tc, cur0, W, H, npairs, stride, TW, TH);
    if (rc) return rc;
    rc = make_tmap(&tr, ref0, W, H, npairs, stride, a.pitch, a.rh);
    if (rc) return rc;
    if (stats) CK(cudaMemsetAsync(stats, 0, sizeof(uint64_t) * 3 * (size_t)npairs, s));
    const dim3 grid(ntx, nty, npairs);
    if (B == 16) launch_bma_b<16, 8, 8>(alg, grid, smem, tc, tr, a, s);
    else launch_bma_b<8, 2, 4>(alg, grid, smem, tc, tr, a, s);
    g_launches++;
    CK(cudaGetLastError());
    return ME_OK;
}

int run_fs(const uint8_t* cur0, const uint8_t* ref0, long long stride, int npairs, int W, int H,
           int block, int p, int16_t* mv, uint32_t* sad, uint16_t* pts, uint64_t* stats,
           cudaStream_t s) {
    me::FsArgs a;
    const int B = block, nbx = W / B, nby = H / B, side = 2 * p + 1;
    a.W = W; a.H = H; a.p = p;
    a.nch = (side + B - 1) / B;
    // tile (measured on B200, profiles/r1b/SUMMARY.md): 8x4 blocks for B=8, 4x4 for B=16,
    // halved while the region exceeds the 256 x 256 TMA box or its 4 byte-phase copies exceed
    // the shared memory of a CTA
    int tbx = B == 16 ? 4 : 8, tby = 4;
    auto fs_smem = [&](int tx, int ty) {
        const int pt = ((tx * B + 2 * p + 31) + 15) & ~15;
        const int nd = side - (a.nch - 1) * B;
        const int rp = 2 * nd <= B ? ty * B + 2 * p : std::max(ty * B + 2 * p, (ty + a.nch) * B - 1);
        return 4 * ((pt * rp + 127 + 128 * 4) & ~127) + tx * ty * B * B + 1024;
    };
    while ((tbx > 1 || tby > 1) &&
           (tbx * B + 2 * p + 31 > 256 || tby * B + 2 * p > 256 || fs_smem(tbx, tby) > g_smem_optin - 1024)) {
        if (tbx >= tby && tbx > 1) tbx /= 2;
        else tby /= 2;
    }
    if (const char* e = getenv("ME_FS_TILE")) {
        int tx = 0, ty = 0;
        if (sscanf(e, "%d,%d", &tx, &ty) == 2 && tx > 0 && ty > 0) { tbx = tx; tby = ty; }
    }
    tbx = std::min(tbx, nbx);
    tby = std::min(tby, nby);
    if ((tbx * B) % 16) tbx = std::min(nbx, ((tbx * B + 15) / 16) * 16 / B);
    a.tbx = tbx; a.tby = tby;
    a.ntx = (nbx + tbx - 1) / tbx;
    const int nty = (nby + tby - 1) / tby;
    const int TW = tbx * B, TH = tby * B;
    a.pitch = ((TW + 2 * p + 31) + 15) & ~15;
    a.rh = TH + 2 * p;
    // a last dy chunk of <= B/2 candidates is scored candidate by candidate and touches rows
    // < rh only; a fuller one runs as a full chunk over padding rows
    const int nd_last = side - (a.nch - 1) * B;
    a.rh_pad = 2 * nd_last <= B ? a.rh : std::max(a.rh, (tby + a.nch) * B - 1);
    // measured on B200 (profiles/r1b): 8x8 blocks keep a (block, dx) item whole; 16x16 blocks
    // (64 cur registers, 16 accumulators per item) split it into one item per dy chunk
    a.nsplit = B == 16 ? a.nch : 1;
    if (const char* e = getenv("ME_FS_SPLIT")) a.nsplit = std::max(1, std::min(a.nch, atoi(e)));
    const int rbytes = a.pitch * a.rh_pad;
    // copy stride: >= region, 128-aligned copy 0, stride/4 = 8 (mod 32) words spreads the copies
    int cs = (rbytes + 127) & ~127;
    while (((cs / 4) & 31) != 8) cs += 16;
    a.cstride = cs;
    a.cur_off = (4 * cs + 127) & ~127;
    a.nbx = nbx; a.nb = nbx * nby;
    a.mv = reinterpret_cast<uint32_t*>(mv); a.sad = sad; a.pts = pts;
    a.stats = reinterpret_cast<unsigned long long*>(stats);
    const size_t smem = 128 + (size_t)a.cur_off + (size_t)TW * TH;
    if ((int)smem > g_smem_optin - 1024) return fail(ME_EINVAL, "FS tile does not fit in shared memory");
    if (tbx * tby > 64) return fail(ME_EINVAL, "FS tile too large");
    CUtensorMap tc, tr;
    int rc = make_tmap(&tc, cur0, W, H, npairs, stride, TW, TH);
    if (rc) return rc;
    rc = make_tmap(&tr, ref0, W, H, npairs, stride, a.pitch, a.rh);
    if (rc) return rc;
    if (stats) CK(cudaMemsetAsync(stats, 0, sizeof(uint64_t) * 3 * (size_t)npairs, s));
    dim3 grid(a.ntx * nty, npairs);
    int nthr = 256;
    if (const char* e = getenv("ME_FS_THREADS")) {  // tuning only
        const int t = atoi(e);
        if (t >= 64 && t <= 512 && t % 32 == 0) nthr = t;
    }
    // column-sweep builds (fs_kernel SIDE) for the bench geometries: 8x8 / +-16 (c3) with 4
    // warps per CTA, 16x16 / +-32 (c4) with 8 (measured on B200, 32 pairs: c3 1.375 ms vs 1.59
    // chunked, c4 18.38 vs 20.10 ms); ME_FS_SWEEP=0 selects the chunked kernel
    const char* sw = getenv("ME_FS_SWEEP");
    const bool sweep = !(sw && atoi(sw) == 0);
    if (sweep && block == 8 && p == 16 && a.pitch == 128 && a.nsplit == 1) {
        if (!getenv("ME_FS_THREADS")) nthr = 128;
        me::fs_kernel<8, 33, 128><<<grid, nthr, smem, s>>>(tc, tr, a);
    } else if (sweep && block == 16 && p == 32 && a.pitch == 160 && !getenv("ME_FS_SPLIT")) {
        a.nsplit = 1;  // one item per (block, dx): the whole column
        me::fs_kernel<16, 65, 160><<<grid, nthr, smem, s>>>(tc, tr, a);
    } else if (block == 16) {
        me::fs_kernel<16><<<grid, nthr, smem, s>>>(tc, tr, a);
    } else {
        me::fs_kernel<8><<<grid, nthr, smem, s>>>(tc, tr, a);
    }
    g_launches++;
    CK(cudaGetLastError());
    return ME_OK;
}

int run_mc_sse(const uint8_t* cur0, const uint8_t* ref0, long long stride, int npairs, int W,
               int H, int block, const int16_t* mv, uint64_t* sse, cudaStream_t s) {
    // frames of at least one DCDS tile: the TMA-staged kernel (the DCDS tile geometry with a
    // fixed halo; larger MVs fall back to clamped global reads inside it); otherwise the
    // warp-per-block kernel
    if (!getenv("ME_MC_LEGACY")) {
        const int hp = block == 16 ? 32 : 16;
        DcdsLaunch L = plan_dcds(W, H, block, hp, npairs);
        if (L.TW == (block == 16 ? 4 : 16) * block && L.TH == (block == 16 ? 8 : 4) * block) {
            L.a.cur0 = cur0; L.a.ref0 = ref0; L.a.stride = stride;
            L.a.stats = reinterpret_cast<unsigned long long*>(sse);
            const size_t smem = (size_t)((L.a.cur_off + L.TW * L.TH + 7) & ~7) + 16;
            CUtensorMap tc, tr;
            int rc = make_tmap(&tc, cur0, W, H, npairs, stride, L.TW, L.TH);
            if (rc) return rc;
            rc = make_tmap(&tr, ref0, W, H, npairs, stride, L.a.pitch, L.a.rh);
            if (rc) return rc;
            CK(cudaMemsetAsync(sse, 0, sizeof(uint64_t) * (size_t)npairs, s));
            const uint32_t* mvf = reinterpret_cast<const uint32_t*>(mv);
            // measured (tools/gpu_mc.sh): 128 threads for 8x8 blocks (c3 0.318 ms vs 0.361 at 256), 256 for
            // 16x16 (c4 4.99 ms vs 5.74 at 128)
            const int nt = getenv("ME_MC_THREADS") ? atoi(getenv("ME_MC_THREADS")) : (block == 16 ? 256 : 128);
            if (block == 16) me::mc_sse_tma_kernel<16><<<L.grid, nt, smem, s>>>(tc, tr, L.a, mvf);
            else me::mc_sse_tma_kernel<8><<<L.grid, nt, smem, s>>>(tc, tr, L.a, mvf);
            g_launches++;
            CK(cudaGetLastError());
            return ME_OK;
        }
    }
    me::McArgs a;
    a.cur0 = cur0; a.ref0 = ref0; a.stride = stride;
    a.W = W; a.H = H; a.B = block;
    a.nbx = W / block; a.nb = a.nbx * (H / block);
    a.mv = reinterpret_cast<const uint32_t*>(mv);
    a.sse = reinterpret_cast<unsigned long long*>(sse);
    CK(cudaMemsetAsync(sse, 0, sizeof(uint64_t) * (size_t)npairs, s));
    const int per_cta = 8 * (32 / block);  // 8 warps, 32 / B blocks per warp
    dim3 grid((a.nb + per_cta - 1) / per_cta, npairs);
    if (block == 16) me::mc_sse_kernel<16><<<grid, 256, 0, s>>>(a);
    else me::mc_sse_kernel<8><<<grid, 256, 0, s>>>(a);
    g_launches++;
    CK(cudaGetLastError());
    return ME_OK;
}

template <typename K>
int allow_smem(K kernel) {
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, kernel));
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            g_smem_optin - (int)fa.sharedSizeBytes));
    return ME_OK;
}

int grow(uint8_t** p, size_t* cap, size_t need) {
    if (*cap >= need) return ME_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    if (cudaMalloc(p, need) != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return fail(ME_ENOMEM, "staging buffer allocation failed");
    }
    *cap = need;
    return ME_OK;
}

}  // namespace

extern "C" {

int me_init(int device) {
    if (g_dev == device) return ME_OK;
    // a different device: release the previous device's streams, scratch and staging first,
    // so nothing of one device is used on another
    if (g_dev >= 0) me_shutdown();
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) return fail(ME_EINVAL, "no such CUDA device");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        snprintf(g_err, sizeof g_err, "device %d is sm_%d%d; libme.so is built for sm_100a only",
                 device, prop.major, prop.minor);
        return ME_ECUDA;
    }
    g_smem_optin = (int)prop.sharedMemPerBlockOptin;
    g_smem_sm = (int)prop.sharedMemPerMultiprocessor;
    g_sms = prop.multiProcessorCount;
    int rc;
#define ME_ALLOW(B, G, V) \
    if ((rc = allow_smem(me::dcds_kernel<B, G, 2, V>))) return rc;             \
    if ((rc = allow_smem(me::dcds_kernel<B, G, 4, V>))) return rc;             \
    if ((rc = allow_smem(me::dcds_kernel<B, G, 8, V>))) return rc;
    ME_DCDS_KERNELS(ME_ALLOW)
#undef ME_ALLOW
    if ((rc = allow_smem(me::dcds_kernel<8, 2, 4, 0, false, true, 192>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<8, 2, 4, 1, false, true, 192>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<16, 8, 8, 0, false, true, 176>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<16, 8, 8, 1, false, true, 176>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<8, 2, 4, 0, false, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<8, 2, 8, 0, false, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<8, 2, 8, 1, false, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<8, 2, 4, 1, false, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<16, 8, 8, 0, false, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<16, 8, 8, 1, false, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<16, 8, 8, 0, false, true, 176, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<16, 8, 8, 1, false, true, 176, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<16, 8, 8, 0, false, true, 0, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<16, 8, 8, 1, false, true, 0, true>))) return rc;
    if ((rc = allow_smem(me::dcds_redo_kernel<16, 8, 0, true>))) return rc;
    if ((rc = allow_smem(me::dcds_redo_kernel<16, 8, 1, true>))) return rc;
    if ((rc = allow_smem(me::dcds_redo_kernel<16, 8, 0, false>))) return rc;
    if ((rc = allow_smem(me::dcds_redo_kernel<16, 8, 1, false>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<8, 2, 4, 0, true, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<8, 2, 4, 1, true, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<16, 8, 8, 0, true, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<16, 8, 8, 1, true, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<8, 2, 4, 0, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<8, 2, 4, 1, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<16, 8, 8, 0, true>))) return rc;
    if ((rc = allow_smem(me::dcds_kernel<16, 8, 8, 1, true>))) return rc;
#define ME_ALLOW_BMA(B, G, NW)                                                           \
    if ((rc = allow_smem(me::bma_kernel<B, G, NW, me::ALG_CDS>))) return rc;            \
    if ((rc = allow_smem(me::bma_kernel<B, G, NW, me::ALG_DS>))) return rc;             \
    if ((rc = allow_smem(me::bma_kernel<B, G, NW, me::ALG_HEXBS_H>))) return rc;        \
    if ((rc = allow_smem(me::bma_kernel<B, G, NW, me::ALG_HEXBS_V>))) return rc;
    ME_ALLOW_BMA(8, 2, 4)
    ME_ALLOW_BMA(16, 8, 8)
#undef ME_ALLOW_BMA
    if ((rc = allow_smem(me::mc_sse_tma_kernel<16>))) return rc;
    if ((rc = allow_smem(me::mc_sse_tma_kernel<8>))) return rc;
    if ((rc = allow_smem(me::fs_kernel<16>))) return rc;
    if ((rc = allow_smem(me::fs_kernel<8>))) return rc;
    if ((rc = allow_smem(me::fs_kernel<8, 33, 128>))) return rc;
    if ((rc = allow_smem(me::fs_kernel<16, 65, 160>))) return rc;
    if (!g_scratch) CK(cudaMalloc(&g_scratch, 64));
    {  // visited-bitmap templates for every p (dcds_kernel.cuh, bm_template_word)
        static uint32_t tmpl[me::BM_TMPL_WORDS];
        for (int q = 1; q <= 32; q++) {
            const int nw = me::bm_nwords(q), off = me::bm_tmpl_off(q);
            for (int t = 0; t < nw; t++) {
                tmpl[off + t] = me::bm_template_word(q, t, false);
                tmpl[off + nw + t] = me::bm_template_word(q, t, true);
            }
        }
        CK(cudaMemcpyToSymbol(me::c_bm_tmpl, tmpl, sizeof tmpl));
    }
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&g_encode),
                                   cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess) return fail(ME_ECUDA, "cuTensorMapEncodeTiled not found");
    }
    for (auto& cs : g_copy_streams)
        if (!cs) CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    if (!g_order_ev) CK(cudaEventCreateWithFlags(&g_order_ev, cudaEventDisableTiming));
    if (!g_ovf_ev) CK(cudaEventCreateWithFlags(&g_ovf_ev, cudaEventDisableTiming));
    for (auto& st : g_stage) {  // me_dcds_batch_host staging: allocated here, not per call
        if ((rc = grow(&st.frames, &st.frames_cap, (size_t)kStageFrames))) return rc;
        if ((rc = grow(&st.out, &st.out_cap, (size_t)kStageFrames / 4))) return rc;  // >= outputs of a full chunk
    }
    g_dev = device;
    g_launches = 0;
    return ME_OK;
}

int me_set_stream(void* stream) {
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    g_stream = reinterpret_cast<cudaStream_t>(stream);
    return ME_OK;
}

int me_dcds_batch(const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride, int npairs, int W,
                  int H, int block, int p, int16_t* mv_out, uint32_t* sad_out,
                  uint16_t* points_out, uint64_t* stats_out) {
    int rc = validate_search(cur0, ref0, pair_stride, npairs, W, H, block, p, mv_out, sad_out,
                             points_out);
    if (rc) return rc;
    if (stats_out && !aligned(stats_out, 8)) return fail(ME_EALIGN, "stats_out must be 8-byte aligned");
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    return run_dcds(cur0, ref0, pair_stride, npairs, W, H, block, p, mv_out, sad_out, points_out,
                    stats_out, 0, g_stream);
}

int me_dcds_s_batch(const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride, int npairs,
                    int W, int H, int block, int p, int16_t* mv_out, uint32_t* sad_out,
                    uint16_t* points_out, uint64_t* stats_out) {
    int rc = validate_search(cur0, ref0, pair_stride, npairs, W, H, block, p, mv_out, sad_out,
                             points_out);
    if (rc) return rc;
    if (stats_out && !aligned(stats_out, 8)) return fail(ME_EALIGN, "stats_out must be 8-byte aligned");
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    return run_dcds(cur0, ref0, pair_stride, npairs, W, H, block, p, mv_out, sad_out, points_out,
                    stats_out, 1, g_stream);
}

int me_dcds_batch_packed(const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride, int npairs,
                         int W, int H, int block, int p, int8_t* mv_out, uint16_t* sad_out,
                         uint16_t* points_out, uint64_t* stats_out) {
    int rc = validate_frames(cur0, ref0, pair_stride, npairs, W, H, block);
    if (rc) return rc;
    if (p < 1 || p > 32) return fail(ME_EINVAL, "p must be in [1, 32]");
    if (!mv_out || !sad_out || !points_out) return fail(ME_EINVAL, "NULL output pointer");
    if (!aligned(mv_out, 2) || !aligned(sad_out, 2) || !aligned(points_out, 2))
        return fail(ME_EALIGN, "packed outputs must be 2-byte aligned");
    if (stats_out && !aligned(stats_out, 8)) return fail(ME_EALIGN, "stats_out must be 8-byte aligned");
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    return run_dcds(cur0, ref0, pair_stride, npairs, W, H, block, p,
                    reinterpret_cast<int16_t*>(mv_out), reinterpret_cast<uint32_t*>(sad_out), points_out,
                    stats_out, 0, g_stream, nullptr, nullptr, 0, true);
}

int me_dcds_trace_batch(int variant, const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride,
                        int npairs, int W, int H, int block, int p, int16_t* mv_out,
                        uint32_t* sad_out, uint16_t* points_out, uint64_t* trace_out, int trace_cap,
                        uint16_t* trace_len_out) {
    if (variant != 0 && variant != 1) return fail(ME_EINVAL, "variant must be 0 (DCDS) or 1 (DCDS^S)");
    int rc = validate_search(cur0, ref0, pair_stride, npairs, W, H, block, p, mv_out, sad_out,
                             points_out);
    if (rc) return rc;
    if (trace_cap < 1 || trace_cap > 255) return fail(ME_EINVAL, "trace_cap must be in [1, 255]");
    if (!trace_out || !trace_len_out) return fail(ME_EINVAL, "NULL trace pointer");
    if (!aligned(trace_out, 8) || !aligned(trace_len_out, 2))
        return fail(ME_EALIGN, "trace_out must be 8-byte aligned, trace_len_out 2-byte");
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    return run_dcds(cur0, ref0, pair_stride, npairs, W, H, block, p, mv_out, sad_out, points_out,
                    nullptr, variant, g_stream, trace_out, trace_len_out, trace_cap);
}

int me_bma_batch(int alg, const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride, int npairs,
                 int W, int H, int block, int p, int16_t* mv_out, uint32_t* sad_out,
                 uint16_t* points_out, uint64_t* stats_out) {
    if (alg < ME_ALG_DCDS || alg > ME_ALG_HEXBS_V) return fail(ME_EINVAL, "unknown algorithm id");
    int rc = validate_search(cur0, ref0, pair_stride, npairs, W, H, block, p, mv_out, sad_out,
                             points_out);
    if (rc) return rc;
    if (stats_out && !aligned(stats_out, 8)) return fail(ME_EALIGN, "stats_out must be 8-byte aligned");
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    if (alg <= ME_ALG_DCDS_S)
        return run_dcds(cur0, ref0, pair_stride, npairs, W, H, block, p, mv_out, sad_out, points_out,
                        stats_out, alg, g_stream);
    return run_bma(alg, cur0, ref0, pair_stride, npairs, W, H, block, p, mv_out, sad_out, points_out,
                   stats_out, g_stream);
}

int me_ideal_nsp_map(int alg, int p, int32_t* nsp_out, int32_t* mvx_out, int32_t* mvy_out) {
    if (alg < ME_ALG_DCDS || alg > ME_ALG_HEXBS_V) return fail(ME_EINVAL, "unknown algorithm id");
    if (p < 1 || p > 32) return fail(ME_EINVAL, "p must be in [1, 32]");
    if (!nsp_out) return fail(ME_EINVAL, "NULL nsp_out");
    if (!aligned(nsp_out, 4) || (mvx_out && !aligned(mvx_out, 4)) || (mvy_out && !aligned(mvy_out, 4)))
        return fail(ME_EALIGN, "int32 outputs must be 4-byte aligned");
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    me::IdealArgs a;
    a.alg = alg; a.p = p; a.nsp = nsp_out; a.mvx = mvx_out; a.mvy = mvy_out;
    for (int r = 0; r < me::NROW_ALL; r++) a.rcode[r] = me::any_row_code(r);
    const int n = (2 * p + 1) * (2 * p + 1);
    me::ideal_kernel<<<(n + 127) / 128, 128, 0, g_stream>>>(a);
    g_launches++;
    CK(cudaGetLastError());
    return ME_OK;
}

int me_mv_hist(const int16_t* mv, int64_t n, int p, uint64_t* hist_out) {
    if ((!mv && n > 0) || !hist_out) return fail(ME_EINVAL, "NULL pointer");
    if (n < 0 || p < 1 || p > 32) return fail(ME_EINVAL, "bad n / p");
    if (!aligned(mv, 4) || !aligned(hist_out, 8)) return fail(ME_EALIGN, "misaligned pointer");
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    const int nbin = (2 * p + 1) * (2 * p + 1);
    CK(cudaMemsetAsync(hist_out, 0, sizeof(uint64_t) * nbin, g_stream));
    if (n > 0) {
        const long long want = (n + 255) / 256;
        const int grid = (int)std::min<long long>(want, 4 * 148);
        me::mv_hist_kernel<<<grid, 256, nbin * sizeof(unsigned int), g_stream>>>(
            reinterpret_cast<const uint32_t*>(mv), n, p, reinterpret_cast<unsigned long long*>(hist_out));
        g_launches++;
    }
    CK(cudaGetLastError());
    return ME_OK;
}

int me_dcds(const uint8_t* cur, const uint8_t* ref, int W, int H, int block, int p,
            int16_t* mv_out, uint32_t* sad_out, uint16_t* points_out) {
    return me_dcds_batch(cur, ref, 0, 1, W, H, block, p, mv_out, sad_out, points_out, nullptr);
}

int me_fullsearch_batch(const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride, int npairs,
                        int W, int H, int block, int p, int16_t* mv_out, uint32_t* sad_out,
                        uint16_t* points_out, uint64_t* stats_out) {
    int rc = validate_search(cur0, ref0, pair_stride, npairs, W, H, block, p, mv_out, sad_out,
                             points_out);
    if (rc) return rc;
    if (stats_out && !aligned(stats_out, 8)) return fail(ME_EALIGN, "stats_out must be 8-byte aligned");
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    return run_fs(cur0, ref0, pair_stride, npairs, W, H, block, p, mv_out, sad_out, points_out,
                  stats_out, g_stream);
}

int me_fullsearch(const uint8_t* cur, const uint8_t* ref, int W, int H, int block, int p,
                  int16_t* mv_out, uint32_t* sad_out, uint16_t* points_out) {
    return me_fullsearch_batch(cur, ref, 0, 1, W, H, block, p, mv_out, sad_out, points_out,
                               nullptr);
}

int me_mc_sse_batch(const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride, int npairs,
                    int W, int H, int block, const int16_t* mv, uint64_t* sse_out) {
    int rc = validate_frames(cur0, ref0, pair_stride, npairs, W, H, block);
    if (rc) return rc;
    if (!mv || !sse_out) return fail(ME_EINVAL, "NULL mv / sse pointer");
    if (!aligned(mv, 4) || !aligned(sse_out, 8)) return fail(ME_EALIGN, "mv / sse_out misaligned");
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    return run_mc_sse(cur0, ref0, pair_stride, npairs, W, H, block, mv, sse_out, g_stream);
}

int me_mc_psnr(const uint8_t* cur, const uint8_t* ref, int W, int H, int block, const int16_t* mv,
               double* psnr_out, uint64_t* sse_out) {
    int rc = validate_frames(cur, ref, 0, 1, W, H, block);
    if (rc) return rc;
    if (!mv || !psnr_out) return fail(ME_EINVAL, "NULL mv / psnr pointer");
    if (!aligned(mv, 4)) return fail(ME_EALIGN, "mv must be 4-byte aligned");
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    rc = run_mc_sse(cur, ref, 0, 1, W, H, block, mv, reinterpret_cast<uint64_t*>(g_scratch), g_stream);
    if (rc) return rc;
    unsigned long long sse = 0;
    CK(cudaMemcpyAsync(&sse, g_scratch, sizeof sse, cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    if (sse_out) *sse_out = sse;
    // PSNR of the compensated frame (P:342 aspect 4; reading C18)
    *psnr_out = sse == 0 ? INFINITY : 10.0 * log10((255.0 * 255.0) * ((double)W * H) / (double)sse);
    return ME_OK;
}

int me_quality_batch(const int16_t* mv, const int16_t* mv_fs, int npairs, int nb, double* out) {
    if (!mv || !mv_fs || !out) return fail(ME_EINVAL, "NULL pointer");
    if (npairs < 1 || nb < 1 || npairs > 65535) return fail(ME_EINVAL, "bad npairs / nb");
    if (!aligned(mv, 4) || !aligned(mv_fs, 4) || !aligned(out, 8)) return fail(ME_EALIGN, "misaligned pointer");
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    me::quality_kernel<<<npairs, 256, 0, g_stream>>>(reinterpret_cast<const uint32_t*>(mv),
                                                     reinterpret_cast<const uint32_t*>(mv_fs), nb, out);
    g_launches++;
    CK(cudaGetLastError());
    return ME_OK;
}

int me_dcds_batch_host(const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride, int npairs,
                       int W, int H, int block, int p, int16_t* mv_out, uint32_t* sad_out,
                       uint16_t* points_out, uint64_t* stats_out) {
    if (!cur0 || !ref0) return fail(ME_EINVAL, "NULL frame pointer");
    if (npairs > 1 && pair_stride < (long long)W * H) return fail(ME_EINVAL, "pair_stride smaller than a frame");
    // host pointers: alignment of the device staging copy is what the kernels need
    int rc = validate_search(reinterpret_cast<const uint8_t*>(16), reinterpret_cast<const uint8_t*>(16),
                             16 * (((long long)W * H + 15) / 16), npairs, W, H, block, p, mv_out, sad_out,
                             points_out);
    if (rc) return rc;
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    // device staging layout per chunk: [n][cur | ref], each frame W*H bytes, pair stride
    // 2*W*H (a multiple of 16: W % 16 == 0).  cur and ref are copied separately, so the two
    // host frames of a pair may be unrelated buffers.
    const long long fsz = (long long)W * H, dstride = 2 * fsz;
    const long long hstride = npairs > 1 ? pair_stride : fsz;  // host pitch (unused for one pair)
    const int nb = (W / block) * (H / block);
    const int chunk = (int)std::max(1ll, std::min<long long>(npairs, (long long)kStageFrames / dstride));
    const size_t fbytes = (size_t)dstride * chunk;
    const size_t obytes = (size_t)chunk * nb * (4 + 4 + 2) + (size_t)chunk * 24 + 64;
    for (auto& st : g_stage) {  // pre-allocated by me_init; grows only for frames > kStageFrames
        if ((rc = grow(&st.frames, &st.frames_cap, fbytes))) return rc;
        if ((rc = grow(&st.out, &st.out_cap, obytes))) return rc;
    }
    // order the copies after whatever the caller queued on the library stream
    CK(cudaEventRecord(g_order_ev, g_stream));
    for (auto cs : g_copy_streams) CK(cudaStreamWaitEvent(cs, g_order_ev, 0));
    auto body = [&]() -> int {
        for (int c0 = 0, ci = 0; c0 < npairs; c0 += chunk, ci++) {
            const int n = std::min(chunk, npairs - c0);
            HostStage& st = g_stage[ci & 1];
            cudaStream_t s = g_copy_streams[ci & 1];
            // n frames of W*H bytes at host pitch hstride -> device pitch 2*W*H
            CK(cudaMemcpy2DAsync(st.frames, (size_t)dstride, cur0 + (size_t)c0 * hstride, (size_t)hstride,
                                 (size_t)fsz, (size_t)n, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpy2DAsync(st.frames + fsz, (size_t)dstride, ref0 + (size_t)c0 * hstride, (size_t)hstride,
                                 (size_t)fsz, (size_t)n, cudaMemcpyHostToDevice, s));
            int16_t* dmv = reinterpret_cast<int16_t*>(st.out);
            uint32_t* dsad = reinterpret_cast<uint32_t*>(st.out + (size_t)n * nb * 4);
            uint64_t* dst = reinterpret_cast<uint64_t*>(st.out + (((size_t)n * nb * 8 + 7) & ~(size_t)7));
            uint16_t* dpts = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(dst) + (size_t)n * 24);
            int r = run_dcds(st.frames, st.frames + fsz, dstride, n, W, H, block, p, dmv, dsad, dpts, dst, 0, s);
            if (r) return r;
            CK(cudaMemcpyAsync(mv_out + (size_t)c0 * nb * 2, dmv, (size_t)n * nb * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(sad_out + (size_t)c0 * nb, dsad, (size_t)n * nb * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(points_out + (size_t)c0 * nb, dpts, (size_t)n * nb * 2, cudaMemcpyDeviceToHost, s));
            if (stats_out)
                CK(cudaMemcpyAsync(stats_out + (size_t)c0 * 3, dst, (size_t)n * 24, cudaMemcpyDeviceToHost, s));
        }
        return ME_OK;
    };
    rc = body();
    // always drain both copy streams: on an error no copy may still be reading or writing the
    // caller's buffers when this returns
    for (auto cs : g_copy_streams) {
        const cudaError_t e = cudaStreamSynchronize(cs);
        if (e != cudaSuccess && rc == ME_OK) rc = set_cuda_err(e, "cudaStreamSynchronize(copy stream)");
    }
    return rc;
}

int64_t me_launch_count(void) { return g_launches; }

int me_dcds_overflow_count(uint64_t* count_out) {
    if (!count_out) return fail(ME_EINVAL, "NULL count_out");
    if (g_dev < 0) return fail(ME_ENOTINIT, "me_init has not succeeded");
    uint32_t c[2] = {0, 0};  // interior + border blocks
    if (g_ovf_used) {
        CK(cudaEventSynchronize(g_ovf_ev));
        CK(cudaMemcpy(c, g_ovf, 8, cudaMemcpyDeviceToHost));
    }
    *count_out = (uint64_t)c[0] + c[1];
    return ME_OK;
}

const char* me_strerror(int status) {
    switch (status) {
        case ME_OK: return "ok";
        case ME_EINVAL: return g_err[0] ? g_err : "invalid argument";
        case ME_EALIGN: return g_err[0] ? g_err : "misaligned argument";
        case ME_ENOTINIT: return "me_init has not succeeded";
        case ME_ECUDA: return g_err[0] ? g_err : "CUDA error";
        case ME_ENOMEM: return g_err[0] ? g_err : "out of device memory";
        default: return "unknown status";
    }
}

void me_shutdown(void) {
    if (g_dev < 0) return;
    for (auto& st : g_stage) {
        if (st.frames) cudaFree(st.frames);
        if (st.out) cudaFree(st.out);
        st = HostStage();
    }
    if (g_scratch) cudaFree(g_scratch);
    g_scratch = nullptr;
    if (g_ovf) cudaFree(g_ovf);
    g_ovf = nullptr;
    g_ovf_cap = 0;
    if (g_rec) cudaFree(g_rec);
    g_rec = nullptr;
    g_rec_cap = 0;
    g_ovf_used = false;
    if (g_ovf_ev) cudaEventDestroy(g_ovf_ev);
    g_ovf_ev = nullptr;
    g_ovf_stream = nullptr;
    for (auto& cs : g_copy_streams) {
        if (cs) cudaStreamDestroy(cs);
        cs = nullptr;
    }
    if (g_order_ev) cudaEventDestroy(g_order_ev);
    g_order_ev = nullptr;
    g_stream = nullptr;
    g_dev = -1;
}

}  // extern "C"
