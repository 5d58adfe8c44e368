/*
 * me.h -- C ABI of libme.so, the B200 (sm_100a) DCDS block-motion-estimation hot path.
 *
 * Paper: Jia & Zhang, "Directional Cross Diamond Search Algorithm for Fast Block Motion
 * Estimation" (arxiv 0806.0689); P:n = PAPER.md line n.  DESIGN.md states the readings.
 *
 * Problem statement: "The frame is partitioned into non-overlapping and equal-sized
 * blocks (8x8) or macroblocks (16x16) ... the motion vector is obtained by finding out the
 * displacement of the best-matched block in the reference frame ... within the search window
 * centered around the original position.  Matching process is performed by minimizing a
 * certain matching criterion."
 *
 * Common conventions (every entry point):
 *   - Frames are 8-bit luma, row-major, pitch = W bytes.  W % block == 0, H % block == 0,
 *     block in {8, 16}; W % 16 == 0 and every frame/base pointer 16-byte aligned
 *     (vectorised loads) -- else ME_EALIGN.
 *   - Blocks are numbered in raster order; nb = (W/block) * (H/block).
 *   - MV convention: cur block at (bx,by) matches ref at (bx+dx, by+dy).  mv arrays hold
 *     int16 pairs (dx, dy) per block ([nb][2]).
 *   - Candidates are limited to |dx|,|dy| <= p with 1 <= p <= 32.  Reference pixels outside
 *     the frame read the edge-replicated reference ref[clamp(y)][clamp(x)] (reading C9), so
 *     every window candidate is scorable.
 *   - SAD = sum over the block of |cur - ref| (integer; the paper's MAD times block^2,
 *     P:342; reading C12).  Ties keep the incumbent; among new points the first in the fixed
 *     pattern order wins (readings C6, C7; FS: centre first then raster, C13).
 *   - Pointers are DEVICE pointers unless marked (host).  The caller owns every buffer and
 *     keeps inputs alive until the stream completes; the library allocates nothing per call
 *     (the _host variant keeps grow-only staging buffers, freed by me_shutdown).
 *   - All launches are asynchronous on the stream set by me_set_stream (default: the legacy
 *     default stream) unless the entry point says it synchronises.
 *   - Errors: a negative me_status; arguments are validated before any device work, and no
 *     partial outputs are promised after an error.  CUDA errors map to ME_ECUDA and
 *     me_strerror() returns the detail of the last error.  Not thread-safe: one host thread
 *     drives the library per process.  There is no CPU fallback.
 */
#ifndef ME_H
#define ME_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ME_OK = 0,
    ME_EINVAL = -1,    /* bad sizes / block / p / npairs / NULL pointer                  */
    ME_EALIGN = -2,    /* W % 16 != 0 or a pointer / stride not 16-byte aligned           */
    ME_ENOTINIT = -3,  /* me_init has not succeeded                                       */
    ME_ECUDA = -4,     /* a CUDA runtime error (see me_strerror)                          */
    ME_ENOMEM = -5     /* device allocation failed (host-buffer variant only)             */
} me_status;

/* Select `device`, check it is sm_100 with enough shared memory, set kernel attributes,
 * and allocate the library's device resources (scratch, copy streams, the staging buffers of
 * me_dcds_batch_host).  Idempotent per device; calling it with another device first releases
 * everything of the previous one (as me_shutdown), so no stream or buffer crosses devices. */
int me_init(int device);

/* cudaStream_t for every later launch (NULL = legacy default stream). */
int me_set_stream(void* cuda_stream);

/* DCDS on one frame pair: Step 1 HCSP with the halfway stop,
 * Step 2 HDSP/VDSP by switching strategy one, Step 3 repeated with switching
 * strategy two until the BMP is the pattern centre (no iteration cap), Step 4
 * the two middle points.  Each position is scored at most once per block
 * (reading C5).
 * Outputs per block: mv_out [nb][2] int16 (dx,dy); sad_out [nb] SAD at that MV;
 * points_out [nb] number of distinct candidates scored (NSP, P:342 aspect 3). */
int me_dcds(const uint8_t* cur, const uint8_t* ref, int W, int H, int block, int p,
            int16_t* mv_out, uint32_t* sad_out, uint16_t* points_out);

/* Full search: all (2p+1)^2 window candidates, (0,0) first then raster (dy outer,
 * dx inner), strict minimum.  points_out = (2p+1)^2 for every block ("225"). */
int me_fullsearch(const uint8_t* cur, const uint8_t* ref, int W, int H, int block, int p,
                  int16_t* mv_out, uint32_t* sad_out, uint16_t* points_out);

/* Motion-compensated PSNR of cur predicted from ref by the mv field (P:342 aspect 4):
 * SSE = sum (cur(x,y) - ref(clamp(x+dx), clamp(y+dy)))^2 (exact, uint64); *psnr_out =
 * 10*log10(255^2*W*H/SSE) in double (+inf when SSE == 0; reading C18).  psnr_out and
 * sse_out are HOST pointers (sse_out may be NULL).  Synchronises the stream. */
int me_mc_psnr(const uint8_t* cur, const uint8_t* ref, int W, int H, int block,
               const int16_t* mv, double* psnr_out /* host */, uint64_t* sse_out /* host */);

/* Throughput path: npairs independent pairs; pair t's frames are cur0 + t*pair_stride and
 * ref0 + t*pair_stride (pair_stride % 16 == 0).  Outputs are concatenated per pair:
 * mv_out [npairs][nb][2], sad_out [npairs][nb], points_out [npairs][nb].
 * stats_out (device, may be NULL): [npairs][3] uint64 = {sum points, sum SAD, SSE of the
 * motion-compensated pair at the DCDS MVs (P:342 aspects 1-4)}; overwritten. */
int me_dcds_batch(const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride, int npairs,
                  int W, int H, int block, int p, int16_t* mv_out, uint32_t* sad_out,
                  uint16_t* points_out, uint64_t* stats_out);

/* me_dcds_batch with the outputs in the 6-byte transport record of the multi-GPU gather
 * (SURVEY 8(e)): mv_out [npairs][nb][2] int8 (dx, dy; |d| <= p <= 32), sad_out [npairs][nb]
 * uint16 (SAD <= 255 * 256), points_out [npairs][nb] uint16 -- the same values as
 * me_dcds_batch's, 40% fewer bytes; stats_out as me_dcds_batch.  Outputs 2-byte aligned
 * (stats 8-byte), else ME_EALIGN; other errors as me_dcds_batch. */
int me_dcds_batch_packed(const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride, int npairs,
                         int W, int H, int block, int p, int8_t* mv_out, uint16_t* sad_out,
                         uint16_t* points_out, uint64_t* stats_out);

/* DCDS^S (Table X): as me_dcds_batch but Step 4 scores only the middle point on the
 * side of the cheaper distant point of the final pattern (an infeasible distant point costs
 * +inf; a tie picks the negative side -- reading C22). */
int me_dcds_s_batch(const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride, int npairs,
                    int W, int H, int block, int p, int16_t* mv_out, uint32_t* sad_out,
                    uint16_t* points_out, uint64_t* stats_out);

/* Diagnostic trace of DCDS (variant 0) / DCDS^S (variant 1): the same search as
 * me_dcds_batch / me_dcds_s_batch (same outputs, bit for bit) from a separately compiled
 * kernel that also records every scoring pass of every block ("trace"), to diff a
 * search against the oracle's point-by-point trace when parity fails.  Default lane-group
 * geometry only (ME_EINVAL when ME_G / ME_NW override it).
 * trace_out (device) [npairs][nb][trace_cap] uint64, one record per pass in search order:
 *   bits 0-7   pass number (0 = Step 1, 1..n = Steps 2-3, n+1 = Step 4)
 *   bits 8-11  pattern: 15 = HCSP (Step 1), 2 = HDSP, 3 = VDSP, 4 / 5 = horizontal / vertical
 *              middle points (Step 4); the DCDS^S distant-point look-up is not a pass
 *   bits 12-19 slots newly scored (bit k = slot k of the pattern in the order of reading C7:
 *              HCSP (0,0) (-1,0) (1,0) (-2,0) (2,0) (0,-1) (0,1); HDSP (-2,0) (2,0) (0,-1)
 *              (0,1); VDSP (-1,0) (1,0) (0,-2) (0,2); middle points (-1,0) (1,0) / (0,-1) (0,1))
 *   bits 20-27 / 28-35  pattern centre dx / dy (int8 two's complement)
 *   bits 36-51 incumbent SAD after the pass
 * trace_len_out (device) [npairs][nb] uint16: passes of each block (records beyond
 * trace_cap are counted but not written).  1 <= trace_cap <= 255; trace_out 8-byte aligned. */
int me_dcds_trace_batch(int variant, const uint8_t* cur0, const uint8_t* ref0,
                        int64_t pair_stride, int npairs, int W, int H, int block, int p,
                        int16_t* mv_out, uint32_t* sad_out, uint16_t* points_out,
                        uint64_t* trace_out, int trace_cap, uint16_t* trace_len_out);

/* Block-matching algorithm ids of me_bma_batch.  DCDS / DCDS^S are the paper's method; the
 * others are the comparison BMAs the paper measures DCDS against (Table VII
 * P:307-324), with the readings of DESIGN.md C23-C26:
 *   CDS     (ref. [13]) 9-point 5x5 cross, first-step stop; the two unchecked central-3x3
 *           points beside the arm of the BMP (a tie moves the BMP there), second-step stop for
 *           a distance-1 BMP; then DS from the BMP.
 *   DS      (ref. [10]) large diamond (9 points, then 8 recentred) until the BMP is its centre,
 *           then the small diamond (4 points).
 *   HEXBS_H (ref. [12], Fig. 2a) horizontal hexagon {(+-2,0),(+-1,+-2)} until centred, then the
 *           4 distance-1 points; HEXBS_V the vertical hexagon (Fig. 2b).
 * All share the conventions above: visited set (each position scored once per block), strict
 * compare, window-only feasibility, edge-replicated reference; points of a pattern are
 * scanned in ascending distance from its centre, ties by (|dy|,|dx|,dy,dx). */
typedef enum {
    ME_ALG_DCDS = 0,
    ME_ALG_DCDS_S = 1,
    ME_ALG_CDS = 2,
    ME_ALG_DS = 3,
    ME_ALG_HEXBS_H = 4,
    ME_ALG_HEXBS_V = 5
} me_alg;

/* Any me_alg over npairs pairs; arguments, layout, outputs (mv, SAD, NSP, stats = {sum points,
 * sum SAD, SSE at the chosen MVs}) and errors exactly as me_dcds_batch (ME_EINVAL for an
 * unknown alg).  ME_ALG_DCDS / ME_ALG_DCDS_S run the me_dcds_batch / me_dcds_s_batch kernels. */
int me_bma_batch(int alg, const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride,
                 int npairs, int W, int H, int block, int p, int16_t* mv_out, uint32_t* sad_out,
                 uint16_t* points_out, uint64_t* stats_out);

/* The ideal condition of P:299-301 (Table VII): for every true MV t of the +-p
 * window, run algorithm `alg` on the unimodal surface whose distortion at candidate q is the
 * Euclidean distance |q - t| (the device uses |q - t|^2, which orders and ties candidates
 * identically), with the same readings as the pixel searches.  Outputs (DEVICE int32 arrays
 * of (2p+1)^2, row-major over (ty, tx), i.e. index (ty+p)*(2p+1) + tx+p): nsp_out = number of
 * search points; mvx_out / mvy_out (may be NULL) = the MV found.  1 <= p <= 32. */
int me_ideal_nsp_map(int alg, int p, int32_t* nsp_out, int32_t* mvx_out, int32_t* mvy_out);

/* MV histogram (the MVP distribution of P:71-98): hist_out[(dy+p)*(2p+1) + dx+p] = number of
 * the n vectors mv[i] = (dx,dy) (DEVICE int16 pairs) inside the +-p window (others are not
 * counted; mv may be NULL when n == 0).  hist_out: DEVICE uint64 [(2p+1)^2], overwritten.
 * 1 <= p <= 32.  Table II / III /
 * Fig. 3 statistics are host arithmetic on this histogram (paper_0806_0689_b200/mvstats.py). */
int me_mv_hist(const int16_t* mv, int64_t n, int p, uint64_t* hist_out);

/* Full search over npairs pairs; same layout as me_dcds_batch (stats: {sum points, sum SAD,
 * SSE at the FS MVs}). */
int me_fullsearch_batch(const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride,
                        int npairs, int W, int H, int block, int p, int16_t* mv_out,
                        uint32_t* sad_out, uint16_t* points_out, uint64_t* stats_out);

/* Motion-compensated SSE of npairs pairs (device sse_out [npairs] uint64, overwritten). */
int me_mc_sse_batch(const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride, int npairs,
                    int W, int H, int block, const int16_t* mv, uint64_t* sse_out);

/* Table-IX-style quality of a motion field against the full-search field (P:342 aspects 5
 * and 6): for each of npairs pairs of nb blocks, out[2k] = number of blocks
 * whose MV equals the FS MV (the "probability of finding the true MV" times nb) and
 * out[2k+1] = sum over blocks of the Euclidean distance |mv - mv_fs| (double; deterministic
 * fixed-order reduction).  mv, mv_fs: device [npairs][nb][2] int16; out: device double
 * [npairs][2], overwritten.  MAD, MSE, NSP and PSNR follow from the stats_out of the searches
 * (MAD = sum SAD / (nb*B*B), MSE = SSE / (W*H), NSP = sum points / nb). */
int me_quality_batch(const int16_t* mv, const int16_t* mv_fs, int npairs, int nb, double* out);

/* End-to-end variant of me_dcds_batch on HOST buffers.  cur0, ref0: host, the frames of
 * pair t at cur0 + t*pair_stride and ref0 + t*pair_stride (W*H bytes each; for npairs == 1
 * pair_stride is ignored and cur / ref may be any two host buffers -- each frame is copied
 * on its own, never the span between them).  Frames are copied to device staging buffers in
 * chunks on two copy streams (cudaMemcpy2DAsync per chunk: cur rows, then ref rows), each
 * chunk's search overlapping the next chunk's copy, and the outputs (host, as me_dcds_batch)
 * copied back.  Synchronises, on success and on error: when it returns no copy touches the
 * caller's buffers.  Pinned host memory gives full copy bandwidth.  The staging buffers are
 * allocated by me_init (128 MiB of frames each); only a pair larger than that grows them,
 * once (ME_ENOMEM if that fails).  No host pointer alignment is required. */
int me_dcds_batch_host(const uint8_t* cur0, const uint8_t* ref0, int64_t pair_stride,
                       int npairs, int W, int H, int block, int p, int16_t* mv_out,
                       uint32_t* sad_out, uint16_t* points_out, uint64_t* stats_out);

/* Number of kernels this library has launched since me_init (for the bench's
 * gpu_launches field). */
int64_t me_launch_count(void);

/* Blocks of the most recent DCDS / DCDS^S batch call (me_dcds_batch, me_dcds_s_batch,
 * me_dcds_batch_packed, me_bma_batch with those algorithms) whose search left the compact
 * visited set and was run again by the overflow pass (DESIGN.md §7 "Compact visited set":
 * 16x16 blocks at p >= 26, or as ME_COMPACT forces); 0 when that call did not use the compact
 * set.  Diagnostic only -- the outputs are the same either way.  *count_out is a HOST
 * pointer; waits for that call's overflow passes, then reads the two list counts (interior and
 * border blocks) from the device.  A call captured into a CUDA graph writes the counts when
 * the graph is replayed; synchronise the replay before asking. */
int me_dcds_overflow_count(uint64_t* count_out);

/* Static description of the last error (never NULL). */
const char* me_strerror(int status);

/* Free library-owned device memory and forget the device. */
void me_shutdown(void);

#ifdef __cplusplus
}
#endif
#endif
