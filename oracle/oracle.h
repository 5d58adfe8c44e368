/*
 * oracle.h -- plain, slow, single-threaded CPU oracle for the DCDS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load or call this library.  The product
 * path (paper_0806_0689_b200/, libme.so) never links, imports or executes it, and
 * it shares no code, header, table or helper with the CUDA path.
 *
 * Paper: Jia & Zhang, "Directional Cross Diamond Search Algorithm for Fast Block
 * Motion Estimation" (arxiv 0806.0689).  P:n = /root/reference/PAPER.md line n.
 *
 * Conventions (SURVEY.md 8(c) ledger C1-C22):
 *   - frames are uint8 luma, row-major, pitch = W, W and H multiples of the block size B;
 *   - blocks are numbered in raster order, nb = (W/B)*(H/B)   ("non-overlapping ... blocks");
 *   - a motion vector (dx,dy) matches cur block (bx,by) with ref at (bx+dx, by+dy);
 *   - candidate q is feasible iff |dx|<=p and |dy|<=p (window only, reading C8/C9);
 *   - reference pixels outside the frame read the edge-replicated reference
 *     R(x,y) = ref[clamp(y,0,H-1)*W + clamp(x,0,W-1)]                 (reading C9);
 *   - comparisons are strict, the incumbent wins ties, and points listed first win
 *     ties among new points (readings C6, C7, C13).
 *
 * All functions return 0 on success, -1 on invalid arguments.
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* SAD of the B x B block at (bx,by) of cur against R at (bx+dx, by+dy).  P:342 (MAD as the
 * BDM; SAD = B*B*MAD, reading C12). */
int oracle_sad(const uint8_t* cur, const uint8_t* ref, int W, int H, int B,
               int bx, int by, int dx, int dy, uint32_t* sad_out);

/* Sum of squared differences of the same pair of blocks (P:342 aspect 2, MSE). */
int oracle_sse_block(const uint8_t* cur, const uint8_t* ref, int W, int H, int B,
                     int bx, int by, int dx, int dy, uint64_t* sse_out);

/* DCDS over every block of one frame pair (Steps 1-4).
 * variant 0 = DCDS; variant 1 = DCDS^S (Step 4 checks only the middle point on the
 * side of the cheaper distant point; reading C22).  The comparison BMAs of the paper run on
 * the same machinery (readings C23-C26): variant 2 = CDS (ref. [13]),
 * 3 = DS (ref. [10]), 4 = h-HEXBS (ref. [12], Fig. 2a), 5 = v-HEXBS (Fig. 2b).
 * mv_out[2*i] = dx, mv_out[2*i+1] = dy; sad_out[i]; points_out[i] = NSP of block i. */
int oracle_dcds(const uint8_t* cur, const uint8_t* ref, int W, int H, int B, int p,
                int variant, int16_t* mv_out, uint32_t* sad_out, uint16_t* points_out);

/* Full search over every block (all (2p+1)^2 window candidates; (0,0) first, then
 * raster dy outer / dx inner; strict minimum -- reading C13). */
int oracle_fullsearch(const uint8_t* cur, const uint8_t* ref, int W, int H, int B, int p,
                      int16_t* mv_out, uint32_t* sad_out, uint16_t* points_out);

/* Single-block versions (sampled parity at full size): block origin (bx,by). */
int oracle_dcds_block(const uint8_t* cur, const uint8_t* ref, int W, int H, int B, int p,
                      int variant, int bx, int by, int16_t* mv_out, uint32_t* sad_out,
                      uint16_t* points_out);
int oracle_fullsearch_block(const uint8_t* cur, const uint8_t* ref, int W, int H, int B, int p,
                            int bx, int by, int16_t* mv_out, uint32_t* sad_out,
                            uint16_t* points_out);

/* Motion-compensated SSE and PSNR (P:342 aspect 4; reading C18):
 * pred(x,y) = R(x+mvx, y+mvy) for the block containing (x,y); SSE = sum (cur-pred)^2;
 * PSNR = 10*log10(255^2 * W*H / SSE), +inf when SSE == 0. */
int oracle_mc_psnr(const uint8_t* cur, const uint8_t* ref, int W, int H, int B,
                   const int16_t* mv, double* psnr_out, uint64_t* sse_out);

/* Quality of a motion field against the full-search field (P:43 / P:342 aspects 5 and 6:
 * "the distance from the true motion vectors (obtained by FS)" and "the probability of
 * finding the true MVs"): over nb blocks, *hits = number of blocks whose MV equals the FS MV
 * and *dist = sum of the Euclidean distances |mv - mv_fs| (double, blocks in order). */
int oracle_quality(const int16_t* mv, const int16_t* mv_fs, int nb, int* hits, double* dist);

/* DCDS (or, by variant, a comparison BMA) on an injected cost function (the ideal
 * unimodal surface).  cost(dx,dy,ctx)
 * is called once per distinct feasible candidate.  trace (may be NULL) receives up to
 * trace_cap records of 4 ints {pass, dx, dy, kind}: pass 0 is Step 1 (HCSP), passes
 * 1..n the intermediate steps (1 = Step 2, 2..n = Step 3 repetitions) and pass n+1 Step 4;
 * kind 0=HCSP 1=HDSP 2=VDSP 3=middle point 4=large diamond 5=small diamond 6=5x5 cross
 * 7=hexagon.  *trace_len receives the number of records written. */
typedef double (*oracle_cost_fn)(int dx, int dy, void* ctx);
int oracle_dcds_cost(oracle_cost_fn cost, void* ctx, int p, int variant,
                     int* mv_dx, int* mv_dy, double* cost_out, int* points_out,
                     int* trace, int trace_cap, int* trace_len);

/* Ideal-surface helper: cost = Euclidean distance |q - t|; returns the NSP map over
 * all (2p+1)^2 placements t, row-major (ty outer, tx inner), and the found MVs. */
int oracle_ideal_nsp_map(int p, int variant, int* nsp_out, int* mvx_out, int* mvy_out);

#ifdef __cplusplus
}
#endif
#endif
