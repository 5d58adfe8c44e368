/* Host sanitizer driver for the oracle (ASan/UBSan on the oracle).  Runs every
 * oracle entry point on small seeded frames -- random, flat and binary textures, every
 * variant, border-heavy sizes and windows from 1 to 32 -- under -fsanitize=address,undefined.
 * Exit status 0 = no finding (the sanitizers abort on the first one). */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "../../oracle/oracle.h"

static uint32_t rng = 806689u;
static uint32_t next(void) { rng = rng * 1664525u + 1013904223u; return rng >> 8; }

static double cost_fn(int dx, int dy, void* ctx) {
    const int* t = (const int*)ctx;
    return (double)((dx - t[0]) * (dx - t[0]) + (dy - t[1]) * (dy - t[1]));
}

int main(void) {
    const int sizes[][2] = {{16, 16}, {48, 32}, {176, 144}};
    const int ps[] = {1, 2, 7, 16, 32};
    for (int si = 0; si < 3; si++) {
        const int W = sizes[si][0], H = sizes[si][1];
        uint8_t* cur = malloc((size_t)W * H);
        uint8_t* ref = malloc((size_t)W * H);
        for (int kind = 0; kind < 3; kind++) {
            for (int i = 0; i < W * H; i++) {
                cur[i] = kind == 0 ? (uint8_t)next() : kind == 1 ? 77 : (uint8_t)((next() & 1) * 255);
                ref[i] = kind == 0 ? (uint8_t)next() : kind == 1 ? 77 : (uint8_t)((next() & 1) * 255);
            }
            for (int B = 8; B <= 16; B += 8) {
                if (W % B || H % B) continue;
                const int nb = (W / B) * (H / B);
                int16_t* mv = malloc(sizeof(int16_t) * 2 * nb);
                uint32_t* sad = malloc(sizeof(uint32_t) * nb);
                uint16_t* pts = malloc(sizeof(uint16_t) * nb);
                for (int pi = 0; pi < 5; pi++) {
                    const int p = ps[pi];
                    for (int v = 0; v <= 5; v++)
                        if (oracle_dcds(cur, ref, W, H, B, p, v, mv, sad, pts)) return 2;
                    if (p <= 16 && oracle_fullsearch(cur, ref, W, H, B, p, mv, sad, pts)) return 3;
                    double ps_db; uint64_t sse;
                    if (oracle_mc_psnr(cur, ref, W, H, B, mv, &ps_db, &sse)) return 4;
                    int16_t m1[2]; uint32_t s1; uint16_t p1;
                    if (oracle_dcds_block(cur, ref, W, H, B, p, 0, W - B, H - B, m1, &s1, &p1)) return 5;
                    if (oracle_fullsearch_block(cur, ref, W, H, B, p, 0, 0, m1, &s1, &p1)) return 6;
                }
                free(mv); free(sad); free(pts);
            }
        }
        free(cur); free(ref);
    }
    for (int p = 1; p <= 32; p *= 2) {
        const int side = 2 * p + 1;
        int* nsp = malloc(sizeof(int) * side * side);
        int* mx = malloc(sizeof(int) * side * side);
        int* my = malloc(sizeof(int) * side * side);
        for (int v = 0; v <= 5; v++)
            if (oracle_ideal_nsp_map(p, v, nsp, mx, my)) return 7;
        int t[2] = {p, -p}, bx, by, np, tl;
        double c;
        int tr[4 * 256];
        for (int v = 0; v <= 1; v++)
            if (oracle_dcds_cost(cost_fn, t, p, v, &bx, &by, &c, &np, tr, 256, &tl)) return 8;
        free(nsp); free(mx); free(my);
    }
    puts("oracle sanitizer run: clean");
    return 0;
}
