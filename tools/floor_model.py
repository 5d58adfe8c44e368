"""Floor model of DCDS kernel designs, replaying real search traces.

Input: per-pass traces of real searches (tools/dump_traces.py -> me_dcds_trace_batch): for
every block the passes (pattern id, new-slot mask, centre).  For each candidate design the
model replays the passes in the design's warp structure (lock-step passes, a warp runs while
any of its searches runs) and counts, per macroblock:

  * lane-loads of the staged reference (LDS.32 lane accesses) and LDS warp-instructions;
  * shared-memory wavefronts: per LDS instruction, max over the 32 banks of the number of
    distinct words its active lanes request (predicated-off lanes issue no access);
  * warp-instructions issued and ALU-pipe warp-instructions, from a per-pass cost table of
    the design's code (counted once per warp-pass, whatever the number of active lanes);

and turns them into a time floor: cycles per block = max(issue / 4, ALU / 2, wavefronts / 1)
per SM (B200: 4 schedulers, a half-rate ALU pipe (VABSDIFF4 / SHF / LOP3 / ISETP / SEL),
one shared-memory wavefront per clock), divided by an achieved fraction of that resource.

Designs:
  D0  the round-1 kernel (v14): G = 2 lanes per block, 16 blocks per warp, 4 slots per pass,
      each slot 8 rows x 3 words; costs calibrated on its ncu capture (168 warp-instr / block).
  D1  one thread per block (32 blocks per warp) with row-shared passes on an axis-transposed
      copy of the region: every DDSP / middle-point pass is the horizontal pattern on either
      the region (HDSP, horizontal middle points) or its transpose (VDSP, vertical middle
      points), so all threads run one code path; a pass loads the 10 reference rows of its
      pattern once (4 words each) and derives all slot windows from them by funnel shifts.

usage: python tools/floor_model.py gpurun_out/r2a/traces_c3.npz [--pairs 1]
"""
from __future__ import annotations

import argparse
import json

import numpy as np

SM, CLK = 148, 1.965e9


def decode_all(tr, tl):
    """[n, nb, P] records -> pid, mask, cx, cy arrays and an active mask."""
    r = tr.astype(np.uint64)
    pid = ((r >> np.uint64(8)) & np.uint64(0xF)).astype(np.int16)
    mask = ((r >> np.uint64(12)) & np.uint64(0xFF)).astype(np.int16)
    cx = ((r >> np.uint64(20)) & np.uint64(0xFF)).astype(np.int16)
    cy = ((r >> np.uint64(28)) & np.uint64(0xFF)).astype(np.int16)
    cx = np.where(cx > 127, cx - 256, cx)
    cy = np.where(cy > 127, cy - 256, cy)
    act = np.arange(tr.shape[-1])[None, :] < tl[..., None].astype(np.int64)
    return pid, mask, cx, cy, act


def wavefronts(words, valid):
    """words [n, L] int64 word addresses, valid [n, L] -> wavefronts per row (n,)"""
    n, L = words.shape
    w = np.where(valid, words, -1)
    w = np.sort(w, axis=1)
    dup = np.zeros_like(valid)
    dup[:, 1:] = w[:, 1:] == w[:, :-1]
    keep = (w >= 0) & ~dup
    bank = np.where(keep, w % 32, 32)
    cnt = np.zeros((n, 33), np.int32)
    np.add.at(cnt, (np.repeat(np.arange(n), L), bank.ravel()), 1)
    return cnt[:, :32].max(axis=1)


def warp_layout(nbx, nby, tbx, tby, wx, wy):
    """block -> (warp id, lane, tile x0 block, tile y0 block, local bx, local by)"""
    ntx = (nbx + tbx - 1) // tbx
    bx = np.arange(nbx)[None, :].repeat(nby, 0)
    by = np.arange(nby)[:, None].repeat(nbx, 1)
    tx, ty = bx // tbx, by // tby
    lx, ly = bx % tbx, by % tby
    wpr = tbx // wx  # warps per tile row
    wid_in = (ly // wy) * wpr + lx // wx
    wpt = (tbx // wx) * (tby // wy)
    wid = (ty * ntx + tx) * wpt + wid_in
    lane = (ly % wy) * wx + lx % wx
    return wid.ravel(), lane.ravel(), (tx * tbx).ravel(), (ty * tby).ravel()


def model_d1(d, pairs, tbx=8, tby=8, wx=8, wy=4, pitch=None, pitchT=None, costs=None):
    """one thread per block, transposed copy, row-shared 10-row passes"""
    W, H, B, p = int(d["W"]), int(d["H"]), int(d["B"]), int(d["p"])
    nbx, nby = W // B, H // B
    TW, TH = tbx * B, tby * B
    pitch = pitch or ((TW + 2 * p + 16 + 15) & ~15)
    rh = TH + 2 * p
    pitchT = pitchT or ((rh + 16 + 15) & ~15)
    tbase = ((pitch * rh + 127) & ~127)
    wid, lane, tx0, ty0 = warp_layout(nbx, nby, tbx, tby, wx, wy)
    nwarp = wid.max() + 1
    nl = wx * wy
    bxs = (np.arange(nbx * nby) % nbx) * B
    bys = (np.arange(nbx * nby) // nbx) * B
    x0 = tx0 * B
    y0 = ty0 * B
    xs = (x0 - p) & ~15
    ys = y0 - p
    ox, oy = bxs - xs, bys - ys  # block origin in region coords
    c = costs or D1_COSTS
    tot = dict(lds=0, wf=0, lane_loads=0, instr=0, alu=0, warp_passes=0)
    for pr in pairs:
        pid, mask, cx, cy, act = decode_all(d["trace"][pr], d["tlen"][pr])
        P = pid.shape[1]
        # lane table [nwarp, nl] -> block index
        tab = -np.ones((nwarp, nl), np.int64)
        tab[wid, lane] = np.arange(nbx * nby)
        okb = tab >= 0
        tabc = np.where(okb, tab, 0)
        npass_w = np.where(okb, d["tlen"][pr][tabc], 0).max(axis=1)
        tot["warp_passes"] += int(npass_w.sum())
        tot["instr"] += nwarp * c["once"] + int(np.maximum(npass_w - 1, 0).sum()) * c["pass_"] + nwarp * c["pass0"]
        tot["alu"] += nwarp * c["once_alu"] + int(np.maximum(npass_w - 1, 0).sum()) * c["pass_alu"] + nwarp * c["pass0_alu"]
        for i in range(P):
            a = act[tabc, i] & okb  # [nwarp, nl]
            if not a.any():
                break
            wsel = a.any(axis=1)
            A = a[wsel]
            blk = tabc[wsel]
            pi, cxi, cyi = pid[blk, i], cx[blk, i], cy[blk, i]
            h = np.where((pi == 2) | (pi == 3), 2, 1)
            T = (pi == 3) | (pi == 5)
            if i == 0:  # HCSP at the window origin, normal region: words O-4 .. O+8
                row0 = oy[blk]
                col = ox[blk] - 4
                rows, nw = range(-1, 9), 4
                base_off = np.zeros_like(row0)
                rp = np.full_like(row0, pitch)
            else:
                row0 = np.where(T, ox[blk] + cxi, oy[blk] + cyi)
                colc = np.where(T, oy[blk] + cyi, ox[blk] + cxi)
                col = (colc - h) & ~3
                rows, nw = range(-1, 9), 4
                base_off = np.where(T, tbase, 0)
                rp = np.where(T, pitchT, pitch)
            for r in rows:
                for w in range(nw):
                    addr = base_off + (row0 + r) * rp + col + 4 * w
                    wf = wavefronts(addr // 4, A)
                    tot["wf"] += int(wf.sum())
                    tot["lds"] += int(A.shape[0])
                    tot["lane_loads"] += int(A.sum())
    nblk = len(pairs) * nbx * nby
    return {k: v / nblk for k, v in tot.items()} | {"pitch": pitch, "pitchT": pitchT, "warp_blocks": nl}


def model_d2(d, pairs, tbx=16, tby=4, wx=16, wy=1, G=2, pitch=None, pitchT=None, s4_reuse=True,
             rows_hdsp=(-1, 9)):
    """G lanes per block (16 blocks per warp for G=2), transposed copy, row-shared passes: lane j
    of a group loads the pattern rows r with (r - r0) % G == j, 4 words each; S4 passes reuse
    the rows of the S3 pass before them (no loads) when s4_reuse."""
    W, H, B, p = int(d["W"]), int(d["H"]), int(d["B"]), int(d["p"])
    nbx, nby = W // B, H // B
    TW, TH = tbx * B, tby * B
    pitch = pitch or ((TW + 2 * p + 16 + 15) & ~15)
    rh = TH + 2 * p
    pitchT = pitchT or ((rh + 16 + 15) & ~15)
    tbase = ((pitch * rh + 127) & ~127)
    wid, lane, tx0, ty0 = warp_layout(nbx, nby, tbx, tby, wx, wy)
    nwarp = wid.max() + 1
    nl = wx * wy
    bxs = (np.arange(nbx * nby) % nbx) * B
    bys = (np.arange(nbx * nby) // nbx) * B
    xs = (tx0 * B - p) & ~15
    ys = ty0 * B - p
    ox, oy = bxs - xs, bys - ys
    tot = dict(lds=0, wf=0, lane_loads=0, warp_passes=0)
    r0, r1 = rows_hdsp
    nrow = r1 - r0
    for pr in pairs:
        pid, mask, cx, cy, act = decode_all(d["trace"][pr], d["tlen"][pr])
        tab = -np.ones((nwarp, nl), np.int64)
        tab[wid, lane] = np.arange(nbx * nby)
        okb = tab >= 0
        tabc = np.where(okb, tab, 0)
        tot["warp_passes"] += int(np.where(okb, d["tlen"][pr][tabc], 0).max(axis=1).sum())
        for i in range(pid.shape[1]):
            a = act[tabc, i] & okb
            if not a.any():
                break
            wsel = a.any(axis=1)
            blk = tabc[wsel]
            A = a[wsel]
            pi, cxi, cyi = pid[blk, i], cx[blk, i], cy[blk, i]
            if s4_reuse and i > 0:
                A = A & (pi != 4) & (pi != 5)
            h = np.where((pi == 2) | (pi == 3), 2, 1)
            T = (pi == 3) | (pi == 5)
            if i == 0:
                row0, col = oy[blk], ox[blk] - 4
                base_off, rp = np.zeros_like(oy[blk]), np.full_like(oy[blk], pitch)
            else:
                row0 = np.where(T, ox[blk] + cxi, oy[blk] + cyi)
                colc = np.where(T, oy[blk] + cyi, ox[blk] + cxi)
                col = (colc - h) & ~3
                base_off = np.where(T, tbase, 0)
                rp = np.where(T, pitchT, pitch)
            nstep = (nrow + G - 1) // G
            for st in range(nstep):
                for w in range(4):
                    addrs, vals = [], []
                    for j in range(G):
                        r = r0 + st * G + j
                        addrs.append((base_off + (row0 + r) * rp + col + 4 * w) // 4)
                        vals.append(A & (r < r1))
                    addr = np.concatenate(addrs, axis=1)
                    val = np.concatenate(vals, axis=1)
                    ws = val.any(axis=1)
                    if not ws.any():
                        continue
                    wf = wavefronts(addr[ws], val[ws])
                    tot["wf"] += int(wf.sum())
                    tot["lds"] += int(ws.sum())
                    tot["lane_loads"] += int(val.sum())
    nblk = len(pairs) * nbx * nby
    return {k: v / nblk for k, v in tot.items()} | {"pitch": pitch, "pitchT": pitchT}


def model_d3(d, pairs, tbx=16, tby=4, wx=16, wy=1, pitch=None, pitchT=None, s4_reuse=True, nwl=3):
    """G = 2, both lanes of a group walk all 10 pattern rows; lane j loads words j .. j+nwl-1 of
    the row's 4-word span (so the two lanes of a group read consecutive words: banks of both
    parities); transposed copy; S4 passes reuse the S3 rows when s4_reuse."""
    W, H, B, p = int(d["W"]), int(d["H"]), int(d["B"]), int(d["p"])
    nbx, nby = W // B, H // B
    TW, TH = tbx * B, tby * B
    pitch = pitch or ((TW + 2 * p + 16 + 15) & ~15)
    rh = TH + 2 * p
    pitchT = pitchT or ((rh + 16 + 15) & ~15)
    tbase = ((pitch * rh + 127) & ~127)
    wid, lane, tx0, ty0 = warp_layout(nbx, nby, tbx, tby, wx, wy)
    nwarp = wid.max() + 1
    nl = wx * wy
    bxs = (np.arange(nbx * nby) % nbx) * B
    bys = (np.arange(nbx * nby) // nbx) * B
    xs = (tx0 * B - p) & ~15
    ys = ty0 * B - p
    ox, oy = bxs - xs, bys - ys
    tot = dict(lds=0, wf=0, lane_loads=0, warp_passes=0)
    for pr in pairs:
        pid, mask, cx, cy, act = decode_all(d["trace"][pr], d["tlen"][pr])
        tab = -np.ones((nwarp, nl), np.int64)
        tab[wid, lane] = np.arange(nbx * nby)
        okb = tab >= 0
        tabc = np.where(okb, tab, 0)
        tot["warp_passes"] += int(np.where(okb, d["tlen"][pr][tabc], 0).max(axis=1).sum())
        for i in range(pid.shape[1]):
            a = act[tabc, i] & okb
            if not a.any():
                break
            wsel = a.any(axis=1)
            blk = tabc[wsel]
            A = a[wsel]
            pi, cxi, cyi = pid[blk, i], cx[blk, i], cy[blk, i]
            if s4_reuse and i > 0:
                A = A & (pi != 4) & (pi != 5)
            h = np.where((pi == 2) | (pi == 3), 2, 1)
            T = (pi == 3) | (pi == 5)
            if i == 0:
                row0, col = oy[blk], ox[blk] - 4
                base_off, rp = np.zeros_like(oy[blk]), np.full_like(oy[blk], pitch)
            else:
                row0 = np.where(T, ox[blk] + cxi, oy[blk] + cyi)
                colc = np.where(T, oy[blk] + cyi, ox[blk] + cxi)
                col = (colc - h) & ~3
                base_off = np.where(T, tbase, 0)
                rp = np.where(T, pitchT, pitch)
            for r in range(-1, 9):
                for k in range(nwl):
                    addr = np.concatenate([(base_off + (row0 + r) * rp + col + 4 * (k + j)) // 4 for j in (0, 1)], axis=1)
                    val = np.concatenate([A, A], axis=1)
                    ws = val.any(axis=1)
                    wf = wavefronts(addr[ws], val[ws])
                    tot["wf"] += int(wf.sum())
                    tot["lds"] += int(ws.sum())
                    tot["lane_loads"] += int(val.sum())
    nblk = len(pairs) * nbx * nby
    return {k: v / nblk for k, v in tot.items()} | {"pitch": pitch, "pitchT": pitchT}


def model_g1(d, pairs, tbx=16, tby=4, wx=16, wy=2, pitch=192):
    """one thread per block, per-slot loads (8 rows x 3 words of each new slot), region as the
    round-1 kernel (no transposed copy); a warp issues a slot's loads if any thread needs it"""
    W, H, B, p = int(d["W"]), int(d["H"]), int(d["B"]), int(d["p"])
    nbx, nby = W // B, H // B
    wid, lane, tx0, ty0 = warp_layout(nbx, nby, tbx, tby, wx, wy)
    nwarp = wid.max() + 1
    nl = wx * wy
    bxs = (np.arange(nbx * nby) % nbx) * B
    bys = (np.arange(nbx * nby) // nbx) * B
    xs = (tx0 * B - p) & ~15
    ys = ty0 * B - p
    ox, oy = bxs - xs, bys - ys
    SL = {2: [(-2, 0), (2, 0), (0, -1), (0, 1)], 3: [(-1, 0), (1, 0), (0, -2), (0, 2)],
          4: [(-1, 0), (1, 0), (0, 0), (0, 0)], 5: [(0, -1), (0, 1), (0, 0), (0, 0)]}
    sdx = np.zeros((16, 4), np.int64)
    sdy = np.zeros((16, 4), np.int64)
    for k, v in SL.items():
        sdx[k] = [o[0] for o in v]
        sdy[k] = [o[1] for o in v]
    tot = dict(lds=0, wf=0, lane_loads=0, warp_passes=0)
    for pr in pairs:
        pid, mask, cx, cy, act = decode_all(d["trace"][pr], d["tlen"][pr])
        tab = -np.ones((nwarp, nl), np.int64)
        tab[wid, lane] = np.arange(nbx * nby)
        okb = tab >= 0
        tabc = np.where(okb, tab, 0)
        tot["warp_passes"] += int(np.where(okb, d["tlen"][pr][tabc], 0).max(axis=1).sum())
        for i in range(1, pid.shape[1]):
            a = act[tabc, i] & okb
            if not a.any():
                break
            wsel = a.any(axis=1)
            blk = tabc[wsel]
            A = a[wsel]
            pi = pid[blk, i]
            for k in range(4):
                need = A & (((mask[blk, i] >> k) & 1) == 1)
                ws = need.any(axis=1)
                if not ws.any():
                    continue
                o = (oy[blk] + cy[blk, i] + sdy[pi, k]) * pitch + ox[blk] + cx[blk, i] + sdx[pi, k]
                for r in range(8):
                    for w in range(3):
                        addr = (o + r * pitch) // 4 + w
                        wf = wavefronts(addr[ws], need[ws])
                        tot["wf"] += int(wf.sum())
                        tot["lds"] += int(ws.sum())
                        tot["lane_loads"] += int(need[ws].sum())
    nblk = len(pairs) * nbx * nby
    return {k: v / nblk for k, v in tot.items()}


def model_d0_refill(d, pairs, pitch=192, nwarps=4, tbx=16, tby=4, refill_at=1):
    """D0's loads (G = 2, 4 slots x 8 rows x 3 words, 16 groups per warp) when groups are
    refilled: a CTA's nwarps warps share the tile's block counter, a group that finished takes
    the next block of the tile (raster order) at the next warp-pass (refill_at: only when at
    least that many groups of the warp are idle).  Returns the slot-load counts and the
    warp-passes per block (the issue / ALU side)."""
    W, H, B, p = int(d["W"]), int(d["H"]), int(d["B"]), int(d["p"])
    nbx, nby = W // B, H // B
    SL = {2: [(-2, 0), (2, 0), (0, -1), (0, 1)], 3: [(-1, 0), (1, 0), (0, -2), (0, 2)],
          4: [(-1, 0), (1, 0), (0, 0), (0, 0)], 5: [(0, -1), (0, 1), (0, 0), (0, 0)]}
    tot = dict(lds=0, wf=0, lane_loads=0, warp_passes=0, refill_events=0)
    for pr in pairs:
        pid, mask, cx, cy, act = decode_all(d["trace"][pr], d["tlen"][pr])
        tl = d["tlen"][pr]
        for ty in range(nby // tby):
            for tx in range(nbx // tbx):
                x0, y0 = tx * tbx * B, ty * tby * B
                xs, ys = (x0 - p) & ~15, y0 - p
                queue = [(y0 // B + a) * nbx + x0 // B + b for a in range(tby) for b in range(tbx)]
                qi = 0
                cur = [[None] * 16 for _ in range(nwarps)]   # (block, pass index)
                while True:
                    alive = False
                    for w in range(nwarps):
                        idle = [g for g in range(16) if cur[w][g] is None]
                        if idle and qi < len(queue) and len(idle) >= min(refill_at, len(queue) - qi):
                            tot["refill_events"] += 1
                            for g in idle:
                                if qi < len(queue):
                                    cur[w][g] = [queue[qi], 0]
                                    qi += 1
                        groups = [(g, c) for g, c in enumerate(cur[w]) if c is not None]
                        if not groups:
                            continue
                        alive = True
                        tot["warp_passes"] += 1
                        for k in range(4):
                            addrs, n = [], 0
                            for g, (blk, i) in groups:
                                if i == 0:
                                    continue  # step 1: aligned loads, not a slot load
                                if not (mask[blk, i] >> k) & 1:
                                    continue
                                dx, dy = SL[int(pid[blk, i])][k]
                                ox = (blk % nbx) * B - xs
                                oy = (blk // nbx) * B - ys
                                o = (oy + int(cy[blk, i]) + dy) * pitch + ox + int(cx[blk, i]) + dx
                                addrs.append(o)
                            if not addrs:
                                continue
                            o = np.array(addrs)
                            for r in range(4):
                                for wd in range(3):
                                    words = np.concatenate([(o + 2 * r * pitch) // 4 + wd, (o + (2 * r + 1) * pitch) // 4 + wd])
                                    tot["wf"] += int(wavefronts(words[None, :], np.ones((1, words.size), bool))[0])
                                    tot["lds"] += 1
                                    tot["lane_loads"] += words.size
                        for g, c in groups:
                            c[1] += 1
                            if c[1] >= tl[c[0]]:
                                cur[w][g] = None
                    if not alive:
                        break
    nblk = len(pairs) * (nbx // tbx * tbx) * (nby // tby * tby)
    return {k: v / nblk for k, v in tot.items()}


def model_d0(d, pairs, pitch=192, swap=None, tbx=16, tby=4, wx=16, wy=1):
    """the round-1 kernel: G=2, 16 blocks per warp (16x4 tiles), 4 slots x 8 rows x 3 words"""
    W, H, B, p = int(d["W"]), int(d["H"]), int(d["B"]), int(d["p"])
    nbx, nby = W // B, H // B
    wid, lane, tx0, ty0 = warp_layout(nbx, nby, tbx, tby, wx, wy)
    nwarp = wid.max() + 1
    bxs = (np.arange(nbx * nby) % nbx) * B
    bys = (np.arange(nbx * nby) // nbx) * B
    xs = (tx0 * B - p) & ~15
    ys = ty0 * B - p
    ox, oy = bxs - xs, bys - ys
    SL = {2: [(-2, 0), (2, 0), (0, -1), (0, 1)], 3: [(-1, 0), (1, 0), (0, -2), (0, 2)],
          4: [(-1, 0), (1, 0), (0, 0), (0, 0)], 5: [(0, -1), (0, 1), (0, 0), (0, 0)]}
    sdx = np.zeros((16, 4), np.int64)
    sdy = np.zeros((16, 4), np.int64)
    for k, v in SL.items():
        sdx[k] = [o[0] for o in v]
        sdy[k] = [o[1] for o in v]
    tot = dict(lds=0, wf=0, lane_loads=0, warp_passes=0)
    for pr in pairs:
        pid, mask, cx, cy, act = decode_all(d["trace"][pr], d["tlen"][pr])
        tab = -np.ones((nwarp, 16), np.int64)
        tab[wid, lane] = np.arange(nbx * nby)
        okb = tab >= 0
        tabc = np.where(okb, tab, 0)
        tot["warp_passes"] += int(np.where(okb, d["tlen"][pr][tabc], 0).max(axis=1).sum())
        for i in range(1, pid.shape[1]):
            a = act[tabc, i] & okb
            if not a.any():
                break
            wsel = a.any(axis=1)
            blk = tabc[wsel]
            A = a[wsel]
            pi = pid[blk, i]
            for k in range(4):
                need = A & (((mask[blk, i] >> k) & 1) == 1)
                if not need.any():
                    continue
                ws = need.any(axis=1)
                o = (oy[blk] + cy[blk, i] + sdy[pi, k]) * pitch + ox[blk] + cx[blk, i] + sdx[pi, k]
                gpar = (np.arange(16)[None, :] % 2) if swap == "g" else (
                    (np.arange(16)[None, :] // 2) % 2 if swap == "g2" else np.zeros((1, 16), np.int64))
                for r in range(4):
                    for w in range(3):
                        # two lanes per group: rows j + 2r, j = 0, 1 (swap: odd groups' lanes
                        # exchange rows, so lane 0 reads row 2r + 1)
                        r0 = 2 * r + gpar
                        r1 = 2 * r + 1 - gpar
                        addr = np.concatenate([(o + r0 * pitch) // 4 + w, (o + r1 * pitch) // 4 + w], axis=1)
                        val = np.concatenate([need, need], axis=1)
                        wf = wavefronts(addr[ws], val[ws])
                        tot["wf"] += int(wf.sum())
                        tot["lds"] += int(ws.sum())
                        tot["lane_loads"] += int(val[ws].sum())
    nblk = len(pairs) * nbx * nby
    return {k: v / nblk for k, v in tot.items()}


# Per-pass cost tables (warp-instructions; ALU = the half-rate pipe).  D1 body per pass:
# 10 rows x 4 LDS, 3 pre-shift + 2 (centre window) + 2 (far window) SHF on rows 0..7 and 2 on
# rows -1 / 8, 64 VABSDIFF4 (4 slots x 8 rows x 2 words, predicated), 16 SEL (current block or
# its transpose), ~12 address / loop; control: visited test-and-set of 4 slots (~6 each),
# packed argmin (~8), state machine (~20), loop vote (~4).  Pass 0 (HCSP at the window
# origin): rows 0..7 x (4 LDS + 8 SHF + 10 VABSDIFF4) + rows -1 / 8 x 4 + control.  Once per
# warp: TMA / barrier / bitmap template / transpose share (~60), current block + its
# transpose (16 LDS + 24 PRMT), SSE at the final MV (8 x (3 LDS + 2 SHF + 2 VABSDIFF4 +
# 2 IDP)), outputs and stats (~20).
D1_COSTS = dict(pass0=204, once=200, pass0_alu=160, once_alu=110,
                pass_=40 + 60 + 64 + 16 + 12 + 24 + 8 + 20 + 4, pass_alu=60 + 64 + 16 + 35)


def floor(instr, alu, wf, eff=0.8):
    cyc = max(instr / 4.0, alu / 2.0, wf / 1.0)
    return cyc / eff, {"issue": instr / 4.0, "alu": alu / 2.0, "smem": wf}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("traces")
    ap.add_argument("--pairs", type=int, default=1)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    d = dict(np.load(args.traces))
    pairs = list(range(min(args.pairs, d["trace"].shape[0])))
    nblk_launch = 239 * 32640
    out = {}
    r0 = model_d0(d, pairs)
    # D0 instruction / ALU counts per block from its ncu capture (profiles/r2/ncu_opcodes_c3_v14.csv)
    r0.update(instr=168.3, alu=82.0)
    out["D0 (round-1 v14, measured instr)"] = r0
    for (tbx, tby, wx, wy) in [(8, 8, 8, 4), (16, 4, 16, 2), (16, 4, 8, 4), (32, 2, 32, 1), (8, 8, 4, 8)]:
        for pitch in (None, 128, 144):
            r = model_d1(d, pairs, tbx, tby, wx, wy, pitch=pitch)
            out[f"D1 tile {tbx}x{tby} warp {wx}x{wy} pitch {r['pitch']}"] = r
    for name, r in out.items():
        cyc, parts = floor(r["instr"], r["alu"], r["wf"])
        ms = nblk_launch * cyc / SM / CLK * 1e3
        r["floor_cycles_per_block"] = cyc
        r["bound_parts"] = parts
        r["c3_ms_at_80pct"] = ms
        print(f"{name:45s} lane-loads {r['lane_loads']:6.1f}  LDS {r['lds']:6.1f}  wf {r['wf']:6.1f}  "
              f"instr {r['instr']:6.1f}  alu {r['alu']:6.1f}  warp-passes/blk {r['warp_passes']:.3f}  "
              f"-> {cyc:5.1f} cyc/blk ({min(parts, key=lambda k: -parts[k])}), c3 {ms:.3f} ms")
    if args.json:
        json.dump(out, open(args.json, "w"), indent=1, default=float)
