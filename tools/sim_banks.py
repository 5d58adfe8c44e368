"""Offline model of the DCDS kernel's candidate-row shared-memory loads (the kernel is bound by
the L1 data pipe, profiles/r1c/SUMMARY.md).  Replays the per-pass traces of real searches
(tools/dump_traces.py -> me_dcds_trace_batch) through the warp structure of the ONE kernel
(16x4-block tiles, warp w = block row w of the tile, group g = block column g, G = 2 lanes)
and counts shared-memory wavefronts of every slot load under alternative layouts:
  wavefronts(LDS.32) = max over the 32 banks of the number of distinct words requested.

usage: python tools/sim_banks.py gpurun_out/traces_c3.npz
"""
import sys

import numpy as np

SLOTS = {2: [(-2, 0), (2, 0), (0, -1), (0, 1)], 3: [(-1, 0), (1, 0), (0, -2), (0, 2)],
         4: [(-1, 0), (1, 0)], 5: [(0, -1), (0, 1)]}


def decode(rec):
    rec = int(rec) & 0xFFFFFFFFFFFFFFFF
    pid, mask = (rec >> 8) & 0xF, (rec >> 12) & 0xFF
    cx, cy = (rec >> 20) & 0xFF, (rec >> 28) & 0xFF
    return pid, mask, cx - 256 if cx > 127 else cx, cy - 256 if cy > 127 else cy


def lane_words(layout, pitch, bofs, cpos_off, slot_off, B=8, G=2):
    """word addresses [lanes, loads] of one slot of one group under a layout"""
    o = bofs + cpos_off + slot_off
    if layout == "row":        # lane j: rows j, j+G, ...; B/4 + 1 words per row
        base = [(o + j * pitch) >> 2 for j in range(G)]
        return [[b + r * (G * pitch >> 2) + w for r in range(B // G) for w in range(B // 4 + 1)] for b in base]
    if layout == "rowpred":    # as row, the last word only when the row is unaligned
        base = [(o + j * pitch) >> 2 for j in range(G)]
        last = B // 4 if (o & 3) else -1
        return [[b + r * (G * pitch >> 2) + w if w != B // 4 or last >= 0 else -1
                 for r in range(B // G) for w in range(B // 4 + 1)] for b in base]
    if layout == "half":       # lane j: rows 4j .. 4j+3
        base = [(o + 4 * j * pitch) >> 2 for j in (0, 1)]
        return [[b + r * (pitch >> 2) + w for r in range(4) for w in range(3)] for b in base]
    if layout == "col":        # lane j: word j of all 8 rows (2 words per row)
        base = [(o + 4 * j) >> 2 for j in (0, 1)]
        return [[b + r * (pitch >> 2) + w for r in range(8) for w in range(2)] for b in base]
    raise ValueError(layout)


def simulate(d, layout="row", pitch=208, warp_shape=(16, 1), G=2, tby=4):
    tr, tl = d["trace"], d["tlen"]
    W, H, B, p = int(d["W"]), int(d["H"]), int(d["B"]), int(d["p"])
    nbx, nby = W // B, H // B
    wx, wy = warp_shape
    total_wf = total_lds = 0
    active_lanes = 0
    for pair in range(tr.shape[0]):
        for wy0 in range(0, nby - wy + 1, wy):
            for wx0 in range(0, nbx - wx + 1, wx):
                blocks = [(wy0 + a) * nbx + wx0 + b for a in range(wy) for b in range(wx)]
                # region offsets as in the kernel: tile rows of 4 blocks; the warp's blocks
                # sit at block rows lby within the tile, columns lbx
                recs = [[decode(tr[pair, blk, i]) for i in range(min(int(tl[pair, blk]), tr.shape[2]))]
                        for blk in blocks]
                npass = max(len(r) for r in recs)
                bofs = []
                for a in range(wy):
                    for b in range(wx):
                        lby = (wy0 + a) % tby
                        bofs.append((lby * B + p) * pitch + ((p + 15) & ~15) + b * B)
                for i in range(1, npass):
                    for k in range(4):
                        lanes = []
                        for g, r in enumerate(recs):
                            if i < len(r):
                                pid, mask, cx, cy = r[i]
                                if (mask >> k) & 1:
                                    dx, dy = SLOTS[pid][k]
                                    lanes += lane_words(layout, pitch, bofs[g], cy * pitch + cx, dy * pitch + dx, B, G)
                        if not lanes:
                            continue
                        L = np.array(lanes)  # [lanes, loads]
                        for q in range(L.shape[1]):
                            col = L[:, q]
                            col = col[col >= 0]       # predicated-off lanes issue no access
                            total_lds += 1
                            active_lanes += L.shape[0]
                            if col.size:
                                words = np.unique(col)
                                total_wf += np.bincount(words % 32, minlength=32).max()
    nblk = tr.shape[0] * nbx * nby
    return total_wf / nblk, total_lds / nblk, active_lanes / max(total_lds, 1)


if __name__ == "__main__":
    d = dict(np.load(sys.argv[1]))
    # subsample: the first 1/4 of each pair's block rows keeps the run short
    d["trace"] = d["trace"][:, : d["trace"].shape[1] // 4]
    d["tlen"] = d["tlen"][:, : d["tlen"].shape[1] // 4]
    d["H"] = int(d["H"]) // 4 // 32 * 32
    for layout, pitch, shape in [("row", 208, (16, 1)), ("row", 192, (16, 1)), ("row", 224, (16, 1)),
                                 ("row", 240, (16, 1)), ("row", 272, (16, 1)), ("half", 208, (16, 1)),
                                 ("col", 208, (16, 1)), ("row", 208, (8, 2)), ("col", 208, (8, 2))]:
        wf, lds, act = simulate(d, layout, pitch, shape)
        print(f"{layout:5s} pitch {pitch} warp {shape}: {wf:6.2f} wavefronts/block, {lds:6.2f} LDS/block, "
              f"{wf / lds:.2f} wf/LDS, {act:.1f} active lanes/LDS")
