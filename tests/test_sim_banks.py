"""The shared-memory bank model (tools/sim_banks.py) that chose the 8x8 region pitch, pinned
on hand-computed cases: one warp of 16 groups (G = 2) at the same candidate (coherent motion)
and a single group."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import sim_banks  # noqa: E402


def rec(step, pid, mask, cx, cy):
    return step | (pid << 8) | (mask << 12) | ((cx & 0xFF) << 20) | ((cy & 0xFF) << 28)


def one_warp(nblocks, slot_mask):
    """16 blocks in one row, every block: Step 1 then one HDSP pass at (0,0) with slot_mask"""
    W, H, B, p = 128, 32, 8, 16
    nb = (W // B) * (H // B)
    tr = np.zeros((1, nb, 4), np.int64)
    tl = np.zeros((1, nb), np.int16)
    for b in range(nblocks):
        tr[0, b, 0] = rec(0, 15, 0x7F, 0, 0)
        tr[0, b, 1] = rec(1, 2, slot_mask, 0, 0)
        tl[0, b] = 2
    return {"trace": tr, "tlen": tl, "W": W, "H": 8, "B": B, "p": p}


def test_single_group_loads_are_conflict_free():
    d = one_warp(1, 0b0001)
    wf, lds, act = sim_banks.simulate(d, "row", 192, (16, 1))
    # one slot: 4 rows x 3 words = 12 loads, 2 lanes 16 banks apart: one wavefront each
    nblk = 16
    assert lds * nblk == 12 and wf * nblk == 12 and act == 2


def test_coherent_warp_two_way_conflicts():
    d = one_warp(16, 0b0001)
    for pitch, expect in ((192, 2), (208, 2), (256, 2)):
        wf, lds, act = sim_banks.simulate(d, "row", pitch, (16, 1))
        # 32 lanes: lane 0 of the 16 groups on the 16 even banks (8 bytes = 2 banks apart),
        # lane 1 one row further -- for any 16-byte-multiple pitch also on even banks
        assert act == 32 and wf / lds == expect, (pitch, wf / lds)
    wf, lds, _ = sim_banks.simulate(d, "col", 192, (16, 1))
    assert wf / lds == 1   # a group's two lanes on adjacent words: all 32 banks
