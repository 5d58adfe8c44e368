"""Host logic of the trace build: decoding of me_dcds_trace_batch records (include/me.h)."""
import numpy as np

from paper_0806_0689_b200.me import decode_trace


def rec(step, pid, mask, cx, cy, best):
    return step | (pid << 8) | (mask << 12) | ((cx & 0xFF) << 20) | ((cy & 0xFF) << 28) | (best << 36)


def test_decode_trace_expands_slots_in_pattern_order():
    r = np.array([rec(0, 15, 0x7F, 0, 0, 900),      # HCSP, all 7 points
                  rec(1, 2, 0b1110, -1, 0, 800),    # HDSP at (-1,0): (-2,0) already visited
                  rec(2, 3, 0b0101, -1, -1, 700),   # VDSP at (-1,-1): slots 0 and 2
                  rec(3, 5, 0b10, -1, -1, 650)],    # vertical middle points: (0,+1) only
                 dtype=np.uint64).view(np.int64)
    got = decode_trace(r, 4)
    assert got == [(0, 0, 0, 0), (0, -1, 0, 0), (0, 1, 0, 0), (0, -2, 0, 0), (0, 2, 0, 0),
                   (0, 0, -1, 0), (0, 0, 1, 0),
                   (1, 1, 0, 1), (1, -1, -1, 1), (1, -1, 1, 1),
                   (2, -2, -1, 2), (2, -1, -3, 2),
                   (3, -1, 0, 3)]


def test_decode_trace_empty_passes_and_count():
    r = np.array([rec(0, 15, 0x67, 0, 0, 5), rec(1, 4, 0, 0, 0, 5), rec(2, 4, 3, 0, 0, 5)],
                 dtype=np.uint64).view(np.int64)
    # p = 1: (-2,0) and (2,0) infeasible; a halfway stop runs an empty Step-4 pass
    assert decode_trace(r, 2) == [(0, 0, 0, 0), (0, -1, 0, 0), (0, 1, 0, 0), (0, 0, -1, 0),
                                  (0, 0, 1, 0)]
    assert decode_trace(r, 0) == []
    assert decode_trace(r, 3)[-2:] == [(2, -1, 0, 3), (2, 1, 0, 3)]


def test_decode_trace_extreme_centres():
    r = np.array([rec(7, 3, 0b1111, -32, 32, 65535)], dtype=np.uint64).view(np.int64)
    assert decode_trace(r, 1) == [(7, -33, 32, 2), (7, -31, 32, 2), (7, -32, 30, 2), (7, -32, 34, 2)]
