"""Oracle pins for the paper's comparison BMAs: CDS, DS, h-/v-HEXBS.

The source papers of these algorithms are not in the container; the oracle follows the
readings C23-C26 of DESIGN.md and is pinned here by the paper's own numbers:
Table VII's CDS and DS blocks (P:307-324, 64 integers each, exact), the first-step pattern
masses of Table VI / Fig. 3, Table VIII distribution 2 and
invariants (true MV on the unimodal surface, FS dominance, transposition symmetry).
"""
import math

import numpy as np
import pytest

import oracle
from paper_0806_0689_b200 import synth
from _golden import golden_matrix, load_golden

pytestmark = pytest.mark.filterwarnings("ignore")


def euclid(t):
    return lambda dx, dy: float(np.hypot(dx - t[0], dy - t[1]))


@pytest.mark.parametrize("alg,fixture", [("cds", "table7_cds.txt"), ("ds", "table7_ds.txt")])
def test_table7_competitor_blocks(alg, fixture):
    """Table VII: the ideal-condition NSP of CDS and DS at every true MV of the
    quarter window equals the published integers exactly (64/64)."""
    nsp, mx, my = oracle.ideal_nsp_map(7, oracle.ALGS[alg])
    np.testing.assert_array_equal(nsp[7:, 7:], golden_matrix(fixture, int))


@pytest.mark.parametrize("alg", ["cds", "ds"])
@pytest.mark.parametrize("p", [7, 15, 32])
def test_unimodal_true_mv_found(alg, p):
    """On the unimodal surface of P:299-301 CDS and DS end on the true MV everywhere."""
    nsp, mx, my = oracle.ideal_nsp_map(p, oracle.ALGS[alg])
    ty, tx = np.mgrid[-p:p + 1, -p:p + 1]
    assert (mx == tx).all() and (my == ty).all()


def test_hexbs_vertical_is_transposed_horizontal():
    """v-HEXBS (Fig. 2b) is h-HEXBS (Fig. 2a) turned by 90 degrees: its ideal NSP map is
    the transpose, and both find the true MV at the same (transposed) placements."""
    h, hx, hy = oracle.ideal_nsp_map(7, oracle.ALGS["hexbs_h"])
    v, vx, vy = oracle.ideal_nsp_map(7, oracle.ALGS["hexbs_v"])
    np.testing.assert_array_equal(v, h.T)
    ty, tx = np.mgrid[-7:8, -7:8]
    hit_h = (hx == tx) & (hy == ty)
    hit_v = (vx == tx) & (vy == ty)
    np.testing.assert_array_equal(hit_v, hit_h.T)


def _first_step_points(alg):
    """Offsets scored in the first step (trace pass 0) on a surface that never moves."""
    _, _, _, tr = oracle.dcds_cost(euclid((0, 0)), 7, oracle.ALGS[alg])
    return sorted({(dx, dy) for step, dx, dy, kind in tr if step == 0})


@pytest.mark.parametrize("alg,mass,n", [("dcds", 0.8248, 7), ("cds", 0.8315, 9),
                                        ("ds", 0.6705, 9), ("hexbs_h", 0.6457, 7)])
def test_first_step_pattern_mass(alg, mass, n):
    """Table VI: eta_1 = P_1 / n_1 of each algorithm's first pattern, with P_1 the
    Fig. 3 probability mass under the pattern; the four-digit values of the paper
    are matched to its rounding (+-2e-4: Fig. 3 cells are themselves rounded)."""
    fig3 = golden_matrix("fig3_regions.txt", float)
    pts = _first_step_points(alg)
    assert len(pts) == n
    got = sum(fig3[dy + 2, dx + 2] for dx, dy in pts)
    assert abs(got - mass) <= 2e-4, (alg, got)


def _ansp(alg):
    t2 = golden_matrix("table2_mvp.txt", float)
    nsp, _, _ = oracle.ideal_nsp_map(7, oracle.ALGS[alg])
    q = nsp[7:, 7:]
    assert (q == nsp[7:, 7::-1]).all() and (q == nsp[7::-1, 7:]).all()
    return float((t2 * q).sum() / t2.sum())


def test_table8_distribution2_competitors():
    """Table VIII distribution 2 (Table II weights): CDS 12.5 and DS 14.8 are matched
    (12.524 and 14.849 before the paper's 0.1 rounding).  HEXBS prints 12.1; this reading
    gives 12.167 for every point order (a recorded 0.07 discrepancy -- weak pin)."""
    printed = {r[0]: float(r[1]) for r in load_golden("table8_ansp.txt")}
    printed = {k: v for k, v in printed.items() if k.endswith("2")}
    assert abs(_ansp("cds") - printed["CDS_distribution2"]) < 0.05
    assert abs(_ansp("ds") - printed["DS_distribution2"]) <= 0.05 + 1e-9
    assert abs(_ansp("hexbs_h") - printed["HEXBS_distribution2"]) < 0.1
    # the paper's ordering of the four algorithms holds: DCDS < HEXBS < CDS < DS
    assert _ansp("dcds") < _ansp("hexbs_h") < _ansp("cds") < _ansp("ds")


@pytest.mark.parametrize("alg,zero_nsp", [("cds", 9), ("ds", 13), ("hexbs_h", 11), ("hexbs_v", 11)])
def test_zero_motion_points(alg, zero_nsp):
    """Identical frames: every block stops on (0,0) after the first pattern (+ the final small
    pattern for DS / HEXBS): CDS 9 (first-step stop), DS 9 + 4 = 13 (Table VII DS (0,0)),
    HEXBS 7 + 4 = 11.  Border blocks too (reading C9)."""
    f = synth.random_pair(48, 32, 3)[0]
    mv, sad, pts = oracle.bma(f, f, 8, 7, alg)
    assert (mv == 0).all() and (sad == 0).all() and (pts == zero_nsp).all()


@pytest.mark.parametrize("alg", ["cds", "ds", "hexbs_h", "hexbs_v"])
def test_dominated_by_full_search_and_consistent(alg):
    """Per block SAD_alg >= SAD_FS (FS is the exhaustive minimum); the returned SAD is
    the SAD at the returned MV; points are within [first pattern, (2p+1)^2]."""
    cur, ref = synth.random_pair(64, 48, 11)
    tex = synth.texture(64, 48, (2.0,), 5).numpy()
    for c, r in [(cur, ref), (synth.translated_pair(tex, 2, -1)[0], tex)]:
        mv, sad, pts = oracle.bma(c, r, 16, 7, alg)
        _, sfs, _ = oracle.fullsearch(c, r, 16, 7)
        assert (sad >= sfs).all()
        for i in range(len(sad)):
            bx, by = (i % 4) * 16, (i // 4) * 16
            assert oracle.sad(c, r, 16, bx, by, int(mv[i, 0]), int(mv[i, 1])) == sad[i]
        assert (pts >= 9 if alg in ("cds", "ds") else pts >= 11).all() and (pts <= 225).all()


@pytest.mark.parametrize("B", [16, 8])
@pytest.mark.parametrize("alg,fixture", [("cds", "table7_cds.txt"), ("ds", "table7_ds.txt")])
def test_pixel_ideal_mosaic_reproduces_table7_competitors(B, alg, fixture):
    """The constructed frames whose SAD surface is B*|q-t|^2 + K give Table VII through the
    pixel SAD path too (SURVEY finding 5)."""
    cur, ref, tile, off, blocks = synth.ideal_mosaic(B, 7)
    mv, sad, pts = oracle.bma(cur, ref, B, 7, alg)
    np.testing.assert_array_equal(pts[blocks][7:, 7:], golden_matrix(fixture, int))


# Fig. 7's six parts are missing; this concentric reading of them -- |d|^2 = 0, [1,5),
# [5,8), [8,17), [17,29), >= 29 -- is weak (one of many partitions that fit).
_PART_EDGES = (1, 5, 8, 17, 29)


def _part(dx, dy):
    d = dx * dx + dy * dy
    return 0 if d == 0 else 1 + sum(d >= e for e in _PART_EDGES[1:])


def _ansp_dist1(alg):
    """Table VIII distribution 1: sum_i P_i * mean NSP over part i of the +-7 window."""
    nsp, _, _ = oracle.ideal_nsp_map(7, oracle.ALGS[alg])
    s, n = np.zeros(6), np.zeros(6)
    for ty in range(-7, 8):
        for tx in range(-7, 8):
            s[_part(tx, ty)] += nsp[ty + 7, tx + 7]
            n[_part(tx, ty)] += 1
    return float((np.array([0.4, 0.2, 0.2, 0.1, 0.1, 0.0]) * s / n).sum())


def test_table8_hexbs_reading():
    """HEXBS (reading C25) against BOTH rows of Table VIII.  The printed HEXBS
    values are this reading's ANSP cut to one decimal in both distributions (13.163 -> 13.1,
    12.163 -> 12.1), while DCDS, CDS and DS match the rounded values (DCDS 11.679 -> 11.7 and
    9.683 -> 9.7 rule out truncation for every column).  A different HEXBS reading would have to
    lower the ANSP by 0.014..0.113 in BOTH distributions at once; the readings tried (DESIGN.md
    C25: 8-point final square, the 2/3-point enhanced inner search, no memo, non-strict ties)
    move it by -2.7..+4 instead.  So the reading stands, pinned weakly: to the printed digits
    under truncation, and to within 0.07 under rounding."""
    printed = {r[0]: float(r[1]) for r in load_golden("table8_ansp.txt")}
    d1 = {a: _ansp_dist1(a) for a in ("dcds", "cds", "ds", "hexbs_h")}
    d2 = {a: _ansp(a) for a in ("dcds", "cds", "ds", "hexbs_h")}
    names = {"dcds": "DCDS", "cds": "CDS", "ds": "DS", "hexbs_h": "HEXBS"}
    for a in ("dcds", "cds", "ds"):
        assert round(d1[a], 1) == printed[names[a] + "_distribution1"], (a, d1[a])
        assert round(d2[a], 1) == printed[names[a] + "_distribution2"], (a, d2[a])
    for d, row in ((d1, "_distribution1"), (d2, "_distribution2")):
        assert math.floor(d["hexbs_h"] * 10) / 10 == printed["HEXBS" + row], d["hexbs_h"]
        assert abs(d["hexbs_h"] - printed["HEXBS" + row]) < 0.07
