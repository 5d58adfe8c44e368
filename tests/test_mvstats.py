"""MVP-statistics host arithmetic (paper_0806_0689_b200/mvstats.py) pinned by the paper's own
tables: fed the published distributions it must return the published derived numbers."""
import numpy as np

from paper_0806_0689_b200 import mvstats
from _golden import golden_matrix


def fig3_as_window():
    """Fig. 3's central 5x5 as a p = 2 window P[dy+2, dx+2]."""
    return golden_matrix("fig3_regions.txt", float)


def test_axis_shares_table2():
    """22.69% of the MVs on the horizontal axis, 7.42% on the vertical (centre excluded),
    from Table II (its cells are rounded to 1e-4, so +-2e-4)."""
    h, v = mvstats.axis_shares(golden_matrix("table2_mvp.txt", float))
    assert abs(h - 0.2269) < 2e-4 and abs(v - 0.0742) < 2e-4


def test_fig3_regional_masses():
    """P_square 0.8745, P_diamond 0.8557, P_cross 0.8315, P_3x3 0.7899, P_5x3 0.8248."""
    r = mvstats.regions(fig3_as_window())
    for k, v in [("square5", 0.8745), ("diamond5", 0.8557), ("cross5", 0.8315),
                 ("square3", 0.7899), ("flat_diamond5x3", 0.8248)]:
        assert abs(r[k] - v) < 3e-4, (k, r[k])


def test_eta1_table6():
    """Table VI from Fig. 3: HCSP 0.8248/7, cross 0.8315/9, 3x3 0.7899/9."""
    P = fig3_as_window()
    hcsp = [(0, 0), (-1, 0), (1, 0), (-2, 0), (2, 0), (0, -1), (0, 1)]
    cross = [(0, 0), (-1, 0), (1, 0), (-2, 0), (2, 0), (0, -1), (0, 1), (0, -2), (0, 2)]
    sq3 = [(dx, dy) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    assert abs(mvstats.eta1(P, hcsp) - 0.1178) < 1e-4
    assert abs(mvstats.eta1(P, cross) - 0.0924) < 1e-4
    assert abs(mvstats.eta1(P, sq3) - 0.0878) < 1e-4


def test_marginals_on_axis_match_table3():
    """Table III Bx(d) for |d| <= 2 is Fig. 3's centre row and By(d) its centre
    column (the same MVs): marginals() of the Fig. 3 window returns them."""
    m = mvstats.marginals(fig3_as_window())
    np.testing.assert_allclose(m["Bx"], [0.0151, 0.0718, 0.5805, 0.0562, 0.0440], atol=1e-9)
    np.testing.assert_allclose(m["By"], [0.0031, 0.0295, 0.5805, 0.0277, 0.0035], atol=1e-9)


def test_quarter_fold_of_table3():
    """Table II (quarter-folded) agrees with Table III: Bx(d) + Bx(-d) is Table II's row 0
    (e.g. 0.0151 + 0.0440 = 0.0591 at |d| = 2) and By(d) + By(-d) its column 0; folding a
    window built from them gives the same axis cells."""
    t2 = golden_matrix("table2_mvp.txt", float)
    bx = np.array([0.0042, 0.0013, 0.0028, 0.0037, 0.0049, 0.0151, 0.0718, 0.5805, 0.0562, 0.0440,
                   0.0121, 0.0035, 0.0026, 0.0013, 0.0034])
    by = np.array([0.0010, 0.0015, 0.0006, 0.0011, 0.0016, 0.0031, 0.0295, 0.5805, 0.0277, 0.0035,
                   0.0015, 0.0011, 0.0006, 0.0008, 0.0006])
    P = np.zeros((15, 15))
    P[7, :] = bx
    P[:, 7] += by
    P[7, 7] = 0.5805
    q = mvstats.quarter(P)
    np.testing.assert_allclose(q[0, :], t2[0, :], atol=2e-4)
    np.testing.assert_allclose(q[:, 0], t2[:, 0], atol=2e-4)


def test_ansp_weights():
    """ANSP of a constant map is the constant; Table II's weights sum to ~1."""
    t2 = golden_matrix("table2_mvp.txt", float)
    assert abs(t2.sum() - 1.0) < 5e-3
    assert abs(mvstats.ansp(np.full((15, 15), 25), t2) - 25.0) < 1e-12
