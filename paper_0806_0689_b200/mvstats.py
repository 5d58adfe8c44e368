"""MVP statistics of a motion field: host arithmetic on the
(2p+1)^2 MV histogram that the GPU reduces (me_mv_hist).  Indexing: P[dy+p, dx+p].

  quarter(P)        Table II layout: [|dy|, |dx|], every sign combination accumulated
  axis_shares(T)    share of MVs on the horizontal / vertical axis, centre excluded
                    ("22.69% ... horizontal ... 7.42% ... vertical")
  marginals(P)      Table III: Ax(d), Ay(d) (all MVs accumulated in the vertical / horizontal
                    direction) and Bx(d), By(d) (MVs on the horizontal / vertical axis), d=-p..p
  regions(P)        Fig. 3 / P:110 regional masses of the central 5x5: square, diamond, cross,
                    3x3 square and the 5x3 flat diamond
  eta1(P, pts)      Eq. 7 / Table VI: first-step search efficiency P_1 / n_1 of a pattern
  ansp(nsp, T)      Table VIII: average NSP over the window under the weights T (quarter map)
"""
from __future__ import annotations

import numpy as np


def normalise(hist) -> np.ndarray:
    h = np.asarray(hist, dtype=np.float64)
    s = h.sum()
    return h / s if s > 0 else h


def quarter(P: np.ndarray) -> np.ndarray:
    p = (P.shape[0] - 1) // 2
    q = np.zeros((p + 1, p + 1))
    for dy in range(-p, p + 1):
        for dx in range(-p, p + 1):
            q[abs(dy), abs(dx)] += P[dy + p, dx + p]
    return q


def axis_shares(T: np.ndarray):
    """(horizontal, vertical) share from a Table-II-layout quarter map."""
    return float(T[0, 1:].sum()), float(T[1:, 0].sum())


def marginals(P: np.ndarray):
    p = (P.shape[0] - 1) // 2
    return {"Ax": P.sum(axis=0), "Ay": P.sum(axis=1), "Bx": P[p, :].copy(), "By": P[:, p].copy(),
            "d": np.arange(-p, p + 1)}


REGIONS = {
    "square5": lambda dx, dy: abs(dx) <= 2 and abs(dy) <= 2,
    "diamond5": lambda dx, dy: abs(dx) + abs(dy) <= 2,
    "cross5": lambda dx, dy: (dx == 0 and abs(dy) <= 2) or (dy == 0 and abs(dx) <= 2),
    "square3": lambda dx, dy: abs(dx) <= 1 and abs(dy) <= 1,
    "flat_diamond5x3": lambda dx, dy: (dy == 0 and abs(dx) <= 2) or (abs(dy) == 1 and dx == 0),
}


def regions(P: np.ndarray):
    p = (P.shape[0] - 1) // 2
    out = {}
    for name, inside in REGIONS.items():
        out[name] = float(sum(P[dy + p, dx + p] for dy in range(-min(p, 2), min(p, 2) + 1)
                              for dx in range(-min(p, 2), min(p, 2) + 1) if inside(dx, dy)))
    return out


def eta1(P: np.ndarray, pts) -> float:
    p = (P.shape[0] - 1) // 2
    pts = list(pts)
    return float(sum(P[dy + p, dx + p] for dx, dy in pts)) / len(pts)


def ansp(nsp: np.ndarray, T: np.ndarray) -> float:
    """nsp: full (2p+1)^2 ideal map (sign-symmetric); T: Table-II-layout weights."""
    p = (nsp.shape[0] - 1) // 2
    q = np.asarray(nsp, dtype=np.float64)[p:, p:][: T.shape[0], : T.shape[1]]
    return float((T * q).sum() / T.sum())
