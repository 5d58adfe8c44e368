"""CPU oracle for the DCDS hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_0806_0689_b200``) never imports it; the two share no code.

Thin ctypes wrapper around ``oracle/liboracle.so`` (plain single-threaded C, ``oracle.c``),
plus numpy conveniences.  Every function of the C file cites the PAPER.md passage it
follows; see ``oracle.h``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

# The flags are stated in DESIGN.md (CPU baseline): -O2, auto-vectorisation left on.
CFLAGS = ["-O2", "-std=c99", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C; no intrinsics)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None
COST_FN = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_void_p)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        i16p = ctypes.POINTER(ctypes.c_int16)
        u16p = ctypes.POINTER(ctypes.c_uint16)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        ip = ctypes.POINTER(ctypes.c_int)
        dp = ctypes.POINTER(ctypes.c_double)
        c_int = ctypes.c_int
        L.oracle_sad.argtypes = [u8p, u8p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, u32p]
        L.oracle_sse_block.argtypes = [u8p, u8p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, u64p]
        L.oracle_dcds.argtypes = [u8p, u8p, c_int, c_int, c_int, c_int, c_int, i16p, u32p, u16p]
        L.oracle_fullsearch.argtypes = [u8p, u8p, c_int, c_int, c_int, c_int, i16p, u32p, u16p]
        L.oracle_dcds_block.argtypes = [u8p, u8p, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                        i16p, u32p, u16p]
        L.oracle_fullsearch_block.argtypes = [u8p, u8p, c_int, c_int, c_int, c_int, c_int, c_int,
                                              i16p, u32p, u16p]
        L.oracle_mc_psnr.argtypes = [u8p, u8p, c_int, c_int, c_int, i16p, dp, u64p]
        L.oracle_dcds_cost.argtypes = [COST_FN, ctypes.c_void_p, c_int, c_int, ip, ip, dp, ip, ip, c_int, ip]
        L.oracle_ideal_nsp_map.argtypes = [c_int, c_int, ip, ip, ip]
        L.oracle_quality.argtypes = [i16p, i16p, c_int, ip, dp]
        for f in (L.oracle_sad, L.oracle_sse_block, L.oracle_dcds, L.oracle_fullsearch,
                  L.oracle_mc_psnr, L.oracle_dcds_cost, L.oracle_ideal_nsp_map,
                  L.oracle_dcds_block, L.oracle_fullsearch_block, L.oracle_quality):
            f.restype = c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _frames(cur, ref):
    cur = np.ascontiguousarray(cur, dtype=np.uint8)
    ref = np.ascontiguousarray(ref, dtype=np.uint8)
    if cur.shape != ref.shape or cur.ndim != 2:
        raise ValueError("cur and ref must be equal-shape 2-D uint8 frames")
    return cur, ref


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"{what}: invalid arguments (rc={rc})")


def sad(cur, ref, B, bx, by, dx, dy) -> int:
    cur, ref = _frames(cur, ref)
    H, W = cur.shape
    out = ctypes.c_uint32()
    _check(lib().oracle_sad(_ptr(cur, ctypes.c_uint8), _ptr(ref, ctypes.c_uint8), W, H, B,
                            bx, by, dx, dy, ctypes.byref(out)), "oracle_sad")
    return out.value


def sse_block(cur, ref, B, bx, by, dx, dy) -> int:
    cur, ref = _frames(cur, ref)
    H, W = cur.shape
    out = ctypes.c_uint64()
    _check(lib().oracle_sse_block(_ptr(cur, ctypes.c_uint8), _ptr(ref, ctypes.c_uint8), W, H, B,
                                  bx, by, dx, dy, ctypes.byref(out)), "oracle_sse_block")
    return out.value


def _search(fn, cur, ref, B, p, *extra):
    cur, ref = _frames(cur, ref)
    H, W = cur.shape
    nb = (W // B) * (H // B) if (W % B == 0 and H % B == 0) else 0
    mv = np.zeros((max(nb, 1), 2), np.int16)
    sad_ = np.zeros(max(nb, 1), np.uint32)
    pts = np.zeros(max(nb, 1), np.uint16)
    _check(fn(_ptr(cur, ctypes.c_uint8), _ptr(ref, ctypes.c_uint8), W, H, B, p, *extra,
              _ptr(mv, ctypes.c_int16), _ptr(sad_, ctypes.c_uint32), _ptr(pts, ctypes.c_uint16)),
           fn.__name__)
    return mv[:nb], sad_[:nb], pts[:nb]


# Algorithm ids of the C oracle (oracle.h): DCDS, DCDS^S and the paper's comparison
# BMAs on the same machinery (readings C23-C26).
ALGS = {"dcds": 0, "dcds_s": 1, "cds": 2, "ds": 3, "hexbs_h": 4, "hexbs_v": 5}


def bma(cur, ref, B, p, alg: str):
    """Any block-matching search of :data:`ALGS` over every block: (mv, sad, points)."""
    return dcds(cur, ref, B, p, ALGS[alg])


def bma_block(cur, ref, B, p, bx, by, alg: str):
    """Single-block version of :func:`bma`: ((dx, dy), sad, points)."""
    return dcds_block(cur, ref, B, p, bx, by, ALGS[alg])


def dcds(cur, ref, B, p, variant: int = 0):
    """DCDS over every block: returns (mv[nb,2] int16, sad[nb] u32, points[nb] u16)."""
    return _search(lib().oracle_dcds, cur, ref, B, p, variant)


def fullsearch(cur, ref, B, p):
    """Full search: returns (mv, sad, points) like :func:`dcds`."""
    return _search(lib().oracle_fullsearch, cur, ref, B, p)


def _block(fn, cur, ref, B, p, bx, by, *extra):
    cur, ref = _frames(cur, ref)
    H, W = cur.shape
    mv = np.zeros(2, np.int16)
    s = np.zeros(1, np.uint32)
    n = np.zeros(1, np.uint16)
    _check(fn(_ptr(cur, ctypes.c_uint8), _ptr(ref, ctypes.c_uint8), W, H, B, p, *extra, bx, by,
              _ptr(mv, ctypes.c_int16), _ptr(s, ctypes.c_uint32), _ptr(n, ctypes.c_uint16)),
           fn.__name__)
    return (int(mv[0]), int(mv[1])), int(s[0]), int(n[0])


def dcds_block(cur, ref, B, p, bx, by, variant: int = 0):
    """DCDS of the single block at (bx, by): ((dx, dy), sad, points)."""
    return _block(lib().oracle_dcds_block, cur, ref, B, p, bx, by, variant)


def fullsearch_block(cur, ref, B, p, bx, by):
    """Full search of the single block at (bx, by): ((dx, dy), sad, points)."""
    return _block(lib().oracle_fullsearch_block, cur, ref, B, p, bx, by)


def mc_psnr(cur, ref, B, mv):
    """Motion-compensated (psnr_db, sse) (P:342 aspect 4)."""
    cur, ref = _frames(cur, ref)
    H, W = cur.shape
    mv = np.ascontiguousarray(mv, dtype=np.int16).reshape(-1, 2)
    if W % B or H % B or mv.shape[0] != (W // B) * (H // B):
        raise ValueError("mc_psnr: mv field does not match the frame")
    ps = ctypes.c_double()
    sse = ctypes.c_uint64()
    _check(lib().oracle_mc_psnr(_ptr(cur, ctypes.c_uint8), _ptr(ref, ctypes.c_uint8), W, H, B,
                                _ptr(mv, ctypes.c_int16), ctypes.byref(ps), ctypes.byref(sse)),
           "oracle_mc_psnr")
    return ps.value, sse.value


def dcds_cost(cost, p, variant: int = 0, trace_cap: int = 4096):
    """DCDS on an injected cost function ``cost(dx, dy) -> float``.

    Returns (mv, cost, points, trace) where trace is a list of (step, dx, dy, kind)."""
    cb = COST_FN(lambda dx, dy, _ctx: float(cost(dx, dy)))
    mx, my, pts, tl = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    c = ctypes.c_double()
    tr = np.zeros((trace_cap, 4), np.int32)
    _check(lib().oracle_dcds_cost(cb, None, p, variant, ctypes.byref(mx), ctypes.byref(my),
                                  ctypes.byref(c), ctypes.byref(pts),
                                  _ptr(tr, ctypes.c_int), trace_cap, ctypes.byref(tl)),
           "oracle_dcds_cost")
    n = min(tl.value, trace_cap)
    return (mx.value, my.value), c.value, pts.value, [tuple(int(v) for v in r) for r in tr[:n]]


def ideal_nsp_map(p, variant: int = 0):
    """NSP and found MV for every true-MV placement on the ideal surface (Table VII).

    Returns (nsp[2p+1, 2p+1], mvx, mvy), indexed [ty+p, tx+p]."""
    side = 2 * p + 1
    nsp = np.zeros(side * side, np.int32)
    mx = np.zeros(side * side, np.int32)
    my = np.zeros(side * side, np.int32)
    _check(lib().oracle_ideal_nsp_map(p, variant, _ptr(nsp, ctypes.c_int), _ptr(mx, ctypes.c_int),
                                      _ptr(my, ctypes.c_int)), "oracle_ideal_nsp_map")
    return nsp.reshape(side, side), mx.reshape(side, side), my.reshape(side, side)


def quality(mv, mv_fs):
    """(hits, sum of Euclidean distances) of an MV field [nb, 2] against the FS field
    (P:342 aspects 5-6)."""
    mv = np.ascontiguousarray(mv, dtype=np.int16)
    mv_fs = np.ascontiguousarray(mv_fs, dtype=np.int16)
    if mv.shape != mv_fs.shape or mv.ndim != 2 or mv.shape[1] != 2:
        raise ValueError("mv and mv_fs must be equal-shape [nb, 2] fields")
    h, d = ctypes.c_int(), ctypes.c_double()
    _check(lib().oracle_quality(_ptr(mv, ctypes.c_int16), _ptr(mv_fs, ctypes.c_int16), mv.shape[0],
                                ctypes.byref(h), ctypes.byref(d)), "oracle_quality")
    return h.value, d.value
