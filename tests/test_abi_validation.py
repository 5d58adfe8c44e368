"""Argument validation of the C ABI (include/me.h), host only: every entry point checks its
arguments before any device work, so bad calls return ME_EINVAL / ME_EALIGN and a valid call
without me_init returns ME_ENOTINIT -- all without a GPU (the pointers are never touched).
me_init is never called in this process, which the ENOTINIT cases rely on."""
import ctypes

import pytest

from paper_0806_0689_b200 import me

OK, EINVAL, EALIGN, ENOTINIT = me.ME_OK, me.ME_EINVAL, me.ME_EALIGN, me.ME_ENOTINIT
A = 1 << 20          # a fake, 16-byte aligned device address (never dereferenced)
W, H = 64, 48        # 16-multiple frame


@pytest.fixture(scope="module")
def lib():
    L = me.load()
    if me._inited:
        pytest.skip("me_init already called in this process")
    return L


def batch_args(**kw):
    a = dict(cur=A, ref=A + W * H, stride=2 * W * H, n=3, W=W, H=H, B=16, p=7, mv=A + (1 << 24),
             sad=A + (2 << 24), pts=A + (3 << 24), stats=A + (4 << 24))
    a.update(kw)
    return (a["cur"], a["ref"], a["stride"], a["n"], a["W"], a["H"], a["B"], a["p"], a["mv"],
            a["sad"], a["pts"], a["stats"])


CASES = [
    ({}, ENOTINIT),
    ({"cur": 0}, EINVAL), ({"ref": 0}, EINVAL),
    ({"W": 0}, EINVAL), ({"H": -16}, EINVAL),
    ({"B": 4}, EINVAL), ({"B": 32}, EINVAL),
    ({"W": 72}, EINVAL),                      # not a multiple of B = 16
    ({"W": 40, "B": 8}, EALIGN),              # multiple of 8, not of 16
    ({"n": 0}, EINVAL), ({"n": 65536}, EINVAL),
    ({"p": 0}, EINVAL), ({"p": 33}, EINVAL),
    ({"mv": 0}, EINVAL), ({"sad": 0}, EINVAL), ({"pts": 0}, EINVAL),
    ({"cur": A + 4}, EALIGN), ({"ref": A + 8}, EALIGN),
    ({"stride": 2 * W * H + 4}, EALIGN),
    ({"stride": W * H - 16}, EINVAL),         # pairs overlap
    ({"mv": A + 2}, EALIGN), ({"sad": A + 2}, EALIGN), ({"pts": A + 1}, EALIGN),
    ({"stats": A + 4}, EALIGN),
    ({"stats": 0}, ENOTINIT),                 # stats are optional
]


@pytest.mark.parametrize("fn", ["me_dcds_batch", "me_dcds_s_batch", "me_fullsearch_batch"])
@pytest.mark.parametrize("kw,rc", CASES, ids=[str(c[0]) or "valid" for c in CASES])
def test_batch_validation(lib, fn, kw, rc):
    assert getattr(lib, fn)(*batch_args(**kw)) == rc


def test_bma_and_trace_validation(lib):
    assert lib.me_bma_batch(6, *batch_args()) == EINVAL        # unknown algorithm
    assert lib.me_bma_batch(-1, *batch_args()) == EINVAL
    for alg in me.ALGS.values():
        assert lib.me_bma_batch(alg, *batch_args()) == ENOTINIT
    args = batch_args()[:-1]
    assert lib.me_dcds_trace_batch(2, *args, A, 16, A) == EINVAL      # variant
    assert lib.me_dcds_trace_batch(0, *args, A, 0, A) == EINVAL       # cap
    assert lib.me_dcds_trace_batch(0, *args, A, 256, A) == EINVAL
    assert lib.me_dcds_trace_batch(0, *args, 0, 16, A) == EINVAL      # NULL trace
    assert lib.me_dcds_trace_batch(0, *args, A + 4, 16, A) == EALIGN
    assert lib.me_dcds_trace_batch(0, *args, A, 16, A + 1) == EALIGN
    assert lib.me_dcds_trace_batch(1, *args, A, 16, A) == ENOTINIT


def test_other_entry_points(lib):
    assert lib.me_ideal_nsp_map(0, 0, A, A, A) == EINVAL
    assert lib.me_ideal_nsp_map(9, 7, A, A, A) == EINVAL
    assert lib.me_ideal_nsp_map(0, 7, 0, A, A) == EINVAL
    assert lib.me_ideal_nsp_map(0, 7, A + 2, A, A) == EALIGN
    assert lib.me_ideal_nsp_map(0, 7, A, None, None) == ENOTINIT
    assert lib.me_mv_hist(A, -1, 7, A) == EINVAL
    assert lib.me_mv_hist(None, 10, 7, A) == EINVAL
    assert lib.me_mv_hist(None, 0, 7, A) == ENOTINIT               # empty field: no mv needed
    assert lib.me_mv_hist(A, 10, 7, A + 4) == EALIGN
    assert lib.me_mc_sse_batch(A, A + W * H, 2 * W * H, 3, W, H, 16, A, A) == ENOTINIT
    assert lib.me_mc_sse_batch(A, A + W * H, 2 * W * H, 3, W, H, 16, 0, A) == EINVAL
    assert lib.me_quality_batch(A, A, 0, 5, A) == EINVAL
    assert lib.me_quality_batch(A, A, 2, 5, A) == ENOTINIT
    psnr = ctypes.c_double()
    assert lib.me_mc_psnr(A, A + W * H, W, H, 16, A, ctypes.byref(psnr), None) == ENOTINIT
    assert lib.me_set_stream(None) == ENOTINIT
    assert lib.me_strerror(EINVAL)  # every status has a message
