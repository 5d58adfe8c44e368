"""Thin Python binding of libme.so (include/me.h) -- argument marshalling only.

Every step of the hot path runs in the sm_100a kernels of libme.so; this module only turns
torch tensors into pointers/sizes and status codes into exceptions.  There is no CPU
fallback: if libme.so is missing or the device is not an sm_100 GPU the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# ME_LIBRARY selects another in-tree build (tests: libme_debug.so, the ME_DEBUG bounds checks)
SO_PATH = os.environ.get("ME_LIBRARY") or os.path.join(_HERE, "libme.so")

ME_OK, ME_EINVAL, ME_EALIGN, ME_ENOTINIT, ME_ECUDA, ME_ENOMEM = 0, -1, -2, -3, -4, -5

# Exported symbols (kept in sync with include/me.h; tests/test_abi.py checks both ways).
SYMBOLS = (
    "me_init", "me_set_stream", "me_dcds", "me_fullsearch", "me_mc_psnr", "me_dcds_batch",
    "me_dcds_s_batch", "me_fullsearch_batch", "me_mc_sse_batch", "me_dcds_batch_host",
    "me_launch_count", "me_strerror", "me_shutdown", "me_quality_batch", "me_bma_batch",
    "me_ideal_nsp_map", "me_mv_hist", "me_dcds_trace_batch", "me_dcds_batch_packed",
    "me_dcds_overflow_count",
)

# me_alg ids (include/me.h)
ALGS = {"dcds": 0, "dcds_s": 1, "cds": 2, "ds": 3, "hexbs_h": 4, "hexbs_v": 5}


class MEError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libme status {status}: {msg}")
        self.status = status


_lib = None


def load() -> ctypes.CDLL:
    """Load the in-tree libme.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise ImportError(f"{SO_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(SO_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    search = [vp, vp, i32, i32, i32, i32, vp, vp, vp]
    batch = [vp, vp, i64, i32, i32, i32, i32, i32, vp, vp, vp, vp]
    L.me_init.argtypes = [i32]
    L.me_set_stream.argtypes = [vp]
    L.me_dcds.argtypes = search
    L.me_fullsearch.argtypes = search
    L.me_mc_psnr.argtypes = [vp, vp, i32, i32, i32, vp, ctypes.POINTER(ctypes.c_double),
                             ctypes.POINTER(ctypes.c_uint64)]
    L.me_dcds_batch.argtypes = batch
    L.me_dcds_s_batch.argtypes = batch
    L.me_dcds_batch_packed.argtypes = batch
    L.me_fullsearch_batch.argtypes = batch
    L.me_dcds_batch_host.argtypes = batch
    L.me_mc_sse_batch.argtypes = [vp, vp, i64, i32, i32, i32, i32, vp, vp]
    L.me_quality_batch.argtypes = [vp, vp, i32, i32, vp]
    L.me_bma_batch.argtypes = [i32] + batch
    L.me_ideal_nsp_map.argtypes = [i32, i32, vp, vp, vp]
    L.me_mv_hist.argtypes = [vp, i64, i32, vp]
    L.me_dcds_trace_batch.argtypes = [i32] + batch[:-1] + [vp, i32, vp]
    L.me_dcds_overflow_count.argtypes = [vp]
    L.me_launch_count.argtypes = []
    L.me_launch_count.restype = i64
    L.me_strerror.argtypes = [i32]
    L.me_strerror.restype = ctypes.c_char_p
    L.me_shutdown.argtypes = []
    L.me_shutdown.restype = None
    for n in SYMBOLS:
        if n not in ("me_launch_count", "me_strerror", "me_shutdown"):
            getattr(L, n).restype = i32
    _lib = L
    return L


def _check(rc: int):
    if rc != ME_OK:
        raise MEError(rc, load().me_strerror(rc).decode())


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


_inited = {}


def me_init(device: int = 0):
    _check(load().me_init(int(device)))
    _inited[device] = True


def me_set_stream(stream=None):
    """stream: a torch.cuda.Stream (or None for the legacy default stream)."""
    _check(load().me_set_stream(None if stream is None else stream.cuda_stream))


def _frame_dims(cur):
    if cur.dtype != torch.uint8:
        raise TypeError("frames must be uint8")
    return cur.shape[-1], cur.shape[-2]


def alloc_outputs(npairs: int, nb: int, device, stats: bool = True):
    """Output tensors of a batched search: mv [n, nb, 2] int16, sad [n, nb] int32 (holding
    uint32), points [n, nb] int16 (holding uint16), stats [n, 3] int64 (holding uint64)."""
    mv = torch.empty(npairs, nb, 2, dtype=torch.int16, device=device)
    sad = torch.empty(npairs, nb, dtype=torch.int32, device=device)
    pts = torch.empty(npairs, nb, dtype=torch.int16, device=device)
    st = torch.empty(npairs, 3, dtype=torch.int64, device=device) if stats else None
    return mv, sad, pts, st


def me_dcds(cur, ref, block, p, mv_out, sad_out, points_out):
    W, H = _frame_dims(cur)
    _check(load().me_dcds(_ptr(cur), _ptr(ref), W, H, block, p, _ptr(mv_out), _ptr(sad_out),
                          _ptr(points_out)))


def me_fullsearch(cur, ref, block, p, mv_out, sad_out, points_out):
    W, H = _frame_dims(cur)
    _check(load().me_fullsearch(_ptr(cur), _ptr(ref), W, H, block, p, _ptr(mv_out),
                                _ptr(sad_out), _ptr(points_out)))


def me_mc_psnr(cur, ref, block, mv):
    """Returns (psnr_db, sse).  Synchronises the library stream."""
    W, H = _frame_dims(cur)
    ps = ctypes.c_double()
    sse = ctypes.c_uint64()
    _check(load().me_mc_psnr(_ptr(cur), _ptr(ref), W, H, block, _ptr(mv), ctypes.byref(ps),
                             ctypes.byref(sse)))
    return ps.value, sse.value


def _batch(fn, frames, block, p, mv, sad, pts, stats):
    """frames: [npairs, 2, H, W] uint8 (cur = [:, 0], ref = [:, 1])."""
    if frames.dim() != 4 or frames.shape[1] != 2 or not frames.is_contiguous():
        raise ValueError("frames must be a contiguous [npairs, 2, H, W] uint8 tensor")
    n, _, H, W = frames.shape
    stride = 2 * H * W
    base = _ptr(frames)
    _check(fn(base, base + H * W, stride, n, W, H, block, p, _ptr(mv), _ptr(sad), _ptr(pts),
              _ptr(stats)))


def me_dcds_batch(frames, block, p, mv, sad, pts, stats=None):
    _batch(load().me_dcds_batch, frames, block, p, mv, sad, pts, stats)


def me_dcds_batch_packed(frames, block, p, mv, sad, pts, stats=None):
    """me_dcds_batch into the 6-byte transport record: mv [n, nb, 2] int8, sad [n, nb] int16
    (holding uint16), pts [n, nb] int16 (holding uint16), stats [n, 3] int64."""
    _batch(load().me_dcds_batch_packed, frames, block, p, mv, sad, pts, stats)


def me_dcds_s_batch(frames, block, p, mv, sad, pts, stats=None):
    _batch(load().me_dcds_s_batch, frames, block, p, mv, sad, pts, stats)


def me_fullsearch_batch(frames, block, p, mv, sad, pts, stats=None):
    _batch(load().me_fullsearch_batch, frames, block, p, mv, sad, pts, stats)


def me_bma_batch(alg, frames, block, p, mv, sad, pts, stats=None):
    """Any block-matching algorithm of :data:`ALGS` (name or id) over a batch of pairs."""
    a = ALGS[alg] if isinstance(alg, str) else int(alg)
    fn = load().me_bma_batch
    _batch(lambda *args: fn(a, *args), frames, block, p, mv, sad, pts, stats)


def me_dcds_trace_batch(variant, frames, block, p, mv, sad, pts, trace, trace_len):
    """DCDS (variant 0) / DCDS^S (1) with a per-pass trace (include/me.h): trace is an int64
    tensor [npairs, nb, cap] (cap <= 255), trace_len an int16 tensor [npairs, nb]."""
    if trace.dtype != torch.int64 or trace.dim() != 3 or not trace.is_contiguous():
        raise ValueError("trace must be a contiguous [npairs, nb, cap] int64 tensor")
    cap = trace.shape[-1]
    fn = load().me_dcds_trace_batch
    _batch(lambda *a: fn(int(variant), *a[:-1], _ptr(trace), cap, _ptr(trace_len)),
           frames, block, p, mv, sad, pts, None)


# slot offsets (dx, dy) of the traced patterns (reading C7; pattern ids of include/me.h)
_TRACE_SLOTS = {
    15: ((0, 0), (-1, 0), (1, 0), (-2, 0), (2, 0), (0, -1), (0, 1)),
    2: ((-2, 0), (2, 0), (0, -1), (0, 1)),
    3: ((-1, 0), (1, 0), (0, -2), (0, 2)),
    4: ((-1, 0), (1, 0)),
    5: ((0, -1), (0, 1)),
}
# pattern id -> trace kind (0 HCSP, 1 HDSP, 2 VDSP, 3 middle point)
_TRACE_KIND = {15: 0, 2: 1, 3: 2, 4: 3, 5: 3}


def decode_trace(records, n):
    """Expand n trace records of one block into the scored points, in scoring order, as
    (step, dx, dy, kind) tuples (step 0 = Step 1; kind 0 HCSP, 1 HDSP, 2 VDSP, 3 middle)."""
    out = []
    for r in [int(x) & 0xFFFFFFFFFFFFFFFF for x in records[:n]]:
        step, pid, mask = r & 0xFF, (r >> 8) & 0xF, (r >> 12) & 0xFF
        cx, cy = ((r >> 20) & 0xFF), ((r >> 28) & 0xFF)
        cx, cy = cx - 256 if cx > 127 else cx, cy - 256 if cy > 127 else cy
        for k, (ox, oy) in enumerate(_TRACE_SLOTS[pid]):
            if (mask >> k) & 1:
                out.append((step, cx + ox, cy + oy, _TRACE_KIND[pid]))
    return out


def me_ideal_nsp_map(alg, p, device="cuda"):
    """Ideal-condition NSP map (Table VII) of an algorithm for every true MV of the
    +-p window: (nsp, mvx, mvy) int32 device tensors of shape [2p+1, 2p+1] indexed [ty+p, tx+p]."""
    a = ALGS[alg] if isinstance(alg, str) else int(alg)
    side = 2 * p + 1
    out = [torch.empty(side, side, dtype=torch.int32, device=device) for _ in range(3)]
    _check(load().me_ideal_nsp_map(a, p, *(_ptr(t) for t in out)))
    return tuple(out)


def me_mv_hist(mv, p, hist=None):
    """Histogram [2p+1, 2p+1] (uint64 as int64) of an int16 MV field [..., 2] on the device."""
    side = 2 * p + 1
    if hist is None:
        hist = torch.empty(side, side, dtype=torch.int64, device=mv.device)
    n = mv.numel() // 2
    _check(load().me_mv_hist(_ptr(mv), n, p, _ptr(hist)))
    return hist


def me_dcds_batch_host(frames, block, p, mv, sad, pts, stats=None):
    """Host-buffer variant: frames and outputs are CPU tensors (pinned for full bandwidth)."""
    _batch(load().me_dcds_batch_host, frames, block, p, mv, sad, pts, stats)


def me_mc_sse_batch(frames, block, mv, sse):
    n, _, H, W = frames.shape
    base = _ptr(frames)
    _check(load().me_mc_sse_batch(base, base + H * W, 2 * H * W, n, W, H, block, _ptr(mv), _ptr(sse)))


def me_quality_batch(mv, mv_fs, out=None):
    """Per pair (hits, sum of Euclidean distances) of mv against mv_fs ([n, nb, 2] int16)."""
    n, nb = mv.shape[0], mv.shape[1]
    if out is None:
        out = torch.empty(n, 2, dtype=torch.float64, device=mv.device)
    _check(load().me_quality_batch(_ptr(mv), _ptr(mv_fs), n, nb, _ptr(out)))
    return out


def me_dcds_overflow_count() -> int:
    """Blocks of the last DCDS / DCDS^S batch that the compact visited set handed to the
    overflow pass (include/me.h; 0 when that call did not use the compact set)."""
    n = ctypes.c_uint64()
    _check(load().me_dcds_overflow_count(ctypes.byref(n)))
    return n.value


def me_launch_count() -> int:
    return int(load().me_launch_count())


def me_shutdown():
    load().me_shutdown()
    _inited.clear()
