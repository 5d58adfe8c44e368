"""GPU parity of the compact visited set (DESIGN.md §7 "Compact visited set"): the 16x16 ONE
kernels keep a bmx x bmy bitmap window instead of the full +-p one; a search whose centre
leaves it is abandoned and its block searched again by the overflow pass (dcds_redo_kernel)
with the full bitmap.  The outputs must be the oracle's whichever path a block took.

ME_COMPACT=bmx,bmy forces small windows so that most searches overflow (both passes and
their hand-off are exercised on every content kind); the default (p >= 26) is checked on
large translations, against ME_COMPACT=0, in the packed record, and through the host-buffer
path (chunks on two streams sharing the overflow list)."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_0806_0689_b200 as me
from paper_0806_0689_b200 import synth

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0") if torch.cuda.is_available() else None


@pytest.fixture(scope="module", autouse=True)
def init():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    me.me_init(0)
    me.me_set_stream(torch.cuda.current_stream())
    yield
    os.environ.pop("ME_COMPACT", None)


def _content(kind, W, H, seed):
    if kind == "noise":
        return synth.random_pair(W, H, seed)
    if kind == "flat":
        return synth.flat_pair(W, H, 77)
    if kind == "binary":
        return synth.binary_pair(W, H, seed)
    tex = synth.texture(W, H, (3.0, 8.0), seed).numpy()
    if kind == "far":  # large translations: the searches travel far from the origin
        return synth.translated_pair(tex, 11 + seed % 9, -(5 + seed % 7))
    rng = np.random.default_rng(seed)
    return synth.translated_pair(tex, int(rng.integers(-6, 7)), int(rng.integers(-4, 5)))


def _search(frames, p, variant, packed=False):
    n, _, H, W = frames.shape
    nb = (W // 16) * (H // 16)
    if packed:
        mv = torch.zeros(n, nb, 2, dtype=torch.int8, device=DEV)
        sad = torch.zeros(n, nb, dtype=torch.int16, device=DEV)
        pts = torch.zeros(n, nb, dtype=torch.int16, device=DEV)
        st = torch.zeros(n, 3, dtype=torch.int64, device=DEV)
        me.me_dcds_batch_packed(frames, 16, p, mv, sad, pts, st)
        torch.cuda.synchronize()
        return (mv.cpu().numpy().astype(np.int16), sad.cpu().numpy().view(np.uint16).astype(np.uint32),
                pts.cpu().numpy().view(np.uint16), st.cpu().numpy().astype(np.uint64))
    mv, sad, pts, st = me.alloc_outputs(n, nb, DEV)
    (me.me_dcds_s_batch if variant else me.me_dcds_batch)(frames, 16, p, mv, sad, pts, st)
    torch.cuda.synchronize()
    return (mv.cpu().numpy(), sad.cpu().numpy().astype(np.uint32), pts.cpu().numpy().astype(np.uint16),
            st.cpu().numpy().astype(np.uint64))


def _check_oracle(host, p, variant, got):
    gmv, gsad, gpts, gst = got
    for t in range(host.shape[0]):
        cur, ref = host[t, 0], host[t, 1]
        omv, osad, opts = oracle.dcds(cur, ref, 16, p, variant)
        bad = np.flatnonzero((gmv[t] != omv).any(1) | (gsad[t] != osad) | (gpts[t] != opts))
        assert bad.size == 0, (f"pair {t} p={p} v={variant}: {bad.size} blocks differ, first {bad[:4]}: "
                               f"gpu {gmv[t][bad[0]]},{gsad[t][bad[0]]},{gpts[t][bad[0]]} "
                               f"oracle {omv[bad[0]]},{osad[bad[0]]},{opts[bad[0]]}")
        sse = oracle.mc_psnr(cur, ref, 16, omv)[1]
        assert tuple(int(x) for x in gst[t]) == (int(opts.astype(np.int64).sum()),
                                                 int(osad.astype(np.int64).sum()), int(sse))


# forced windows: (bmx, bmy) with 4 <= bmx, 2 <= bmy, both <= p - 2
FORCED = [((4, 2), 7), ((5, 3), 8), ((6, 6), 15), ((9, 4), 16), ((12, 10), 32), ((24, 20), 32),
          ((4, 30), 32), ((30, 2), 32)]


@pytest.mark.parametrize("win,p", FORCED, ids=[f"w{w[0]}x{w[1]}-p{p}" for w, p in FORCED])
@pytest.mark.parametrize("variant", [0, 1], ids=["dcds", "dcds_s"])
def test_forced_window_parity(monkeypatch, win, p, variant):
    monkeypatch.setenv("ME_COMPACT", f"{win[0]},{win[1]}")
    W, H = 208, 176  # 13 x 11 blocks: ragged 4x8 tiles in both directions
    kinds = ["far", "texture", "noise", "binary", "flat", "far"]
    host = np.stack([np.stack(_content(k, W, H, 31 * p + i)) for i, k in enumerate(kinds)])
    frames = torch.from_numpy(host).to(DEV)
    got = _search(frames, p, variant)
    nov = me.me_dcds_overflow_count()
    _check_oracle(host, p, variant, got)
    if win[0] <= 9:  # the far translations leave these windows
        assert nov > 0, "the overflow pass was not exercised"
    assert nov <= len(kinds) * (W // 16) * (H // 16)


def test_forced_window_tiny_frames(monkeypatch):
    """frames of one block / one block row / one block column (tiles clipped to the frame)"""
    monkeypatch.setenv("ME_COMPACT", "4,2")
    for (W, H) in [(16, 16), (64, 16), (16, 128), (48, 32)]:
        host = np.stack([np.stack(_content(k, W, H, 5 + i)) for i, k in enumerate(["far", "noise", "texture"])])
        got = _search(torch.from_numpy(host).to(DEV), 7, 0)
        _check_oracle(host, 7, 0, got)


# (window or None = default, p, ME_REC_CAP or None = default)
WARM = [(None, 32, None), (None, 32, 3), (None, 32, 0), ((6, 4), 12, None), ((5, 3), 16, 5), ((4, 2), 7, None)]


@pytest.mark.parametrize("win,p,cap", WARM, ids=[f"w{c[0]}-p{c[1]}-cap{c[2]}" for c in WARM])
@pytest.mark.parametrize("variant", [0, 1], ids=["dcds", "dcds_s"])
def test_warm_start_parity(monkeypatch, win, p, cap, variant):
    """abandoned interior searches continue in the overflow pass from their warm-start records
    (ME_REC_CAP: only the first few get one, the rest restart from the window origin): every
    output is still the oracle's"""
    if win is None:
        monkeypatch.delenv("ME_COMPACT", raising=False)
    else:
        monkeypatch.setenv("ME_COMPACT", f"{win[0]},{win[1]}")
    if cap is None:
        monkeypatch.delenv("ME_REC_CAP", raising=False)
    else:
        monkeypatch.setenv("ME_REC_CAP", str(cap))
    W, H = 320, 256
    kinds = ["far", "texture", "noise", "far", "binary", "flat"]
    host = np.stack([np.stack(_content(k, W, H, 7 * p + i)) for i, k in enumerate(kinds)])
    frames = torch.from_numpy(host).to(DEV)
    got = _search(frames, p, variant)
    nov = me.me_dcds_overflow_count()
    _check_oracle(host, p, variant, got)
    assert nov > 0, "nothing reached the overflow passes"


def test_invalid_forced_window_falls_back_to_full(monkeypatch):
    """an out-of-range ME_COMPACT window is ignored (full bitmap): no overflow list in use"""
    monkeypatch.setenv("ME_COMPACT", "3,2")  # bmx < 4
    host = np.stack([np.stack(_content("far", 128, 128, 3))])
    got = _search(torch.from_numpy(host).to(DEV), 7, 0)
    assert me.me_dcds_overflow_count() == 0
    _check_oracle(host, 7, 0, got)


@pytest.mark.parametrize("variant", [0, 1], ids=["dcds", "dcds_s"])
def test_default_window_p32_far_motion(monkeypatch, variant):
    """p = 32 uses the compact set by default; translations up to 31 px make searches
    leave the 51 x 45 window; parity with the oracle and with ME_COMPACT=0"""
    monkeypatch.delenv("ME_COMPACT", raising=False)
    W, H = 320, 256
    tex = synth.texture(W, H, (6.0, 12.0), 4242).numpy()
    shifts = [(29, 3), (-30, -2), (4, 27), (-26, -25), (12, -8), (0, 0)]
    host = np.stack([np.stack(synth.translated_pair(tex, dx, dy)) for dx, dy in shifts])
    frames = torch.from_numpy(host).to(DEV)
    got = _search(frames, 32, variant)
    nov = me.me_dcds_overflow_count()
    assert nov > 0, "expected searches to leave the default compact window"
    _check_oracle(host, 32, variant, got)
    monkeypatch.setenv("ME_COMPACT", "0")
    full = _search(frames, 32, variant)
    assert me.me_dcds_overflow_count() == 0
    for a, b in zip(got, full):
        np.testing.assert_array_equal(a, b)


def test_default_window_c4_pairs_packed_and_full():
    """c4 pairs: the default compact set, ME_COMPACT=0 and the packed record agree, and the
    overflow fraction is of the measured order (tools/excursion.py: 0.14 %)"""
    cfg = synth.CONFIGS["c4"]
    frames = synth.make_sequence(cfg, device=DEV, pairs=range(1, 9))
    os.environ.pop("ME_COMPACT", None)
    got = _search(frames, cfg.p, 0)
    nov = me.me_dcds_overflow_count()
    packed = _search(frames, cfg.p, 0, packed=True)
    os.environ["ME_COMPACT"] = "0"
    try:
        full = _search(frames, cfg.p, 0)
    finally:
        os.environ.pop("ME_COMPACT", None)
    for a, b in zip(got, full):
        np.testing.assert_array_equal(a, b)
    for a, b in zip(got, packed):
        np.testing.assert_array_equal(a, b)
    assert 0 < nov < 0.01 * frames.shape[0] * cfg.nb


def test_host_path_chunks_share_the_overflow_list():
    """me_dcds_batch_host at c4 (8 pairs per 128 MiB staging chunk, chunks alternating over
    two copy streams, each with its own overflow pass): equal to the device search"""
    cfg = synth.CONFIGS["c4"]
    n = 19
    os.environ.pop("ME_COMPACT", None)
    frames = synth.make_sequence(cfg, device=DEV, pairs=range(40, 40 + n))
    dev = _search(frames, cfg.p, 0)
    hfr = frames.cpu().pin_memory()
    hmv, hsad, hpts, hst = [x.pin_memory() for x in me.alloc_outputs(n, cfg.nb, "cpu")]
    me.me_dcds_batch_host(hfr, cfg.B, cfg.p, hmv, hsad, hpts, hst)
    np.testing.assert_array_equal(hmv.numpy(), dev[0])
    np.testing.assert_array_equal(hsad.numpy().astype(np.uint32), dev[1])
    np.testing.assert_array_equal(hpts.numpy().astype(np.uint16), dev[2])
    np.testing.assert_array_equal(hst.numpy().astype(np.uint64), dev[3])


def test_cuda_graph_capture_and_replay():
    """the compact path (memset, main kernel, two overflow passes) captured into a CUDA graph
    on torch's capture stream and replayed: outputs equal the eager call's"""
    os.environ.pop("ME_COMPACT", None)
    W, H = 320, 256
    tex = synth.texture(W, H, (6.0, 12.0), 777).numpy()
    host = np.stack([np.stack(synth.translated_pair(tex, dx, dy)) for dx, dy in [(30, 2), (-3, 1), (5, -28)]])
    frames = torch.from_numpy(host).to(DEV)
    eager = _search(frames, 32, 0)
    assert me.me_dcds_overflow_count() > 0
    n, nb = frames.shape[0], (W // 16) * (H // 16)
    mv, sad, pts, st = me.alloc_outputs(n, nb, DEV)
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g):
            me.me_set_stream(torch.cuda.current_stream())
            me.me_dcds_batch(frames, 16, 32, mv, sad, pts, st)
    finally:
        me.me_set_stream(torch.cuda.current_stream())
    for _ in range(2):
        mv.zero_(); sad.zero_(); pts.zero_()
        g.replay()
        torch.cuda.synchronize()
        got = (mv.cpu().numpy(), sad.cpu().numpy().astype(np.uint32), pts.cpu().numpy().astype(np.uint16),
               st.cpu().numpy().astype(np.uint64))
        for a, b in zip(got, eager):
            np.testing.assert_array_equal(a, b)
    # eager calls on another stream after the capture (the capture recorded no ordering event)
    side = torch.cuda.Stream()
    me.me_set_stream(side)
    try:
        with torch.cuda.stream(side):
            again = _search(frames, 32, 0)
    finally:
        me.me_set_stream(torch.cuda.current_stream())
    for a, b in zip(again, eager):
        np.testing.assert_array_equal(a, b)
    assert me.me_dcds_overflow_count() > 0
    again = _search(frames, 32, 0)
    for a, b in zip(again, eager):
        np.testing.assert_array_equal(a, b)
