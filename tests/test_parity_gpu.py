"""GPU parity: libme.so (sm_100a) against the CPU oracle, through the C ABI.

Integer outputs (mv, SAD, points, SSE) must be bit-identical; PSNR within 1e-9 dB
(BASELINE.json north_star).  Sizes span several tiles with ragged tails; the full-size
configs c3/c4 run in the bench's launch configuration (one batched launch over all pairs)
and are checked on whole sampled pairs plus sampled blocks the oracle computes one by one.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle
import paper_0806_0689_b200 as me
from paper_0806_0689_b200 import synth
from _golden import golden_matrix

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0") if torch.cuda.is_available() else None


@pytest.fixture(scope="module", autouse=True)
def init():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    me.me_init(0)
    me.me_set_stream(torch.cuda.current_stream())
    yield


def to_np(t):
    return t.cpu().numpy()


def gpu_search(frames, B, p, kind="dcds"):
    n, _, H, W = frames.shape
    nb = (W // B) * (H // B)
    mv, sad, pts, st = me.alloc_outputs(n, nb, frames.device)
    fn = {"dcds": me.me_dcds_batch, "dcds_s": me.me_dcds_s_batch, "fs": me.me_fullsearch_batch}.get(kind)
    if fn is None:  # a comparison BMA
        me.me_bma_batch(kind, frames, B, p, mv, sad, pts, st)
    else:
        fn(frames, B, p, mv, sad, pts, st)
    torch.cuda.synchronize()
    return (to_np(mv), to_np(sad).astype(np.uint32), to_np(pts).astype(np.uint16),
            to_np(st).astype(np.uint64))


def assert_pair_equal(host_pair, B, p, mv, sad, pts, kind="dcds", tag=""):
    cur, ref = host_pair[0], host_pair[1]
    if kind == "fs":
        omv, osad, opts = oracle.fullsearch(cur, ref, B, p)
    else:
        omv, osad, opts = oracle.bma(cur, ref, B, p, kind)
    bad = np.flatnonzero((mv != omv).any(1) | (sad != osad) | (pts != opts))
    assert bad.size == 0, (f"{tag} {kind} B={B} p={p}: {bad.size} blocks differ, first {bad[:5]}: "
                           f"gpu {mv[bad[0]]},{sad[bad[0]]},{pts[bad[0]]} "
                           f"oracle {omv[bad[0]]},{osad[bad[0]]},{opts[bad[0]]}")
    return omv, osad, opts


def frames_from_np(cur, ref):
    return torch.from_numpy(np.stack([cur, ref])[None].copy()).to(DEV)


# ---------------------------------------------------------------------------------------

def test_smoke_entry():
    import __graft_entry__
    __graft_entry__.smoke()


def test_c0_c1_all_pairs_dcds_fs_psnr():
    for name in ("c0", "c1"):
        cfg = synth.CONFIGS[name]
        fr = synth.make_sequence(cfg, device=DEV)
        host = to_np(fr)
        mv, sad, pts, st = gpu_search(fr, cfg.B, cfg.p)
        fmv, fsad, fpts, fst = gpu_search(fr, cfg.B, cfg.p, "fs")
        sse_dev = torch.empty(cfg.npairs, dtype=torch.int64, device=DEV)
        me.me_mc_sse_batch(fr, cfg.B, torch.from_numpy(mv).to(DEV), sse_dev)
        sse_dev = to_np(sse_dev)
        for t in range(cfg.npairs):
            omv, osad, opts = assert_pair_equal(host[t], cfg.B, cfg.p, mv[t], sad[t], pts[t], tag=f"{name}/{t}")
            assert_pair_equal(host[t], cfg.B, cfg.p, fmv[t], fsad[t], fpts[t], "fs", tag=f"{name}/{t}")
            ops, osse = oracle.mc_psnr(host[t, 0], host[t, 1], cfg.B, omv)
            assert st[t].tolist() == [int(opts.sum()), int(osad.sum()), osse]
            assert int(sse_dev[t]) == osse
            ps, sse = me.me_mc_psnr(fr[t, 0], fr[t, 1], cfg.B, torch.from_numpy(mv[t]).to(DEV))
            assert sse == osse and abs(ps - ops) <= 1e-9
            fo = oracle.fullsearch(host[t, 0], host[t, 1], cfg.B, cfg.p)
            assert fst[t].tolist() == [int(fo[2].astype(np.int64).sum()), int(fo[1].astype(np.int64).sum()),
                                       oracle.mc_psnr(host[t, 0], host[t, 1], cfg.B, fo[0])[1]]
            assert (fsad[t] <= sad[t]).all()


def test_c2_pairs():
    cfg = synth.CONFIGS["c2"]
    pairs = list(range(1, 300, 13))
    fr = synth.make_sequence(cfg, device=DEV, pairs=pairs)
    host = to_np(fr)
    mv, sad, pts, st = gpu_search(fr, cfg.B, cfg.p)
    for k in range(len(pairs)):
        assert_pair_equal(host[k], cfg.B, cfg.p, mv[k], sad[k], pts[k], tag=f"c2/{pairs[k]}")
    fmv, fsad, fpts, _ = gpu_search(fr[:3].contiguous(), cfg.B, cfg.p, "fs")
    for k in range(3):
        assert_pair_equal(host[k], cfg.B, cfg.p, fmv[k], fsad[k], fpts[k], "fs", tag=f"c2/{pairs[k]}")


def _sampled_full_size(name, n_full, n_blocks, fs_pairs, seed):
    """Full sequence on the GPU in one batched launch (the bench's configuration); whole
    pairs and random blocks checked against the oracle; stats checked against the outputs
    at every pair (a property that holds at any size)."""
    cfg = synth.CONFIGS[name]
    fr = synth.make_sequence(cfg, device=DEV)
    mv, sad, pts, st = gpu_search(fr, cfg.B, cfg.p)
    # stats == sums of the per-block outputs, every pair
    np.testing.assert_array_equal(st[:, 0], pts.astype(np.int64).sum(1))
    np.testing.assert_array_equal(st[:, 1], sad.astype(np.int64).sum(1))
    sse_dev = torch.empty(cfg.npairs, dtype=torch.int64, device=DEV)
    me.me_mc_sse_batch(fr, cfg.B, torch.from_numpy(mv).to(DEV), sse_dev)
    np.testing.assert_array_equal(st[:, 2], to_np(sse_dev))
    assert (pts >= 7).all()   # border blocks too (reading C9), p >= 2
    rng = np.random.default_rng(seed)
    full = sorted(set([0, cfg.npairs - 1] + list(rng.integers(0, cfg.npairs, n_full - 2))))
    for t in full:
        host = to_np(fr[t])
        omv, osad, opts = assert_pair_equal(host, cfg.B, cfg.p, mv[t], sad[t], pts[t], tag=f"{name}/{t}")
        assert int(st[t, 2]) == oracle.mc_psnr(host[0], host[1], cfg.B, omv)[1]
    nbx = cfg.W // cfg.B
    ts = rng.integers(0, cfg.npairs, n_blocks)
    bs = rng.integers(0, cfg.nb, n_blocks)
    cache = {}
    for t, b in zip(ts, bs):
        if t not in cache:
            cache[t] = to_np(fr[t])
        host = cache[t]
        bx, by = (b % nbx) * cfg.B, (b // nbx) * cfg.B
        omv, osad, opts = oracle.dcds_block(host[0], host[1], cfg.B, cfg.p, bx, by)
        assert (tuple(mv[t, b]), sad[t, b], pts[t, b]) == (omv, osad, opts), (t, b)
    # FS on a few pairs, sampled blocks (the oracle FS is (2p+1)^2 B^2 per block)
    fsel = fr[fs_pairs].contiguous()
    fmv, fsad, fpts, _ = gpu_search(fsel, cfg.B, cfg.p, "fs")
    for k, t in enumerate(fs_pairs):
        host = to_np(fr[t])
        for b in list(rng.integers(0, cfg.nb, 40)) + [0, nbx - 1, cfg.nb - nbx, cfg.nb - 1]:
            bx, by = (b % nbx) * cfg.B, (b // nbx) * cfg.B
            omv, osad, opts = oracle.fullsearch_block(host[0], host[1], cfg.B, cfg.p, bx, by)
            assert (tuple(fmv[k, b]), fsad[k, b], fpts[k, b]) == (omv, osad, opts), (t, b)
            assert fsad[k, b] <= sad[t, b]
    del fr
    torch.cuda.empty_cache()


def test_c3_full_size_sampled():
    _sampled_full_size("c3", 4, 3000, [0, 118], seed=3)


@pytest.mark.slow
def test_c4_full_size_sampled():
    _sampled_full_size("c4", 2, 1000, [0], seed=4)


@pytest.mark.parametrize("B", [16, 8])
def test_ideal_mosaic_table7(B):
    """Pixel-ideal mosaic (SAD = B|q-t|^2 + K): the GPU kernel reproduces Table VII
     and the full ideal NSP map, with the true MV everywhere."""
    cur, ref, tile, off, blocks = synth.ideal_mosaic(B, 7)
    mv, sad, pts, _ = gpu_search(frames_from_np(cur, ref), B, 7)
    got = pts[0][blocks]
    np.testing.assert_array_equal(got[7:, 7:], golden_matrix("table7_dcds.txt", int))
    nsp, mx, my = oracle.ideal_nsp_map(7)
    np.testing.assert_array_equal(got, nsp)
    np.testing.assert_array_equal(mv[0][blocks][..., 0], mx)
    np.testing.assert_array_equal(mv[0][blocks][..., 1], my)
    assert_pair_equal(np.stack([cur, ref]), B, 7, mv[0], sad[0], pts[0], tag="mosaic")


SPECIAL = [
    ("flat", 176, 144), ("binary", 176, 144), ("random", 176, 144), ("texture", 176, 144),
    ("border16", 48, 48), ("border8", 32, 24), ("tiny", 16, 16), ("wide", 400, 32),
]


def special_pair(kind, W, H, seed=0):
    if kind == "flat":
        return synth.flat_pair(W, H, 77)
    if kind == "binary":
        return synth.binary_pair(W, H, seed + 1)
    if kind == "texture":
        tex = synth.texture(W, H, (2.0,), seed + 2).numpy()
        return synth.translated_pair(tex, 3, -1)
    return synth.random_pair(W, H, seed + 3)


@pytest.mark.parametrize("kind,W,H", SPECIAL)
@pytest.mark.parametrize("B", [16, 8])
@pytest.mark.parametrize("p", [1, 2, 7, 15, 16, 32])
def test_special_inputs(kind, W, H, B, p):
    if W % B or H % B:
        pytest.skip("frame not divisible by block")
    cur, ref = special_pair(kind, W, H, seed=p * 3 + B)
    fr = frames_from_np(cur, ref)
    host = np.stack([cur, ref])
    for k in ("dcds", "dcds_s"):
        mv, sad, pts, st = gpu_search(fr, B, p, k)
        assert_pair_equal(host, B, p, mv[0], sad[0], pts[0], k, tag=kind)
    if p <= 16 or W * H <= 48 * 48:
        mv, sad, pts, st = gpu_search(fr, B, p, "fs")
        assert_pair_equal(host, B, p, mv[0], sad[0], pts[0], "fs", tag=kind)


def test_dcds_s_c1():
    cfg = synth.CONFIGS["c1"]
    fr = synth.make_sequence(cfg, device=DEV, pairs=range(1, 12))
    host = to_np(fr)
    mv, sad, pts, _ = gpu_search(fr, cfg.B, cfg.p, "dcds_s")
    dmv, dsad, dpts, _ = gpu_search(fr, cfg.B, cfg.p, "dcds")
    for t in range(fr.shape[0]):
        assert_pair_equal(host[t], cfg.B, cfg.p, mv[t], sad[t], pts[t], "dcds_s")
    assert (pts <= dpts).all()


def test_single_pair_entry_points():
    cfg = synth.CONFIGS["c0"]
    fr = synth.make_sequence(cfg, device=DEV)
    cur, ref = fr[0, 0], fr[0, 1]
    mv = torch.empty(cfg.nb, 2, dtype=torch.int16, device=DEV)
    sad = torch.empty(cfg.nb, dtype=torch.int32, device=DEV)
    pts = torch.empty(cfg.nb, dtype=torch.int16, device=DEV)
    me.me_dcds(cur, ref, cfg.B, cfg.p, mv, sad, pts)
    torch.cuda.synchronize()
    host = to_np(fr[0])
    assert_pair_equal(host, cfg.B, cfg.p, to_np(mv), to_np(sad).astype(np.uint32),
                      to_np(pts).astype(np.uint16))
    me.me_fullsearch(cur, ref, cfg.B, cfg.p, mv, sad, pts)
    torch.cuda.synchronize()
    assert_pair_equal(host, cfg.B, cfg.p, to_np(mv), to_np(sad).astype(np.uint32),
                      to_np(pts).astype(np.uint16), "fs")
    ps, sse = me.me_mc_psnr(ref, ref, cfg.B, torch.zeros(cfg.nb, 2, dtype=torch.int16, device=DEV))
    assert sse == 0 and math.isinf(ps)


def test_host_buffer_variant_matches_device():
    cfg = synth.CONFIGS["c1"]
    fr = synth.make_sequence(cfg, device=DEV)
    mv, sad, pts, st = gpu_search(fr, cfg.B, cfg.p)
    hfr = fr.cpu().pin_memory()
    hmv, hsad, hpts, hst = me.alloc_outputs(cfg.npairs, cfg.nb, "cpu")
    me.me_dcds_batch_host(hfr, cfg.B, cfg.p, hmv, hsad, hpts, hst)
    np.testing.assert_array_equal(hmv.numpy(), mv)
    np.testing.assert_array_equal(hsad.numpy().astype(np.uint32), sad)
    np.testing.assert_array_equal(hpts.numpy().astype(np.uint16), pts)
    np.testing.assert_array_equal(hst.numpy().astype(np.uint64), st)


def test_host_buffer_variant_chunks_and_padded_stride():
    """me_dcds_batch_host over several staging chunks (128 MiB of frames per chunk: 32 c3 pairs)
    with a host pair stride larger than 2*W*H (padding between pairs): equal to the device
    search of the same pairs."""
    import ctypes
    cfg = synth.CONFIGS["c3"]
    n = 35
    fr = synth.make_sequence(cfg, device=DEV, pairs=range(1, n + 1))
    mv, sad, pts, st = gpu_search(fr, cfg.B, cfg.p)
    fsz = cfg.W * cfg.H
    stride = 2 * fsz + 4096 + 7  # padded, odd: the ABI copies each frame on its own
    host = torch.zeros(n * stride + 64, dtype=torch.uint8).pin_memory()
    hf = fr.cpu().reshape(n, 2 * fsz)
    for t in range(n):
        host[t * stride: t * stride + fsz] = hf[t, :fsz]
        host[t * stride + fsz + 5: t * stride + 2 * fsz + 5] = hf[t, fsz:]
    hmv, hsad, hpts, hst = [x.pin_memory() for x in me.alloc_outputs(n, cfg.nb, "cpu")]
    L = me.load()
    base = host.data_ptr()
    rc = L.me_dcds_batch_host(base, base + fsz + 5, stride, n, cfg.W, cfg.H, cfg.B, cfg.p,
                              hmv.data_ptr(), hsad.data_ptr(), hpts.data_ptr(), hst.data_ptr())
    assert rc == 0, L.me_strerror(rc)
    np.testing.assert_array_equal(hmv.numpy(), mv)
    np.testing.assert_array_equal(hsad.numpy().astype(np.uint32), sad)
    np.testing.assert_array_equal(hpts.numpy().astype(np.uint16), pts)
    np.testing.assert_array_equal(hst.numpy().astype(np.uint64), st)


def test_host_buffer_variant_unrelated_single_pair():
    """me_dcds_batch_host with npairs == 1 and cur / ref in two unrelated host buffers (the
    ABI copies each frame on its own, never the span between them), odd pointer
    offsets, and a re-init cycle (me_shutdown + me_init re-allocates the staging)."""
    import ctypes
    cfg = synth.CONFIGS["c0"]
    fr = synth.make_sequence(cfg, device=DEV).cpu().numpy()
    # the two frames far apart and at odd byte offsets inside their buffers
    bc = np.zeros(cfg.W * cfg.H + 7, np.uint8)
    br = np.zeros(cfg.W * cfg.H + 3 + (1 << 20), np.uint8)
    cur = bc[7:]
    ref = br[3 + (1 << 20):]
    cur[:] = fr[0, 0].ravel()
    ref[:] = fr[0, 1].ravel()
    omv, osad, opts = oracle.dcds(fr[0, 0], fr[0, 1], cfg.B, cfg.p)
    for cycle in range(2):
        if cycle:
            me.load().me_shutdown()
            me.me_init(0)
            me.me_set_stream(torch.cuda.current_stream())
        hmv, hsad, hpts, hst = me.alloc_outputs(1, cfg.nb, "cpu")
        L = me.load()
        rc = L.me_dcds_batch_host(cur.ctypes.data, ref.ctypes.data, 0, 1, cfg.W, cfg.H, cfg.B, cfg.p,
                                  hmv.data_ptr(), hsad.data_ptr(), hpts.data_ptr(), hst.data_ptr())
        assert rc == 0, L.me_strerror(rc)
        np.testing.assert_array_equal(hmv[0].numpy(), omv)
        np.testing.assert_array_equal(hsad[0].numpy().astype(np.uint32), osad)
        np.testing.assert_array_equal(hpts[0].numpy().astype(np.uint16), opts)
        assert int(hst[0, 0]) == int(opts.sum()) and int(hst[0, 1]) == int(osad.sum())


def test_user_stream_and_launch_count():
    cfg = synth.CONFIGS["c1"]
    fr = synth.make_sequence(cfg, device=DEV, pairs=[1, 2])
    s = torch.cuda.Stream()
    n0 = me.me_launch_count()
    with torch.cuda.stream(s):
        me.me_set_stream(s)
        out = me.alloc_outputs(2, cfg.nb, DEV)
        me.me_dcds_batch(fr, cfg.B, cfg.p, *out)
    s.synchronize()
    me.me_set_stream(torch.cuda.current_stream())
    assert me.me_launch_count() == n0 + 1
    ref = gpu_search(fr, cfg.B, cfg.p)
    np.testing.assert_array_equal(to_np(out[0]), ref[0])


def test_errors_raise():
    fr = torch.zeros(1, 2, 32, 40, dtype=torch.uint8, device=DEV)
    out = me.alloc_outputs(1, 20, DEV)
    with pytest.raises(me.MEError):
        me.me_dcds_batch(fr, 16, 7, *out)     # 40 % 16 != 0


def test_nccl_gather_single_rank():
    """The NCCL gather path of bench.py (world size 1 on one GPU: the collective runs, and the
    gathered fields equal the local ones byte for byte)."""
    import socket
    import torch.distributed as dist
    from paper_0806_0689_b200 import dist as mdist
    if dist.is_initialized():
        pytest.skip("process group already initialised")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=DEV)
    try:
        cfg = synth.CONFIGS["c1"]
        fr = synth.make_sequence(cfg, device=DEV, pairs=range(1, 6))
        out = me.alloc_outputs(5, cfg.nb, DEV)
        me.me_dcds_batch(fr, cfg.B, cfg.p, *out)
        g = mdist.gather_fields(*out, 5)
        for a, b in zip(g, out):
            assert torch.equal(a, b)
    finally:
        dist.destroy_process_group()


def test_quality_kernel_examples_and_parity():
    """me_quality_batch: S:480-488 examples (field vs itself -> (0, 1); one of two blocks off by
    (1,0) -> (0.5, 0.5); all off by (3,4) -> (5, 0)) and c1 DCDS-vs-FS against the oracle's
    quality function (oracle_quality) pair by pair."""
    z = torch.zeros(1, 2, 2, dtype=torch.int16, device=DEV)
    one = z.clone()
    one[0, 1, 0] = 1
    far = z.clone()
    far[..., 0] = 3
    far[..., 1] = 4
    q = me.me_quality_batch(torch.cat([z, one, far]), torch.cat([z, z, z])).cpu().numpy()
    np.testing.assert_allclose(q[:, 0] / 2, [1.0, 0.5, 0.0])
    np.testing.assert_allclose(q[:, 1] / 2, [0.0, 0.5, 5.0], rtol=1e-15)
    cfg = synth.CONFIGS["c1"]
    fr = synth.make_sequence(cfg, device=DEV)
    mv, _, _, _ = gpu_search(fr, cfg.B, cfg.p)
    fmv, _, _, _ = gpu_search(fr, cfg.B, cfg.p, "fs")
    q = me.me_quality_batch(torch.from_numpy(mv).to(DEV), torch.from_numpy(fmv).to(DEV)).cpu().numpy()
    for t in range(mv.shape[0]):  # against the oracle's quality function, pair by pair
        h, dist = oracle.quality(mv[t], fmv[t])
        assert q[t, 0] == h and abs(q[t, 1] - dist) <= 1e-9 * max(1.0, dist)
    from paper_0806_0689_b200 import report
    rep = report.compare_dcds_fs(fr, cfg.B, cfg.p)
    assert rep["FS"]["prob"] == 1.0 and rep["FS"]["dist"] == 0.0 and rep["FS"]["nsp"] == 225.0
    assert rep["FS"]["mad"] <= rep["DCDS"]["mad"] and rep["DCDS"]["nsp"] < 225.0


# ---------------------------------------------------------------------------------------
# Comparison BMAs: CDS, DS, h-/v-HEXBS through me_bma_batch.
# ---------------------------------------------------------------------------------------
BMAS = ["cds", "ds", "hexbs_h", "hexbs_v"]


@pytest.mark.parametrize("alg", BMAS)
def test_bma_c0_c1_c2(alg):
    for name, pairs in (("c0", None), ("c1", range(0, 29, 4)), ("c2", range(1, 300, 37))):
        cfg = synth.CONFIGS[name]
        fr = synth.make_sequence(cfg, device=DEV, pairs=pairs)
        host = to_np(fr)
        mv, sad, pts, st = gpu_search(fr, cfg.B, cfg.p, alg)
        for t in range(fr.shape[0]):
            omv, osad, opts = assert_pair_equal(host[t], cfg.B, cfg.p, mv[t], sad[t], pts[t], alg,
                                                tag=f"{name}/{t}")
            _, osse = oracle.mc_psnr(host[t, 0], host[t, 1], cfg.B, omv)
            assert st[t].tolist() == [int(opts.astype(np.int64).sum()), int(osad.astype(np.int64).sum()), osse]


@pytest.mark.parametrize("alg", BMAS)
@pytest.mark.parametrize("kind,W,H", [("flat", 176, 144), ("binary", 176, 144), ("random", 176, 144),
                                      ("border16", 48, 48), ("tiny", 16, 16), ("wide", 400, 32)])
@pytest.mark.parametrize("B", [16, 8])
@pytest.mark.parametrize("p", [1, 2, 7, 32])
def test_bma_special_inputs(alg, kind, W, H, B, p):
    if W % B or H % B:
        pytest.skip("frame not divisible by block")
    cur, ref = special_pair(kind, W, H, seed=p * 5 + B)
    mv, sad, pts, _ = gpu_search(frames_from_np(cur, ref), B, p, alg)
    assert_pair_equal(np.stack([cur, ref]), B, p, mv[0], sad[0], pts[0], alg, tag=kind)


@pytest.mark.parametrize("B", [16, 8])
@pytest.mark.parametrize("alg,fixture", [("cds", "table7_cds.txt"), ("ds", "table7_ds.txt")])
def test_bma_ideal_mosaic_table7(B, alg, fixture):
    """The kernels reproduce Table VII's CDS and DS blocks through pixels."""
    cur, ref, tile, off, blocks = synth.ideal_mosaic(B, 7)
    mv, sad, pts, _ = gpu_search(frames_from_np(cur, ref), B, 7, alg)
    np.testing.assert_array_equal(pts[0][blocks][7:, 7:], golden_matrix(fixture, int))
    assert_pair_equal(np.stack([cur, ref]), B, 7, mv[0], sad[0], pts[0], alg, tag="mosaic")


@pytest.mark.parametrize("alg", BMAS + ["dcds_s"])
def test_bma_c3_c4_sampled(alg):
    """Full-size frames, bench launch configuration (all pairs of a chunk in one launch),
    checked on sampled blocks computed one by one by the oracle (DCDS^S included: the DCDS
    kernels' VARIANT 1 at the bench shapes)."""
    rng = np.random.default_rng(17)
    for name, pairs in (("c3", [0, 57, 123]), ("c4", [0, 311])):
        cfg = synth.CONFIGS[name]
        fr = synth.make_sequence(cfg, device=DEV, pairs=pairs)
        host = to_np(fr)
        mv, sad, pts, _ = gpu_search(fr, cfg.B, cfg.p, alg)
        nbx = cfg.W // cfg.B
        for t in range(len(pairs)):
            for i in rng.choice(cfg.nb, 150, replace=False):
                bx, by = (i % nbx) * cfg.B, (i // nbx) * cfg.B
                omv, osad, opts = oracle.bma_block(host[t, 0], host[t, 1], cfg.B, cfg.p, bx, by, alg)
                assert (tuple(mv[t, i]), sad[t, i], pts[t, i]) == (omv, osad, opts), (name, t, i)


def test_bma_unknown_alg_rejected():
    fr = synth.make_sequence(synth.CONFIGS["c0"], device=DEV)
    mv, sad, pts, st = me.alloc_outputs(1, 99, DEV)
    with pytest.raises(me.MEError):
        me.me_bma_batch(6, fr, 16, 7, mv, sad, pts, st)


# ---------------------------------------------------------------------------------------
# ideal-condition simulator and MV histogram on the GPU.
# ---------------------------------------------------------------------------------------
ALL_ALGS = ["dcds", "dcds_s", "cds", "ds", "hexbs_h", "hexbs_v"]


@pytest.mark.parametrize("alg", ALL_ALGS)
@pytest.mark.parametrize("p", [1, 2, 7, 15, 16, 32])
def test_ideal_map_matches_oracle(alg, p):
    nsp, mx, my = (to_np(t) for t in me.me_ideal_nsp_map(alg, p))
    onsp, omx, omy = oracle.ideal_nsp_map(p, oracle.ALGS[alg])
    np.testing.assert_array_equal(nsp, onsp)
    np.testing.assert_array_equal(mx, omx)
    np.testing.assert_array_equal(my, omy)


@pytest.mark.parametrize("alg,fixture", [("dcds", "table7_dcds.txt"), ("cds", "table7_cds.txt"),
                                         ("ds", "table7_ds.txt")])
def test_ideal_map_table7_and_table8(alg, fixture):
    """Table VII out of the GPU simulator, and Table VIII distribution 2."""
    from paper_0806_0689_b200 import mvstats
    nsp = to_np(me.me_ideal_nsp_map(alg, 7)[0])
    np.testing.assert_array_equal(nsp[7:, 7:], golden_matrix(fixture, int))
    printed = {"dcds": 9.7, "cds": 12.5, "ds": 14.8}[alg]
    assert abs(mvstats.ansp(nsp, golden_matrix("table2_mvp.txt", float)) - printed) <= 0.05 + 1e-9


def test_mv_hist_matches_numpy():
    rng = np.random.default_rng(3)
    for n, p in [(0, 7), (1, 1), (12345, 7), (1 << 20, 32)]:
        mv = rng.integers(-p - 2, p + 3, size=(n, 2)).astype(np.int16)
        h = to_np(me.me_mv_hist(torch.from_numpy(mv).to(DEV), p))
        side = 2 * p + 1
        ok = (np.abs(mv) <= p).all(axis=1)
        ref = np.bincount(((mv[ok, 1] + p) * side + mv[ok, 0] + p).astype(np.int64),
                          minlength=side * side).reshape(side, side)
        np.testing.assert_array_equal(h, ref)


def test_mvp_statistics_of_fs_fields():
    """Table II/III-style statistics of the FS motion fields of c1 (the paper computes them on
    FS fields): GPU FS + GPU histogram equal the oracle's FS fields counted in numpy."""
    from paper_0806_0689_b200 import mvstats
    cfg = synth.CONFIGS["c1"]
    fr = synth.make_sequence(cfg, device=DEV, pairs=range(1, 6))
    mv, sad, pts, st = gpu_search(fr, cfg.B, cfg.p, "fs")
    h = to_np(me.me_mv_hist(torch.from_numpy(mv).to(DEV), cfg.p)).astype(np.float64)
    host = to_np(fr)
    ref = np.zeros_like(h)
    for t in range(host.shape[0]):
        omv, _, _ = oracle.fullsearch(host[t, 0], host[t, 1], cfg.B, cfg.p)
        for dx, dy in omv:
            ref[dy + cfg.p, dx + cfg.p] += 1
    np.testing.assert_array_equal(h, ref)
    P = mvstats.normalise(h)
    hs, vs = mvstats.axis_shares(mvstats.quarter(P))
    assert 0 < vs < hs < 1  # the synthetic mix is horizontally biased (2:1, BASELINE configs)


def test_per_frame_series_matches_oracle():
    """report.pair_series (the per-frame PSNR / NSP series of P:387-413) on c1: every DCDS row
    equals the oracle's per-pair MAD, MSE, NSP and PSNR; distance / probability against the
    oracle's FS field; FS against itself is (0, 1)."""
    from paper_0806_0689_b200 import report
    cfg = synth.CONFIGS["c1"]
    fr = synth.make_sequence(cfg, device=DEV, pairs=range(1, 7))
    rows = report.pair_series(fr, cfg.B, cfg.p, ("dcds", "fs"), first_frame=1)
    host = fr.cpu().numpy()
    assert [r["frame"] for r in rows if r["algorithm"] == "dcds"] == list(range(1, 7))
    for t in range(6):
        omv, osad, opts = oracle.dcds(host[t, 0], host[t, 1], cfg.B, cfg.p)
        fmv, _, _ = oracle.fullsearch(host[t, 0], host[t, 1], cfg.B, cfg.p)
        ps, sse = oracle.mc_psnr(host[t, 0], host[t, 1], cfg.B, omv)
        d = next(r for r in rows if r["frame"] == t + 1 and r["algorithm"] == "dcds")
        assert d["nsp"] == opts.astype(np.int64).sum() / cfg.nb
        assert d["mad"] == osad.astype(np.int64).sum() / (cfg.nb * cfg.B * cfg.B)
        assert d["mse"] == sse / (cfg.W * cfg.H) and abs(d["psnr_db"] - ps) <= 1e-9
        hits, dist = oracle.quality(omv, fmv)
        assert d["prob"] == hits / cfg.nb and abs(d["dist"] - dist / cfg.nb) < 1e-12
        f = next(r for r in rows if r["frame"] == t + 1 and r["algorithm"] == "fs")
        assert f["prob"] == 1.0 and f["dist"] == 0.0 and f["nsp"] == (2 * cfg.p + 1) ** 2
    csv = report.series_csv(rows)
    assert csv.splitlines()[0] == "frame,algorithm,mad,mse,nsp,psnr_db,dist,prob" and len(csv.splitlines()) == 13
