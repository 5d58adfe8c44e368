"""GPU trace build (me_dcds_trace_batch): the same search as the production kernels, bit for
bit, and a per-pass record that expands to the oracle's point-by-point trace (scored points,
their order, step numbers and pattern kinds, readings C5-C7, C22).

The oracle side drives oracle.dcds_cost with the pixel SAD of the block (oracle.sad), so the
comparison is against the oracle's own search order, not against the kernel's.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_0806_0689_b200 as me
from paper_0806_0689_b200 import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0") if torch.cuda.is_available() else None
CAP = 64


@pytest.fixture(scope="module", autouse=True)
def init():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    me.me_init(0)
    me.me_set_stream(torch.cuda.current_stream())
    yield


def run_trace(frames, B, p, variant):
    n, _, H, W = frames.shape
    nb = (W // B) * (H // B)
    mv, sad, pts, _ = me.alloc_outputs(n, nb, DEV, stats=False)
    tr = torch.zeros(n, nb, CAP, dtype=torch.int64, device=DEV)
    tl = torch.zeros(n, nb, dtype=torch.int16, device=DEV)
    me.me_dcds_trace_batch(variant, frames, B, p, mv, sad, pts, tr, tl)
    mv2, sad2, pts2, _ = me.alloc_outputs(n, nb, DEV, stats=False)
    (me.me_dcds_s_batch if variant else me.me_dcds_batch)(frames, B, p, mv2, sad2, pts2)
    torch.cuda.synchronize()
    assert torch.equal(mv, mv2) and torch.equal(sad, sad2) and torch.equal(pts, pts2)
    return mv.cpu().numpy(), sad.cpu().numpy(), pts.cpu().numpy(), tr.cpu().numpy(), tl.cpu().numpy()


def check_blocks(host, B, p, variant, out, blocks):
    mv, sad, pts, tr, tl = out
    cur, ref = host[0], host[1]
    nbx = cur.shape[1] // B
    for b in blocks:
        bx, by = (b % nbx) * B, (b // nbx) * B  # block origin in pixels
        omv, ocost, opts, otrace = oracle.dcds_cost(
            lambda dx, dy: oracle.sad(cur, ref, B, bx, by, dx, dy), p, variant)
        n = int(tl[b])
        assert n <= CAP
        got = me.decode_trace(tr[b], n)
        assert got == otrace, f"B={B} p={p} v={variant} block {b}: gpu {got} oracle {otrace}"
        assert tuple(mv[b]) == omv and sad[b] == ocost and pts[b] == opts == len(got)
        # the last record carries the final SAD
        assert (int(tr[b][n - 1]) >> 36) & 0xFFFF == sad[b]


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("B,p", [(8, 7), (16, 7), (8, 16), (16, 32), (8, 1), (16, 2)])
def test_trace_matches_oracle_trace(variant, B, p):
    cfg = synth.CONFIGS["c0"]
    fr = synth.make_sequence(cfg, device=DEV)[:2].contiguous()
    host = fr.cpu().numpy()
    nb = (fr.shape[3] // B) * (fr.shape[2] // B)
    rng = np.random.default_rng(B * 100 + p + variant)
    for t in range(fr.shape[0]):
        out = run_trace(fr[t:t + 1], B, p, variant)
        blocks = rng.choice(nb, size=min(nb, 48), replace=False)
        check_blocks(host[t], B, p, variant, tuple(o[0] for o in out), blocks)


@pytest.mark.parametrize("kind", ["flat", "random"])
def test_trace_special_inputs(kind):
    W, H = 176, 144
    cur, ref = synth.flat_pair(W, H, 77) if kind == "flat" else synth.random_pair(W, H, 5)
    fr = torch.from_numpy(np.stack([cur, ref])[None].copy()).to(DEV)
    for B in (8, 16):
        out = run_trace(fr, B, 7, 0)
        nb = (W // B) * (H // B)
        check_blocks(np.stack([cur, ref]), B, 7, 0, tuple(o[0] for o in out), range(0, nb, 7))


def test_trace_cap_counts_beyond_capacity():
    cfg = synth.CONFIGS["c0"]
    fr = synth.make_sequence(cfg, device=DEV)[:1].contiguous()
    nb = cfg.nb
    mv, sad, pts, _ = me.alloc_outputs(1, nb, DEV, stats=False)
    tr = torch.zeros(1, nb, 1, dtype=torch.int64, device=DEV)
    tl = torch.zeros(1, nb, dtype=torch.int16, device=DEV)
    me.me_dcds_trace_batch(0, fr, cfg.B, cfg.p, mv, sad, pts, tr, tl)
    torch.cuda.synchronize()
    assert (tl.cpu().numpy() >= 2).all()  # Step 1 plus at least the Step-4 pass
    assert ((tr.cpu().numpy()[0, :, 0] >> 8) & 0xF == 15).all()  # record 0 is Step 1


def test_trace_rejects_bad_cap():
    cfg = synth.CONFIGS["c0"]
    fr = synth.make_sequence(cfg, device=DEV)[:1].contiguous()
    mv, sad, pts, _ = me.alloc_outputs(1, cfg.nb, DEV, stats=False)
    tl = torch.zeros(1, cfg.nb, dtype=torch.int16, device=DEV)
    for cap in (0, 256):
        tr = torch.zeros(1, cfg.nb, cap, dtype=torch.int64, device=DEV)
        with pytest.raises(me.MEError):
            me.me_dcds_trace_batch(0, fr, cfg.B, cfg.p, mv, sad, pts, tr, tl)


@pytest.mark.parametrize("B,tile", [(8, "16,8"), (16, "8,8")])
def test_trace_handout_kernels_match_oracle(B, tile):
    """The trace build of the hand-out kernels (tiles with more blocks than lane groups)."""
    import os
    old = os.environ.get("ME_TILE")
    os.environ["ME_TILE"] = tile
    try:
        cfg = synth.CONFIGS["c1"]
        fr = synth.make_sequence(cfg, device=DEV, pairs=[3])
        host = fr.cpu().numpy()
        nb = (fr.shape[3] // B) * (fr.shape[2] // B)
        for variant in (0, 1):
            out = run_trace(fr, B, 7, variant)
            check_blocks(host[0], B, 7, variant, tuple(o[0] for o in out), range(0, nb, 5))
    finally:
        if old is None:
            os.environ.pop("ME_TILE", None)
        else:
            os.environ["ME_TILE"] = old
