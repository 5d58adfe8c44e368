"""Seeded fuzz parity: random frame sizes (every tile shape, ragged edge tiles, frames smaller
than a tile), windows 1..32, both block sizes and mixed content (noise, smooth texture with
noise, translated texture, binary ties, flat), several pairs per launch -- every algorithm of
the library against the oracle, bit for bit, and the batch statistics against the outputs."""
import numpy as np
import pytest
import torch

import oracle
import paper_0806_0689_b200 as me
from paper_0806_0689_b200 import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0") if torch.cuda.is_available() else None
ALGS = ["dcds", "dcds_s", "cds", "ds", "hexbs_h", "hexbs_v"]


@pytest.fixture(scope="module", autouse=True)
def init():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    me.me_init(0)
    me.me_set_stream(torch.cuda.current_stream())
    yield


def make_pair(rng, W, H, kind, seed):
    if kind == "noise":
        return synth.random_pair(W, H, seed)
    if kind == "flat":
        return synth.flat_pair(W, H, int(rng.integers(0, 256)))
    if kind == "binary":
        return synth.binary_pair(W, H, seed)
    tex = synth.texture(W, H, (1.5, 4.0), seed).numpy()
    if kind == "translated":
        return synth.translated_pair(tex, int(rng.integers(-6, 7)), int(rng.integers(-6, 7)))
    cur = np.clip(tex.astype(np.int16) + rng.integers(-6, 7, tex.shape), 0, 255).astype(np.uint8)
    ref = np.roll(tex, (int(rng.integers(-3, 4)), int(rng.integers(-9, 10))), (0, 1))
    return cur, np.ascontiguousarray(ref)


@pytest.mark.parametrize("case", range(96))
def test_fuzz_parity(case):
    rng = np.random.default_rng(806689 + case)
    B = int(rng.choice([8, 16]))
    W = 16 * int(rng.integers(1, 21))
    H = B * int(rng.integers(1, 22 if B == 8 else 12))
    p = int(rng.choice([1, 2, 3, 5, 7, 8, 12, 15, 16, 17, 24, 31, 32]))
    npairs = int(rng.integers(1, 4))
    kinds = rng.choice(["noise", "flat", "binary", "translated", "texture"], npairs)
    pairs = [make_pair(rng, W, H, k, 1000 * case + i) for i, k in enumerate(kinds)]
    host = np.stack([np.stack(pr) for pr in pairs])             # [n, 2, H, W]
    fr = torch.from_numpy(host.copy()).to(DEV)
    nb = (W // B) * (H // B)
    tag = f"case {case}: {W}x{H} B={B} p={p} {list(kinds)}"
    for alg in ALGS:
        mv, sad, pts, st = me.alloc_outputs(npairs, nb, DEV)
        me.me_bma_batch(alg, fr, B, p, mv, sad, pts, st)
        torch.cuda.synchronize()
        mv, sad = mv.cpu().numpy(), sad.cpu().numpy().astype(np.uint32)
        pts, st = pts.cpu().numpy().astype(np.uint16), st.cpu().numpy()
        for t in range(npairs):
            omv, osad, opts = oracle.bma(host[t, 0], host[t, 1], B, p, alg)
            bad = np.flatnonzero((mv[t] != omv).any(1) | (sad[t] != osad) | (pts[t] != opts))
            assert bad.size == 0, f"{tag} {alg} pair {t}: {bad.size} blocks differ, first {bad[:4]}"
            assert st[t, 0] == opts.astype(np.int64).sum() and st[t, 1] == osad.astype(np.int64).sum()
            assert int(st[t, 2]) == oracle.mc_psnr(host[t, 0], host[t, 1], B, omv)[1], f"{tag} {alg} SSE"
    if p <= 16 and W * H <= 160 * 160:  # full search: (2p+1)^2 candidates per block in the oracle
        mv, sad, pts, st = me.alloc_outputs(npairs, nb, DEV)
        me.me_fullsearch_batch(fr, B, p, mv, sad, pts, st)
        torch.cuda.synchronize()
        mv, sad, pts = mv.cpu().numpy(), sad.cpu().numpy().astype(np.uint32), pts.cpu().numpy().astype(np.uint16)
        for t in range(npairs):
            omv, osad, opts = oracle.fullsearch(host[t, 0], host[t, 1], B, p)
            bad = np.flatnonzero((mv[t] != omv).any(1) | (sad[t] != osad) | (pts[t] != opts))
            assert bad.size == 0, f"{tag} fs pair {t}: {bad.size} blocks differ"
