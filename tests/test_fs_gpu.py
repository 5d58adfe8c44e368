"""GPU parity of the full-search builds (reading C13 tie order): the column-sweep builds
for the bench geometries (8x8 / +-16 and 16x16 / +-32, whole tiles of 8x4 / 4x4 blocks plus
ragged ones) and the chunked kernel (ME_FS_SWEEP=0) on the same frames, whole pairs against
the oracle's full search, bit for bit (MV, SAD, NSP, per-pair statistics)."""
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
    os.environ.pop("ME_FS_SWEEP", None)


def _pair(kind, W, H, seed):
    if kind == "flat":
        return synth.flat_pair(W, H, 91)
    if kind == "binary":
        return synth.binary_pair(W, H, seed)
    if kind == "noise":
        return synth.random_pair(W, H, seed)
    tex = synth.texture(W, H, (2.0, 6.0), seed).numpy()
    rng = np.random.default_rng(seed)
    return synth.translated_pair(tex, int(rng.integers(-9, 10)), int(rng.integers(-9, 10)))


# (B, p, W, H): the sweep builds need the bench tile width (8 blocks of 8 / 4 blocks of 16)
CASES = [(8, 16, 128, 64), (8, 16, 208, 88), (16, 32, 128, 96), (16, 32, 96, 80)]


@pytest.mark.parametrize("B,p,W,H", CASES, ids=[f"B{c[0]}p{c[1]}-{c[2]}x{c[3]}" for c in CASES])
@pytest.mark.parametrize("sweep", ["1", "0"], ids=["sweep", "chunked"])
def test_fullsearch_builds(monkeypatch, B, p, W, H, sweep):
    monkeypatch.setenv("ME_FS_SWEEP", sweep)
    kinds = ["texture", "noise", "binary", "flat", "texture"]
    host = np.stack([np.stack(_pair(k, W, H, 17 * B + i)) for i, k in enumerate(kinds)])
    frames = torch.from_numpy(host).to(DEV)
    n, nb = host.shape[0], (W // B) * (H // B)
    mv, sad, pts, st = me.alloc_outputs(n, nb, DEV)
    me.me_fullsearch_batch(frames, B, p, mv, sad, pts, st)
    torch.cuda.synchronize()
    mv, sad, pts, st = (mv.cpu().numpy(), sad.cpu().numpy().astype(np.uint32),
                        pts.cpu().numpy().astype(np.uint16), st.cpu().numpy().astype(np.uint64))
    for t in range(n):
        omv, osad, opts = oracle.fullsearch(host[t, 0], host[t, 1], B, p)
        bad = np.flatnonzero((mv[t] != omv).any(1) | (sad[t] != osad) | (pts[t] != opts))
        assert bad.size == 0, (kinds[t], bad[:5], mv[t][bad[0]], omv[bad[0]], sad[t][bad[0]], osad[bad[0]])
        sse = oracle.mc_psnr(host[t, 0], host[t, 1], B, omv)[1]
        assert tuple(int(x) for x in st[t]) == (int(opts.astype(np.int64).sum()), int(osad.astype(np.int64).sum()),
                                               int(sse))
