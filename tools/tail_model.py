"""How much of a DCDS CTA's lifetime is its slowest search?  Runs the trace build over a config
(in chunks), takes every block's number of scoring passes, groups the blocks as the ONE kernel
does (tile of TBX x TBY blocks per CTA, 32/G groups per warp), and reports the mean over CTAs
of (max passes in the CTA) against the mean passes per block, plus the same with searches cut
at K passes (the model of handing searches longer than K to an overflow pass).

  python tools/tail_model.py [--config c4] [--out f.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--chunk", type=int, default=40)
    ap.add_argument("--cap", type=int, default=128)
    ap.add_argument("--pairs", type=int, default=200)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import paper_0806_0689_b200 as me
    from paper_0806_0689_b200 import synth
    me.me_init(0)
    me.me_set_stream(torch.cuda.current_stream())
    cfg = synth.CONFIGS[args.config]
    npairs = min(args.pairs, cfg.npairs)
    fr_all = synth.make_sequence(cfg, device="cuda:0", pairs=range(1, npairs + 1))
    tl_all = []
    for c0 in range(0, npairs, args.chunk):
        fr = fr_all[c0:c0 + args.chunk].contiguous()
        n = fr.shape[0]
        mv, sad, pts, _ = me.alloc_outputs(n, cfg.nb, "cuda:0", stats=False)
        tr = torch.zeros(n, cfg.nb, args.cap, dtype=torch.int64, device="cuda:0")
        tl = torch.zeros(n, cfg.nb, dtype=torch.int16, device="cuda:0")
        me.me_dcds_trace_batch(0, fr, cfg.B, cfg.p, mv, sad, pts, tr, tl)
        tl_all.append(tl.cpu().numpy().astype(np.int64))
    tl = np.concatenate(tl_all)  # [pairs, nb] passes per block (Step 1 included)
    nbx, nby = cfg.W // cfg.B, cfg.H // cfg.B
    tbx, tby = (4, 8) if cfg.B == 16 else (16, 4)
    bpw = 4 if cfg.B == 16 else 16  # blocks per warp (32 / G)
    t = tl.reshape(-1, nby, nbx)
    # pad to whole tiles with zeros (missing blocks)
    ty, tx = -(-nby // tby), -(-nbx // tbx)
    pad = np.zeros((t.shape[0], ty * tby, tx * tbx), np.int64)
    pad[:, :nby, :nbx] = t
    tiles = pad.reshape(t.shape[0], ty, tby, tx, tbx).transpose(0, 1, 3, 2, 4).reshape(-1, tby * tbx)
    res = {"config": cfg.name, "pairs": npairs, "mean_passes": float(tl.mean()),
           "p99_passes": float(np.percentile(tl, 99)), "max_passes": int(tl.max()), "cut": []}
    for K in [None, 40, 30, 24, 20, 16, 14, 12, 10]:
        c = tiles if K is None else np.minimum(tiles, K)
        cta = c.max(1).mean()
        warp = c.reshape(c.shape[0], -1, bpw).max(2).mean()
        frac = 0.0 if K is None else float((tl > K).mean())
        res["cut"].append({"K": K, "cta_max_mean": float(cta), "warp_max_mean": float(warp),
                           "block_mean": float(c.mean()), "blocks_cut_frac": frac})
        print(K, round(cta, 2), round(warp, 2), round(float(c.mean()), 2), round(frac, 5), flush=True)
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
