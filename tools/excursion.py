"""How far do the DCDS searches of a config wander?  Runs the trace build over every pair
(in chunks), takes each block's pattern centres (every scoring pass: the points it tests lie
within 2 of them), and reports the fraction of blocks whose centres leave a given compact
visited-set window -- the blocks the compact-set kernel hands to its overflow passes
(DESIGN.md §7 "Compact visited set").

  python tools/excursion.py [--configs c3,c4] [--variant 0] [--out f.json]

Window (px, py): the bitmap layout of the full window over half-widths px x py (row length
2px + 3, no border); the centres that keep every pattern point inside it are cx in
[-px, px - 2], cy in [-py, py].
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
    ap.add_argument("--configs", default="c3,c4")
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=40)
    ap.add_argument("--cap", type=int, default=96)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import paper_0806_0689_b200 as me
    from paper_0806_0689_b200 import synth
    me.me_init(0)
    me.me_set_stream(torch.cuda.current_stream())
    res = {}
    for name in args.configs.split(","):
        cfg = synth.CONFIGS[name]
        fr_all = synth.make_sequence(cfg, device="cuda:0")
        lo = []
        hi = []
        over_cap = 0
        for c0 in range(0, cfg.npairs, args.chunk):
            fr = fr_all[c0:c0 + args.chunk].contiguous()
            n = fr.shape[0]
            mv, sad, pts, _ = me.alloc_outputs(n, cfg.nb, "cuda:0", stats=False)
            tr = torch.zeros(n, cfg.nb, args.cap, dtype=torch.int64, device="cuda:0")
            tl = torch.zeros(n, cfg.nb, dtype=torch.int16, device="cuda:0")
            me.me_dcds_trace_batch(args.variant, fr, cfg.B, cfg.p, mv, sad, pts, tr, tl)
            cx = ((tr >> 20) & 0xFF).to(torch.int16)
            cy = ((tr >> 28) & 0xFF).to(torch.int16)
            cx = torch.where(cx > 127, cx - 256, cx)
            cy = torch.where(cy > 127, cy - 256, cy)
            k = torch.arange(args.cap, device="cuda:0")[None, None, :]
            valid = k < tl.to(torch.int64)[..., None]
            big = torch.full_like(cx, 1000)
            lo.append(torch.stack([torch.where(valid, cx, big).amin(-1),
                                   torch.where(valid, cy, big).amin(-1)], -1).reshape(-1, 2).cpu())
            hi.append(torch.stack([torch.where(valid, cx, -big).amax(-1),
                                   torch.where(valid, cy, -big).amax(-1)], -1).reshape(-1, 2).cpu())
            over_cap += int((tl.to(torch.int64) >= args.cap).sum())
        lo = torch.cat(lo).numpy().astype(np.int64)
        hi = torch.cat(hi).numpy().astype(np.int64)
        nbk = lo.shape[0]
        out = {"blocks": nbk, "over_cap": over_cap, "p": cfg.p, "windows": []}
        for px in range(8, cfg.p - 1):
            for py in range(8, cfg.p - 1):
                words = ((2 * py + 5) * (2 * px + 3) + 2 + 31) // 32
                esc = (lo[:, 0] < -px) | (hi[:, 0] > px - 2) | (lo[:, 1] < -py) | (hi[:, 1] > py)
                out["windows"].append({"px": px, "py": py, "words": words,
                                       "escape_frac": float(esc.mean())})
        # the best window per word budget
        best = {}
        for w in out["windows"]:
            for budget in (32, 40, 48, 56, 64, 72, 80, 96):
                if w["words"] <= budget and (budget not in best or w["escape_frac"] < best[budget]["escape_frac"]):
                    best[budget] = w
        out["best_per_budget"] = {str(k): v for k, v in sorted(best.items())}
        hx = np.maximum(-lo[:, 0], hi[:, 0])
        hy = np.maximum(-lo[:, 1], hi[:, 1])
        out["abs_cx_max_hist"] = np.bincount(np.clip(hx, 0, 40), minlength=41).tolist()
        out["abs_cy_max_hist"] = np.bincount(np.clip(hy, 0, 40), minlength=41).tolist()
        res[name] = {k: v for k, v in out.items() if k != "windows"}
        print(name, json.dumps(res[name]["best_per_budget"]), "over_cap", over_cap, flush=True)
        del fr_all
        torch.cuda.empty_cache()
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
