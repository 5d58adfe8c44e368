"""Table-IX-style comparison of DCDS, DCDS^S, CDS, DS, h-/v-HEXBS and FS on the
seeded synthetic sequences (the paper's 18 sequences are unavailable).

  python tools/table9.py [--configs c1,c2,c3] [--pairs 16] [--out profiles/r1/table9_synthetic.md]

Runs on the GPU through the C ABI (me_bma_batch, me_fullsearch_batch, me_quality_batch).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_0806_0689_b200 as me  # noqa: E402
from paper_0806_0689_b200 import report, synth  # noqa: E402

NAMES = {"dcds": "DCDS", "dcds_s": "DCDS^S", "cds": "CDS", "ds": "DS", "hexbs_h": "h-HEXBS",
         "hexbs_v": "v-HEXBS", "fs": "FS"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3")
    ap.add_argument("--pairs", type=int, default=16)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    me.me_init(0)
    me.me_set_stream(torch.cuda.current_stream())
    lines = ["| config | BMA | MAD | MSE | NSP | PSNR (dB) | distance | probability | NSP / NSP(DCDS) - 1 | blocks/s |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    res = {}
    for name in args.configs.split(","):
        cfg = synth.CONFIGS[name]
        n = min(cfg.npairs, args.pairs)
        pairs = range(1, cfg.npairs + 1, max(1, cfg.npairs // n))[:n]
        fr = synth.make_sequence(cfg, device="cuda:0", pairs=pairs)
        rows = report.compare_bmas(fr, cfg.B, cfg.p, reps=3)
        res[name] = rows
        for alg, r in rows.items():
            bps = f"{r['blocks_per_s']:.3e}" if "blocks_per_s" in r else "-"
            lines.append(f"| {name} ({len(pairs)} pairs) | {NAMES[alg]} | {r['mad']:.4f} | {r['mse']:.3f} | "
                         f"{r['nsp']:.3f} | {r['psnr_db']:.3f} | {r['dist']:.5f} | {100 * r['prob']:.3f}% | "
                         f"{100 * r['nsp_speedup_of_dcds']:.1f}% | {bps} |")
    text = "\n".join(lines)
    print(text)
    if args.out:
        with open(args.out, "w") as f:
            f.write("# Table-IX-style comparison on the synthetic sequences (tools/table9.py)\n\n")
            f.write("Sequence values are means of per-pair values (reading C18).  FS is the true-MV\n")
            f.write("reference of distance/probability (P:43 aspects 5-6).  The paper's own Table IX\n")
            f.write("(P:344-385) is on its 18 natural sequences and is context only.\n\n")
            f.write(text + "\n")
        with open(os.path.splitext(args.out)[0] + ".json", "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
