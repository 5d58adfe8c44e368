"""Per-frame PSNR / NSP series (the paper's frame-wise comparison, Figs. 8-9, whose
images are missing) on the seeded synthetic sequences: DCDS, DCDS^S and FS (and optionally
every BMA), one row per pair and algorithm, written as SPEC's per-frame CSV plus a
markdown summary (sequence means = means of the per-frame values, reading C18).

  python tools/series.py [--configs c1,c2] [--algs dcds,dcds_s,fs] [--outdir profiles/r2]

Runs on the GPU through the C ABI (me_bma_batch, me_fullsearch_batch, me_quality_batch).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_0806_0689_b200 as me  # noqa: E402
from paper_0806_0689_b200 import report, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2")
    ap.add_argument("--algs", default="dcds,dcds_s,cds,ds,hexbs_h,fs")
    ap.add_argument("--outdir", default=os.path.join(ROOT, "profiles", "r2"))
    args = ap.parse_args()
    me.me_init(0)
    me.me_set_stream(torch.cuda.current_stream())
    algs = tuple(args.algs.split(","))
    md = ["# Per-frame series on the synthetic sequences (tools/series.py)", "",
          "P:387-413 (Figs. 8-9) plot PSNR and NSP frame by frame on the paper's sequences; these",
          "are the same series on the seeded synthetic configs (SURVEY 8(d)).  One CSV row per",
          "frame and algorithm (SPEC S:510 layout); below, per config, the sequence means and the",
          "per-frame range.", ""]
    for name in args.configs.split(","):
        cfg = synth.CONFIGS[name]
        fr = synth.make_sequence(cfg, device="cuda:0")
        rows = report.pair_series(fr, cfg.B, cfg.p, algs)
        path = os.path.join(args.outdir, f"series_{name}.csv")
        with open(path, "w") as f:
            f.write(report.series_csv(rows))
        md += [f"## {name}: {cfg.W}x{cfg.H}, {cfg.npairs} pairs, B={cfg.B}, +-{cfg.p} (`{os.path.basename(path)}`)", "",
               "| algorithm | mean PSNR (dB) | min..max PSNR | mean NSP | min..max NSP | mean dist | mean prob |",
               "|---|---|---|---|---|---|---|"]
        for alg in algs:
            rs = [r for r in rows if r["algorithm"] == alg]
            m = report.sequence_means(rs)
            ps = [r["psnr_db"] for r in rs]
            ns = [r["nsp"] for r in rs]
            md.append(f"| {alg} | {m['psnr_db']:.3f} | {min(ps):.2f}..{max(ps):.2f} | {m['nsp']:.3f} | "
                      f"{min(ns):.2f}..{max(ns):.2f} | {m['dist']:.4f} | {m['prob']:.4f} |")
        md.append("")
    with open(os.path.join(args.outdir, "series.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
