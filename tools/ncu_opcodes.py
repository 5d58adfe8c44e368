"""Per-opcode instruction mix of one kernel from an ncu report (SURVEY 8(d) evidence: the
instruction budget per block, executed VABSDIFF4 lane-ops against the algorithmic ones).

usage: python tools/ncu_opcodes.py <report.ncu-rep> [--blocks N] [--csv out.csv]
Reads `ncu -i <rep> --page source --csv --print-source sass` (per-SASS-instruction metrics)
and sums warp-level instructions, thread-level instructions and shared-memory wavefronts per
opcode (the mnemonic without modifiers)."""
import argparse
import collections
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--blocks", type=float, default=None, help="macroblocks per launch (per-block columns)")
ap.add_argument("--csv", default=None)
ap.add_argument("--kernel", default=None, help="regex of the kernel (default: the first)")
args = ap.parse_args()
cmd = ["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "sass"]
if args.kernel:
    cmd += ["-k", "regex:" + args.kernel]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
ci, ct, cw = h.index("Instructions Executed"), h.index("Thread Instructions Executed"), h.index("L1 Wavefronts Shared")
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for r in data:
    src = r[1].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1]
    op = src.split()[0].split(".")[0] if src else "?"
    a = agg[op]
    a[0] += float(r[ci] or 0); a[1] += float(r[ct] or 0); a[2] += float(r[cw] or 0)
tot = [sum(v[i] for v in agg.values()) for i in range(3)]
nb = args.blocks or 1.0
lines = [("opcode", "warp_instr", "thread_instr", "active_lanes", "smem_wavefronts", "share_pct",
          "warp_instr_per_block", "wavefronts_per_block")]
for op, (wi, ti, wf) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    lines.append((op, int(wi), int(ti), round(ti / wi, 2) if wi else 0, int(wf), round(100 * wi / tot[0], 2),
                  round(wi / nb, 3), round(wf / nb, 3)))
lines.append(("TOTAL", int(tot[0]), int(tot[1]), round(tot[1] / tot[0], 2), int(tot[2]), 100.0,
              round(tot[0] / nb, 2), round(tot[2] / nb, 2)))
w = csv.writer(open(args.csv, "w") if args.csv else io.StringIO())
for ln in lines:
    w.writerow(ln)
for ln in lines[:40] + lines[-1:]:
    print("  ".join(f"{x:>12}" if not isinstance(x, str) else f"{x:<14}" for x in ln))
