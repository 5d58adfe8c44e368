"""Attribute ncu per-SASS-instruction metrics of one kernel to CUDA source lines.

usage: python tools/ncu_bylines.py <report.ncu-rep> <cubin> <mangled-kernel-name> [column]
Uses nvdisasm -g (line info from -lineinfo builds) to map SASS offsets to source lines."""
import collections, csv, re, subprocess, sys

rep, cubin, fn = sys.argv[1:4]
col = sys.argv[4] if len(sys.argv) > 4 else "Instructions Executed"
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
sec = dis.split("//--------------------- .text." + fn + " ")[1].split("//--------------------- ")[0]
line_of = {}
cur = None
for ln in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
ia, ic = h.index("Address"), h.index(col)
base = int(data[0][ia], 16)
agg = collections.Counter()
tot = 0.0
for r in data:
    off = int(r[ia], 16) - base
    v = float(r[ic] or 0)
    tot += v
    agg[line_of.get(off, ("?", 0))] += v
src = {}
texts = {}
for (f, l), v in agg.most_common(int(sys.argv[5]) if len(sys.argv) > 5 else 40):
    if f != "?" and f not in texts:
        import glob
        cand = glob.glob("/root/repo/**/" + f, recursive=True)
        texts[f] = open(cand[0]).read().splitlines() if cand else []
    t = texts.get(f, [])
    print(f"{v / tot * 100:5.1f}%  {f}:{l:<5d} {t[l-1].strip()[:90] if 0 < l <= len(t) else ''}")
