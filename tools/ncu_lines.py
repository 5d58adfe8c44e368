"""Top SASS lines of an ncu report by a source-page column (default: shared wavefronts)."""
import csv, subprocess, sys
rep = sys.argv[1]
col = sys.argv[2] if len(sys.argv) > 2 else "L1 Wavefronts Shared"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
ic, isrc, ie = h.index(col), h.index("Source"), h.index("Instructions Executed")
iid = h.index("L1 Wavefronts Shared Ideal") if "L1 Wavefronts Shared Ideal" in h else None
tot = sum(float(r[ic] or 0) for r in data)
print("total", tot)
for k, r in sorted(enumerate(data), key=lambda kr: -float(kr[1][ic] or 0))[:top]:
    ideal = r[iid] if iid is not None else ""
    print(f"{k:5d} {float(r[ic] or 0)/tot*100:5.1f}%  inst={r[ie]:>10s} ideal={ideal:>10s}  {r[isrc].strip()[:70]}")

# aggregate by opcode
agg = {}
for r in data:
    op = r[isrc].strip().split()
    if not op: continue
    o = op[1] if op[0].startswith("@") else op[0]
    a = agg.setdefault(o, [0.0, 0.0])
    a[0] += float(r[ic] or 0); a[1] += float(r[ie] or 0)
print("by opcode (column, instructions):")
for o, (w, n) in sorted(agg.items(), key=lambda t: -t[1][0])[:15]:
    print(f"  {o:24s} {w/tot*100:5.1f}%  {w:14.0f} {n:14.0f}")
