"""Top CUDA source lines of an ncu source page (ncu -i rep --page source --csv
--print-source cuda) by warp-stall samples: python scripts/cuda_lines.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
# the csv holds one table per source file: a "File"/"#" header row precedes each
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = []
hdr = None
fname = "?"
for r in rows:
    if not r:
        continue
    if "Warp Stall Sampling (All Samples)" in r:
        hdr = r
        continue
    if hdr is None:
        if len(r) == 1:
            fname = r[0]
        continue
    if len(r) != len(hdr):
        if len(r) == 1:
            fname = r[0]
        continue
    try:
        v = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        continue
    line = r[hdr.index("#")] if "#" in hdr else "?"
    src = r[hdr.index("Source")].strip()[:90]
    ex = r[hdr.index("Instructions Executed")] if "Instructions Executed" in hdr else ""
    out.append((v, fname.split("/")[-1], line, ex, src))
tot = sum(o[0] for o in out) or 1.0
print("total samples", tot)
for v, f, line, ex, src in sorted(out, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}%  {f}:{line}  ex={ex}  {src}")
