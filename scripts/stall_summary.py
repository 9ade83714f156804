"""Aggregate the warp-stall samples of an ncu source page (--page source --csv
--print-source sass) by reason and by SASS opcode: python scripts/stall_summary.py src.csv"""
import csv, sys, re
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; data=rows[2:]
ia=hdr.index("Source"); iss=hdr.index("Warp Stall Sampling (All Samples)"); iex=hdr.index("Instructions Executed")
sc=[i for i,h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot=defaultdict(float); byop=defaultdict(lambda: defaultdict(float)); cnt=defaultdict(float)
T=0
for r in data:
    try: s=float(r[iss])
    except: continue
    op=r[ia].strip().split()[0] if r[ia].strip() else '?'
    if op.startswith('@'): op=r[ia].strip().split()[1]
    op=op.split('.')[0]
    T+=s
    cnt[op]+=float(r[iex] or 0)
    for i in sc:
        v=float(r[i] or 0); tot[hdr[i]]+=v; byop[op][hdr[i]]+=v
print("total samples",T)
for k,v in sorted(tot.items(), key=lambda x:-x[1])[:10]: print(f"  {k:24s} {v/T*100:5.1f}%")
print("by opcode (samples%, inst executed):")
agg=sorted(byop.items(), key=lambda x:-sum(x[1].values()))
for op,d in agg[:14]:
    s=sum(d.values()); top=sorted(d.items(), key=lambda x:-x[1])[:3]
    print(f"  {op:8s} {s/T*100:5.1f}%  n={cnt[op]:.3g}  "+", ".join(f"{k[6:]}={v/T*100:.1f}" for k,v in top))
