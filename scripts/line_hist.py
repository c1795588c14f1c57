"""Per-CUDA-line instruction / stall shares from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
agg = defaultdict(lambda: [0.0, 0.0, ""])
fname = ""
line = None
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ii = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= ii:
        continue
    if r[0]:
        line = (fname, r[0], r[1][:90])
    try:
        v, s = float(r[ii] or 0), float(r[ss] or 0)
    except ValueError:
        continue
    if line:
        a = agg[line[:2]]
        a[0] += v
        a[1] += s
        a[2] = line[2]
tv = sum(a[0] for a in agg.values()) or 1
ts = sum(a[1] for a in agg.values()) or 1
for k, (v, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100 * v / tv:5.1f}% inst {100 * s / ts:5.1f}% stall  {k[0]}:{k[1]:5s} {src.strip()}")
