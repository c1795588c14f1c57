"""Opcode histogram (instructions executed, stall samples) from an ncu --page source --csv SASS export."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
hdr = rows[hi]
si, ii, ss = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
agg = defaultdict(lambda: [0.0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= ii:
        continue
    try:
        v, s = float(r[ii]), float(r[ss])
    except ValueError:
        continue
    op = r[si].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    agg[o.split(".")[0]][0] += v
    agg[o.split(".")[0]][1] += s
tv = sum(a[0] for a in agg.values())
ts = sum(a[1] for a in agg.values())
for k, (v, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{k:12s} {100 * v / tv:6.2f}% inst  {100 * s / ts:6.2f}% stall")
print(f"total warp inst {tv:.3e}")
