"""Attribute ncu source-page stall samples of a convtc kernel to code roles
(producer / MMA / epilogue), via nvdisasm line info of the built cubin.
python scripts/ncu_roles.py report.ncu-rep kernel_mangled_name"""
import collections
import csv
import io
import os
import re
import subprocess
import sys

rep, kname = sys.argv[1], sys.argv[2]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.makedirs("/tmp/cub", exist_ok=True)
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2604_16834_b200/libhe_sm100.so")], cwd="/tmp/cub",
               capture_output=True)
sass = subprocess.run(["nvdisasm", "-g", "-c", "/tmp/cub/convtc.sm_100a.cubin"], capture_output=True, text=True).stdout
lines = sass.split("\n")
start = [i for i, l in enumerate(lines) if f".text.{kname}:" in l][0]
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith("//----") and ".text." in lines[i]), len(lines))
addr2 = {}
owner = None
for l in lines[start:end]:
    m = re.search(r'//## File "(.*)", line (\d+)', l)
    if m and m.group(1).endswith("convtc.cu"):
        owner = int(m.group(2))
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", l)
    if m:
        addr2[int(m.group(1), 16)] = (owner, m.group(3))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
base = int(data[0][0], 16)
stc = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in stc}
i_ex = h.index("Instructions Executed")
src = open(os.path.join(ROOT, "paper_2604_16834_b200/csrc/convtc.cu")).read().split("\n")
# roles by the comment markers in the kernel
marks = [(i + 1, t) for i, l in enumerate(src) for t in ("producers", "MMA issuer", "epilogue") if "=====" in l and t in l]


def role(ln):
    if ln is None:
        return "other"
    r = "setup/helpers"
    for mln, t in marks:
        if ln >= mln:
            r = t
    return r


agg = collections.defaultdict(collections.Counter)
ins = collections.Counter()
for r in data:
    own, op = addr2.get(int(r[0], 16) - base, (None, "?"))
    ro = role(own)
    for c, j in idx.items():
        agg[ro][c] += int(r[j] or 0)
    ins[ro] += int(r[i_ex] or 0)
tot = sum(sum(v.values()) for v in agg.values())
for ro, cnt in agg.items():
    t = sum(cnt.values())
    print(f"{ro:14s} samples {t:8d} ({100 * t / tot:4.1f}%) instr {ins[ro]:12d} ",
          {k[6:]: v for k, v in cnt.most_common(6)})
