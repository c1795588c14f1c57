"""Digest of one ncu --set full report: duration, issue, pipes, stalls, DRAM bytes.

python scripts/ncu_digest.py report.ncu-rep [launch index]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, row = rows[0], rows[2 + idx]
d = dict(zip(hdr, row))


def f(k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")


print("kernel:", d.get("Kernel Name", "?")[:100])
print(f"duration {f('gpu__time_duration.sum'):.3f} ms   regs {d.get('launch__registers_per_thread')}  "
      f"warps/SM {f('sm__warps_active.avg.per_cycle_active'):.1f}  issue {f('sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f}%")
print(f"dram read {f('dram__bytes_read.sum'):.3f} GB  write {f('dram__bytes_write.sum'):.3f} GB  (units as ncu prints them)")
pipes = sorted(((f(k), k.split("pipe_")[1].split(".")[0]) for k in hdr
                if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active")),
               reverse=True)
print("pipes:", ", ".join(f"{n} {v:.1f}%" for v, n in pipes[:8] if v == v))
st = [(f(k), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in hdr
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
tot = sum(v for v, _ in st if v == v)
print("stalls:", ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in sorted(st, reverse=True)[:8] if v == v))
