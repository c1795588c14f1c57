"""Time encrypt_batch of one config-3 group (3072 x 32768 values, 9 limbs) and list its kernels."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16834_b200 import configs  # noqa: E402
import torch  # noqa: E402

from paper_2604_16834_b200.engine import GpuEngine  # noqa: E402

eng = GpuEngine(configs.context(3, seed=1))
v = torch.rand((3072, 32768), dtype=torch.float64, device="cuda")
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(2):
    eng.release(*eng.encrypt_batch(v, level=8))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t = time.perf_counter()
e0.record()
for _ in range(reps):
    eng.release(*eng.encrypt_batch(v, level=8))
e1.record()
th = time.perf_counter() - t
torch.cuda.synchronize()
print(f"encrypt_batch 3072 cts at 9 limbs: {e0.elapsed_time(e1) / reps:.2f} ms/call (host enqueue {1e3 * th / reps:.1f} ms)")
