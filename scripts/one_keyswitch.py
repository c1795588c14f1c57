"""Run a few batched relinearisation key switches (config-2 or config-3 ring) -- ncu target."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16834_b200 import _lib, configs  # noqa: E402  (selects the allocator first)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_16834_b200.engine import GpuEngine  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
eng = GpuEngine(configs.context(cfg, seed=7))
L, N = eng.context.n_q, eng.N
x = torch.empty((B, 3, L, N), dtype=torch.int64, device=eng.device)
for i, q in enumerate(eng.moduli[:L]):
    x[:, :, i] = torch.randint(0, q, (B, 3, N), device=eng.device, dtype=torch.int64)
out = torch.empty((B, 2, L, N), dtype=torch.int64, device=eng.device)
eng._ensure_relin()
pi = _lib.ptr_array([x[i].data_ptr() for i in range(B)])
po = _lib.ptr_array([out[i].data_ptr() for i in range(B)])
for _ in range(reps):
    _lib.check(eng._L.he_relin(eng._h, _lib.addr(pi), _lib.addr(po), B, L, eng.stream))
torch.cuda.synchronize()
print("ok")
