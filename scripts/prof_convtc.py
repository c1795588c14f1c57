"""One conv1-tile launch of the tcgen05 fused conv (for ncu): config 3 shape, 9 limbs.
python scripts/prof_convtc.py [conv1|conv2] [launches]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16834_b200 import _lib, configs  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_16834_b200.engine import GpuEngine  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "conv1"
launches = int(sys.argv[2]) if len(sys.argv) > 2 else 2
eng = GpuEngine(configs.context(3, seed=7))
N, L = eng.N, eng._L
if which == "conv1":
    p, H, W, M, pool, y0, y1, ell, wbits, nci = 3, 32, 32, 16, 1, 0, 8, 9, 20, 2
else:
    p, H, W, M, pool, y0, y1, ell, wbits, nci = 16, 16, 16, 32, 0, 0, 16, 9, 14, 3
x = torch.empty((p * H * W, nci, ell, N), dtype=torch.int64, device=eng.device)
for i, q in enumerate(eng.moduli[:ell]):
    x[:, :, i] = torch.randint(0, q, (p * H * W, nci, N), device=eng.device, dtype=torch.int64)
nwin = ((y1 - y0) // 2) * (W // 2) if pool else 1
out = torch.empty((M * nwin, 2 * nci - 1, ell, N), dtype=torch.int64, device=eng.device)
pi = _lib.ptr_array([x[i].data_ptr() for i in range(p * H * W)])
po = _lib.ptr_array([out[i].data_ptr() for i in range(M * nwin)])
w = np.random.default_rng(0).integers(-(1 << wbits), 1 << wbits, size=(M, 9 * p), dtype=np.int64)
for _ in range(launches):
    _lib.check(L.he_conv_square_sum_n(eng._h, _lib.addr(pi), nci, p, H, W, _lib.addr(po), M, pool, y0, y1,
                                      _lib.addr(w), None, None, ell, torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("ok", which)
