"""Probe he_conv_square_sum_n on small shapes (debug helper): args cfg H bias(0/1) wbits."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16834_b200 import _lib, configs  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_16834_b200.engine import GpuEngine  # noqa: E402

cfg, H, wb, wbits = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
eng = GpuEngine(configs.context(cfg, seed=7))
N, ell, p, M, W = eng.N, 3, 16, 32, H
rng = np.random.default_rng(0)
x = torch.empty((p * H * W, 3, ell, N), dtype=torch.int64, device=eng.device)
for i, q in enumerate(eng.moduli[:ell]):
    x[:, :, i] = torch.randint(0, q, (p * H * W, 3, N), device=eng.device, dtype=torch.int64)
out = torch.empty((M, 5, ell, N), dtype=torch.int64, device=eng.device)
pi = _lib.ptr_array([x[i].data_ptr() for i in range(p * H * W)])
po = _lib.ptr_array([out[i].data_ptr() for i in range(M)])
w = rng.integers(-(1 << wbits), 1 << wbits, size=(M, 9 * p), dtype=np.int64)
bres = np.array([[int(rng.integers(0, q)) for q in eng.moduli[:ell]] for _ in range(M)], np.uint64) if wb else None
rc = eng._L.he_conv_square_sum_n(eng._h, _lib.addr(pi), 3, p, H, W, _lib.addr(po), M, 0, 0, H, _lib.addr(w),
                                 _lib.addr(bres) if wb else None, None, ell, eng.stream)
torch.cuda.synchronize()
print(f"cfg {cfg} H {H} bias {wb} wbits {wbits}: rc {rc}", eng._L.he_last_error() if rc else "", flush=True)
