"""Time he_conv_square_sum on config 3's two layer shapes (uniform residues).

python scripts/time_convsq.py [reps]
  conv1: 3 -> 16 channels, 32x32, one 8-row tile + 2x2 pool, 14 limbs
  conv2: 16 -> 32 channels, 16x16, all rows + GAP, 12 limbs
  conv2 (carry plan): 3-component inputs, 14 limbs, 5-component GAP sums
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16834_b200 import _lib, configs  # noqa: E402  (selects the allocator first)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_16834_b200.engine import GpuEngine  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
eng = GpuEngine(configs.context(3, seed=7))
N = eng.N
rng = np.random.default_rng(0)


def case(p, H, W, M, pool, y0, y1, ell, wbits, nci=2):
    x = torch.empty((p * H * W, nci, ell, N), dtype=torch.int64, device=eng.device)
    for i, q in enumerate(eng.moduli[:ell]):
        x[:, :, i] = torch.randint(0, q, (p * H * W, nci, N), device=eng.device, dtype=torch.int64)
    nwin = ((y1 - y0) // 2) * (W // 2) if pool else 1
    out = torch.empty((M * nwin, 2 * nci - 1, ell, N), dtype=torch.int64, device=eng.device)
    pi = _lib.ptr_array([x[i].data_ptr() for i in range(p * H * W)])
    po = _lib.ptr_array([out[i].data_ptr() for i in range(M * nwin)])
    w = rng.integers(-(1 << wbits), 1 << wbits, size=(M, 9 * p), dtype=np.int64)

    def run():
        _lib.check(eng._L.he_conv_square_sum_n(eng._h, _lib.addr(pi), nci, p, H, W, _lib.addr(po), M, pool, y0,
                                               y1, _lib.addr(w), None, None, ell, eng.stream))

    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pairs = M * (y1 - y0) * W * ell * N
    print(f"nci={nci} p={p} M={M} {H}x{W} rows[{y0},{y1}) pool={pool} ell={ell}: {ms:.2f} ms  "
          f"{ms * 1e6 / pairs:.3f} ns per (channel, pixel, coeff)", flush=True)
    del x, out
    torch.cuda.empty_cache()


case(3, 32, 32, 16, 1, 0, 8, 14, 19)
case(16, 16, 16, 32, 0, 0, 16, 12, 14)
case(16, 16, 16, 32, 0, 0, 16, 14, 14, nci=3)
