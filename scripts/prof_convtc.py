"""One conv1-tile launch of the tcgen05 fused conv (for ncu): config 3 shape, 9 limbs.
python scripts/prof_convtc.py [conv1|conv2] [launches]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16834_b200 import _lib, configs  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_16834_b200.engine import GpuEngine  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "conv1"   # conv1 | conv2 | conv1pl | conv2pl (planar carry)
launches = int(sys.argv[2]) if len(sys.argv) > 2 else 2
eng = GpuEngine(configs.context(3, seed=7))
N, L = eng.N, eng._L
if which.endswith("pl"):
    ell = 9
    pl = torch.empty(ell * (N // 8) * 16 * 16 * 1920, dtype=torch.uint8, device=eng.device)
    st = torch.cuda.current_stream().cuda_stream
    if which == "conv1pl":
        x = torch.empty((3 * 1024, 2, ell, N), dtype=torch.int64, device=eng.device)
        for i, q in enumerate(eng.moduli[:ell]):
            x[:, :, i] = torch.randint(0, q, (3 * 1024, 2, N), device=eng.device, dtype=torch.int64)
        pi = _lib.ptr_array([x[i].data_ptr() for i in range(3 * 1024)])
        w = np.random.default_rng(0).integers(-(1 << 20), 1 << 20, size=(16, 27), dtype=np.int64)
        f = lambda: L.he_conv_square_sum_pl(eng._h, _lib.addr(pi), 2, 3, 32, 32, None, 16, 1, 0, 8, _lib.addr(w), None,
                                            None, ell, None, pl.data_ptr(), st)
    else:
        pl.random_(0, 256)
        out = torch.empty((32, 5, ell, N), dtype=torch.int64, device=eng.device)
        po = _lib.ptr_array([out[i].data_ptr() for i in range(32)])
        w = np.random.default_rng(0).integers(-(1 << 14), 1 << 14, size=(32, 144), dtype=np.int64)
        f = lambda: L.he_conv_square_sum_pl(eng._h, None, 3, 16, 16, 16, _lib.addr(po), 32, 0, 0, 16, _lib.addr(w),
                                            None, None, ell, pl.data_ptr(), None, st)
    for _ in range(launches):
        _lib.check(f())
    torch.cuda.synchronize()
    if os.environ.get("CONVTC_ROLES"):  # per-role / per-phase cycle counters of one more launch
        _lib.check(L.he_convtc_profile(1, None))
        _lib.check(f())
        torch.cuda.synchronize()
        r = np.zeros(7)
        _lib.check(L.he_convtc_profile(0, r.ctypes.data))
        print(which, "counters (M cycles per CTA):", [round(v / 148 / 1e6, 2) for v in r])
    print("ok", which)
    sys.exit(0)
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
