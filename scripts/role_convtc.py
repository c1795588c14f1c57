"""Per-role cycle breakdown of the tcgen05 conv kernels (he_convtc_profile)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16834_b200 import _lib, configs  # noqa
import numpy as np, torch
from paper_2604_16834_b200.engine import GpuEngine
def ev_ms(run, reps=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
eng = GpuEngine(configs.context(3, seed=7)); N, L = eng.N, eng._L
for name, (p, H, W, M, pool, y0, y1, ell, wbits, nci) in {
        "conv1 tile": (3, 32, 32, 16, 1, 0, 8, 9, 20, 2), "conv2": (16, 16, 16, 32, 0, 0, 16, 9, 14, 3)}.items():
    x = torch.empty((p * H * W, nci, ell, N), dtype=torch.int64, device=eng.device)
    for i, q in enumerate(eng.moduli[:ell]):
        x[:, :, i] = torch.randint(0, q, (p * H * W, nci, N), device=eng.device, dtype=torch.int64)
    nwin = ((y1 - y0) // 2) * (W // 2) if pool else 1
    out = torch.empty((M * nwin, 2 * nci - 1, ell, N), dtype=torch.int64, device=eng.device)
    pi = _lib.ptr_array([x[i].data_ptr() for i in range(p * H * W)]); po = _lib.ptr_array([out[i].data_ptr() for i in range(M * nwin)])
    w = np.random.default_rng(0).integers(-(1 << wbits), 1 << wbits, size=(M, 9 * p), dtype=np.int64)
    run = lambda: _lib.check(L.he_conv_square_sum_n(eng._h, _lib.addr(pi), nci, p, H, W, _lib.addr(po), M, pool, y0, y1, _lib.addr(w), None, None, ell, torch.cuda.current_stream().cuda_stream))
    run(); torch.cuda.synchronize()
    ms = ev_ms(run)
    _lib.check(L.he_convtc_profile(1, None))
    run(); torch.cuda.synchronize()
    r = np.zeros(7); _lib.check(L.he_convtc_profile(0, r.ctypes.data))
    r /= 148
    names = ["prod wait-empty", "prod total", "mma wait-full", "mma wait-dempty", "mma total", "epi wait-dfull", "epi total"]
    print(name, f"{ms:.2f} ms (no timers)", {n: f"{v/1e6:.2f}M" for n, v in zip(names, r)}, flush=True)
    del x, out; torch.cuda.empty_cache()
# planar conv2
ell = 9
pl = torch.empty(ell * (N // 8) * 16 * 16 * 1920, dtype=torch.uint8, device=eng.device)
w2 = np.random.default_rng(0).integers(-(1 << 14), 1 << 14, size=(32, 144), dtype=np.int64)
out2 = torch.empty((32, 5, ell, N), dtype=torch.int64, device=eng.device)
po2 = _lib.ptr_array([out2[i].data_ptr() for i in range(32)])
run = lambda: _lib.check(L.he_conv_square_sum_pl(eng._h, None, 3, 16, 16, 16, _lib.addr(po2), 32, 0, 0, 16, _lib.addr(w2), None, None, ell, pl.data_ptr(), None, torch.cuda.current_stream().cuda_stream))
run(); torch.cuda.synchronize()
ms = ev_ms(run)
_lib.check(L.he_convtc_profile(1, None)); run(); torch.cuda.synchronize()
r = np.zeros(7); _lib.check(L.he_convtc_profile(0, r.ctypes.data)); r /= 148
names = ["prod wait-empty", "prod total", "mma wait-full", "mma wait-dempty", "mma total", "epi wait-dfull", "epi total"]
print("conv2 planar", f"{ms:.2f} ms (no timers)", {n: f"{v/1e6:.2f}M" for n, v in zip(names, r)}, flush=True)
