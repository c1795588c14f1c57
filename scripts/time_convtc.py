"""Time the fused conv kernels at config 3's benchmark shapes (9 limbs, uniform
residues): tcgen05 (convtc.cu) vs mma.sync (convsq_kernel.cuh).

python scripts/time_convtc.py [reps]
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
L = eng._L


def case(p, H, W, M, pool, y0, y1, ell, wbits, nci=2):
    x = torch.empty((p * H * W, nci, ell, N), dtype=torch.int64, device=eng.device)
    for i, q in enumerate(eng.moduli[:ell]):
        x[:, :, i] = torch.randint(0, q, (p * H * W, nci, N), device=eng.device, dtype=torch.int64)
    nwin = ((y1 - y0) // 2) * (W // 2) if pool else 1
    out = torch.empty((M * nwin, 2 * nci - 1, ell, N), dtype=torch.int64, device=eng.device)
    pi = _lib.ptr_array([x[i].data_ptr() for i in range(p * H * W)])
    po = _lib.ptr_array([out[i].data_ptr() for i in range(M * nwin)])
    w = rng.integers(-(1 << wbits), 1 << wbits, size=(M, 9 * p), dtype=np.int64)
    stream = torch.cuda.current_stream().cuda_stream
    res = {}
    for tc in (1, 0):
        L.he_set_conv_tc(tc)

        def run():
            _lib.check(L.he_conv_square_sum_n(eng._h, _lib.addr(pi), nci, p, H, W, _lib.addr(po), M, pool, y0,
                                              y1, _lib.addr(w), None, None, ell, stream))

        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        res[tc] = e0.elapsed_time(e1) / reps
        if tc:
            snap = out.clone()
        else:
            same = torch.equal(snap, out)
    L.he_set_conv_tc(1)
    rows = (y1 - y0)
    bytes_ = (p * (rows + 2) * W * nci + M * (rows // 2 if pool else 1) * (W // 2 if pool else 1) * (2 * nci - 1)) \
        * ell * N * 8
    print(f"nci={nci} p={p} M={M} {H}x{W} rows[{y0},{y1}) pool={pool} ell={ell} wbits={wbits}: "
          f"tcgen05 {res[1]:.2f} ms, mma.sync {res[0]:.2f} ms, bit-identical={same}, "
          f"tcgen05 HBM {bytes_ / res[1] / 1e6:.0f} GB/s", flush=True)
    del x, out, snap
    torch.cuda.empty_cache()


case(3, 32, 32, 16, 1, 0, 8, 9, 20)
case(3, 32, 32, 16, 1, 0, 32, 9, 20)
case(16, 16, 16, 32, 0, 0, 16, 9, 14, nci=3)


def planar_case(reps=3):
    """conv1 -> planar carry -> conv2 (the run_cnn chain) at config 3's shapes, 9 limbs."""
    ell = 9
    p1, H, W, M1 = 3, 32, 32, 16
    x = torch.empty((p1 * H * W, 2, ell, N), dtype=torch.int64, device=eng.device)
    for i, q in enumerate(eng.moduli[:ell]):
        x[:, :, i] = torch.randint(0, q, (p1 * H * W, 2, N), device=eng.device, dtype=torch.int64)
    pi = _lib.ptr_array([x[i].data_ptr() for i in range(p1 * H * W)])
    pl = torch.empty(ell * (N // 8) * 16 * 16 * 1920, dtype=torch.uint8, device=eng.device)
    w1 = rng.integers(-(1 << 20), 1 << 20, size=(M1, 27), dtype=np.int64)
    w2 = rng.integers(-(1 << 14), 1 << 14, size=(32, 144), dtype=np.int64)
    out2 = torch.empty((32, 5, ell, N), dtype=torch.int64, device=eng.device)
    po2 = _lib.ptr_array([out2[i].data_ptr() for i in range(32)])
    stream = torch.cuda.current_stream().cuda_stream

    def c1():
        _lib.check(L.he_conv_square_sum_pl(eng._h, _lib.addr(pi), 2, p1, H, W, None, M1, 1, 0, H, _lib.addr(w1),
                                           None, None, ell, None, pl.data_ptr(), stream))

    def c2():
        _lib.check(L.he_conv_square_sum_pl(eng._h, None, 3, 16, 16, 16, _lib.addr(po2), 32, 0, 0, 16,
                                           _lib.addr(w2), None, None, ell, pl.data_ptr(), None, stream))

    for name, f in (("conv1 -> planar (32 rows)", c1), ("planar -> conv2 (16 rows)", c2)):
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name}: {e0.elapsed_time(e1) / reps:.2f} ms", flush=True)


planar_case(reps)
