"""Time batched relinearisation (+ joint rescale) at config 3's top level: us per ciphertext.

python scripts/time_relin.py [B] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16834_b200 import _lib, configs  # noqa: E402  (selects the allocator first)
import torch  # noqa: E402

from paper_2604_16834_b200.engine import GpuEngine  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
eng = GpuEngine(configs.context(3, seed=7))
L, N = eng.context.n_q, eng.N
x = torch.empty((B, 3, L, N), dtype=torch.int64, device=eng.device)
for i, q in enumerate(eng.moduli[:L]):
    x[:, :, i] = torch.randint(0, q, (B, 3, N), device=eng.device, dtype=torch.int64)
eng._ensure_relin()
pi = _lib.ptr_array([x[i].data_ptr() for i in range(B)])
for extra in (2, 0):
    out = torch.empty((B, 2, L - extra, N), dtype=torch.int64, device=eng.device)
    po = _lib.ptr_array([out[i].data_ptr() for i in range(B)])

    def run():
        if extra:
            _lib.check(eng._L.he_relin_rescale(eng._h, _lib.addr(pi), _lib.addr(po), B, L, extra, eng.stream))
        else:
            _lib.check(eng._L.he_relin(eng._h, _lib.addr(pi), _lib.addr(po), B, L, eng.stream))

    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / (reps * B)
    print(f"{'relin_rescale(extra=2)' if extra else 'relin'} at ell={L}: {us:.1f} us/ct (B={B})", flush=True)
    del out
