"""Host-side cost of config-3 network passes: wall time of every allocation
(engine._alloc) in passes following a device synchronize vs. back-to-back."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16834_b200 import configs  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_16834_b200.engine import GpuEngine  # noqa: E402
from paper_2604_16834_b200.featuremajor import run_cnn  # noqa: E402
from paper_2604_16834_b200.packing import pack_features  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

spec = configs.CNN3
wts = spec.make_weights(1234)
eng = GpuEngine(configs.context(3, seed=42))
x = pack_features(eng, np.random.default_rng(0).uniform(0, 1, size=(32768, 3072)))
eng._ensure_relin()
_, pool = rt.cudaDeviceGetDefaultMemPool(0)
log = []
orig = eng._alloc


def timed_alloc(count, n_comp, limbs):
    t = time.perf_counter()
    r = orig(count, n_comp, limbs)
    log.append((count * n_comp * limbs * eng.N * 8 / 2 ** 30, 1e3 * (time.perf_counter() - t)))
    return r


eng._alloc = timed_alloc
G = 2 ** 30
for rep in range(5):
    if rep in (0, 3):
        torch.cuda.synchronize()
    log.clear()
    t = time.perf_counter()
    eng.release(*run_cnn(eng, x, spec, wts, release_inputs=False))
    t1 = time.perf_counter()
    _, thr = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold)
    _, res = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
    _, used = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrUsedMemHigh)
    slow = [(round(g, 1), round(ms, 1)) for g, ms in log if ms > 1]
    print(f"pass {rep} (sync before: {rep in (0, 3)}): host {1e3 * (t1 - t):.1f} ms, slow allocs (GB, ms) {slow}, "
          f"threshold {int(thr)}, reserved {int(res) / G:.1f} GB, used high {int(used) / G:.1f} GB", flush=True)
torch.cuda.synchronize()
