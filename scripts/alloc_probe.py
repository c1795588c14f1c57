"""Probe: cost of large stream-ordered allocations under the shared cudaMallocAsync pool."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16834_b200 import configs  # noqa: E402,F401  (sets the allocator backend)
import torch  # noqa: E402

print(torch.cuda.get_allocator_backend())
from cuda.bindings import runtime as rt  # noqa: E402

err, pool = rt.cudaDeviceGetDefaultMemPool(0)
err, thr = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold)
print("default pool release threshold", err, thr)
err, cur = rt.cudaDeviceGetMemPool(0)
print("current pool is default:", int(cur) == int(pool))
G = 1 << 30
keep = torch.empty(45 * G // 8, dtype=torch.int64, device="cuda")
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    bufs = [torch.empty(22 * G // 8, dtype=torch.int64, device="cuda") for _ in range(4)]
    t1 = time.perf_counter()
    del bufs
    torch.cuda.synchronize()
    err, thr = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
    print(f"rep {rep}: 4 x 22 GB torch.empty {1e3 * (t1 - t):.1f} ms; pool reserved {int(thr) / G:.1f} GB")
