"""Quick timing probe: one encrypted forward pass with a per-C-ABI-call breakdown.

usage: python scripts/probe_cfg.py [cfg=3] [reps=1]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16834_b200 import configs  # first: selects torch's allocator backend
import numpy as np
import torch

from paper_2604_16834_b200.engine import GpuEngine
from paper_2604_16834_b200.featuremajor import run_cnn, run_mlp
from paper_2604_16834_b200.packing import pack_features

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
eng = GpuEngine(configs.context(cfg, seed=1))
rng = np.random.default_rng(0)
t0 = time.time()
if cfg == 1:
    spec = configs.MLP1
    x = rng.uniform(0, 1, (2048, 64))
else:
    spec = configs.CNN3 if cfg == 3 else configs.CNN4
    x = rng.uniform(0, 1, (32768, 3 * 32 * 32))
wts = spec.make_weights(2)
cts = pack_features(eng, x)
eng._ensure_relin()
torch.cuda.synchronize()
print(f"setup+encrypt {time.time() - t0:.2f}s", flush=True)
for r in range(reps):
    eng.enable_timing(True)
    torch.cuda.synchronize()
    t = time.time()
    if cfg == 1:
        out = run_mlp(eng, cts, spec, wts) if r == reps - 1 else run_mlp(eng, [c for c in cts], spec, wts)
    else:
        out = run_cnn(eng, cts, spec, wts, release_inputs=False)
    torch.cuda.synchronize()
    dt = time.time() - t
    summ = eng.timing_summary()
    tot = sum(v[1] for v in summ.values())
    print(f"rep {r}: wall {dt:.3f}s  sum-of-calls {tot / 1e3:.3f}s  samples/s {x.shape[0] / dt:.1f}")
    for k, (n, ms, units) in sorted(summ.items(), key=lambda kv: -kv[1][1]):
        gbs = units[0] / (ms * 1e6) if ms else 0
        gmac = units[1] / (ms * 1e6) if ms else 0
        print(f"   {k:12s} calls {n:6d}  {ms:9.1f} ms  {gbs:8.1f} GB/s(alg)  {gmac:9.1f} GMAC/s")
    eng.release(*out)
print("peak mem GB", torch.cuda.max_memory_allocated() / 1e9)
