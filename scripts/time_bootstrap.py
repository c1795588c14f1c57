"""Per-phase and per-op timing of GpuEngine.bootstrap (synchronised wall
clock around every backend op; diagnostics only).
usage: python scripts/time_bootstrap.py [ring] (rings of tests/helpers.py)"""
import collections
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
from helpers import PARAMS, engine_context  # noqa: E402

from paper_2604_16834_b200 import bootstrap as B  # noqa: E402
from paper_2604_16834_b200.engine import GpuEngine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "boot16s"
spec = PARAMS[name]
depth = B.BootPlan(N=1 << spec[0], q0=1, hamming=spec[5] if len(spec) > 5 else 0).depth
eng = GpuEngine(engine_context(name, bootstrap_reserve=depth))
x = np.random.default_rng(1).uniform(-1, 1, eng.context.n)
ct = eng.drop_level_batch([eng.encrypt_batch(x[None])[0]], 0)[0]
eng.bootstrap(ct)
torch.cuda.synchronize()

stats = collections.defaultdict(lambda: [0, 0.0])
orig = {}
for op in ("mod_raise", "rotate_hoisted", "rotate", "conj", "mul_monomial", "add", "sub", "add_const", "mul_int",
           "mult_ct", "lincomb", "lincomb_plain"):
    orig[op] = getattr(B.GpuBootOps, op)

    def wrap(f, op=op):
        def g(self, *a, **k):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = f(self, *a, **k)
            torch.cuda.synchronize()
            stats[op][0] += 1
            stats[op][1] += (time.perf_counter() - t0) * 1e3
            return r
        return g
    setattr(B.GpuBootOps, op, wrap(orig[op]))

phases = {}
for ph in ("coeff_to_slot", "eval_mod", "slot_to_coeff"):
    f = getattr(B.Bootstrapper, ph)

    def wp(f, ph=ph):
        def g(self, *a, **k):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = f(self, *a, **k)
            torch.cuda.synchronize()
            phases[ph] = phases.get(ph, 0.0) + (time.perf_counter() - t0) * 1e3
            return r
        return g
    setattr(B.Bootstrapper, ph, wp(f))

n0 = eng._L.he_launch_count()
t0 = time.perf_counter()
out = eng.bootstrap(ct)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) * 1e3
print(f"{name}: bootstrap {tot:.1f} ms (synchronised per op), launches {eng._L.he_launch_count() - n0}, "
      f"err {np.max(np.abs(eng.decrypt(out) - x)):.2e}")
for k, v in phases.items():
    print(f"  phase {k:15s} {v:8.1f} ms")
for k, (c, ms) in sorted(stats.items(), key=lambda kv: -kv[1][1]):
    print(f"  op {k:15s} {c:4d} calls {ms:8.1f} ms  {ms / c:7.2f} ms/call")
