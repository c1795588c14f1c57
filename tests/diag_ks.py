"""Diagnostic (not collected by pytest): localise GPU key-switch mismatches."""
import sys

sys.path.insert(0, "tests")
sys.path.insert(0, "oracle")
sys.path.insert(0, ".")
import numpy as np
import torch

from helpers import engine_context, from_np, oracle_for, rand_residues, to_np
from paper_2604_16834_b200.engine import GpuEngine

for name in sys.argv[1:] or ["tiny"]:
    eng = GpuEngine(engine_context(name))
    orc = oracle_for(name)
    eng._ensure_relin()
    key = orc.switch_key(0)
    rng = np.random.default_rng(3)
    L = eng.context.n_q
    for ell in (L, 1):
        for kind in ("zero", "limb0", "rand"):
            d = rand_residues(rng, eng.moduli[:ell], (1,), eng.N)[0]
            if kind == "zero":
                d[:] = 0
            elif kind == "limb0":
                d[1:] = 0
            td = from_np(d, eng.device)
            o0 = torch.empty_like(td)
            o1 = torch.empty_like(td)
            P = lambda ts: np.array([t.data_ptr() for t in ts], np.uint64)
            a, b, c = P([td]), P([o0]), P([o1])
            rc = eng._L.he_keyswitch(eng._h, 0, a.ctypes.data, b.ctypes.data, c.ctypes.data, 1, ell, None)
            r0, r1 = orc.keyswitch(d, key)
            g0, g1 = to_np(o0), to_np(o1)
            print(name, "ell", ell, kind, "rc", rc, "o0 limbs equal", [bool(np.array_equal(g0[i], r0[i])) for i in range(ell)],
                  "o1 limbs equal", [bool(np.array_equal(g1[i], r1[i])) for i in range(ell)])
            if not np.array_equal(g0, r0):
                i = next(i for i in range(ell) if not np.array_equal(g0[i], r0[i]))
                diff = (g0[i].astype(object) - r0[i].astype(object)) % eng.moduli[i]
                print("   first bad limb", i, "gpu", g0[i][:4], "orc", r0[i][:4], "diff mod q", diff[:4])
