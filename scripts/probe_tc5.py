"""tcgen05 kind::i8 MMA cost vs N and the A operand's shared-memory layout."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_16834_b200 import _lib
L = _lib.load()
for n in (16, 32, 64, 96, 112, 128):
    for sbo, lbo in ((0, 0), (256, 256), (640, 640), (1920, 1920), (1920, 128), (128, 1920)):
        r = np.zeros(2)
        rc = L.he_microbench_tc5_strided(0, n, sbo, lbo, r.ctypes.data)
        if rc:
            print(n, sbo, lbo, "rc", rc, L.he_last_error()); continue
        print(f"N={n:3d} A sbo={sbo:5d} lbo={lbo:5d}: {r[1]:6.1f} cycles/MMA  {r[0]/1e12:7.1f} TMAC/s", flush=True)
