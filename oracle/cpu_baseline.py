"""CPU baseline: the C oracle (ckks_oracle.c, OpenMP + one ciphertext per host
thread) timed on a bounded sample of the config-3 network and extrapolated
with that network's exact operation counts.

TEST / MEASUREMENT INFRASTRUCTURE ONLY: used by bench.py's cpu_baseline leg
and ``bench.py --impl reference``.  The reference package has no compiled
CPU implementation of this path (hebatch is a float64 simulator without
cryptography), so the oracle port stands in for it ("kind": "port").
"""

from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle as O  # noqa: E402


def cfg3_op_counts():
    """Exact per-group op counts of the frozen config-3 plan (featuremajor.run_cnn):
    conv1 at 14 limbs (deferred rescale) -> square+pool sums -> relin with a
    joint 2-limb ModDown at 14 -> conv2 at 12 -> square+GAP sums -> relin with a
    joint 2-limb ModDown at 12 -> dense at 10 limbs -> rescale."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2604_16834_b200.featuremajor import conv3x3_csr

    N = 1 << 16
    nnz1 = len(conv3x3_csr(3, range(16), 32, 32)[1])
    nnz2 = len(conv3x3_csr(16, range(32), 16, 16)[1])
    return {
        # modular MACs over 2 components (conv1, conv2, dense)
        "lincomb_macs": nnz1 * 2 * 14 * N + nnz2 * 2 * 12 * N + 320 * 2 * 10 * N,
        # squares summed into pools / GAP: 4 modular products per coefficient
        "square_macs": 16384 * 4 * 14 * N + 8192 * 4 * 12 * N,
        "relin_rescale2": [(4096, 14), (32, 12)],
        "rescale": [(10, 10)],
    }


def measure(seconds_budget: float = 20.0, threads: int | None = None, seed: int = 0) -> dict:
    """Time the oracle on a bounded sample; returns samples/s for one 32768-sample group."""
    threads = threads or len(os.sched_getaffinity(0))
    orc = O.Oracle(16, [40] * 14, [42] * 3, 3, seed=seed, scale=2.0 ** 40)
    rng = np.random.default_rng(seed)
    N = orc.N
    mods = orc.moduli

    def rand_ct(ell, nc=2):
        out = np.empty((nc, ell, N), np.uint64)
        for i in range(ell):
            out[:, i] = rng.integers(0, mods[i], (nc, N), dtype=np.uint64)
        return out

    ops = cfg3_op_counts()
    res = {"threads": threads}
    # 1. linear combination throughput (OpenMP over outputs)
    n_out, k = 8 * threads, 27
    ins = [rand_ct(14) for _ in range(k)]
    rows = np.arange(n_out + 1) * k
    cols = np.tile(np.arange(k), n_out)
    w = rng.integers(-(2 ** 41), 2 ** 41, len(cols))
    t = time.perf_counter()
    orc.lincomb(ins, rows, cols, w, n_threads=threads)
    dt = time.perf_counter() - t
    res["lincomb_mac_per_s"] = len(cols) * 2 * 14 * N / dt
    # 2. relinearisation + joint 2-limb ModDown of 3-component ciphertexts, one per host thread
    rk = orc.switch_key(0)
    per_relin = {}
    for ell in (14, 12):
        a = [rand_ct(ell, 3) for _ in range(threads)]
        t = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda c: orc.relin_rescale(c, rk, 2), a))
        per_relin[ell] = (time.perf_counter() - t) / threads
    res["relin_s"] = per_relin
    # 3. rescale
    per_rs = {}
    for ell in (10,):
        a = [rand_ct(ell) for _ in range(threads)]
        t = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(orc.rescale, a))
        per_rs[ell] = (time.perf_counter() - t) / threads
    res["rescale_s"] = per_rs
    # 4. tensor products (the squares summed into pools)
    a = [rand_ct(14) for _ in range(threads)]
    t = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda c: orc.tensor(c, c), a))
    res["square_mac_per_s"] = threads * 4 * 14 * N / (time.perf_counter() - t)
    total = ops["lincomb_macs"] / res["lincomb_mac_per_s"] + ops["square_macs"] / res["square_mac_per_s"]
    total += sum(cnt * per_relin[ell] for cnt, ell in ops["relin_rescale2"])
    total += sum(cnt * per_rs[ell] for cnt, ell in ops["rescale"])
    res["group_seconds_extrapolated"] = total
    res["samples_per_s"] = 32768.0 / total
    res["sample"] = (f"oracle on {threads} host threads running the same plan as the GPU: {n_out}x{k}-term lincomb "
                     f"at 14 limbs, {threads} relinearisations with a joint 2-limb ModDown at 14 and 12 limbs, "
                     f"{threads} rescales at 10 limbs, {threads} tensor products; extrapolated with the exact config-3 op counts of one "
                     f"32768-sample group")
    return res


if __name__ == "__main__":
    import json

    print(json.dumps(measure(), default=str))
