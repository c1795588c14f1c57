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


ELL = 9  # input limbs of the plan (featuremajor.min_input_level for config 3)


def cfg3_op_counts(ell: int = ELL):
    """Exact per-group op counts of the config-3 carry plan (featuremajor.run_cnn
    with inputs at `ell` limbs): conv1 (deferred rescale) over 2-component inputs
    -> squares summed into 2x2 pools, NOT relinearised (3 components) -> conv2
    over those 3-component squares -> squares (6 products) summed into the GAP ->
    32 five-component relinearisations with a joint 6-limb ModDown -> dense at
    ell - 6 limbs -> rescale."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2604_16834_b200.featuremajor import conv3x3_csr

    N = 1 << 16
    nnz1 = len(conv3x3_csr(3, range(16), 32, 32)[1])
    nnz2 = len(conv3x3_csr(16, range(32), 16, 16)[1])
    return {
        # modular MACs (conv1 over 2 components, conv2 over 3, dense over 2)
        "lincomb_macs": nnz1 * 2 * ell * N + nnz2 * 3 * ell * N + 320 * 2 * (ell - 6) * N,
        # window sums of squares: 3 products per conv1 output coefficient, 6 per conv2 output
        "square_macs": 16384 * 3 * ell * N + 8192 * 6 * ell * N,
        "relin5": [(32, ell, 6)],
        "rescale": [(10, ell - 6)],
    }


def measure(seconds_budget: float = 20.0, threads: int | None = None, seed: int = 0, ell: int = ELL) -> dict:
    """Time the oracle on a bounded sample; returns samples/s for one 32768-sample group."""
    threads = threads or len(os.sched_getaffinity(0))
    wall0 = time.perf_counter()
    orc = O.Oracle(16, [40] * 14, [42] * 3, 3, seed=seed, scale=2.0 ** 40)
    rng = np.random.default_rng(seed)
    N = orc.N
    mods = orc.moduli

    def rand_ct(ell, nc=2):
        out = np.empty((nc, ell, N), np.uint64)
        for i in range(ell):
            out[:, i] = rng.integers(0, mods[i], (nc, N), dtype=np.uint64)
        return out

    ops = cfg3_op_counts(ell)
    res = {"threads": threads}
    # 1. linear combination throughput (OpenMP over outputs)
    n_out, k = 8 * threads, 27
    ins = [rand_ct(ell) for _ in range(k)]
    rows = np.arange(n_out + 1) * k
    cols = np.tile(np.arange(k), n_out)
    w = rng.integers(-(2 ** 41), 2 ** 41, len(cols))
    t = time.perf_counter()
    orc.lincomb(ins, rows, cols, w, n_threads=threads)
    dt = time.perf_counter() - t
    res["lincomb_mac_per_s"] = len(cols) * 2 * ell * N / dt
    # 2. five-component relinearisation + joint 6-limb ModDown, one per host thread
    keys = [orc.switch_key(O.power_key_elt(p)) for p in (2, 3, 4)]
    a = [rand_ct(ell, 5) for _ in range(threads)]
    t = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda c: orc.relin_rescale_n(c, keys, 6), a))
    per_relin = (time.perf_counter() - t) / threads
    res["relin5_s"] = per_relin
    # 3. rescale
    a = [rand_ct(ell - 6) for _ in range(threads)]
    t = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(orc.rescale, a))
    per_rs = (time.perf_counter() - t) / threads
    res["rescale_s"] = per_rs
    # 4. tensor products (the squares summed into pools): 4 modular products per coefficient
    a = [rand_ct(ell) for _ in range(threads)]
    t = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda c: orc.tensor(c, c), a))
    res["square_mac_per_s"] = threads * 4 * ell * N / (time.perf_counter() - t)
    total = ops["lincomb_macs"] / res["lincomb_mac_per_s"] + ops["square_macs"] / res["square_mac_per_s"]
    total += sum(cnt * per_relin for cnt, _, _ in ops["relin5"])
    total += sum(cnt * per_rs for cnt, _ in ops["rescale"])
    res["group_seconds_extrapolated"] = total
    res["samples_per_s"] = 32768.0 / total
    res["wall_s"] = time.perf_counter() - wall0          # the measured sample (incl. key generation)
    res["extrapolation_factor"] = total / res["wall_s"]
    res["sample"] = (f"oracle on {threads} host threads running the GPU's plan at {ell} limbs: {n_out}x{k}-term "
                     f"lincomb, {threads} five-component relinearisations with a joint 6-limb ModDown, {threads} "
                     f"rescales at {ell - 6} limbs, {threads} tensor products; extrapolated with the exact config-3 op "
                     f"counts of one 32768-sample group")
    return res


if __name__ == "__main__":
    import json

    print(json.dumps(measure(), default=str))
