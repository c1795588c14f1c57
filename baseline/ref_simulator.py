"""R1 of BASELINE.md section 2: the REFERENCE itself (hebatch.SimulatorEngine, the
float64 slot simulator of /root/reference/pkg/src/hebatch/engine.py:229-420, no
cryptography) timed on config 3's feature-major network, through the
reference's own public primitives (constant / mult_plain / add / add_plain /
mult_ct, engine.py:276-313) -- the call pattern of tests/golden/make_golden.py.

The package is installed unmodified into baseline/_ref:
    python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
        --target baseline/_ref <copy of /root/reference/pkg> --no-deps
(--no-deps: its matplotlib dependency is absent and unused on this path).

A full config-3 group is ~10^6 simulator calls (minutes), so one bounded slice
per layer is timed on one host thread (the simulator is GIL-bound) and every
layer is scaled by its exact term / output count; the measured wall time and
the extrapolation factor are both reported.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")


def available() -> str | None:
    """None if hebatch imports from baseline/_ref, else the reason."""
    if not os.path.isdir(os.path.join(REF, "hebatch")):
        return "baseline/_ref/hebatch not installed"
    return None


def _conv_terms(p, H, W, rows, chans):
    t = 0
    for _ in chans:
        for y in rows:
            for x in range(W):
                for dy in (-1, 0, 1):
                    for dx in (-1, 0, 1):
                        if 0 <= y + dy < H and 0 <= x + dx < W:
                            t += p
    return t


def _measure_once(seed: int = 0) -> dict:
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from hebatch.engine import EngineContext, SimulatorEngine

    n = 32768
    rng = np.random.default_rng(seed)
    eng = SimulatorEngine(EngineContext(n=n, max_level=13, bootstrap_reserve=1))
    c0, c1, c2 = 0.25, 0.5, 0.125
    w1 = rng.normal(0.0, np.sqrt(1 / 27), (16, 3, 3, 3))
    w2 = rng.normal(0.0, np.sqrt(1 / 144), (32, 16, 3, 3))
    wd = rng.normal(0.0, np.sqrt(1 / 32), (10, 32))
    layers = {}
    wall0 = time.perf_counter()

    def conv_act(x, w, p, H, W, rows, chans):
        out = {}
        t0 = time.perf_counter()
        conv = {}
        for o in chans:
            for y in rows:
                for xx in range(W):
                    acc = None
                    for i in range(p):
                        for dy in (-1, 0, 1):
                            for dx in (-1, 0, 1):
                                yy, xs = y + dy, xx + dx
                                if 0 <= yy < H and 0 <= xs < W:
                                    t = eng.mult_plain(x[(i, yy, xs)], eng.constant(w[o, i, dy + 1, dx + 1]))
                                    acc = t if acc is None else eng.add(acc, t)
                    conv[(o, y, xx)] = acc
        t1 = time.perf_counter()
        for k, v in conv.items():
            sq = eng.mult_plain(eng.mult_ct(v, v), eng.constant(c2))
            lin = eng.mult_plain(v, eng.constant(c1))
            out[k] = eng.add_plain(eng.add(sq, lin), eng.constant(c0))
        t2 = time.perf_counter()
        return out, t1 - t0, t2 - t1

    # inputs: 3 channels x rows 0..2 (what conv1 rows 0..1 read)
    x = {(c, y, xx): eng.encrypt(rng.uniform(0.0, 1.0, n)) for c in range(3) for y in range(3) for xx in range(32)}
    a1, tc1, ta1 = conv_act(x, w1, 3, 32, 32, [0, 1], [0])
    layers["conv1"] = (tc1, _conv_terms(3, 32, 32, range(32), range(16)) / _conv_terms(3, 32, 32, [0, 1], [0]))
    layers["act1"] = (ta1, 16 * 1024 / len(a1))
    t0 = time.perf_counter()
    pooled = {}
    for xx in range(16):
        s = None
        for a in (0, 1):
            for b in (0, 1):
                t = eng.mult_plain(a1[(0, a, 2 * xx + b)], eng.constant(0.25))
                s = t if s is None else eng.add(s, t)
        pooled[(0, 0, xx)] = s
    layers["pool1"] = (time.perf_counter() - t0, 16 * 256 / 16)
    # conv2 row 0 of output channel 0 reads pooled rows 0..1 of all 16 channels
    x2 = {(c, y, xx): (pooled[(0, 0, xx)] if (c, y) == (0, 0) else eng.encrypt(rng.uniform(0.0, 1.0, n)))
          for c in range(16) for y in range(2) for xx in range(16)}
    a2, tc2, ta2 = conv_act(x2, w2, 16, 16, 16, [0], [0])
    layers["conv2"] = (tc2, _conv_terms(16, 16, 16, range(16), range(32)) / _conv_terms(16, 16, 16, [0], [0]))
    layers["act2"] = (ta2, 32 * 256 / len(a2))
    t0 = time.perf_counter()
    s = None
    for xx in range(16):
        t = eng.mult_plain(a2[(0, 0, xx)], eng.constant(1.0 / 256))
        s = t if s is None else eng.add(s, t)
    layers["gap"] = (time.perf_counter() - t0, 32 * 256 / 16)
    gap = [s] * 32
    t0 = time.perf_counter()
    logits = []
    for k in range(10):
        acc = None
        for o in range(32):
            t = eng.mult_plain(gap[o], eng.constant(wd[k, o]))
            acc = t if acc is None else eng.add(acc, t)
        logits.append(eng.decrypt(acc))
    layers["dense+decrypt"] = (time.perf_counter() - t0, 1.0)
    wall = time.perf_counter() - wall0
    measured = sum(t for t, _ in layers.values())
    group = sum(t * f for t, f in layers.values())
    return {"samples_per_s": n / group, "group_seconds_extrapolated": group, "measured_s": measured,
            "wall_s": wall, "extrapolation_factor": group / measured, "threads": 1,
            "layers": {k: {"measured_s": round(t, 4), "factor": round(f, 2)} for k, (t, f) in layers.items()},
            "sample": "reference hebatch.SimulatorEngine (float64 slots, no cryptography) on config 3's "
                      "feature-major CNN through its own constant/mult_plain/add/mult_ct calls: one slice per "
                      "layer (conv1 channel 0 rows 0-1, its activation and pool, conv2 channel 0 row 0, "
                      "activation, GAP partial, dense + decrypt), each scaled by its exact term/output count"}


def measure(seed: int = 0, repeats: int = 5) -> dict:
    """Median (by extrapolated group time) of ``repeats`` slice measurements."""
    runs = sorted((_measure_once(seed + k) for k in range(repeats)), key=lambda r: r["group_seconds_extrapolated"])
    r = dict(runs[len(runs) // 2])
    r["repeats"] = repeats
    r["wall_s"] = sum(x["wall_s"] for x in runs)
    return r


if __name__ == "__main__":
    import json

    print(json.dumps(measure()))
