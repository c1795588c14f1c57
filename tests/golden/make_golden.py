"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Imports the reference package (hebatch, /root/reference/pkg/src -- a float64
slot simulator) in this container and records its outputs for seeded inputs.
The reference cannot travel to the GPU box, so its results are committed as
small fixtures; tests compare against them (tests/test_golden.py, and the
GPU API tests).  Re-run:  python tests/golden/make_golden.py

Fixtures:
  cfg1_mlp.npz      BASELINE config 1 through the reference call sequence
                    (pack_inputs -> conv_forward k=1 -> mult_ct -> conv_forward
                    -> decrypt), plus its operation counters.
  fm_cnn_small.npz  a small feature-major CNN (conv3x3 + act 0.125x^2+0.5x+0.25
                    + 2x2 avg pool + GAP + dense) written with the reference's
                    own constant / mult_plain / add / mult_ct primitives.
  fm_cnn2_small.npz two conv blocks (2->3 channels at 4x4 + act + 2x2 avg pool,
                    3->4 at 2x2 + act + GAP, dense 4->5), the shape of config 3's
                    network, for the carry-plan replay (tests/test_golden.py).
  spec_examples.json  results of the SPEC.md operation examples on the reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from hebatch.conv import ConvSpec, conv_forward, conv_keys  # noqa: E402
from hebatch.engine import EngineContext, SimulatorEngine  # noqa: E402
from hebatch.errors import LengthExceedsSlots, LevelExhausted, MissingRotationKey  # noqa: E402
from hebatch.packing import PackingLayout, pack_inputs  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def cfg1():
    rng = np.random.default_rng(0)
    images = rng.uniform(0.0, 1.0, size=(2048, 8, 8))
    wr = np.random.default_rng(1)
    W1 = wr.normal(0.0, np.sqrt(1 / 64), (32, 64))
    W2 = wr.normal(0.0, np.sqrt(1 / 32), (10, 32))
    eng = SimulatorEngine(EngineContext(n=2048, max_level=4, bootstrap_reserve=1))
    lay = PackingLayout(n=2048, H=1, W=1, b=2048, p=64)
    cts = pack_inputs(eng, [im.reshape(64, 1, 1) for im in images], lay)
    h = conv_forward(eng, cts, ConvSpec(W1[:, :, None, None], np.zeros(32), lay))
    h2 = [eng.mult_ct(x, x) for x in h]
    out = conv_forward(eng, h2, ConvSpec(W2[:, :, None, None], np.zeros(10), lay.with_channels(32)))
    logits = np.stack([eng.decrypt(c) for c in out], axis=1)
    c = eng.snapshot_counters()
    np.savez_compressed(os.path.join(HERE, "cfg1_mlp.npz"), W1=W1, W2=W2, logits=logits,
                        images_digest=np.array(digest(images)), out_level=np.array(out[0].level),
                        counters=np.array([c.plain_mults, c.adds, c.ct_mults, c.rotations]))


def fm_cnn_small():
    """Feature-major CNN with the reference primitives: ciphertext (c, y, x)
    holds pixel (c, y, x) of n samples."""
    n, p, q, H, W = 16, 2, 3, 4, 4
    rng = np.random.default_rng(3)
    imgs = rng.uniform(0.0, 1.0, size=(n, p, H, W))
    w1 = rng.normal(0.0, np.sqrt(1 / (9 * p)), (q, p, 3, 3))
    w2 = rng.normal(0.0, np.sqrt(1 / q), (5, q))
    eng = SimulatorEngine(EngineContext(n=n, max_level=6, bootstrap_reserve=1))
    x = {(c, y, xx): eng.encrypt(imgs[:, c, y, xx]) for c in range(p) for y in range(H) for xx in range(W)}
    conv = {}
    for o in range(q):
        for y in range(H):
            for xx in range(W):
                acc = None
                for i in range(p):
                    for dy in (-1, 0, 1):
                        for dx in (-1, 0, 1):
                            yy, xs = y + dy, xx + dx
                            if 0 <= yy < H and 0 <= xs < W:
                                t = eng.mult_plain(x[(i, yy, xs)], eng.constant(w1[o, i, dy + 1, dx + 1]))
                                acc = t if acc is None else eng.add(acc, t)
                conv[(o, y, xx)] = acc
    act = {}
    for k, v in conv.items():   # 0.125 v^2 + 0.5 v + 0.25
        sq = eng.mult_plain(eng.mult_ct(v, v), eng.constant(0.125))
        lin = eng.mult_plain(v, eng.constant(0.5))
        act[k] = eng.add_plain(eng.add(sq, lin), eng.constant(0.25))
    pooled = {}
    for o in range(q):
        for y in range(H // 2):
            for xx in range(W // 2):
                s = None
                for a in (0, 1):
                    for b in (0, 1):
                        t = eng.mult_plain(act[(o, 2 * y + a, 2 * xx + b)], eng.constant(0.25))
                        s = t if s is None else eng.add(s, t)
                pooled[(o, y, xx)] = s
    gap = []
    for o in range(q):
        s = None
        for y in range(H // 2):
            for xx in range(W // 2):
                t = eng.mult_plain(pooled[(o, y, xx)], eng.constant(1.0 / ((H // 2) * (W // 2))))
                s = t if s is None else eng.add(s, t)
        gap.append(s)
    logits = []
    for k in range(5):
        s = None
        for o in range(q):
            t = eng.mult_plain(gap[o], eng.constant(w2[k, o]))
            s = t if s is None else eng.add(s, t)
        logits.append(eng.decrypt(s))
    np.savez_compressed(os.path.join(HERE, "fm_cnn_small.npz"), images=imgs, w1=w1, w2=w2,
                        logits=np.stack(logits, axis=1))


def _ref_conv_act(eng, x, w, p, q, H, W):
    """conv3x3 (pad 1) + 0.125 v^2 + 0.5 v + 0.25 with the reference primitives."""
    act = {}
    for o in range(q):
        for y in range(H):
            for xx in range(W):
                acc = None
                for i in range(p):
                    for dy in (-1, 0, 1):
                        for dx in (-1, 0, 1):
                            yy, xs = y + dy, xx + dx
                            if 0 <= yy < H and 0 <= xs < W:
                                t = eng.mult_plain(x[(i, yy, xs)], eng.constant(w[o, i, dy + 1, dx + 1]))
                                acc = t if acc is None else eng.add(acc, t)
                sq = eng.mult_plain(eng.mult_ct(acc, acc), eng.constant(0.125))
                lin = eng.mult_plain(acc, eng.constant(0.5))
                act[(o, y, xx)] = eng.add_plain(eng.add(sq, lin), eng.constant(0.25))
    return act


def fm_cnn2_small():
    """Two conv blocks in the reference primitives (config 3's layer sequence)."""
    n, p, q1, q2, H, W = 16, 2, 3, 4, 4, 4
    rng = np.random.default_rng(5)
    imgs = rng.uniform(0.0, 1.0, size=(n, p, H, W))
    w1 = rng.normal(0.0, np.sqrt(1 / (9 * p)), (q1, p, 3, 3))
    w2 = rng.normal(0.0, np.sqrt(1 / (9 * q1)), (q2, q1, 3, 3))
    wd = rng.normal(0.0, np.sqrt(1 / q2), (5, q2))
    eng = SimulatorEngine(EngineContext(n=n, max_level=12, bootstrap_reserve=1))
    x = {(c, y, xx): eng.encrypt(imgs[:, c, y, xx]) for c in range(p) for y in range(H) for xx in range(W)}
    a1 = _ref_conv_act(eng, x, w1, p, q1, H, W)
    pooled = {}
    for o in range(q1):
        for y in range(H // 2):
            for xx in range(W // 2):
                s = None
                for a in (0, 1):
                    for b in (0, 1):
                        t = eng.mult_plain(a1[(o, 2 * y + a, 2 * xx + b)], eng.constant(0.25))
                        s = t if s is None else eng.add(s, t)
                pooled[(o, y, xx)] = s
    a2 = _ref_conv_act(eng, pooled, w2, q1, q2, H // 2, W // 2)
    gap = []
    for o in range(q2):
        s = None
        for y in range(H // 2):
            for xx in range(W // 2):
                t = eng.mult_plain(a2[(o, y, xx)], eng.constant(1.0 / ((H // 2) * (W // 2))))
                s = t if s is None else eng.add(s, t)
        gap.append(s)
    logits = []
    for k in range(5):
        s = None
        for o in range(q2):
            t = eng.mult_plain(gap[o], eng.constant(wd[k, o]))
            s = t if s is None else eng.add(s, t)
        logits.append(eng.decrypt(s))
    np.savez_compressed(os.path.join(HERE, "fm_cnn2_small.npz"), images=imgs, w1=w1, w2=w2, wd=wd,
                        logits=np.stack(logits, axis=1))


def spec_examples():
    out = {}
    e = SimulatorEngine(EngineContext(n=4, max_level=25, bootstrap_reserve=10))
    out["encrypt_pad"] = e.decrypt(e.encrypt([1, 2])).tolist()
    out["encrypt_level"] = e.encrypt([1, 2]).level
    out["encrypt_empty"] = e.decrypt(e.encrypt([])).tolist()
    try:
        e.encrypt([1, 2, 3, 4, 5])
        out["encrypt_too_long"] = "ok"
    except LengthExceedsSlots:
        out["encrypt_too_long"] = "LengthExceedsSlots"
    e.register_rotation_keys([1, -1])
    ct = e.encrypt([1, 2, 3, 4])
    out["rotate_1"] = e.decrypt(e.rotate(ct, 1)).tolist()
    out["rotate_-3"] = e.decrypt(e.rotate(ct, -3)).tolist()
    out["rotate_0_same_handle"] = e.rotate(ct, 0) is ct
    try:
        e.rotate(ct, 2)
        out["rotate_missing"] = "ok"
    except MissingRotationKey as err:
        out["rotate_missing"] = ["MissingRotationKey", err.offset]
    out["add"] = e.decrypt(e.add(e.encrypt([1, 1]), e.encrypt([2, 3]))).tolist()
    m = e.mult_plain(e.encrypt([2, 3]), e.plain([1, 1, 1, 1]))
    out["mult_plain_ones"] = [e.decrypt(m).tolist(), m.level]
    out["mask"] = e.decrypt(e.mult_plain(e.encrypt([5, 6, 7, 8]), e.plain([1, 1, 0, 0]))).tolist()
    out["square"] = e.decrypt(e.mult_ct(e.encrypt([2, -3]), e.encrypt([2, -3]))).tolist()
    e2 = SimulatorEngine(EngineContext(n=4, max_level=2, bootstrap_reserve=1))
    c2 = e2.encrypt([1])
    c2 = e2.mult_plain(c2, e2.constant(1.0))
    c2 = e2.mult_plain(c2, e2.constant(1.0))
    try:
        e2.mult_plain(c2, e2.constant(1.0))
        out["level_exhausted"] = "ok"
    except LevelExhausted:
        out["level_exhausted"] = "LevelExhausted"
    e3 = SimulatorEngine(EngineContext(n=16, max_level=25, bootstrap_reserve=10))
    e3.register_rotation_keys([-1, 1, -8, 8])
    out["register_4"] = e3.resident_key_count
    kl = e3.snapshot_counters().key_loads
    e3.register_rotation_keys([1, -1])
    out["register_idempotent"] = [e3.resident_key_count, e3.snapshot_counters().key_loads - kl]
    out["conv_keys_W32"] = sorted(conv_keys(PackingLayout(n=4096, H=32, W=32, b=4, p=1)))
    e4 = SimulatorEngine(EngineContext(n=1024, max_level=25, bootstrap_reserve=10))
    lay = PackingLayout(n=1024, H=8, W=8, b=4, p=3)
    e4.register_rotation_keys(conv_keys(lay))
    rng = np.random.default_rng(5)
    cts = pack_inputs(e4, [rng.normal(size=(3, 8, 8)) for _ in range(4)], lay)
    before = e4.snapshot_counters()
    conv_forward(e4, cts, ConvSpec(rng.normal(size=(16, 3, 3, 3)), np.zeros(16), lay))
    d = e4.snapshot_counters().delta(before)
    out["conv_p3_q16_counts"] = [d.plain_mults, d.rotations]
    with open(os.path.join(HERE, "spec_examples.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    cfg1()
    fm_cnn_small()
    fm_cnn2_small()
    spec_examples()
    print("golden fixtures written to", HERE)
