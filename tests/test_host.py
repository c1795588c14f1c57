"""Host-side logic (no GPU): API dataclasses and validation, the layer CSR
builders against a direct convolution, activation folding algebra, and the
reference's slot semantics replayed on a numpy slot engine (which stands in
for the simulator so the generic conv_forward / compact_strided paths can be
exercised on CPU)."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from paper_2604_16834_b200 import configs
from paper_2604_16834_b200.conv import (ConvSpec, compact_strided, compaction_offsets, conv_forward, conv_keys)
from paper_2604_16834_b200.engine import CipherVec, EngineContext, OpCounters, PlainVec, RotationKeySet
from paper_2604_16834_b200.errors import (HebatchError, LengthExceedsSlots, MissingRotationKey, OverlappingRanges,
                                          ShapeMismatch, SlotConstraintViolated, UnsupportedKernel, UnsupportedStride)
from paper_2604_16834_b200.featuremajor import (Activation, conv3x3_csr, conv3x3_groups, gap_csr, pool2x2_csr)
from paper_2604_16834_b200.packing import (PackingLayout, encode_kernel_tap, encode_replicated, make_segment_mask,
                                           pack_inputs, unpack_outputs, TapOffset)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class SlotEngine:
    """numpy slot engine with the reference's semantics (test double)."""

    def __init__(self, n, max_level=25):
        self.context = EngineContext(n=n, max_level=max_level, bootstrap_reserve=1)
        self.keys = RotationKeySet(n)
        self.rot = 0
        self._id = 0

    def _ct(self, v, level):
        self._id += 1
        return CipherVec(data=np.asarray(v, float), level=level, scale_bits=40, id=self._id, n_slots=len(v))

    def encrypt(self, values):
        v = np.zeros(self.context.n)
        values = np.asarray(values, float).ravel()
        if len(values) > self.context.n:
            raise LengthExceedsSlots("too long")
        v[: len(values)] = values
        return self._ct(v, self.context.max_level)

    def decrypt(self, ct):
        return ct.data.copy()

    def rotate(self, ct, k):
        if k % self.context.n == 0:
            return ct
        if not self.keys.holds(k):
            raise MissingRotationKey(k)
        self.rot += 1
        return self._ct(np.roll(ct.data, -k), ct.level)

    def add(self, a, b):
        return self._ct(a.data + b.data, min(a.level, b.level))

    def add_plain(self, a, p):
        return self._ct(a.data + p.slots, a.level)

    def mult_plain(self, ct, p):
        return self._ct(ct.data * p.slots, ct.level - 1)

    def release(self, *cts):
        pass

    def register_rotation_keys(self, offs):
        self.keys.register(offs)


def test_engine_context_validation_matches_reference():
    with pytest.raises(ValueError):
        EngineContext(n=3)
    with pytest.raises(ValueError):
        EngineContext(n=8, max_level=4)          # default reserve 10 >= max_level (engine.py:58-59)
    with pytest.raises(ValueError):
        EngineContext(n=8, max_level=4, bootstrap_reserve=1, mult_level_cost=0)
    c = configs.context(3)
    assert (c.ring_degree, c.n_q, c.alpha, c.q_chain_bits[:2], c.p_chain_bits) == (65536, 14, 3, (40, 40), (42,) * 3)
    c1 = configs.context(1)
    assert (c1.n_q, c1.alpha, c1.p_chain_bits, c1.scale) == (5, 1, (60,), 2.0 ** 40)
    c2 = configs.context(2)
    assert (c2.n_q, c2.alpha, len(c2.p_chain_bits), c2.scale) == (24, 4, 4, 2.0 ** 50)


def test_rotation_keyset_and_counters():
    ks = RotationKeySet(16)
    assert ks.register([-1, 1, -8, 8]) == 3 and ks.resident == frozenset({1, 8, 15})
    assert len(ks) == 3 and ks.register([1]) == 0 and ks.generation_count == 3
    assert ks.unload([1]) is None
    assert not ks.holds(1) and ks.holds(-1)
    a, b = OpCounters(rotations=5, adds=3, peak_live_ciphertexts=9), OpCounters(rotations=2, adds=1)
    assert a.delta(b) == OpCounters(rotations=3, adds=2, peak_live_ciphertexts=9)


def test_packing_layout_and_encoders():
    with pytest.raises(SlotConstraintViolated):
        PackingLayout(n=16, H=2, W=2, b=5)
    with pytest.raises(ShapeMismatch):
        PackingLayout(n=16, H=0, W=2, b=1)
    lay = PackingLayout(n=32, H=3, W=3, b=2, p=2)
    tap = encode_kernel_tap(2.0, TapOffset(-1, -1), lay).plain.slots
    assert np.count_nonzero(tap[:9]) == 4 and np.count_nonzero(tap) == 8 and tap[4] == 2.0
    r = encode_replicated([1, 2], 4, 12)
    assert list(r.slots) == [1, 2, 0, 0] * 3
    with pytest.raises(LengthExceedsSlots):
        encode_replicated([1, 2, 3], 2, 8)
    with pytest.raises(OverlappingRanges):
        make_segment_mask([(0, 4), (3, 6)], 8)
    eng = SlotEngine(32)
    imgs = [np.arange(18, dtype=float).reshape(2, 3, 3) + 100 * j for j in range(2)]
    cts = pack_inputs(eng, imgs, lay)
    assert np.array_equal(cts[1].data[:18], np.concatenate([imgs[0][1].ravel(), imgs[1][1].ravel()]))
    assert np.array_equal(unpack_outputs(cts[0], lay, engine=eng)[1], imgs[1][0].ravel())
    with pytest.raises(ShapeMismatch):
        pack_inputs(eng, imgs[:1], lay)


def test_conv_forward_generic_path_counts_match_reference():
    ex = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    eng = SlotEngine(1024)
    lay = PackingLayout(n=1024, H=8, W=8, b=4, p=3)
    eng.register_rotation_keys(conv_keys(lay))
    rng = np.random.default_rng(5)
    imgs = [rng.normal(size=(3, 8, 8)) for _ in range(4)]
    w = rng.normal(size=(16, 3, 3, 3))
    outs = conv_forward(eng, pack_inputs(eng, imgs, lay), ConvSpec(w, np.zeros(16), lay))
    assert eng.rot == ex["conv_p3_q16_counts"][1]
    # slot values equal a direct zero-padded convolution
    x = np.stack(imgs)
    xp = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)))
    ref = sum(np.einsum("oi,bihw->bohw", w[:, :, dy, dx], xp[:, :, dy:dy + 8, dx:dx + 8])
              for dy in range(3) for dx in range(3))
    got = np.stack([unpack_outputs(o.data, lay) for o in outs], axis=1)   # [b, q, 64]
    assert np.max(np.abs(got - ref.reshape(4, 16, 64))) < 1e-9
    with pytest.raises(UnsupportedKernel):
        ConvSpec(np.zeros((1, 1, 5, 5)), np.zeros(1), lay)
    with pytest.raises(UnsupportedStride):
        ConvSpec(np.zeros((1, 1, 3, 3)), np.zeros(1), lay, stride=3)


def test_compact_strided_works_on_slot_engine():
    """The reference stub raises NotImplementedError (conv.py:274); ours gathers
    the stride-2 samples into contiguous m/4 segments."""
    lay = PackingLayout(n=64, H=4, W=4, b=2)
    eng = SlotEngine(64, max_level=30)
    eng.register_rotation_keys(compaction_offsets(lay))
    v = np.arange(64, dtype=float) + 1
    v[32:] = 0
    out = compact_strided(eng, eng.encrypt(v), lay).data
    want = np.zeros(64)
    for j in range(2):
        for y in range(2):
            for x in range(2):
                want[j * 4 + y * 2 + x] = v[j * 16 + 2 * y * 4 + 2 * x]
    assert np.array_equal(out, want)


def test_conv_csr_builders_equal_direct_convolution():
    rng = np.random.default_rng(1)
    p, q, H, W, S = 3, 4, 6, 5, 7
    x = rng.normal(size=(S, p, H, W))
    w = rng.normal(size=(q, p, 3, 3))
    feats = x.reshape(S, -1).T                       # feature-major: [p*H*W, samples]
    xp = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)))
    ref = sum(np.einsum("oi,sihw->sohw", w[:, :, dy, dx], xp[:, :, dy:dy + H, dx:dx + W])
              for dy in range(3) for dx in range(3)).reshape(S, -1).T
    rp, cols, widx = conv3x3_csr(p, range(q), H, W)
    out = np.array([(w.reshape(-1)[widx[a:b]][:, None] * feats[cols[a:b]]).sum(0) for a, b in zip(rp[:-1], rp[1:])])
    assert np.allclose(out, ref)
    tp, col, tap, npix = conv3x3_groups(p, H, W, rows=[2, 3, 5])
    wm = w.reshape(q, -1)
    for m in range(q):
        for gi, (y, xx) in enumerate([(r, c) for r in (2, 3, 5) for c in range(W)]):
            v = sum(wm[m, tap[t]] * feats[col[t]] for t in range(tp[gi], tp[gi + 1]))
            assert np.allclose(v, ref[m * H * W + y * W + xx])
    from paper_2604_16834_b200.featuremajor import conv3x3_fulltaps

    full = conv3x3_fulltaps(p, H, W, rows=[2, 3, 5])
    for gi in range(full.shape[0]):
        valid = [(t, int(full[gi, t])) for t in range(p * 9) if full[gi, t] >= 0]
        assert valid == [(int(tap[t]), int(col[t])) for t in range(tp[gi], tp[gi + 1])]
    rp, cols = pool2x2_csr(2, 4, 4)
    assert list(cols[:4]) == [0, 1, 4, 5] and len(rp) == 2 * 4 + 1
    rp, cols = gap_csr(2, 9, channel_offset=0)
    assert list(cols[9:12]) == [9, 10, 11]


def test_activation_folding_algebra():
    act = Activation((0.25, 0.5, 0.125))
    a, b = act.fold()
    x = np.linspace(-3, 3, 11)
    c = 0.25 - 0.5 ** 2 / (4 * 0.125)
    assert np.allclose((a * x + b) ** 2 + c, act(x))
    cub = Activation((0.5, 0.5, 0.0, 0.0625))
    a, _ = cub.fold()
    y = a * x
    assert np.allclose(y * (y * y + 0.5 / a) + 0.5, cub(x))
    assert configs.CNN3.levels_needed() == 5 and configs.CNN4.levels_needed() == 13


class HoistSlotEngine(SlotEngine):
    """SlotEngine with the batched rotate_hoisted entry (out[j][i] = rotate(cts[i], ks[j]))."""

    def __init__(self, n):
        super().__init__(n)
        self.hoist_calls = []

    def rotate_hoisted(self, cts, ks):
        self.hoist_calls.append((len(cts), tuple(ks)))
        return [[self.rotate(c, k) for c in cts] for k in ks]


def test_align_inputs_hoisted_path_matches_rotation_path():
    """conv.align_inputs on an engine with rotate_hoisted: two hoisted calls (+-1 on
    the input, +-W on the three row copies), the same nine aligned slot vectors and
    the same 8 rotations as the reference's rotation loop."""
    from paper_2604_16834_b200.conv import align_inputs

    lay = PackingLayout(n=256, H=8, W=8, b=2, p=1)
    plain, hoisted = SlotEngine(256), HoistSlotEngine(256)
    for e in (plain, hoisted):
        e.register_rotation_keys(conv_keys(lay))
    v = np.random.default_rng(1).normal(size=256)
    a = align_inputs(plain, plain.encrypt(v), lay)
    b = align_inputs(hoisted, hoisted.encrypt(v), lay)
    assert hoisted.hoist_calls == [(1, (-1, 1)), (3, (-8, 8))]
    assert plain.rot == hoisted.rot == 8
    for key in a:
        assert np.array_equal(a[key].data, b[key].data), key


def test_accumulator_eq29_on_slot_engine():
    """Eq. 29: g compacted blocks land in slots [i*sts', (i+1)*sts') of one
    ciphertext (SPEC.md:435-442 examples), inputs consumed incrementally; the
    stride-2 compaction + accumulator pipeline equals the concatenation of the
    compacted images; OccupancyOverflow / MissingRotationKey before any work."""
    from paper_2604_16834_b200.conv import Accumulator, accumulate, accumulator_offsets
    from paper_2604_16834_b200.errors import OccupancyOverflow

    n = 64
    eng = SlotEngine(n, max_level=30)
    blocks = [np.arange(4, dtype=float) + 10 * (i + 1) for i in range(4)]
    cts = [eng.encrypt(np.concatenate([b, np.full(n - 4, 7.0)])) for b in blocks]   # junk beyond sts'
    with pytest.raises(MissingRotationKey):
        accumulate(eng, cts, 4)
    eng.register_rotation_keys(accumulator_offsets(4, 4, n))
    assert accumulator_offsets(4, 4, n) == frozenset({60, 56, 52})
    out = accumulate(eng, cts, 4).data
    want = np.zeros(n)
    want[:16] = np.concatenate(blocks)
    assert np.array_equal(out, want)                      # [A|B|C|D], junk masked away
    assert accumulate(eng, [eng.encrypt(np.arange(n, dtype=float))], 8).data[:8].tolist() == list(range(8))
    with pytest.raises(OccupancyOverflow):
        Accumulator(eng, 5, 16)
    # compaction of 4 stride-2 tiles (2 images of 4x4 each), then the accumulator: effective batch x4
    lay = PackingLayout(n=n, H=4, W=4, b=2)
    eng.register_rotation_keys(compaction_offsets(lay))
    sts_p = lay.b * (lay.H // 2) * (lay.W // 2)          # 8 slots after compaction
    eng.register_rotation_keys(accumulator_offsets(4, sts_p, n))
    rng = np.random.default_rng(5)
    tiles = [np.concatenate([rng.uniform(size=32), np.zeros(32)]) for _ in range(4)]
    acc = Accumulator(eng, 4, sts_p)
    for t in tiles:
        acc.add(compact_strided(eng, eng.encrypt(t), lay))
    got = acc.result().data
    for i, t in enumerate(tiles):
        for j in range(2):
            for y in range(2):
                for x in range(2):
                    assert got[i * sts_p + j * 4 + y * 2 + x] == t[j * 16 + 2 * y * 4 + 2 * x]
    assert not got[4 * sts_p:].any()
