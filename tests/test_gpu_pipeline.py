"""The paper's slot-reclaiming pipeline on the B200 engine:
stride-2 compaction (compact_strided; the reference's stub raises,
/root/reference/pkg/src/hebatch/conv.py:233-291) feeding the Eq. 29
accumulator, compared
limb for limb with the same layer code run on an oracle-backed engine (every
mult_plain / rotate / add an oracle call), and at decrypt level with the
expected slot permutation.
"""

from __future__ import annotations

import numpy as np
import pytest

from helpers import engine_context, oracle_for, to_np

pytestmark = pytest.mark.gpu


class _OCt:
    def __init__(self, data, level, scale):
        self.data, self.level, self.scale = data, level, scale


class OracleEngine:
    """The engine operations compact_strided / Accumulator call, restated on the
    CPU oracle with GpuEngine's exact encodings (full-width plaintexts encoded
    at q_last and rescaled; constants as round(c q_last); rotations through the
    Galois key of 5^k)."""

    def __init__(self, orc, context):
        from paper_2604_16834_b200.engine import RotationKeySet

        self.orc, self.context = orc, context
        self.keys = RotationKeySet(context.n)

    def register_rotation_keys(self, offs):
        self.keys.register(offs)

    def release(self, *cts):
        pass

    def mult_plain(self, ct, p):
        orc = self.orc
        ell = ct.level + 1
        ql = orc.moduli[ell - 1]
        v = np.asarray(p.slots, np.float64)
        if np.all(v == v[0]):
            val = int(np.rint(float(v[0]) * ql))
            prod = orc.mul_const(ct.data, np.array([val % q for q in orc.moduli[:ell]], np.uint64))
        else:
            prod = orc.mul_plain(ct.data, orc.plain_to_ntt(orc.encode(v, float(ql)), ell))
        return _OCt(orc.rescale(prod), ct.level - 1, ct.scale)

    def rotate(self, ct, k):
        from paper_2604_16834_b200.errors import MissingRotationKey

        c = k % self.context.n
        if c == 0:
            return ct
        if not self.keys.holds(c):
            raise MissingRotationKey(c)
        g = pow(5, c, 2 * self.orc.N)
        return _OCt(self.orc.rotate(np.ascontiguousarray(ct.data), g, self.orc.switch_key(g)), ct.level, ct.scale)

    def add(self, a, b):
        ell = min(a.level, b.level) + 1
        return _OCt(self.orc.add(np.ascontiguousarray(a.data[:, :ell]), np.ascontiguousarray(b.data[:, :ell])),
                    ell - 1, a.scale)


def test_compaction_and_accumulator_bit_exact_vs_oracle():
    from paper_2604_16834_b200.conv import Accumulator, accumulator_offsets, compact_strided, compaction_offsets
    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.packing import PackingLayout

    eng = GpuEngine(engine_context("cfg4s", seed=2))
    orc = oracle_for("cfg4s", seed=2)
    n = eng.context.n
    lay = PackingLayout(n=n, H=4, W=4, b=8)          # 8 images of 4x4 per ciphertext
    g, sts_p = 4, 8 * 4                                # after stride 2: 32 slots per tile, 4 tiles merged
    offs = compaction_offsets(lay) | accumulator_offsets(g, sts_p, n)
    eng.register_rotation_keys(offs)
    oe = OracleEngine(orc, eng.context)
    oe.register_rotation_keys(offs)
    rng = np.random.default_rng(6)
    tiles = [np.concatenate([rng.uniform(-1, 1, lay.occupied), np.zeros(n - lay.occupied)]) for _ in range(g)]
    acc_g, acc_o = Accumulator(eng, g, sts_p), Accumulator(oe, g, sts_p)
    for t in tiles:
        c = eng.encrypt(t)
        co = _OCt(to_np(c.data), c.level, c.scale)
        cg = compact_strided(eng, c, lay)
        cr = compact_strided(oe, co, lay)
        assert cg.level == cr.level
        assert np.array_equal(to_np(cg.data), cr.data)   # compaction limbs
        eng.release(c)
        acc_g.add(cg)
        acc_o.add(cr)
    out_g, out_o = acc_g.result(), acc_o.result()
    assert out_g.level == out_o.level
    assert np.array_equal(to_np(out_g.data), out_o.data)  # Eq. 29 merge limbs
    got = eng.decrypt(out_g)
    want = np.zeros(n)
    for i, t in enumerate(tiles):
        for j in range(lay.b):
            for y in range(2):
                for x in range(2):
                    want[i * sts_p + j * 4 + y * 2 + x] = t[j * 16 + 2 * y * 4 + 2 * x]
    assert np.max(np.abs(got - want)) < 1e-6
    c = eng.snapshot_counters()
    assert c.rotations > 0 and c.plain_mults > 0


def test_cbc_batched_fold_bit_exact_vs_oracle_and_counters():
    """The batched CBC 3x3 layer (conv_forward k=3 on GpuEngine: hoisted
    alignment + ONE he_lincomb_plain fold + one rescale per output + bias):
    limbs equal the oracle's replay of the same semantics (every product
    oc_mul_plain, sums oc_add, oc_rescale once, bias plaintext added to c0);
    decrypts to the direct convolution; counters advance as the reference fold's
    (reference conv.py:137-166)."""
    from paper_2604_16834_b200 import configs
    from paper_2604_16834_b200.conv import ConvSpec, align_inputs, cbc_plaintexts, conv_forward, conv_keys
    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.packing import PackingLayout, pack_inputs, unpack_outputs

    eng = GpuEngine(configs.context(1, seed=2))
    orc = oracle_for("cfg1", seed=2)
    lay = PackingLayout(n=2048, H=8, W=8, b=4, p=3)
    eng.register_rotation_keys(conv_keys(lay))
    rng = np.random.default_rng(7)
    imgs = [rng.uniform(-1, 1, size=(3, 8, 8)) for _ in range(4)]
    w = rng.normal(0, 0.3, size=(4, 3, 3, 3))
    bias = rng.normal(0, 0.1, size=4)
    spec = ConvSpec(w, bias, lay)
    cts = pack_inputs(eng, imgs, lay)
    c0 = eng.snapshot_counters()
    outs = conv_forward(eng, cts, spec)
    c1 = eng.snapshot_counters()
    assert c1.plain_mults - c0.plain_mults == 4 * 3 * 9
    assert c1.adds - c0.adds == 4 * (27 - 1) + 4
    assert c1.rotations - c0.rotations == 3 * 8
    # oracle replay of the batched semantics on the same aligned inputs
    taps = [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    al = [align_inputs(eng, ct, lay) for ct in cts]
    flat = [to_np(a[t].data) for a in al for t in taps]
    ell = cts[0].level + 1
    ql = float(orc.moduli[ell - 1])
    P = cbc_plaintexts(spec)
    for o in range(4):
        acc = None
        for j, a in enumerate(flat):
            prod = orc.mul_plain(a, orc.plain_to_ntt(orc.encode(P[o, j], ql), ell))
            acc = prod if acc is None else orc.add(acc, prod)
        r = orc.rescale(acc)
        bslots = np.zeros(lay.n)
        bslots[: lay.occupied] = bias[o]
        pt = orc.plain_to_ntt(orc.encode(bslots, cts[0].scale), ell - 1)
        r[0] = orc.add(r[:1], pt[None])[0]
        assert np.array_equal(to_np(outs[o].data), r), o
    x = np.stack(imgs)
    xp = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)))
    ref = sum(np.einsum("oi,bihw->bohw", w[:, :, dy, dx], xp[:, :, dy:dy + 8, dx:dx + 8])
              for dy in range(3) for dx in range(3)) + bias[None, :, None, None]
    got = np.stack([unpack_outputs(o, lay, engine=eng) for o in outs], axis=1)
    assert np.max(np.abs(got - ref.reshape(4, 4, 64))) < 1e-6
