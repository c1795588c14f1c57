"""Bit-exact parity of the full-width plaintext and ciphertext-ciphertext
element-wise ops against the CPU oracle.

Reference operations (/root/reference/pkg/src/hebatch/engine.py):
  plain / constant   :389-402   -> he_encode_plain (FFT encode at a scale + NTT)
  add                :284-289   -> he_add / he_sub (2, 3 or 5 components)
  add_plain          :291-296   -> he_encode_plain at the ciphertext's scale + he_add on c0
  mult_plain         :298-304   -> he_encode_plain at q_last + he_mul_plain + rescale
Every limb is compared with the oracle's restatement (oc_encode, oc_plain_to_ntt,
oc_add, oc_sub, oc_mul_plain, oc_mul_const, oc_rescale) on the same inputs.
"""

from __future__ import annotations

import numpy as np
import pytest

from helpers import engine_context, from_np, oracle_for, rand_residues, to_np

pytestmark = pytest.mark.gpu

NAMES = ["tiny", "cfg1", "cfg3", "cfg2", "p15"]


@pytest.fixture(scope="module", params=NAMES)
def pair(request):
    from paper_2604_16834_b200.engine import GpuEngine

    name = request.param
    return name, GpuEngine(engine_context(name)), oracle_for(name)


def _oracle_pt(orc, vals, scale, ell):
    return orc.plain_to_ntt(orc.encode(vals, scale), ell)


def _mod_add(a, b, moduli):
    out = np.empty_like(a)
    for i, q in enumerate(moduli):
        s = a[i].astype(np.uint64) + b[i].astype(np.uint64)
        out[i] = np.where(s >= np.uint64(q), s - np.uint64(q), s)
    return out


def test_encode_plain_full_width_bit_exact(pair):
    import torch

    name, eng, orc = pair
    rng = np.random.default_rng(21)
    n = eng.context.n
    L = eng.context.n_q
    for scale, ell in ((eng.context.scale, L), (float(eng.moduli[L - 2]), L - 1)):
        vals = rng.uniform(-1, 1, n)
        pt = torch.empty((ell, eng.N), dtype=torch.int64, device=eng.device)
        vv = torch.as_tensor(vals, device=eng.device)
        assert eng._L.he_encode_plain(eng._h, vv.data_ptr(), n, scale, ell, pt.data_ptr(), None) == 0
        torch.cuda.synchronize()
        assert np.array_equal(to_np(pt), _oracle_pt(orc, vals, scale, ell)), (scale, ell)
    # a short vector is zero-padded (reference plain(): engine.py:389-397)
    vals = rng.uniform(-1, 1, max(1, n // 3))
    pt = torch.empty((L, eng.N), dtype=torch.int64, device=eng.device)
    vv = torch.as_tensor(vals, device=eng.device)
    assert eng._L.he_encode_plain(eng._h, vv.data_ptr(), vals.size, eng.context.scale, L, pt.data_ptr(), None) == 0
    torch.cuda.synchronize()
    full = np.zeros(n)
    full[: vals.size] = vals
    assert np.array_equal(to_np(pt), _oracle_pt(orc, full, eng.context.scale, L))


@pytest.mark.parametrize("nc", [2, 3])
def test_add_sub_bit_exact(pair, nc):
    name, eng, orc = pair
    rng = np.random.default_rng(22 + nc)
    L = eng.context.n_q
    ell = max(1, L - 1)
    a = rand_residues(rng, eng.moduli[:ell], (nc,), eng.N)
    b = rand_residues(rng, eng.moduli[:ell], (nc,), eng.N)
    ca = eng._wrap([from_np(a, eng.device)], ell - 1, [eng.context.scale])[0]
    cb = eng._wrap([from_np(b, eng.device)], ell - 1, [eng.context.scale])[0]
    s = eng.add(ca, cb)
    d = eng._add_batch([ca], [cb], sub=True)[0]
    assert np.array_equal(to_np(s.data), orc.add(a, b))
    assert np.array_equal(to_np(d.data), orc.sub(a, b))
    # mixed levels: the higher operand is read at the lower level (reference add: min level)
    hi = rand_residues(rng, eng.moduli[:L], (nc,), eng.N)
    ch = eng._wrap([from_np(hi, eng.device)], L - 1, [eng.context.scale])[0]
    s2 = eng.add(ch, cb)
    assert s2.level == ell - 1
    assert np.array_equal(to_np(s2.data), orc.add(np.ascontiguousarray(hi[:, :ell]), b))


def test_add_plain_full_width_bit_exact_and_decrypt(pair):
    name, eng, orc = pair
    rng = np.random.default_rng(31)
    n = eng.context.n
    x, pv = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    ct = eng.encrypt_batch(x[None])[0]
    out = eng.add_plain(ct, eng.plain(pv))
    ell = ct.level + 1
    pt = _oracle_pt(orc, pv, ct.scale, ell)
    ref = to_np(ct.data).copy()
    ref[0] = _mod_add(ref[0], pt, eng.moduli[:ell])
    assert np.array_equal(to_np(out.data), ref)
    assert np.max(np.abs(eng.decrypt(out) - (x + pv))) < 1e-6


def test_mult_plain_full_width_and_constant_bit_exact(pair):
    name, eng, orc = pair
    if eng.context.n_q < 2:
        pytest.skip("needs a level to rescale")
    rng = np.random.default_rng(41)
    n = eng.context.n
    x, pv = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    ct = eng.encrypt_batch(x[None])[0]
    ell = ct.level + 1
    ql = eng.moduli[ell - 1]
    out = eng.mult_plain(ct, eng.plain(pv))
    pt = _oracle_pt(orc, pv, float(ql), ell)
    ref = orc.rescale(orc.mul_plain(to_np(ct.data), pt))
    assert out.level == ct.level - 1
    assert np.array_equal(to_np(out.data), ref)
    assert abs(out.scale / ct.scale - 1.0) < 1e-12    # encoded at q_last: the scale comes back
    assert np.max(np.abs(eng.decrypt(out) - x * pv)) < 1e-5
    # scalar fast path (constant): the same residue at every NTT point
    c = 0.3125
    oc = eng.mult_plain(ct, eng.constant(c))
    v = int(np.rint(c * ql))
    res = np.array([v % q for q in eng.moduli[:ell]], np.uint64)
    refc = orc.rescale(orc.mul_const(to_np(ct.data), res))
    assert np.array_equal(to_np(oc.data), refc)
    assert np.max(np.abs(eng.decrypt(oc) - c * x)) < 1e-5


def test_add_plain_constant_bit_exact(pair):
    name, eng, orc = pair
    rng = np.random.default_rng(51)
    n = eng.context.n
    x = rng.uniform(-1, 1, n)
    ct = eng.encrypt_batch(x[None])[0]
    ell = ct.level + 1
    c = -0.75
    out = eng.add_plain(ct, eng.constant(c))
    v = int(np.rint(c * ct.scale))
    res = np.array([v % q for q in eng.moduli[:ell]], np.uint64)
    assert np.array_equal(to_np(out.data), orc.add_const(to_np(ct.data), res))
    assert np.max(np.abs(eng.decrypt(out) - (x + c))) < 1e-6


def test_multi_component_guards(pair):
    """Ops defined on 2-component ciphertexts refuse unrelinearised ones."""
    from paper_2604_16834_b200.errors import HebatchError

    name, eng, orc = pair
    rng = np.random.default_rng(61)
    n = eng.context.n
    a, b = eng.encrypt_batch(rng.uniform(-1, 1, (2, n)))
    t = eng.tensor_batch([a], [b])[0]
    with pytest.raises(HebatchError):
        eng.decrypt(t)
    with pytest.raises(HebatchError):
        eng.register_rotation_keys([1])
        eng.rotate(t, 1)
