"""CPU oracle self-checks (no GPU).

* Philox4x32-10 against the published Random123 known-answer vectors;
* the C oracle against the independent pure-Python big-int restatement
  (oracle/pyref.py) on every primitive at a tiny ring;
* algebraic identities that hold for any correct RNS-CKKS: NTT products are
  negacyclic convolutions, INTT o NTT = id, rotation = slot roll, etc.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O
import pyref as R

ARGS = (5, [60, 40, 40, 40], [60, 60], 2)


def test_philox_known_answers():
    kat = [
        ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
        ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
        ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
         [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
    ]
    for ctr, key, want in kat:
        assert O.philox(ctr, key) == want
        assert R.philox(ctr, key) == want


@pytest.fixture(scope="module")
def both():
    return O.Oracle(*ARGS, seed=7), R.PyRef(*ARGS, seed=7)


def test_params_and_keys_match_bigint(both):
    o, p = both
    assert o.moduli == p.mod and o.psi == p.psi
    for q in o.moduli:
        assert (q - 1) % (2 * o.N) == 0
    sk = o.secret_key()
    assert all(list(map(int, sk[m])) == p.sk_ntt(m) for m in range(len(o.moduli)))
    for g in (0, 5, 25, O.power_key_elt(3), O.power_key_elt(4)):
        assert np.array_equal(o.switch_key(g), np.array(p.switch_key(g), np.uint64))


def test_ntt_matches_definition_and_negacyclic_product(both):
    o, p = both
    rng = np.random.default_rng(1)
    for m in range(len(o.moduli)):
        q = o.moduli[m]
        a = [int(v) for v in rng.integers(0, q, o.N, dtype=np.uint64)]
        b = [int(v) for v in rng.integers(0, q, o.N, dtype=np.uint64)]
        A, B = o.ntt(np.array(a, np.uint64), m), o.ntt(np.array(b, np.uint64), m)
        assert list(map(int, A)) == p.ntt(a, m)
        assert list(map(int, o.intt(A, m))) == a
        prod = [(int(x) * int(y)) % q for x, y in zip(A, B)]
        assert list(map(int, o.intt(np.array(prod, np.uint64), m))) == p.negacyclic(a, b, q)


def test_encode_encrypt_keyswitch_rescale_match_bigint(both):
    o, p = both
    rng = np.random.default_rng(2)
    v = rng.uniform(-1, 1, 16)
    assert list(o.encode(v)) == p.encode(v, 2.0 ** 40)
    ct = o.encrypt(v, 3)
    assert np.array_equal(ct, np.array(p.encrypt(v, 3), np.uint64))
    for g in (0, 5):
        k, pk = o.switch_key(g), p.switch_key(g)
        for ell in (4, 3, 1):
            d = ct[1, :ell].copy()
            o0, o1 = o.keyswitch(d, k)
            p0, p1 = p.keyswitch([list(map(int, x)) for x in d], pk, ell)
            assert np.array_equal(o0, np.array(p0, np.uint64)) and np.array_equal(o1, np.array(p1, np.uint64))
    pc = [[list(map(int, l)) for l in c] for c in ct]
    assert np.array_equal(o.rescale(ct), np.array(p.rescale(pc), np.uint64))
    assert list(o.decrypt_coeffs(ct)) == [float(x) for x in p.decrypt_coeffs(pc)]
    assert list(o.decode(o.decrypt_coeffs(ct), 2.0 ** 40)) == p.decode([float(x) for x in p.decrypt_coeffs(pc)],
                                                                        2.0 ** 40)


def test_homomorphic_identities_cfg1_ring():
    o = O.Oracle(12, [60, 40, 40, 40, 40], [60], 1, seed=1)
    rng = np.random.default_rng(0)
    a, b = rng.uniform(-1, 1, o.n), rng.uniform(-1, 1, o.n)
    ca, cb = o.encrypt(a, 0), o.encrypt(b, 1)
    s = o.scale
    assert np.max(np.abs(o.decrypt(ca, s) - a)) < 1e-7
    assert np.max(np.abs(o.decrypt(o.add(ca, cb), s) - (a + b))) < 1e-7
    m = o.mult_ct(ca, cb, o.switch_key(0))
    assert np.max(np.abs(o.decrypt(m, s * s / o.moduli[4]) - a * b)) < 1e-6
    for k in (1, 7, o.n - 1):
        g = O.galois_elt(k, o.N)
        r = o.rotate(ca, g, o.switch_key(g))
        assert np.max(np.abs(o.decrypt(r, s) - np.roll(a, -k))) < 1e-5
    # scalar plaintext product encoded at the dropped prime keeps the scale
    c = 0.37
    res = [int(np.rint(c * o.moduli[4])) % q for q in o.moduli[:5]]
    r = o.rescale(o.mul_const(ca, res))
    assert np.max(np.abs(o.decrypt(r, s) - c * a)) < 1e-7
    # lincomb is linear and exact
    w = np.array([3, -5, 7], np.int64)
    cs = [o.encrypt(rng.uniform(-1, 1, o.n), 10 + i) for i in range(3)]
    out = o.lincomb(cs, [0, 3], [0, 1, 2], w)[0]
    manual = o.add(o.add(o.mul_const(cs[0], [3 % q for q in o.moduli]),
                         o.mul_const(cs[1], [(-5) % q for q in o.moduli])),
                   o.mul_const(cs[2], [7 % q for q in o.moduli]))
    assert np.array_equal(out, manual)


def test_five_component_relin_rescale():
    """oc_relin_rescale_n: the 3-component form equals oc_relin_rescale bit for bit,
    and a 5-component square-of-square (keys s^2, s^3, s^4) decrypts to a^4 after
    the joint ModDown over P and the dropped limbs."""
    o = O.Oracle(12, [60, 40, 40, 40, 40, 40, 40], [60, 60], 2, seed=3)
    rng = np.random.default_rng(4)
    a = rng.uniform(-1, 1, o.n)
    ca = o.encrypt(a, 0)
    keys = [o.switch_key(O.power_key_elt(k)) for k in (2, 3, 4)]
    d3 = o.tensor_sq(ca)
    assert np.array_equal(d3, o.tensor(ca, ca))
    assert np.array_equal(o.relin_rescale_n(d3, keys[:1], 2), o.relin_rescale(d3, keys[0], 2))
    d5 = o.tensor_sq(d3)
    assert d5.shape[0] == 5
    s = o.scale ** 4
    for extra in (2, 3):  # final scale 2^80 / 2^40 (decrypt CRTs two limbs)
        r = o.relin_rescale_n(d5, keys, extra)
        sc = s
        for k in range(extra):
            sc /= o.moduli[6 - k]
        assert np.max(np.abs(o.decrypt(r, sc) - a ** 4)) < 1e-5


def test_hoisted_rotation_contract():
    """oc_rotate_hoisted: KS of the unrotated c1 with sigma_g^-1(key_g), + c0, then
    sigma_g -- decrypts to np.roll like the plain rotation, and equals that
    composition of the oracle's own keyswitch / automorphism."""
    o = O.Oracle(12, [60, 40, 40, 40, 40], [60], 1, seed=4)
    rng = np.random.default_rng(3)
    a = rng.uniform(-1, 1, o.n)
    ca = o.encrypt(a, 0)
    ell = ca.shape[1]
    for k in (1, 5, o.n - 3):
        g = O.galois_elt(k, o.N)
        hk = o.hoist_key(o.switch_key(g), g)
        r = o.rotate_hoisted(ca, g, hk)
        assert np.max(np.abs(o.decrypt(r, o.scale) - np.roll(a, -k))) < 1e-5
        k0, k1 = o.keyswitch(ca[1].copy(), hk)
        t = np.stack([o.add(ca[:1], k0[None])[0], k1])
        assert np.array_equal(r, o.automorphism(t, g).reshape(2, ell, o.N))
