"""Pins the plaintext references and the CPU oracle to the REFERENCE's outputs.

Fixtures in tests/golden/ were produced by running the reference simulator
(hebatch.SimulatorEngine, /root/reference) through its own public API
(tests/golden/make_golden.py).  These CPU tests check:
  * the float64 forward passes used by the GPU tests (MlpSpec / CnnSpec
    .forward_plain) reproduce the reference to 1e-9;
  * the CPU RNS-CKKS oracle running the frozen feature-major level plan
    decrypts to the reference's outputs within 1e-3 (BASELINE tolerance).
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from helpers import oracle_for

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _cfg1():
    g = np.load(os.path.join(GOLD, "cfg1_mlp.npz"))
    images = np.random.default_rng(0).uniform(0.0, 1.0, size=(2048, 8, 8))
    assert hashlib.sha256(images.tobytes()).hexdigest()[:16] == str(g["images_digest"])
    return g, images


def test_cfg1_plaintext_forward_matches_reference():
    from paper_2604_16834_b200 import configs

    g, images = _cfg1()
    wts = [(g["W1"], np.zeros(32)), (g["W2"], np.zeros(10))]
    ref = configs.MLP1.forward_plain(wts, images.reshape(2048, 64))
    assert np.max(np.abs(ref - g["logits"])) < 1e-9
    assert list(g["counters"]) == [2368, 2368, 32, 0] and int(g["out_level"]) == 1


def test_cfg1_oracle_ckks_decrypts_to_reference():
    """Config 1 end to end in RNS-CKKS on the CPU oracle (N = 2^12, 60+4x40
    bits): dense -> x^2 -> dense, same plan as featuremajor.run_mlp."""
    import oracle_nets as ON

    g, images = _cfg1()
    orc = oracle_for("cfg1", seed=11)
    rk = orc.switch_key(0)
    x = ON.encrypt_features(orc, images.reshape(2048, 64))
    s = orc.scale
    rows = np.arange(33) * 64
    cols = np.tile(np.arange(64), 32)
    h = ON.lincomb(orc, x, rows, cols, g["W1"].reshape(-1), bias=np.zeros(32), out_scale=s)
    h = ON.activation(orc, rk, h, (0.0, 0.0, 1.0))
    rows = np.arange(11) * 32
    cols = np.tile(np.arange(32), 10)
    out = ON.lincomb(orc, h, rows, cols, g["W2"].reshape(-1), bias=np.zeros(10), out_scale=s)
    got = np.stack([orc.decrypt(o.data, o.scale) for o in out], axis=1)
    assert out[0].ell - 1 == int(g["out_level"])             # same level as the reference (1 of max 4)
    assert np.max(np.abs(got - g["logits"])) < 1e-3


def _small_cnn_spec():
    from paper_2604_16834_b200.featuremajor import Activation, CnnSpec, CnnWeights

    g = np.load(os.path.join(GOLD, "fm_cnn_small.npz"))
    spec = CnnSpec(channels=(2, 3), H=4, W=4, act=Activation((0.25, 0.5, 0.125)), pool_after=(0,), n_classes=5)
    wts = CnnWeights([(g["w1"], np.zeros(3))], (g["w2"], np.zeros(5)))
    return g, spec, wts


def test_small_cnn_plaintext_forward_matches_reference():
    g, spec, wts = _small_cnn_spec()
    ref = spec.forward_plain(wts, g["images"])
    assert np.max(np.abs(ref - g["logits"])) < 1e-9


def test_small_cnn_oracle_ckks_decrypts_to_reference():
    """Feature-major conv3x3 + folded activation + pool sum + GAP sum + dense,
    in RNS-CKKS on the oracle (tiny ring, n = 16 samples)."""
    import oracle_nets as ON

    from paper_2604_16834_b200.featuremajor import gap_csr, pool2x2_csr

    g, spec, wts = _small_cnn_spec()
    orc = oracle_for("tiny", seed=4)
    rk = orc.switch_key(0)
    imgs = g["images"]
    x = ON.encrypt_features(orc, imgs.reshape(16, -1))
    s = orc.scale
    w1 = wts.convs[0][0]
    y = ON.conv3x3(orc, x, w1, np.zeros(3), 4, 4, ON.fold(spec.act.coeffs), s)
    rows = np.arange(6) * 3
    cols = np.tile(np.arange(3), 5)
    # eager plan: relinearise + rescale every activation, then pool and GAP
    z = ON.activation(orc, rk, y, spec.act.coeffs)
    rp, cols_p = pool2x2_csr(3, 4, 4)
    pz = ON.lincomb_int(orc, z, rp, cols_p, 4 * z[0].scale)
    rp, cols_g = gap_csr(3, 4)
    gz = ON.lincomb_int(orc, pz, rp, cols_g, 4 * pz[0].scale)
    out = ON.lincomb(orc, gz, rows, cols, wts.dense[0].reshape(-1), bias=np.zeros(5), out_scale=s)
    got = np.stack([orc.decrypt(o.data, o.scale) for o in out], axis=1)
    assert np.max(np.abs(got - g["logits"])) < 1e-3
    # lazy plan (run_cnn's last block): unrelinearised squares summed by the
    # GAP over all 16 pixels, ONE relin + rescale per channel, then dense
    zl = ON.activation_lazy(orc, y, spec.act.coeffs)
    rp, cols_g = gap_csr(3, 16)
    gl = ON.lincomb_int(orc, zl, rp, cols_g, 16 * zl[0].scale)
    gl = [ON.relin_rescale(orc, rk, c) for c in gl]
    out = ON.lincomb(orc, gl, rows, cols, wts.dense[0].reshape(-1), bias=np.zeros(5), out_scale=s)
    got = np.stack([orc.decrypt(o.data, o.scale) for o in out], axis=1)
    assert np.max(np.abs(got - g["logits"])) < 1e-3
    # deferred-rescale plan (run_cnn default): conv at weight scale ~2^20, no
    # rescale; lazy square; GAP; relin; drop two primes; dense
    yd = ON.conv3x3_deferred(orc, x, w1, np.zeros(3), 4, 4, ON.fold(spec.act.coeffs), s)
    assert yd[0].ell == 4
    zd = ON.activation_lazy(orc, yd, spec.act.coeffs)
    gd = ON.lincomb_int(orc, zd, rp, cols_g, 16 * zd[0].scale)
    gd = [ON.relin_rescale2(orc, rk, c) for c in gd]
    out = ON.lincomb(orc, gd, rows, cols, wts.dense[0].reshape(-1), bias=np.zeros(5), out_scale=s)
    got = np.stack([orc.decrypt(o.data, o.scale) for o in out], axis=1)
    assert out[0].ell == 1
    assert np.max(np.abs(got - g["logits"])) < 1e-3


def test_spec_examples_fixture_is_the_reference_behaviour():
    ex = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    assert ex["rotate_1"] == [2.0, 3.0, 4.0, 1.0]
    assert ex["rotate_-3"] == ex["rotate_1"]
    assert ex["conv_p3_q16_counts"] == [432, 24]
    assert ex["mult_plain_ones"][1] == 24


def test_carry_plan_oracle_replay_decrypts_to_reference():
    """The plan bench.py times (run_cnn's fused carry plan: conv1 + square + pool
    kept as 3-component sums, conv2 over them + square + GAP as 5-component sums,
    ONE 5-component relinearisation dropping carried_drops primes, dense +
    rescale) replayed on the oracle end to end decrypts to the reference
    simulator's two-block CNN (fm_cnn2_small.npz) within 1e-3.  The same replay
    (oracle_nets.carry_plan_convs_sampled) is the limb-level checker of the GPU
    network in tests/test_gpu_networks.py."""
    import oracle as O
    import oracle_nets as ON

    from paper_2604_16834_b200.featuremajor import Activation, CnnSpec, CnnWeights, dense_csr

    g = np.load(os.path.join(GOLD, "fm_cnn2_small.npz"))
    spec = CnnSpec(channels=(2, 3, 4), H=4, W=4, act=Activation((0.25, 0.5, 0.125)), pool_after=(0,), n_classes=5)
    wts = CnnWeights([(g["w1"], np.zeros(3)), (g["w2"], np.zeros(4))], (g["wd"], np.zeros(5)))
    assert np.max(np.abs(spec.forward_plain(wts, g["images"]) - g["logits"])) < 1e-9
    orc = oracle_for("carry9", seed=6)
    x = [o.data for o in ON.encrypt_features(orc, g["images"].reshape(16, -1))]
    b0, s0, gap, sg, drops = ON.carry_plan_convs_sampled(orc, orc.moduli, orc.scale, x, orc.scale, spec, wts)
    assert len(b0) == 3 * 2 * 2 and b0[0].shape[0] == 3 and gap[0].shape[0] == 5
    assert drops == 6                      # config 3's level plan: 9 limbs -> 3 after the relinearisation
    keys = [orc.switch_key(O.power_key_elt(k)) for k in (2, 3, 4)]
    rel = []
    for c in gap:
        s = sg
        for k in range(drops):
            s /= orc.moduli[c.shape[1] - 1 - k]
        rel.append(ON.OracleCts(orc.relin_rescale_n(c, keys, drops), s))
    rp, cols = dense_csr(5, 4)
    out = ON.lincomb(orc, rel, rp, cols, wts.dense[0].reshape(-1), bias=np.zeros(5), out_scale=orc.scale)
    assert out[0].ell == 2
    got = np.stack([orc.decrypt(o.data, o.scale) for o in out], axis=1)[:16]
    assert np.max(np.abs(got - g["logits"])) < 1e-3
