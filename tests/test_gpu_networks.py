"""End-to-end encrypted networks on the B200 vs the float64 reference forward
pass (decrypt-level, 1e-3 max-abs as BASELINE.json requires) and vs the CPU
oracle (bit-exact, layerwise sampled: the oracle recomputes chosen output
ciphertexts from the GPU's own layer inputs)."""

from __future__ import annotations

import numpy as np
import pytest

from helpers import oracle_for, to_np

pytestmark = pytest.mark.gpu

TOL = 1e-3


def _cfg1_data(seed=0):
    from paper_2604_16834_b200 import configs

    rng = np.random.default_rng(seed)
    images = rng.uniform(0.0, 1.0, size=(2048, 8, 8))
    wts = configs.MLP1.make_weights(seed + 1)
    return images, wts


def test_cfg1_through_reference_api_matches_plaintext_and_counters():
    """pack_inputs -> conv_forward(k=1) -> mult_ct (x^2) -> conv_forward -> decrypt,
    the reference call sequence of SURVEY.md 3.A, on the GPU engine."""
    from paper_2604_16834_b200 import configs
    from paper_2604_16834_b200.conv import ConvSpec, conv_forward
    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.packing import PackingLayout, pack_inputs

    images, ((W1, b1), (W2, b2)) = _cfg1_data()
    eng = GpuEngine(configs.context(1, seed=3))
    lay1 = PackingLayout(n=2048, H=1, W=1, b=2048, p=64)
    cts = pack_inputs(eng, [im.reshape(64, 1, 1) for im in images], lay1)
    h = conv_forward(eng, cts, ConvSpec(W1[:, :, None, None], b1, lay1))
    h2 = [eng.mult_ct(x, x) for x in h]
    out = conv_forward(eng, h2, ConvSpec(W2[:, :, None, None], b2, lay1.with_channels(32)))
    got = np.stack([eng.decrypt(c) for c in out], axis=1)             # [samples, 10]
    ref = configs.MLP1.forward_plain([(W1, b1), (W2, b2)], images.reshape(2048, 64))
    assert np.max(np.abs(got - ref)) < TOL
    c = eng.snapshot_counters()
    assert (c.plain_mults, c.adds, c.ct_mults, c.rotations) == (2368, 2368, 32, 0)
    assert out[0].level == 1


def test_cfg1_fm_runner_bit_exact_vs_oracle():
    from paper_2604_16834_b200 import configs
    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.featuremajor import run_mlp
    from paper_2604_16834_b200.packing import pack_features

    images, wts = _cfg1_data(1)
    eng = GpuEngine(configs.context(1, seed=5))
    x = pack_features(eng, images.reshape(2048, 64))
    x_np = [to_np(c.data) for c in x]
    out = run_mlp(eng, x, configs.MLP1, wts)
    got = eng.decrypt_batch(out).T
    ref = configs.MLP1.forward_plain(wts, images.reshape(2048, 64))
    assert np.max(np.abs(got - ref)) < TOL
    # oracle replays the whole MLP with the same integer encodings
    orc = oracle_for("cfg1", seed=5)
    rk = orc.switch_key(0)
    moduli = orc.moduli
    cur, scales = x_np, [eng.context.scale] * 64
    (W1, b1), (W2, b2) = wts
    a, b = configs.MLP1.act.fold()
    for k, (w, bias, fold) in enumerate([(W1, b1, (a, b)), (W2, b2, (1.0, 0.0))]):
        ell = cur[0].shape[1]
        ql = moduli[ell - 1]
        q, p = w.shape
        rows = np.arange(q + 1) * p
        cols = np.tile(np.arange(p), q)
        s_out = eng.context.scale
        wf = (fold[0] * w.reshape(-1)) * (ql * s_out) / np.asarray(scales)[cols]
        acc = orc.lincomb(cur, rows, cols, np.rint(wf).astype(np.int64))
        nxt = []
        for o in range(q):
            r = orc.rescale(acc[o])
            bv = fold[0] * bias[o] + fold[1]
            r = orc.add_const(r, [int(np.rint(bv * s_out)) % m for m in moduli[: ell - 1]])
            nxt.append(r)
        cur, scales = nxt, [s_out] * q
        if k == 0:
            ql2 = moduli[ell - 2]
            cur = [orc.mult_ct(c, c, rk) for c in cur]
            scales = [s * s / ql2 for s in scales]
    for o in range(10):
        assert np.array_equal(to_np(out[o].data), cur[o]), o


@pytest.mark.slow
def test_cfg3_network_decrypt_and_sampled_bit_exact():
    from paper_2604_16834_b200 import configs
    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.featuremajor import fm_conv3x3, run_cnn
    from paper_2604_16834_b200.packing import pack_features

    rng = np.random.default_rng(7)
    spec = configs.CNN3
    images = rng.uniform(0.0, 1.0, size=(32768, 3, 32, 32)).astype(np.float64)
    wts = spec.make_weights(11)
    eng = GpuEngine(configs.context(3, seed=9))
    x = pack_features(eng, images.reshape(32768, -1))
    # sampled bit-exact check of conv1 + activation on a few outputs
    orc = oracle_for("cfg3", seed=9)
    a, b = spec.act.fold()
    w1, b1 = wts.convs[0]
    y = fm_conv3x3(eng, x, w1, b1, 32, 32, out_channels=[5], fold=(a, b))
    for (yy, xx) in [(0, 0), (13, 31), (31, 7)]:
        o = yy * 32 + xx
        terms = [(i, yy + dy, xx + dx, dy, dx) for i in range(3) for dy in (-1, 0, 1) for dx in (-1, 0, 1)
                 if 0 <= yy + dy < 32 and 0 <= xx + dx < 32]
        ins = [to_np(x[i * 1024 + py * 32 + px].data) for (i, py, px, _, _) in terms]
        ell = 14
        ql = eng.moduli[ell - 1]
        s = eng.context.scale
        wv = np.array([a * w1[5, i, dy + 1, dx + 1] for (i, _, _, dy, dx) in terms])
        wi = np.rint(wv * (ql * s) / s).astype(np.int64)
        acc = orc.lincomb(ins, [0, len(terms)], list(range(len(terms))), wi)[0]
        r = orc.rescale(acc)
        r = orc.add_const(r, [int(np.rint((a * b1[5] + b) * s)) % m for m in eng.moduli[:13]])
        assert np.array_equal(to_np(y[o].data), r), (yy, xx)
    rk = orc.switch_key(0)
    sq = eng.mult_ct_batch([y[0]], [y[0]])
    assert np.array_equal(to_np(sq[0].data), orc.mult_ct(to_np(y[0].data), to_np(y[0].data), rk))
    # lazy activation + pool window (0, 0): tensor, +c, sum of 4, relin, rescale
    import oracle_nets as ON

    win = [y[0], y[1], y[32], y[33]]
    c = 0.25 - 0.5 ** 2 / (4 * 0.125)
    t = eng.add_const_batch(eng.tensor_batch(win, win), [c] * 4)
    p = eng.lincomb_int(t, [0, 4], [0, 1, 2, 3], np.ones(4, np.int64), out_scale=4 * t[0].scale)
    r = eng.relin_rescale_batch(p)[0]
    oc = [ON.OracleCts(to_np(v.data), v.scale) for v in win]
    ot = [ON.add_const(orc, ON.tensor(orc, v, v), c) for v in oc]
    op = ON.lincomb_int(orc, ot, [0, 4], [0, 1, 2, 3], 4 * ot[0].scale)[0]
    orr = ON.relin_rescale(orc, rk, op)
    assert np.array_equal(to_np(r.data), orr.data) and r.scale == orr.scale
    eng.release(*y, *sq)
    # deferred-rescale conv (run_cnn's default for layers feeding pool / GAP)
    from paper_2604_16834_b200.featuremajor import deferred_weight_scale

    dw = deferred_weight_scale(eng, x)
    yd = fm_conv3x3(eng, x, w1, b1, 32, 32, out_channels=[5], fold=(a, b), weight_scale=dw)
    yy, xx = 13, 31
    terms = [(i, yy + dy, xx + dx, dy, dx) for i in range(3) for dy in (-1, 0, 1) for dx in (-1, 0, 1)
             if 0 <= yy + dy < 32 and 0 <= xx + dx < 32]
    ins = [to_np(x[i * 1024 + py * 32 + px].data) for (i, py, px, _, _) in terms]
    wi = np.rint(np.array([a * w1[5, i, dy + 1, dx + 1] for (i, _, _, dy, dx) in terms]) * dw).astype(np.int64)
    acc = orc.lincomb(ins, [0, len(terms)], list(range(len(terms))), wi)[0]
    so = x[0].scale * dw
    acc = orc.add_const(acc, [int(np.rint((a * b1[5] + b) * so)) % m for m in eng.moduli[:14]])
    assert yd[yy * 32 + xx].level == 13 and yd[0].scale == so
    assert np.array_equal(to_np(yd[yy * 32 + xx].data), acc)
    eng.release(*yd)
    # full network, decrypt-level
    out = run_cnn(eng, x, spec, wts)
    got = eng.decrypt_batch(out).T
    ref = spec.forward_plain(wts, images[:256])
    assert np.max(np.abs(got[:256] - ref)) < TOL


def test_cfg4_layout_sharded_runner_world1_bit_exact_vs_run_cnn():
    """sharded_cnn (config 4's output-channel layout) at world size 1 on the
    GPU equals featuremajor.run_cnn's non-lazy plan bit for bit (partial sums
    over the ring added mod q == the full sum), and decrypts to the float64
    forward pass: a degree-3 CNN on config 4's prime sizes (small ring)."""
    from helpers import engine_context

    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.featuremajor import Activation, CnnSpec, run_cnn
    from paper_2604_16834_b200.packing import pack_features
    from paper_2604_16834_b200.sharded_cnn import run_cnn_sharded

    spec = CnnSpec(channels=(3, 4, 4), H=8, W=8, act=Activation((0.5, 0.5, 0.0, 0.0625)), pool_after=(0, 1))
    wts = spec.make_weights(5)
    eng = GpuEngine(engine_context("cfg4s", seed=3))
    n = eng.context.n
    rng = np.random.default_rng(2)
    images = rng.uniform(0.0, 1.0, size=(n, 3 * 64))
    x = pack_features(eng, images)
    ref_out = run_cnn(eng, x, spec, wts, release_inputs=False, lazy_relin=False)
    sh_out = run_cnn_sharded(eng, x, spec, wts, 0, 1, release_inputs=False, tensor_cores=False)
    for o in range(10):
        assert np.array_equal(to_np(sh_out[o].data), to_np(ref_out[o].data)), o
        assert sh_out[o].scale == ref_out[o].scale and sh_out[o].level == ref_out[o].level
    got = eng.decrypt_batch(sh_out).T
    ref = spec.forward_plain(wts, images.reshape(n, 3, 8, 8))
    assert np.max(np.abs(got - ref)) < TOL
    # the tensor-core form (split-scale weights): same levels and scales, decrypts alike
    tc_out = run_cnn_sharded(eng, x, spec, wts, 0, 1, release_inputs=False, tensor_cores=True)
    for o in range(10):
        assert tc_out[o].scale == ref_out[o].scale and tc_out[o].level == ref_out[o].level
    assert np.max(np.abs(eng.decrypt_batch(tc_out).T - ref)) < TOL


@pytest.mark.gpu
def test_cfg3_min_level_encryption_and_network():
    """Inputs encrypted directly at featuremajor.min_input_level (config 3: 9 of
    14 limbs): the limbs equal the first 9 of the top-level encryption bit for
    bit, and the whole network decrypts to the float64 forward pass within TOL."""
    from paper_2604_16834_b200 import configs
    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.featuremajor import min_input_level, run_cnn
    from paper_2604_16834_b200.packing import pack_features

    rng = np.random.default_rng(21)
    spec = configs.CNN3
    images = rng.uniform(0.0, 1.0, size=(32768, 3 * 32 * 32))
    wts = spec.make_weights(5)
    eng = GpuEngine(configs.context(3, seed=4))
    lv = min_input_level(eng, spec)
    assert lv == 8
    few = np.ascontiguousarray(images[:, :4].T)
    top = eng.encrypt_batch(few)
    eng._enc_counter -= 4  # same randomness indices for the low-level encryption
    low = eng.encrypt_batch(few, level=lv)
    for t, lo in zip(top, low):
        assert lo.level == lv
        assert np.array_equal(to_np(lo.data), to_np(t.data)[:, :lv + 1])
    eng.release(*top, *low)
    x = pack_features(eng, images, level=lv)
    out = run_cnn(eng, x, spec, wts)
    assert out[0].level == lv - 7
    got = eng.decrypt_batch(out).T
    ref = spec.forward_plain(wts, images[:512].reshape(512, 3, 32, 32))
    assert np.max(np.abs(got[:512] - ref)) < TOL


def test_cbc_conv_forward_hoisted_rotations_cfg1_ring():
    """The reference's CBC 3x3 layer (conv_forward k=3: align_inputs' 8 rotations
    from 4 keys, here hoisted) through GpuEngine: decrypts to the direct
    zero-padded convolution, rotation count as the reference loop's."""
    from paper_2604_16834_b200 import configs
    from paper_2604_16834_b200.conv import ConvSpec, conv_forward, conv_keys
    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.packing import PackingLayout, pack_inputs, unpack_outputs

    eng = GpuEngine(configs.context(1, seed=2))
    lay = PackingLayout(n=2048, H=8, W=8, b=4, p=3)
    eng.register_rotation_keys(conv_keys(lay))
    rng = np.random.default_rng(5)
    imgs = [rng.uniform(-1, 1, size=(3, 8, 8)) for _ in range(4)]
    w = rng.normal(0, 0.3, size=(4, 3, 3, 3))
    before = eng.snapshot_counters().rotations
    outs = conv_forward(eng, pack_inputs(eng, imgs, lay), ConvSpec(w, np.zeros(4), lay))
    assert eng.snapshot_counters().rotations - before == 3 * 8
    x = np.stack(imgs)
    xp = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)))
    ref = sum(np.einsum("oi,bihw->bohw", w[:, :, dy, dx], xp[:, :, dy:dy + 8, dx:dx + 8])
              for dy in range(3) for dx in range(3))
    got = np.stack([unpack_outputs(o, lay, engine=eng) for o in outs], axis=1)
    assert np.max(np.abs(got - ref.reshape(4, 4, 64))) < TOL


@pytest.mark.slow
def test_cfg3_carry_plan_every_layer_bit_exact_vs_oracle_replay():
    """The exact path bench.py times -- config 3 at full size, inputs encrypted at
    min_input_level (9 limbs), run_cnn's fused carry plan on the kernels the bench
    launches (tcgen05 conv1 tiles with pooled 3-component squares, tcgen05 conv2 +
    5-component GAP sums, 5-component relinearisation dropping 6 primes, dense) --
    compared layer by layer with the oracle:
      * conv layers: every limb of 24 sampled evaluation points of EVERY output
        ciphertext, replayed from the encrypted inputs by the oracle's element-wise
        operations (oracle_nets.carry_plan_convs_sampled on Oracle.coeff_view; the
        same replay decrypts to the reference's two-block CNN in test_golden.py);
      * relinearisation: full polynomials, oc_relin_rescale_n on the GPU's GAP sums;
      * dense head: full polynomials, the oracle lincomb on the GPU's relinearised sums;
    and the logits decrypt to the float64 forward pass within 1e-3."""
    import torch

    import oracle as O
    import oracle_nets as ON
    from paper_2604_16834_b200 import configs
    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.featuremajor import dense_csr, min_input_level, run_cnn
    from paper_2604_16834_b200.packing import pack_features

    spec = configs.CNN3
    wts = spec.make_weights(11)
    rng = np.random.default_rng(17)
    images = rng.uniform(0.0, 1.0, size=(32768, 3 * 32 * 32))
    eng = GpuEngine(configs.context(3, seed=9))
    orc = oracle_for("cfg3", seed=9)
    level = min_input_level(eng, spec)
    assert level == 8
    x = pack_features(eng, images, level=level)
    idx = np.unique(np.concatenate([[0, eng.N - 1], rng.choice(eng.N, 22, replace=False)]))
    tidx = torch.as_tensor(idx, device=eng.device)

    def samp(cts):
        return torch.stack([c.data.index_select(-1, tidx) for c in cts]).cpu().numpy().view(np.uint64)

    xs = samp(x)
    rec = {"block0": {}, "scales": {}}

    def trace(stage, cts, info):
        if stage == "block" and info["blk"] == 0:
            rows = info["rows"]
            nr, Wo = len(rows) // 2, 16
            s = samp(cts)
            for o in range(16):
                for r in range(nr):
                    for xx in range(Wo):
                        rec["block0"][o * 256 + (rows[0] // 2 + r) * Wo + xx] = s[(o * nr + r) * Wo + xx]
            rec["scales"]["block0"] = cts[0].scale
            assert all(c.level == level for c in cts) and eng._ncomp(cts) == 3
        elif stage == "planar":
            # decode the documented layout [limb][N/8][y][x][component][byte plane][8 coeffs][16 channels]
            pc = cts
            assert (pc.channels, pc.H, pc.W, pc.level) == (16, 16, 16, level)
            d = pc.data.view(pc.limbs, eng.N // 8, 16, 16, 3, 5, 8, 16)
            ch, jj = torch.as_tensor(idx // 8, device=eng.device), torch.as_tensor(idx % 8, device=eng.device)
            t = d[:, ch, :, :, :, :, jj, :].to(torch.int64)           # [S][limb][y][x][comp][plane][channel]
            v = sum(t[:, :, :, :, :, k] << (8 * k) for k in range(5))  # [S][limb][y][x][comp][channel]
            v = v.permute(5, 2, 3, 4, 1, 0).reshape(4096, 3, pc.limbs, len(idx))
            v = v.cpu().numpy().view(np.uint64)
            for k in range(4096):
                rec["block0"][k] = v[k]
            rec["scales"]["block0"] = pc.scale
            rec["planar"] = True
        elif stage in ("gap", "relin", "dense"):
            rec[stage] = ([to_np(c.data) for c in cts], [c.scale for c in cts], info)

    out = run_cnn(eng, x, spec, wts, trace=trace)
    view = orc.coeff_view(len(idx))
    b0, s0, gap, sg, drops = ON.carry_plan_convs_sampled(view, orc.moduli, orc.scale, list(xs), eng.context.scale,
                                                         spec, wts)
    # conv1 + square + pool (3-component carry, planar layout on the tcgen05 path), every output
    assert rec.get("planar"), "the bench path carries conv1's squares in the planar layout"
    assert len(rec["block0"]) == len(b0) == 4096
    assert rec["scales"]["block0"] == s0
    for k in range(4096):
        assert np.array_equal(rec["block0"][k], b0[k]), ("block0", k)
    # conv2 + square + GAP (5 components), every output ciphertext
    g_gpu, g_sc, g_info = rec["gap"]
    assert g_info["drops"] == drops == 6 and len(g_gpu) == len(gap) == 32
    for k in range(32):
        assert g_sc[k] == sg
        assert np.array_equal(g_gpu[k][..., idx], gap[k]), ("gap", k)
    # 5-component relinearisation + joint ModDown over P u {6 dropped primes}
    keys = [orc.switch_key(O.power_key_elt(k)) for k in (2, 3, 4)]
    r_gpu, r_sc, _ = rec["relin"]
    for k in (0, 13, 31):
        assert np.array_equal(r_gpu[k], orc.relin_rescale_n(g_gpu[k], keys, drops)), ("relin", k)
    # dense head (lincomb + rescale + bias) on the GPU's relinearised sums
    rp, cols = dense_csr(10, 32)
    ref = ON.lincomb(orc, [ON.OracleCts(r, s) for r, s in zip(r_gpu, r_sc)], rp, cols, wts.dense[0].reshape(-1),
                     bias=np.asarray(wts.dense[1], np.float64), out_scale=eng.context.scale)
    d_gpu, d_sc, _ = rec["dense"]
    for k in range(10):
        assert d_sc[k] == ref[k].scale and np.array_equal(d_gpu[k], ref[k].data), ("dense", k)
    got = eng.decrypt_batch(out).T
    want = spec.forward_plain(wts, images[:256].reshape(256, 3, 32, 32))
    assert np.max(np.abs(got[:256] - want)) < TOL
