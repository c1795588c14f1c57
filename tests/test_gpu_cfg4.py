"""Config 4 at its defined shape on one B200: the deep CNN (3 -> 16 -> 32 -> 64 ->
64 conv3x3 blocks, degree-3 activations, pools after blocks 2 and 4, dense 64 -> 10)
on 32x32 maps of 32768 samples, 24 x 50-bit limbs, streamed over image rows
(sharded_cnn.run_cnn_sharded, world size 1).

Reference counterpart: the conv / activation / pool chain of
/root/reference/pkg/src/hebatch/conv.py:109-173 on the feature-major layout.

Parity, layer by layer, on the GPU's own layer inputs:
  * every block's first tile: the exact conv sums (before the rescale; the
    tensor-core path with split-scale integer weights W 2^k) at 24 sampled
    evaluation points of EVERY output of the tile, replayed by the oracle's
    lincomb with the same integer weights on the sampled inputs (Oracle.coeff_view);
  * one output per block: rescale + degree-3 activation (two ct x ct products
    with relinearisation and rescale, constant adds) on full polynomials;
  * pooled rows: the next block's window inputs == the sums of the 4 activation
    outputs (sampled);
  * the dense head on full polynomials from the GPU's GAP sums;
and the logits decrypt to the float64 forward pass within 1e-3.
"""

from __future__ import annotations

import numpy as np
import pytest

from helpers import oracle_for, to_np

pytestmark = pytest.mark.gpu

TOL = 1e-3


def test_cfg4_full_shape_streamed_layerwise_bit_exact_vs_oracle():
    import torch

    import oracle_nets as ON
    from paper_2604_16834_b200 import configs
    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.featuremajor import dense_csr
    from paper_2604_16834_b200.packing import pack_features
    from paper_2604_16834_b200.sharded_cnn import conv3x3_window_groups, plan_input_level, run_cnn_sharded

    spec = configs.CNN4
    wts = spec.make_weights(1234)
    rng = np.random.default_rng(29)
    images = rng.uniform(0.0, 1.0, size=(32768, 3 * 32 * 32))
    eng = GpuEngine(configs.context(4, seed=5))
    orc = oracle_for("cfg4", seed=5)
    level = plan_input_level(spec)
    assert level == 14
    base = eng._enc_counter
    x = pack_features(eng, images, level=level)
    # inputs: the first 15 limbs of the top-level encryption, bit for bit
    for k in (0, 3071):
        ref = orc.encrypt(images[:, k], base + k)
        assert np.array_equal(to_np(x[k].data), ref[:, : level + 1]), k
    idx = np.unique(np.concatenate([[0, eng.N - 1], rng.choice(eng.N, 22, replace=False)]))
    tidx = torch.as_tensor(idx, device=eng.device)
    view = orc.coeff_view(len(idx))

    def samp(cts):
        return torch.stack([c.data.index_select(-1, tidx) for c in cts]).cpu().numpy().view(np.uint64)

    seen, rec = set(), {}
    H = {0: 32, 1: 32, 2: 16, 3: 16}

    def trace(stage, cts, info):
        if stage in ("gap", "dense"):
            rec[stage] = ([to_np(c.data) for c in cts], [c.scale for c in cts])
            return
        blk = info["blk"]
        if (stage, blk) in seen:
            return
        seen.add((stage, blk))
        if stage == "acc":
            r0, r1 = info["rows"]
            ya, yb = info["window"]
            ins = info["inputs"]
            rec[("acc", blk)] = dict(out=samp(cts), ins=samp(ins), in_scale=ins[0].scale, in_level=ins[0].level,
                                     rows=(r0, r1), window=(ya, yb), w=info["weights"].copy(),
                                     full0=to_np(cts[5].data), out_scale=cts[0].scale)
        else:  # act
            pre = info["pre"]
            assert info["channels"][0] == 0
            rec[("act", blk)] = dict(pre=to_np(pre[5].data), pre_scale=pre[5].scale, y=to_np(cts[5].data),
                                     y_scale=cts[5].scale, ys=samp(cts), n=len(cts), chans=info["channels"])

    out = run_cnn_sharded(eng, x, spec, wts, 0, 1, trace=trace)
    assert len(out) == 10
    rk = orc.switch_key(0)
    a_fold, _ = ON.fold(spec.act.coeffs)
    chans = spec.channels
    for blk in range(4):
        A = rec[("acc", blk)]
        p, q = chans[blk], chans[blk + 1]
        Hb = H[blk]
        Wb = Hb
        r0, r1 = A["rows"]
        ya, yb = A["window"]
        # --- exact conv sums of the tile (every output, 24 evaluation points)
        tp, col, tap, npix = conv3x3_window_groups(p, Hb, Wb, r0, r1, ya, yb)
        limbs = A["in_level"] + 1
        ql = orc.moduli[limbs - 1]
        # the tensor-core path's split-scale integer weights W * 2^k, per launch of <= 32 channels
        mult = ql * eng.context.scale / A["in_scale"]
        wi = np.zeros(A["w"].shape, np.int64)
        for c0 in range(0, q, 32):
            W_, F_ = GpuEngine.split_scale_weights(A["w"][c0:c0 + 32], mult)
            wi[c0:c0 + 32] = W_ * F_
            assert np.abs(W_).max() < 2 ** 23 and np.max(np.abs(W_ * F_ - A["w"][c0:c0 + 32] * mult)) <= F_ / 2
        rows, cols, ws = [0], [], []
        for m in range(q):
            for g in range(npix):
                for t in range(tp[g], tp[g + 1]):
                    cols.append(col[t])
                    ws.append(wi[m, tap[t]])
                rows.append(len(cols))
        ref = view.lincomb([np.ascontiguousarray(a) for a in A["ins"]], rows, cols, np.asarray(ws, np.int64))
        assert len(ref) == A["out"].shape[0] == q * npix
        for k in range(len(ref)):
            assert np.array_equal(A["out"][k], ref[k]), ("acc", blk, k)
        assert A["out_scale"] == ql * eng.context.scale
        # --- rescale + activation of output 5 on full polynomials
        C = rec[("act", blk)]
        z = orc.rescale(A["full0"])
        assert np.array_equal(C["pre"], z), ("rescale", blk)
        assert C["pre_scale"] == eng.context.scale
        y = ON.activation(orc, rk, [ON.OracleCts(z, C["pre_scale"])], spec.act.coeffs)[0]
        assert np.array_equal(C["y"], y.data), ("activation", blk)
        assert C["y_scale"] == y.scale
        # --- pooled row 0 feeds the next block's first window
        if blk in (1, 3) and blk + 1 < 4:
            nxt = rec[("acc", blk + 1)]
            ys, Wc = C["ys"], Wb
            for o in range(C["chans"][1]):   # the first channel chunk of the tile
                for xo in range(Wc // 2):
                    four = [ys[(o * 2 + dy) * Wc + 2 * xo + dx] for dy in (0, 1) for dx in (0, 1)]
                    s = four[0]
                    for f in four[1:]:
                        s = view.add(s, f)
                    nwin = nxt["window"][1] - nxt["window"][0]
                    got = nxt["ins"][o * nwin * (Wc // 2) + xo]
                    assert np.array_equal(got, s), ("pool", blk, o, xo)
    assert a_fold > 0
    # --- dense head on the GPU's GAP sums
    g, gs = rec["gap"]
    rp, cols = dense_csr(10, 64)
    ref = ON.lincomb(orc, [ON.OracleCts(a, s) for a, s in zip(g, gs)], rp, cols, wts.dense[0].reshape(-1),
                     bias=np.asarray(wts.dense[1], np.float64), out_scale=eng.context.scale)
    d, ds = rec["dense"]
    for k in range(10):
        assert ds[k] == ref[k].scale and np.array_equal(d[k], ref[k].data), ("dense", k)
    got = eng.decrypt_batch(out).T[:64]
    want = spec.forward_plain(wts, images[:64].reshape(64, 3, 32, 32))
    assert np.max(np.abs(got - want)) < TOL
