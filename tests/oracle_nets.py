"""The frozen feature-major level plan, replayed with the CPU oracle.

Test infrastructure: mirrors paper_2604_16834_b200.featuremajor (same CSR
builders, same integer weight encodings, same activation folding, same
rescale / constant-add order) but every arithmetic step is an oracle call, so
the GPU networks can be checked bit-exactly and the plan itself can be checked
at decrypt level against the reference simulator's golden outputs.
"""

from __future__ import annotations

import math

import numpy as np


class OracleCts:
    """A ciphertext as (numpy [2][ell][N] array, exact scale)."""

    def __init__(self, data, scale):
        self.data = data
        self.scale = scale

    @property
    def ell(self):
        return self.data.shape[1]


def residues(value_int, moduli, ell):
    return [int(value_int) % q for q in moduli[:ell]]


def lincomb(orc, ins, rows, cols, w, bias=None, out_scale=None):
    """engine.lincomb restated: integer weights at q_last * s_out / s_in, rescale, bias."""
    ell = min(c.ell for c in ins)
    arrs = [np.ascontiguousarray(c.data[:, :ell]) for c in ins]
    ql = orc.moduli[ell - 1]
    s_out = out_scale if out_scale is not None else ins[0].scale
    in_scale = np.array([c.scale for c in ins])
    wf = np.asarray(w, np.float64) * (ql * s_out) / in_scale[np.asarray(cols)]
    wi = np.rint(wf).astype(np.int64)
    acc = orc.lincomb(arrs, rows, cols, wi)
    outs = []
    for o, a in enumerate(acc):
        r = orc.rescale(a)
        if bias is not None:
            r = orc.add_const(r, residues(np.rint(bias[o] * s_out), orc.moduli, ell - 1))
        outs.append(OracleCts(r, s_out))
    return outs


def lincomb_int(orc, ins, rows, cols, out_scale):
    arrs = [np.ascontiguousarray(c.data) for c in ins]
    acc = orc.lincomb(arrs, rows, cols, np.ones(len(cols), np.int64))
    return [OracleCts(a, out_scale) for a in acc]


def mult_ct(orc, rk, a, b):
    ell = min(a.ell, b.ell)
    ql = orc.moduli[ell - 1]
    out = orc.mult_ct(np.ascontiguousarray(a.data[:, :ell]), np.ascontiguousarray(b.data[:, :ell]), rk)
    return OracleCts(out, a.scale * b.scale / ql)


def add_const(orc, a, v):
    """constant added to component 0 (works for 2- and 3-component ciphertexts)."""
    res = residues(np.rint(v * a.scale), orc.moduli, a.ell)
    out = a.data.copy()
    c0 = orc.add_const(np.ascontiguousarray(a.data[:2]), res)[0]
    out[0] = c0
    return OracleCts(out, a.scale)


def tensor(orc, a, b):
    """engine.tensor_batch: 3-component product, no relin / rescale, scale s_a s_b."""
    ell = min(a.ell, b.ell)
    return OracleCts(orc.tensor(np.ascontiguousarray(a.data[:, :ell]), np.ascontiguousarray(b.data[:, :ell])),
                     a.scale * b.scale)


def _relin_drops(orc, rk, a, drops):
    """engine.relin_rescale_batch: at N = 2^16 one joint ModDown over P u
    {dropped limbs} (oc_relin_rescale), else relin followed by `drops` rescales."""
    s = a.scale
    for k in range(drops):
        s /= orc.moduli[a.ell - 1 - k]
    if orc.N == 1 << 16:
        return OracleCts(orc.relin_rescale(np.ascontiguousarray(a.data), rk, drops), s)
    r = orc.relin(np.ascontiguousarray(a.data), rk)
    for _ in range(drops):
        r = orc.rescale(r)
    return OracleCts(r, s)


def relin_rescale(orc, rk, a):
    """engine.relin_rescale_batch(drops=1)."""
    return _relin_drops(orc, rk, a, 1)


def activation_lazy(orc, cts, coeffs):
    """apply_activation(lazy=True) for degree 2: tensor + constant (3 components)."""
    c0, c1, c2 = coeffs
    c = c0 - c1 * c1 / (4 * c2)
    out = [tensor(orc, x, x) for x in cts]
    return [add_const(orc, y, c) for y in out] if c != 0 else out


def activation(orc, rk, cts, coeffs):
    """featuremajor.apply_activation restated (inputs carry the folded affine map)."""
    if len(coeffs) == 3:
        c0, c1, c2 = coeffs
        c = c0 - c1 * c1 / (4 * c2)
        out = [mult_ct(orc, rk, x, x) for x in cts]
        return [add_const(orc, y, c) for y in out] if c != 0 else out
    c0, c1, c2, c3 = coeffs
    a = float(np.cbrt(c3))
    d = c1 / a
    sq = [mult_ct(orc, rk, x, x) for x in cts]
    sq = [add_const(orc, y, d) for y in sq] if d else sq
    cub = [mult_ct(orc, rk, x, y) for x, y in zip(cts, sq)]
    return [add_const(orc, y, c0) for y in cub] if c0 else cub


def fold(coeffs):
    if len(coeffs) == 3:
        c0, c1, c2 = coeffs
        a = math.sqrt(c2)
        return a, c1 / (2 * a)
    return float(np.cbrt(coeffs[3])), 0.0


def conv3x3(orc, ins, w, bias, H, W, fold_ab, out_scale):
    """fm_conv3x3 restated through the same pixel groups, expanded to CSR."""
    from paper_2604_16834_b200.featuremajor import conv3x3_groups

    q, p = w.shape[:2]
    a, b = fold_ab
    tp, col, tap, npix = conv3x3_groups(p, H, W)
    wm = a * w.reshape(q, p * 9)
    rows, cols, ws = [0], [], []
    for m in range(q):
        for g in range(npix):
            for t in range(tp[g], tp[g + 1]):
                cols.append(col[t])
                ws.append(wm[m, tap[t]])
            rows.append(len(cols))
    # engine.lincomb_grouped encodes wm (not per-term) -- identical floats
    bias_out = np.repeat(a * np.asarray(bias, np.float64) + b, npix)
    return lincomb(orc, ins, rows, cols, ws, bias=bias_out, out_scale=out_scale)


def conv3x3_deferred(orc, ins, w, bias, H, W, fold_ab, target_scale):
    """fm_conv3x3(weight_scale=deferred_weight_scale(...)) restated: integer
    weights round(a w dw), NO rescale, bias at s_in dw."""
    from paper_2604_16834_b200.featuremajor import conv3x3_groups

    q, p = w.shape[:2]
    a, b = fold_ab
    ell = ins[0].ell
    s_in = ins[0].scale
    dw = math.sqrt(target_scale * orc.moduli[ell - 1] * orc.moduli[ell - 2]) / s_in
    tp, col, tap, npix = conv3x3_groups(p, H, W)
    wi = np.rint((a * w.reshape(q, p * 9)) * dw).astype(np.int64)
    rows, cols, ws = [0], [], []
    for m in range(q):
        for g in range(npix):
            for t in range(tp[g], tp[g + 1]):
                cols.append(col[t])
                ws.append(wi[m, tap[t]])
            rows.append(len(cols))
    acc = orc.lincomb([np.ascontiguousarray(c.data) for c in ins], rows, cols, ws)
    s_out = s_in * dw
    bias_out = np.repeat(a * np.asarray(bias, np.float64) + b, npix)
    return [OracleCts(orc.add_const(x, residues(np.rint(bias_out[o] * s_out), orc.moduli, ell)), s_out)
            for o, x in enumerate(acc)]


def relin_rescale2(orc, rk, a):
    """engine.relin_rescale_batch(drops=2) after a deferred-rescale conv."""
    return _relin_drops(orc, rk, a, 2)


def encrypt_features(orc, feats, base_index=0):
    """feature-major packing: column f of feats -> ciphertext f."""
    return [OracleCts(orc.encrypt(feats[:, f], base_index + f), orc.scale) for f in range(feats.shape[1])]


# ---------------------------------------------------------------- the carry plan (bench path)
def _deferred_dw(moduli, delta, limbs, s_in, drops):
    """featuremajor.deferred_weight_scale restated: (s_in dw)^2 / (q_{l-1}..q_{l-drops}) = Delta."""
    prod = 1.0
    for k in range(drops):
        prod *= moduli[limbs - 1 - k]
    return math.sqrt(delta * prod) / s_in


def _carried_drops(moduli, delta, limbs, s_in, min_scale=2.0 ** 16):
    """featuremajor.carried_drops restated: the fewest primes giving an integer weight scale >= 2^16."""
    for d in range(2, limbs):
        if _deferred_dw(moduli, delta, limbs, s_in, d) >= min_scale:
            return d
    raise AssertionError("no level budget for the carried activation")


def _fulltaps(p, H, W):
    """[pixel][9p] input index per tap slot i*9 + (dy+1)*3 + (dx+1) (-1 outside), pixels row-major."""
    out = np.full((H * W, 9 * p), -1, np.int64)
    for y in range(H):
        for x in range(W):
            for i in range(p):
                for k in range(9):
                    yy, xx = y + k // 3 - 1, x + k % 3 - 1
                    if 0 <= yy < H and 0 <= xx < W:
                        out[y * W + x, i * 9 + k] = i * H * W + yy * W + xx
    return out


def conv_square_sum_sampled(view, ins, p, H, W, wi, bres, cres, pool):
    """engine.conv_square_sum restated on sampled evaluation points (view =
    Oracle.coeff_view): deferred conv (integer weights, no rescale) -> + bias on
    component 0 -> square (oc_tensor_sq: 3 components from 2, 5 from 3) -> sum
    over each 2x2 window (pool) or every pixel (GAP) -> + the window constant on
    component 0.  ins: p*H*W arrays [nc][ell][S]; returns [M][nwin] (pool,
    window-major per channel) or [M] (GAP) arrays [2nc-1][ell][S]."""
    M = wi.shape[0]
    taps = _fulltaps(p, H, W)
    rows, cols, ws = [0], [], []
    for m in range(M):
        for px in range(H * W):
            for t in np.nonzero(taps[px] >= 0)[0]:
                cols.append(int(taps[px, t]))
                ws.append(int(wi[m, t]))
            rows.append(len(cols))
    conv = view.lincomb(ins, rows, cols, ws)
    nc = ins[0].shape[0]
    sq = []
    for k, o in enumerate(conv):
        m = k // (H * W)
        if bres is not None:
            o = o.copy()
            o[:2] = view.add_const(np.ascontiguousarray(o[:2]), [int(v) for v in bres[m]])
        sq.append(view.tensor_sq(o) if nc == 3 else view.tensor(o, o))
    if pool:
        wins = [[(2 * wy + a) * W + 2 * wx + b for a in (0, 1) for b in (0, 1)]
                for wy in range(H // 2) for wx in range(W // 2)]
    else:
        wins = [list(range(H * W))]
    out = []
    for m in range(M):
        for win in wins:
            acc = sq[m * H * W + win[0]]
            for px in win[1:]:
                acc = view.add(acc, sq[m * H * W + px])
            acc = acc.copy()
            acc[:2] = view.add_const(np.ascontiguousarray(acc[:2]), [int(v) for v in cres])
            out.append(acc)
    return out


def carry_plan_convs_sampled(view, moduli, delta, x_samp, x_scale, spec, wts):
    """featuremajor.run_cnn's fused carry plan (config 3: conv1 + square + 2x2
    pool left UNrelinearised, conv2 over the 3-component squares + square + GAP
    as 5-component sums) restated with the oracle on sampled evaluation points.

    x_samp: the C0*H*W input ciphertexts' sampled points [2][ell][S].  Returns
    (block-0 outputs [16*(H/2)*(W/2)] in run_cnn's (o, y, x) order, their scale,
    GAP outputs [32], their scale, the relinearisation's drop count)."""
    assert len(wts.convs) == 2 and spec.pool_after == (0,) and spec.act.degree == 2
    c0, c1, c2 = spec.act.coeffs
    a = math.sqrt(c2)
    b = c1 / (2 * a)
    cst = c0 - c1 * c1 / (4 * c2)
    H, W = spec.H, spec.W
    ell = x_samp[0].shape[1]
    res = []
    cur, s_in = x_samp, x_scale
    drops = 2
    for blk, (w, bias) in enumerate(wts.convs):
        q, p = w.shape[:2]
        pool = blk == 0
        if blk == 1:
            drops = _carried_drops(moduli, delta, ell, s_in)
        dw = _deferred_dw(moduli, delta, ell, s_in, drops)
        wi = np.rint((a * w.reshape(q, p * 9)) * float(dw)).astype(np.int64)
        assert np.abs(wi).max() < 2 ** 23
        s_out = s_in * float(dw)
        bv = a * np.asarray(bias, np.float64) + b
        bres = (np.array([[int(np.rint(v * s_out)) % m for m in moduli[:ell]] for v in bv], np.uint64)
                if np.any(bv != 0) else None)
        npix = 4 if pool else H * W
        C = int(np.rint(cst * (s_out * s_out)))
        cres = [npix * C % m for m in moduli[:ell]]
        out = conv_square_sum_sampled(view, cur, p, H, W, wi, bres, cres, pool)
        s_next = s_out * s_out * npix
        res.append((out, s_next))
        cur, s_in = out, s_next
        if pool:
            H, W = H // 2, W // 2
    (b0, s0), (g, sg) = res
    return b0, s0, g, sg, drops
