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
