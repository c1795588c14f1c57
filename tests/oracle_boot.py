"""The bootstrap circuit's backend on the CPU oracle (test infrastructure).

paper_2604_16834_b200.bootstrap.Bootstrapper runs unchanged on this backend:
every call restates the matching GpuEngine path with the oracle's functions
(oc_mod_raise restated in oracle.mod_raise, oc_encode_c, oc_mul_plain,
oc_rotate, oc_rotate_hoisted, oc_mult_ct, oc_lincomb, oc_rescale), with the
engine's exact encodings, so the GPU bootstrap can be compared limb for limb.
"""

from __future__ import annotations

import numpy as np

import oracle_nets as ON


class OCt:
    """A ciphertext on the oracle: data [2][level+1][N] (numpy uint64), exact scale."""

    def __init__(self, data, scale):
        self.data = np.ascontiguousarray(data, dtype=np.uint64)
        self.scale = float(scale)

    @property
    def level(self):
        return self.data.shape[1] - 1

    @property
    def ell(self):
        return self.data.shape[1]


class OracleBootOps:
    """List-in, list-out backend (the circuit batches every step)."""

    def __init__(self, orc):
        self.orc = orc
        self.moduli = orc.moduli
        self._keys = {}
        self._hkeys = {}

    def key(self, g):
        if g not in self._keys:
            self._keys[g] = self.orc.switch_key(g)
        return self._keys[g]

    def _res(self, v, ell):
        return np.array([int(v) % q for q in self.moduli[:ell]], np.uint64)

    def mod_raise(self, cts, ell_out):
        return [OCt(self.orc.mod_raise(c.data[:, :1], ell_out), c.scale) for c in cts]

    def rotate_hoisted(self, cts, ks):
        orc, n = self.orc, self.orc.n
        outs = []
        for k in ks:
            if k % n == 0:
                outs.append(list(cts))
                continue
            g = pow(5, k % n, 2 * orc.N)
            if g not in self._hkeys:
                self._hkeys[g] = orc.hoist_key(self.key(g), g)
            outs.append([OCt(orc.rotate_hoisted(c.data, g, self._hkeys[g]), c.scale) for c in cts])
        return outs

    def rotate(self, cts, k):
        n = self.orc.n
        if k % n == 0:
            return list(cts)
        g = pow(5, k % n, 2 * self.orc.N)
        return [OCt(self.orc.rotate(c.data, g, self.key(g)), c.scale) for c in cts]

    def conj(self, cts):
        g = 2 * self.orc.N - 1
        return [OCt(self.orc.rotate(c.data, g, self.key(g)), c.scale) for c in cts]

    def mul_monomial(self, cts, power):
        orc, out = self.orc, []
        for ct in cts:
            e = np.zeros(orc.N, np.uint64)
            e[power % orc.N] = 1
            pt = np.stack([orc.ntt(e if (power // orc.N) % 2 == 0 else np.where(e == 1, np.uint64(q - 1), e), l)
                           for l, q in enumerate(self.moduli[:ct.ell])])
            out.append(OCt(orc.mul_plain(ct.data, pt), ct.scale))
        return out

    def _add(self, a, b, sub):
        ell = min(a.ell, b.ell)
        f = self.orc.sub if sub else self.orc.add
        return OCt(f(np.ascontiguousarray(a.data[:, :ell]), np.ascontiguousarray(b.data[:, :ell])), a.scale)

    def add(self, A, B):
        return [self._add(a, b, False) for a, b in zip(A, B)]

    def sub(self, A, B):
        return [self._add(a, b, True) for a, b in zip(A, B)]

    def add_const(self, cts, v):
        return [OCt(self.orc.add_const(c.data, self._res(np.rint(v * c.scale), c.ell)), c.scale) for c in cts]

    def mul_int(self, cts, k, out_scale):
        return [OCt(self.orc.rescale(self.orc.mul_const(c.data, self._res(k, c.ell))), out_scale) for c in cts]

    def mult_ct(self, A, B):
        rk = self.key(0)
        ell = min(min(c.ell for c in A), min(c.ell for c in B))  # GpuEngine: one level per batch
        out = []
        for a, b in zip(A, B):
            r = ON.mult_ct(self.orc, rk, ON.OracleCts(a.data[:, :ell], a.scale), ON.OracleCts(b.data[:, :ell], b.scale))
            out.append(OCt(r.data, r.scale))
        return out

    def lincomb(self, groups, weights, bias, out_scale):
        out = []
        ell = min(c.ell for g in groups for c in g)  # GpuEngine.lincomb: inputs read at the minimum level
        for g in groups:
            n = len(g)
            r = ON.lincomb(self.orc, [ON.OracleCts(c.data[:, :ell], c.scale) for c in g], [0, n], list(range(n)),
                           list(weights), [bias], out_scale)[0]
            out.append(OCt(r.data, r.scale))
        return out

    def lincomb_plain(self, ins, plains, pt_scale=1.0, key=None):
        orc = self.orc
        ell = ins[0].ell
        ql = float(self.moduli[ell - 1]) * pt_scale
        outs = []
        for row in plains:
            acc = None
            for c, p in zip(ins, row):
                pt = orc.plain_to_ntt(orc.encode_complex(p, ql), ell)
                prod = orc.mul_plain(c.data, pt)
                acc = prod if acc is None else orc.add(acc, prod)
            outs.append(OCt(orc.rescale(acc), ins[0].scale * pt_scale))
        return outs
