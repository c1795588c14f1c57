"""A float slot engine for CPU tests of the multi-rank layer logic.

Implements the engine methods that featuremajor / sharded_cnn call, on
plaintext float64 slot vectors held in torch CPU tensors (so gloo can move
them).  It has no cryptography: it checks data movement and partial-sum
bookkeeping, not arithmetic (the GPU parity tests do that).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class _Ctx:
    scale: float = 2.0 ** 40


@dataclass(eq=False)
class ToyCt:
    data: object          # torch float64 [n_slots]
    level: int
    scale: float


class ToyEngine:
    def __init__(self, n_slots: int, level: int = 30):
        self.context = _Ctx()
        self.n = n_slots
        self.level0 = level
        self.live = 0

    def _ct(self, v, level, scale=2.0 ** 40):
        self.live += 1
        return ToyCt(torch.as_tensor(np.asarray(v, np.float64)), level, scale)

    def encrypt_batch(self, values):
        return [self._ct(v, self.level0) for v in np.asarray(values, np.float64)]

    def decrypt_batch(self, cts):
        return [c.data.numpy().copy() for c in cts]

    def release(self, *cts):
        for c in cts:
            if c.data is not None:
                self.live -= 1
            c.data = None

    # -- layer primitives
    def lincomb_grouped(self, inputs, term_ptr, col, tap, out_base, out_stride, weights, n_out, bias=None,
                        out_scale=None, weight_scale=None, skip_rescale=False):
        w = np.asarray(weights, np.float64)
        out = [np.zeros(self.n) for _ in range(n_out)]
        for g in range(len(out_base)):
            for t in range(term_ptr[g], term_ptr[g + 1]):
                x = inputs[col[t]].data.numpy()
                for m in range(w.shape[0]):
                    out[out_base[g] + m * out_stride] += w[m, tap[t]] * x
        lvl = inputs[0].level
        return [self._ct(v, lvl if skip_rescale else lvl - 1) for v in out]

    def add_batch(self, A, B):
        return [self._ct(a.data.numpy() + b.data.numpy(), min(a.level, b.level)) for a, b in zip(A, B)]

    def rescale_batch(self, cts, out_scale=None):
        return [self._ct(c.data.numpy(), c.level - 1) for c in cts]

    def add_const_batch(self, cts, values, count=True):
        return [self._ct(c.data.numpy() + v, c.level) for c, v in zip(cts, values)]

    def mult_ct_batch(self, A, B):
        return [self._ct(a.data.numpy() * b.data.numpy(), min(a.level, b.level) - 1) for a, b in zip(A, B)]

    def lincomb_int(self, inputs, row_ptr, col, int_weights, out_scale, count_adds=True):
        # unit sums declared at scale k*s decrypt to the mean: slot values scale by s_in / out_scale
        f = inputs[0].scale / out_scale
        out = []
        for o in range(len(row_ptr) - 1):
            v = np.zeros(self.n)
            for t in range(row_ptr[o], row_ptr[o + 1]):
                v += int_weights[t] * inputs[col[t]].data.numpy()
            out.append(self._ct(v * f, inputs[0].level, out_scale))
        return out

    def lincomb(self, inputs, row_ptr, col, weights, bias=None, out_scale=None, count_as_conv=True):
        out = []
        for o in range(len(row_ptr) - 1):
            v = np.zeros(self.n)
            for t in range(row_ptr[o], row_ptr[o + 1]):
                v += weights[t] * inputs[col[t]].data.numpy()
            if bias is not None:
                v += bias[o]
            out.append(self._ct(v, inputs[0].level - 1))
        return out

    # -- collectives payload
    def pack_batch(self, cts):
        return torch.stack([c.data for c in cts]), cts[0].level, cts[0].scale

    def unpack_batch(self, t, level, scale):
        return [self._ct(t[i].numpy(), level, scale) for i in range(t.shape[0])]
