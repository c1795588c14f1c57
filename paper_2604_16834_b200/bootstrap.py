"""CKKS bootstrapping on the B200 engine.

The reference's ``bootstrap`` (/root/reference/pkg/src/hebatch/engine.py:315-319)
is accounting only: the level is reset to ``max_level - bootstrap_reserve``,
the ``bootstraps`` counter advances and the slots are copied.
states the contract; the circuit itself is out of the reference's scope
(SPEC.md:8, :134).  Here it is a real CKKS bootstrap composed from the
engine's bit-exact primitives, so that ``GpuEngine.bootstrap`` keeps the
reference's contract (same slots up to the bootstrap's approximation error,
level ``max_level - bootstrap_reserve``, one ``bootstraps`` count):

1. **ModRaise** (``he_mod_raise``): the ciphertext read at level 0 is lifted
   centred from q_0 to the full chain; it now decrypts to m + q_0 I(X) with a
   small integer polynomial I (|I_j| <= K).
2. **CoeffToSlot**: with u_j = t_j + i t_{j+n} (t the plaintext coefficients;
   slots z = V u, V[i][j] = zeta^{5^i j}, zeta = e^{i pi / N}, V^-1 = V^H / n),
   two baby-step / giant-step linear transforms with complex diagonals
   (V^H / n and -i V^H / n) share one set of hoisted baby rotations and one
   plaintext-weighted lincomb (``he_lincomb_plain``); each result plus its
   conjugate (Galois element 2N - 1) holds 2 Re(.), i.e. the coefficients
   t_j and t_{j+n} as real slots.  A constant product then scales them to
   theta_j = a (t_j / q_0 - 1/4) with a = 2 pi / 2^r.  Two levels.
3. **EvalMod**: z = e^{i theta} = cos(theta) + i sin(theta) from the degree-14 /
   -15 Taylor polynomials (Paterson-Stockmeyer over theta, theta^2 .. theta^8:
   six levels; i sin as the monomial product X^n sin, exact and free since
   zeta_t^n = i at every slot root), then r squarings z <- z^2 (r levels):
   z = e^{i 2^r theta} = e^{i (2 pi t / q_0 - pi / 2)}, and z + conj(z) =
   2 sin(2 pi t / q_0) ~ 4 pi (t mod q_0) / q_0 = 4 pi m / q_0.  Squaring a
   unit complex number doubles an error; the real double-angle recurrence
   c <- 2 c^2 - 1 would quadruple it.
4. **SlotToCoeff**: one BSGS transform with diagonals of c2 V and c2 i V
   (c2 = q_0 / (4 pi scale)) over both EvalMod outputs.  One level.

Depth 2 + 6 + r + 1.  K is the 6-sigma bound of |I| for the engine's dense
ternary secret (sigma = sqrt(2N/3 / 12)); r makes |theta| <= 1.25.  Precision
needs q_0 / scale ~ 2^10 (so that sin(x) ~ x on the message) and a scale of
~2^50: e.g. q_0 of 60 bits with 50-bit rescale primes.

The circuit is written once against a small backend interface (``ops``):
``GpuBootOps`` drives the CUDA engine; the tests drive the same circuit on
the CPU oracle (tests/oracle_boot.py) and compare every limb.  Constants and
the Taylor / Paterson-Stockmeyer weights go through exact-scale encodings
(each constant's integer and the resulting scale are computed here, so both
backends see identical integers).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import HebatchError

THETA_MAX = 1.25     # |theta| bound for the degree-14 Taylor cosine
CTS_PT_BITS = 20     # CoeffToSlot diagonals (|d| = 1/n) are encoded at q_l 2^20: their
                     # plaintext coefficients (~ q_l / n^1.5) keep ~55 bits
TAYLOR_TERMS = 8     # cos / sin(theta): 8 Taylor terms each (degrees 14 / 15)


def secret_bound(N: int, sigma_mult: float = 6.0) -> float:
    """Bound K on |I_j| after ModRaise for the dense ternary secret (each
    coefficient of c1 s is a sum of ~2N/3 terms uniform in (-q_0/2, q_0/2])."""
    return sigma_mult * math.sqrt((2.0 * N / 3.0) / 12.0) + 1.0


@dataclass
class BootPlan:
    """Static parameters of one bootstrap circuit (ring degree N, n = N/2 slots)."""

    N: int
    q0: int
    K: float = 0.0
    r: int = 0
    baby: int = 0
    giant: int = 0
    taylor: list = field(default_factory=list)

    def __post_init__(self) -> None:
        n = self.N // 2
        if not self.K:
            self.K = secret_bound(self.N)
        if not self.r:
            self.r = max(0, math.ceil(math.log2(2 * math.pi * (self.K + 0.25) / THETA_MAX)))
        if not self.baby:
            self.baby = 1 << ((n.bit_length() - 1 + 1) // 2)  # ~ sqrt(n), power of two
        self.baby = min(self.baby, n)
        self.giant = n // self.baby
        self.taylor = [(-1.0) ** k / math.factorial(2 * k) for k in range(TAYLOR_TERMS)]

    @property
    def n(self) -> int:
        return self.N // 2

    @property
    def a(self) -> float:
        return 2.0 * math.pi / (1 << self.r)

    @property
    def depth(self) -> int:
        return 2 + 6 + self.r + 1

    def rotation_offsets(self) -> list[int]:
        """Baby steps 1..b-1 and giant steps b g (g = 1..G-1)."""
        return list(range(1, self.baby)) + [self.baby * g for g in range(1, self.giant)]


# ------------------------------------------------------------------ DFT diagonals
def _pow5(n: int, N: int) -> np.ndarray:
    out = np.empty(n, np.int64)
    g = 1
    for i in range(n):
        out[i] = g
        g = (g * 5) % (2 * N)
    return out


def _zeta(exps: np.ndarray, N: int) -> np.ndarray:
    e = np.mod(exps, 2 * N).astype(np.float64)
    return np.exp(1j * np.pi * e / N)


def cts_diagonals(N: int) -> np.ndarray:
    """Diagonals of V^-1 = V^H / n: d[k][i] = conj(V[(i+k) % n][i]) / n."""
    n = N // 2
    p5 = _pow5(n, N)
    i = np.arange(n, dtype=np.int64)
    out = np.empty((n, n), np.complex128)
    for k in range(n):
        j = (i + k) % n
        out[k] = _zeta(-(p5[j] * i), N) / n
    return out


def stc_diagonals(N: int) -> np.ndarray:
    """Diagonals of V: d[k][i] = V[i][(i+k) % n] = zeta^(5^i ((i+k) % n))."""
    n = N // 2
    p5 = _pow5(n, N)
    i = np.arange(n, dtype=np.int64)
    out = np.empty((n, n), np.complex128)
    for k in range(n):
        j = (i + k) % n
        out[k] = _zeta(p5 * j, N)
    return out


def bsgs_plains(diags: np.ndarray, baby: int, giant: int) -> np.ndarray:
    """BSGS plaintexts p[g][j] = roll(diag[b g + j], b g) so that
    M z = sum_g rot_{b g}( sum_j p[g][j] (.) rot_j(z) )."""
    n = diags.shape[1]
    out = np.empty((giant, baby, n), np.complex128)
    for g in range(giant):
        for j in range(baby):
            out[g, j] = np.roll(diags[baby * g + j], baby * g)
    return out


# ------------------------------------------------------------------ the circuit
class Bootstrapper:
    """Runs the bootstrap circuit on a backend ``ops`` (GpuBootOps or the
    tests' oracle backend).  Diagonal plaintext values are built once per
    instance; encodings happen inside ``ops.lincomb_plain`` at each level."""

    def __init__(self, ops, plan: BootPlan):
        self.ops, self.plan = ops, plan
        b, G = plan.baby, plan.giant
        inv = bsgs_plains(cts_diagonals(plan.N), b, G)                       # [G][b][n]
        # CoeffToSlot: outputs (t, g), t = 0: V^-1, t = 1: -i V^-1 (Re -> Im(u))
        self._cts = np.concatenate([inv, -1j * inv], axis=0)                 # [2G][b][n]
        fwd = bsgs_plains(stc_diagonals(plan.N), b, G)                       # [G][b][n]
        self._stc_fwd = fwd

    # -- helpers
    def _exact_const(self, ct, v: float, target_scale: float):
        """ct * v landing near ``target_scale``: the constant's integer is
        k = rint(v q_l target / s) and the declared output scale is the exact
        s k / (q_l v), so the rounding of k costs no precision."""
        ql = self.ops.moduli[ct.level]
        k = int(np.rint(v * ql * target_scale / ct.scale))
        if abs(k) < (1 << 8):
            raise HebatchError("bootstrap constant underflows its encoding")
        return self.ops.mul_int(ct, k, ct.scale * k / (ql * v))

    def _bsgs(self, cts, plains, pt_scale: float = 1.0):
        """sum_g rot_{b g}(lincomb_plain(babies, plains[o])) for every output
        row o of plains [n_out][n_in = b * len(cts)][n]; giant index g = o % G."""
        ops, b, G = self.ops, self.plan.baby, self.plan.giant
        babies = ops.rotate_hoisted(cts, list(range(b)))                     # [b][len(cts)]
        ins = [babies[j][c] for j in range(b) for c in range(len(cts))]
        partial = ops.lincomb_plain(ins, plains, pt_scale)
        outs = []
        for t in range(len(partial) // G):
            acc = None
            for g in range(G):
                p = partial[t * G + g]
                p = ops.rotate(p, b * g) if g else p
                acc = p if acc is None else ops.add(acc, p)
            outs.append(acc)
        return outs

    def coeff_to_slot(self, raised):
        """-> [theta_lo, theta_hi]: theta = a (t / q_0 - 1/4) for the coefficient
        halves t_j, t_{j+n} (j < n) of the raised plaintext."""
        plan, ops = self.plan, self.ops
        n_out = self._cts.shape[0]
        # |d| = 1/n: plaintext coefficients stay below q_l 2^k / n < 2^60 (int64 encode)
        ql_bits = self.ops.moduli[raised.level].bit_length()
        k = max(0, min(CTS_PT_BITS, 60 - ql_bits + plan.n.bit_length() - 1))
        w = self._bsgs([raised], self._cts.reshape(n_out, plan.baby, plan.n), float(1 << k))
        re2 = [ops.add(x, ops.conj(x)) for x in w]                          # 2 t / s
        c = plan.a * raised.scale / (2.0 * plan.q0)
        th = [self._exact_const(x, c, raised.scale) for x in re2]           # a t / q_0
        return [ops.add_const(x, -plan.a / 4.0) for x in th]

    def eval_mod(self, theta):
        """[theta_i] -> [2 sin(2 pi t / q_0)]: z = e^{i theta} = C + i S from the
        Taylor cosine and sine (i S as the monomial X^n S: free and exact),
        r squarings z <- z^2 (error growth 2 per step, against 4 for the
        cosine double angle), then z + conj(z) = 2 Re(e^{i (2 pi x - pi/2)})."""
        ops = self.ops
        cc = [(-1.0) ** k / math.factorial(2 * k) for k in range(TAYLOR_TERMS)]
        sc = [(-1.0) ** k / math.factorial(2 * k + 1) for k in range(TAYLOR_TERMS)]
        y = ops.mult_ct(theta, theta)                                   # theta^2
        y2 = ops.mult_ct(y, y)
        t1 = ops.mult_ct(theta, y)                                      # theta^3
        y3 = ops.mult_ct(y, y2)
        y4 = ops.mult_ct(y2, y2)
        t2 = ops.mult_ct(theta, y2)                                     # theta^5
        t3 = ops.mult_ct(theta, y3)                                     # theta^7
        zs = []
        for i in range(len(theta)):
            target = y3[i].scale
            mc, ms = y3[i].level - 1, t3[i].level - 1                  # levels of the y^4 products
            q0c = ops.lincomb([y[i], y2[i], y3[i]], cc[1:4], cc[0], target)
            q1c = ops.lincomb([y[i], y2[i], y3[i]], cc[5:8], cc[4], target * ops.moduli[mc] / y4[i].scale)
            cos_t = ops.add(q0c, ops.mult_ct([y4[i]], [q1c])[0])
            odd = [theta[i], t1[i], t2[i], t3[i]]
            q0s = ops.lincomb(odd, sc[0:4], 0.0, target)
            q1s = ops.lincomb(odd, sc[4:8], 0.0, target * ops.moduli[ms] / y4[i].scale)
            sin_t = ops.add(q0s, ops.mult_ct([y4[i]], [q1s])[0])
            zs.append(ops.add(cos_t, ops.mul_monomial(sin_t, self.plan.n)))  # cos + i sin
        for _ in range(self.plan.r):
            zs = ops.mult_ct(zs, zs)
        return [ops.add(z, ops.conj(z)) for z in zs]

    def slot_to_coeff(self, sines, s_in: float):
        plan = self.plan
        c2 = plan.q0 / (4.0 * math.pi * s_in)      # the EvalMod outputs hold 2 sin(2 pi t / q_0)
        fwd = self._stc_fwd
        # inputs ordered (j, t): babies[j][0] = rot_j(sin_lo), babies[j][1] = rot_j(sin_hi)
        pl = np.stack([c2 * fwd, (1j * c2) * fwd], axis=2).reshape(plan.giant, 2 * plan.baby, plan.n)
        return self._bsgs(sines, pl)[0]

    def run(self, ct, ell_top: int):
        """Bootstrap ``ct`` (any level): ModRaise to ell_top limbs, CtS, EvalMod, StC."""
        s_in = ct.scale
        raised = self.ops.mod_raise(ct, ell_top)
        theta = self.coeff_to_slot(raised)
        sines = self.eval_mod(theta)
        return self.slot_to_coeff(sines, s_in)


class GpuBootOps:
    """The circuit's backend on GpuEngine: every call is one of the engine's
    batched C-ABI paths; no counters move (the caller accounts one bootstrap)."""

    def __init__(self, eng):
        self.e = eng
        self.moduli = eng.moduli

    def mod_raise(self, ct, ell_out):
        e = self.e
        out = e._alloc(1, 2, ell_out)
        from . import _lib

        src, dst = e._ptrs([ct]), e._tptrs(out)
        _lib.check(e._call("mod_raise", e._L.he_mod_raise, e._h, _lib.addr(src), ct.level + 1, _lib.addr(dst), 1,
                           ell_out, e.stream), "mod_raise")
        return e._wrap_batch(out, ell_out - 1, [ct.scale])[0]

    def rotate_hoisted(self, cts, ks):
        return self.e._rotate_hoisted_internal(cts, ks)

    def rotate(self, ct, k):
        return self.e._rotate_batch([ct], k)[0] if k % self.e.context.n else ct

    def conj(self, ct):
        return self.e._automorph_batch([ct], 2 * self.e.N - 1)[0]

    def mul_monomial(self, ct, power):
        return self.e._mul_monomial_batch([ct], power)[0]

    def add(self, a, b):
        return self.e._add_batch([a], [b])[0]

    def add_const(self, ct, v):
        return self.e.add_const_batch([ct], [v], count=False)[0]

    def mul_int(self, ct, k, out_scale):
        return self.e._mul_int_batch([ct], [k], [out_scale])[0]

    def mult_ct(self, A, B):
        return self.e._mult_ct_batch(A, B)

    def lincomb(self, ins, weights, bias, out_scale):
        n = len(ins)
        return self.e.lincomb(ins, [0, n], list(range(n)), list(weights), bias=[bias], out_scale=out_scale,
                              count_as_conv=False)[0]

    def lincomb_plain(self, ins, plains, pt_scale=1.0):
        return self.e.lincomb_plain(ins, plains, len(plains), pt_scale)
