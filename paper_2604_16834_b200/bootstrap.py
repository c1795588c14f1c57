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

THETA_MAX = 1.25     # |theta| bound for the degree-14 / -15 Taylor cosine / sine
PT_BITS = 60         # encoded DFT diagonals: |coefficient| < 2^60 (int64 encode), see _pt_scale
CTS_GROWTH_BITS = 20  # total scale growth allowed to CoeffToSlot's plaintext encodings
TAYLOR_TERMS = 8     # cos / sin(theta): 8 Taylor terms each (degrees 14 / 15)


def secret_bound(N: int, hamming: int = 0, sigma_mult: float = 6.0) -> float:
    """Bound K on |I_j| after ModRaise: each coefficient of c1 s is a sum of
    h terms uniform in (-q_0/2, q_0/2] (h ~ 2N/3 for the dense ternary secret,
    the expected weight plus 4 standard deviations for a sparse one)."""
    h = 2.0 * N / 3.0 if hamming <= 0 else hamming + 4.0 * math.sqrt(hamming)
    return sigma_mult * math.sqrt(h / 12.0) + 1.0


# ------------------------------------------------------------------ the factored DFT
# Slots z = V u with u_j = t_j + i t_{j+n} and V[i][j] = zeta^{5^i j}.  Splitting
# u into even / odd j halves the problem: the roots zeta^{5^i} square to the
# half-size roots and zeta^{5^{i + n/2}} = -zeta^{5^i}, so
#     V = B_m ... B_1 R        (m = log2 n, R = bit reversal of j)
# where stage B_k (block size 2^k, h = 2^(k-1)) is the butterfly
#     y_i = x_i + w_i x_{i+h},  y_{i+h} = x_i - w_i x_{i+h}   (i mod 2^k < h)
# with w_i = zeta^{5^i n / 2^k}: a map with three diagonals (rotations 0, +h, -h).
# SlotToCoeff applies B_1 .. B_m to bit-reversed coefficients and CoeffToSlot
# applies B_m^-1 .. B_1^-1 (leaving the coefficients bit-reversed, which the
# slot-wise EvalMod does not mind); consecutive stages are merged into a few
# levels of 2^(t+1) - 1 diagonals each.


def _pow5(n: int, N: int) -> np.ndarray:
    out = np.empty(n, np.int64)
    g = 1
    for i in range(n):
        out[i] = g
        g = (g * 5) % (2 * N)
    return out


def _rot(x: np.ndarray, k: int) -> np.ndarray:
    return np.roll(x, -k)


def compose(A: dict, B: dict, n: int) -> dict:
    """Diagonal form of A after B: (A B) x = sum_{r,s} (A_r (.) rot_r(B_s)) (.) rot_{r+s}(x)."""
    out: dict = {}
    for r, a in A.items():
        for s_, b in B.items():
            o = (r + s_) % n
            out[o] = out.get(o, 0) + a * _rot(b, r)
    return out


def apply_map(D: dict, x: np.ndarray) -> np.ndarray:
    return sum(d * _rot(x, o) for o, d in D.items())


def butterfly_stages(N: int, inverse: bool = False) -> list[dict]:
    """[B_1 .. B_m] (inverse: [B_1^-1 .. B_m^-1]) as {offset: diagonal} maps."""
    n = N // 2
    m = n.bit_length() - 1
    p5 = _pow5(n, N)
    i = np.arange(n)
    out = []
    for k in range(1, m + 1):
        blk, h = 1 << k, 1 << (k - 1)
        w = np.exp(1j * np.pi * ((p5 * (n // blk)) % (2 * N)) / N)
        lo = (i % blk) < h
        wl = np.roll(w, h)                           # w_{i-h} at the upper rows
        if not inverse:
            d0 = np.where(lo, 1.0 + 0j, -wl)
            dp = np.where(lo, w, 0j)
            dm = np.where(lo, 0j, 1.0 + 0j)
        else:                                        # x_i = (y_i + y_{i+h}) / 2, x_{i+h} = (y_i - y_{i+h}) / (2 w_i)
            d0 = np.where(lo, 0.5 + 0j, -0.5 / wl)
            dp = np.where(lo, 0.5 + 0j, 0j)
            dm = np.where(lo, 0j, 0.5 / wl)
        if h == n - h:
            out.append({0: d0, h: dp + dm})
        else:
            out.append({0: d0, h: dp, n - h: dm})
    return out


def dft_groups(N: int, levels: int, inverse: bool) -> list[tuple[int, dict]]:
    """Merged stage groups in application order, each as (h0, map): SlotToCoeff
    applies B_1 .. B_m, CoeffToSlot B_m^-1 .. B_1^-1; h0 is the group's
    smallest butterfly distance (every offset is a multiple of it)."""
    n = N // 2
    st = butterfly_stages(N, inverse)
    m = len(st)
    order = list(range(m)) if not inverse else list(range(m - 1, -1, -1))
    levels = max(1, min(levels, m))
    bounds = [round(g * m / levels) for g in range(levels + 1)]
    out = []
    for g in range(levels):
        idx = order[bounds[g]:bounds[g + 1]]
        M = st[idx[0]]
        for k in idx[1:]:
            M = compose(st[k], M, n)
        out.append((1 << min(idx), {o: d for o, d in M.items() if np.any(d != 0)}))
    return out


@dataclass
class BsgsStage:
    """One merged DFT level as a baby-step / giant-step plan: offsets
    o = (base + g b + j) h0 (j < b baby steps, g < G giant steps) and the
    plaintexts p[g][j] = roll(D[o], (base + g b) h0)."""

    h0: int
    base: int
    baby: int
    giant: int
    rows: list             # giant steps with a nonzero plaintext
    plains: np.ndarray     # [len(rows)][b][n] complex
    dmax: float            # max |plaintext slot value|
    tag: str = ""

    @staticmethod
    def build(h0: int, D: dict, n: int, scale: complex = 1.0) -> "BsgsStage":
        span_n = n // h0
        cs = []
        for o in D:
            c = o // h0
            cs.append(c - span_n if c > span_n // 2 else c)
        lo, hi = min(cs), max(cs)
        span = hi - lo + 1
        b = 1 << max(0, math.ceil(math.log2(span) / 2))
        G = -(-span // b)
        P = np.zeros((G, b, n), np.complex128)
        for g in range(G):
            for j in range(b):
                o = ((lo + g * b + j) * h0) % n
                if o in D:
                    P[g, j] = np.roll(D[o] * scale, ((lo + g * b) * h0) % n)
        rows = [g for g in range(G) if np.any(P[g] != 0)]
        P = np.ascontiguousarray(P[rows])
        return BsgsStage(h0=h0, base=lo, baby=b, giant=G, rows=rows, plains=P, dmax=float(np.max(np.abs(P))))

    def rotations(self, n: int) -> list[int]:
        r = [(j * self.h0) % n for j in range(1, self.baby)]
        r += [((self.base + g * self.baby) * self.h0) % n for g in range(self.giant)]
        return [x for x in r if x]


@dataclass
class BootPlan:
    """Static parameters of one bootstrap circuit (ring degree N, n = N/2 slots)."""

    N: int
    q0: int
    hamming: int = 0
    K: float = 0.0
    r: int = 0
    dft_levels: int = 0

    def __post_init__(self) -> None:
        m = (self.N // 2).bit_length() - 1
        if not self.K:
            self.K = secret_bound(self.N, self.hamming)
        if not self.r:
            self.r = max(0, math.ceil(math.log2(2 * math.pi * (self.K + 0.25) / THETA_MAX)))
        if not self.dft_levels:
            self.dft_levels = max(1, -(-m // 6))
        self.dft_levels = min(self.dft_levels, m)

    @property
    def n(self) -> int:
        return self.N // 2

    @property
    def a(self) -> float:
        return 2.0 * math.pi / (1 << self.r)

    @property
    def depth(self) -> int:
        return self.dft_levels + 1 + 6 + self.r + self.dft_levels

    def _groups(self, inverse: bool) -> list:
        cache = self.__dict__.setdefault("_group_cache", {})
        if inverse not in cache:
            cache[inverse] = dft_groups(self.N, self.dft_levels, inverse)
        return cache[inverse]

    def stages(self, c2: float = 1.0) -> tuple[list[BsgsStage], list[BsgsStage]]:
        """(CoeffToSlot stages, SlotToCoeff stages); c2 scales the first SlotToCoeff level."""
        n = self.n
        cts = [BsgsStage.build(h0, D, n) for h0, D in self._groups(True)]
        stc = [BsgsStage.build(h0, D, n, c2 if g == 0 else 1.0) for g, (h0, D) in enumerate(self._groups(False))]
        for i, st in enumerate(cts):
            st.tag = f"cts{i}"
        for i, st in enumerate(stc):
            st.tag = f"stc{i}"
        return cts, stc

    def rotation_offsets(self) -> list[int]:
        if "_offsets" not in self.__dict__:
            cts, stc = self.stages()
            self._offsets = sorted({r for st in cts + stc for r in st.rotations(self.n)})
        return self._offsets


# ------------------------------------------------------------------ the circuit
class Bootstrapper:
    """Runs the bootstrap circuit on a backend ``ops`` (GpuBootOps or the
    tests' oracle backend) over a batch of ciphertexts of one level and scale.
    Every backend op takes and returns lists, so each step is one batched
    call for the whole batch.  The DFT plans are built once per instance;
    encodings happen inside ``ops.lincomb_plain`` at each level."""

    def __init__(self, ops, plan: BootPlan, s_in: float):
        self.ops, self.plan, self.s_in = ops, plan, s_in
        # SlotToCoeff's input holds 2 sin(2 pi t / q_0) ~ 4 pi m / q_0: c2 = q_0 / (4 pi s_in)
        self.cts, self.stc = plan.stages(plan.q0 / (4.0 * math.pi * s_in))

    # -- helpers
    def _exact_const(self, cts, v: float, target_scale: float):
        """cts * v landing near ``target_scale``: the constant's integer is
        k = rint(v q_l target / s) and the declared output scale is the exact
        s k / (q_l v), so the rounding of k costs no precision."""
        ql = self.ops.moduli[cts[0].level]
        s_ = cts[0].scale
        k = int(np.rint(v * ql * target_scale / s_))
        if abs(k) < (1 << 8):
            raise HebatchError("bootstrap constant underflows its encoding")
        return self.ops.mul_int(cts, k, s_ * k / (ql * v))

    def _pt_scale(self, st: BsgsStage, level: int, grow: bool) -> float:
        """2^k with max|d| q_l 2^k < 2^PT_BITS.  CoeffToSlot (grow) raises k so
        its 2^-t-sized diagonals keep their bits (the exact constant product
        that follows restores the scale); SlotToCoeff only lowers it when a
        diagonal would overflow, so its output keeps the input's scale."""
        ql = float(self.ops.moduli[level])
        k = math.floor(PT_BITS - math.log2(ql) - math.log2(st.dmax))
        if grow:  # at most CTS_GROWTH_BITS over all CoeffToSlot levels (the constant product stays >= 2^12)
            return 2.0 ** min(k, CTS_GROWTH_BITS // self.plan.dft_levels)
        return 2.0 ** min(k, 0)

    def _bsgs(self, cts, st: BsgsStage, grow: bool = False):
        """sum_g rot_{(base + g b) h0}( lincomb_plain(rot_{j h0}(ct), p[g]) ) per ct."""
        ops, n = self.ops, self.plan.n
        babies = ops.rotate_hoisted(cts, [j * st.h0 for j in range(st.baby)])     # [b][B]
        pts = self._pt_scale(st, cts[0].level, grow)
        partial = [ops.lincomb_plain([babies[j][c] for j in range(st.baby)], st.plains, pts, key=st.tag)
                   for c in range(len(cts))]                                       # [B][rows]
        acc = None
        for gi, g in enumerate(st.rows):
            col = [p[gi] for p in partial]
            k = ((st.base + g * st.baby) * st.h0) % n
            col = ops.rotate(col, k) if k else col
            acc = col if acc is None else ops.add(acc, col)
        return acc

    def coeff_to_slot(self, raised):
        """-> theta (2B cts: the B low halves, then the B high halves): theta =
        a (t / q_0 - 1/4) for the coefficients t_j, t_{j+n} (j < n, bit-reversed)."""
        plan, ops = self.plan, self.ops
        w = raised
        for st in self.cts:
            w = self._bsgs(w, st, grow=True)                             # R u / s (complex)
        wc = ops.conj(w)
        lo = ops.add(w, wc)                                              # 2 Re: t_j
        hi = ops.mul_monomial(ops.sub(w, wc), 3 * plan.n)                # -i (w - conj w) = 2 Im: t_{j+n}
        c = plan.a * raised[0].scale / (2.0 * plan.q0)
        th = self._exact_const(lo + hi, c, raised[0].scale)              # a t / q_0
        return ops.add_const(th, -plan.a / 4.0)

    def eval_mod(self, theta):
        """theta -> 2 sin(2 pi t / q_0): z = e^{i theta} = C + i S from the
        Taylor cosine and sine (i S as the monomial X^n S: free and exact),
        r squarings z <- z^2 (error growth 2 per step, against 4 for the
        cosine double angle), then z + conj(z) = 2 Re(e^{i (2 pi x - pi/2)})."""
        ops, m = self.ops, len(theta)
        cc = [(-1.0) ** k / math.factorial(2 * k) for k in range(TAYLOR_TERMS)]
        sc = [(-1.0) ** k / math.factorial(2 * k + 1) for k in range(TAYLOR_TERMS)]
        y = ops.mult_ct(theta, theta)                                   # theta^2
        r1 = ops.mult_ct(y + theta, y + y)
        y2, t1 = r1[:m], r1[m:]                                         # theta^4, theta^3
        r2 = ops.mult_ct(y + y2 + theta, y2 + y2 + y2)
        y3, y4, t2 = r2[:m], r2[m:2 * m], r2[2 * m:]                    # theta^6, theta^8, theta^5
        t3 = ops.mult_ct(theta, y3)                                     # theta^7
        target = y3[0].scale
        mc, ms = y3[0].level - 1, t3[0].level - 1                      # levels of the y^4 products
        even = [[y[i], y2[i], y3[i]] for i in range(m)]
        odd = [[theta[i], t1[i], t2[i], t3[i]] for i in range(m)]
        q0c = ops.lincomb(even, cc[1:4], cc[0], target)
        q1c = ops.lincomb(even, cc[5:8], cc[4], target * ops.moduli[mc] / y4[0].scale)
        q0s = ops.lincomb(odd, sc[0:4], 0.0, target)
        q1s = ops.lincomb(odd, sc[4:8], 0.0, target * ops.moduli[ms] / y4[0].scale)
        cos_t = ops.add(q0c, ops.mult_ct(y4, q1c))
        sin_t = ops.add(q0s, ops.mult_ct(y4, q1s))
        z = ops.add(cos_t, ops.mul_monomial(sin_t, self.plan.n))       # cos + i sin
        for _ in range(self.plan.r):
            z = ops.mult_ct(z, z)
        return ops.add(z, ops.conj(z))

    def slot_to_coeff(self, sines):
        """2 sin for the B low halves then the B high halves (bit-reversed
        coefficient order) -> the B message ciphertexts."""
        ops, plan = self.ops, self.plan
        B = len(sines) // 2
        x = ops.add(sines[:B], ops.mul_monomial(sines[B:], plan.n))      # lo + i hi
        for st in self.stc:
            x = self._bsgs(x, st)
        return x

    def run(self, cts, ell_top: int):
        """Bootstrap ``cts`` (one level; scale this instance's s_in): ModRaise
        to ell_top limbs, CoeffToSlot, EvalMod, SlotToCoeff.  Returns a list."""
        if any(c.scale != self.s_in for c in cts) or len({c.level for c in cts}) != 1:
            raise HebatchError("Bootstrapper: a batch needs one level and this instance's input scale")
        raised = self.ops.mod_raise(cts, ell_top)
        return self.slot_to_coeff(self.eval_mod(self.coeff_to_slot(raised)))


class GpuBootOps:
    """The circuit's backend on GpuEngine: every call is one batched C-ABI
    path over a list of ciphertexts; no counters move (the caller accounts
    the bootstraps)."""

    def __init__(self, eng):
        self.e = eng
        self.moduli = eng.moduli
        self._pts = {}  # (stage tag, limbs, pt_scale) -> encoded diagonals [rows * b][limbs][N]

    def mod_raise(self, cts, ell_out):
        from . import _lib

        e = self.e
        out = e._alloc(len(cts), 2, ell_out)
        src, dst = e._ptrs(cts), e._tptrs(out)
        _lib.check(e._call("mod_raise", e._L.he_mod_raise, e._h, _lib.addr(src), cts[0].level + 1, _lib.addr(dst),
                           len(cts), ell_out, e.stream), "mod_raise")
        return e._wrap_batch(out, ell_out - 1, [c.scale for c in cts])

    def rotate_hoisted(self, cts, ks):
        return self.e._rotate_hoisted_internal(cts, ks)

    def rotate(self, cts, k):
        return self.e._rotate_batch(cts, k) if k % self.e.context.n else list(cts)

    def conj(self, cts):
        return self.e._automorph_batch(cts, 2 * self.e.N - 1)

    def mul_monomial(self, cts, power):
        return self.e._mul_monomial_batch(cts, power)

    def add(self, A, B):
        return self.e._add_batch(A, B)

    def sub(self, A, B):
        return self.e._add_batch(A, B, sub=True)

    def add_const(self, cts, v):
        return self.e.add_const_batch(cts, [v] * len(cts), count=False)

    def mul_int(self, cts, k, out_scale):
        return self.e._mul_int_batch(cts, [k] * len(cts), [out_scale] * len(cts))

    def mult_ct(self, A, B):
        return self.e._mult_ct_batch(A, B)

    def lincomb(self, groups, weights, bias, out_scale):
        """out[i] = sum_t weights[t] groups[i][t] + bias, one launch for all groups."""
        k = len(groups[0])
        ins = [c for g in groups for c in g]
        return self.e.lincomb(ins, list(range(0, len(ins) + 1, k)), list(range(len(ins))), list(weights) * len(groups),
                              bias=[bias] * len(groups), out_scale=out_scale, count_as_conv=False)

    def lincomb_plain(self, ins, plains, pt_scale=1.0, key=None):
        """DFT levels: the encoded diagonals are cached on the device per (stage, level, scale)."""
        e = self.e
        if key is None:
            return e.lincomb_plain(ins, plains, len(plains), pt_scale)
        limbs = ins[0].level + 1
        ck = (key, limbs, pt_scale)
        if ck not in self._pts:
            self._pts[ck] = e.encode_plains(plains.reshape(-1, plains.shape[-1]), limbs, pt_scale)
        return e.lincomb_plain_encoded(ins, self._pts[ck], len(plains), pt_scale)
