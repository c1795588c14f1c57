"""Pure-Python big-integer restatement of the convention contract (small N only).

TEST INFRASTRUCTURE ONLY.  This is the independent second implementation the
C oracle (ckks_oracle.c) is checked against: it shares no code with it and
uses the textbook definitions wherever the C oracle uses a fast algorithm:

  * NTT by direct evaluation out[k] = a(psi^(2*brv(k)+1)), O(N^2);
  * ring products by schoolbook negacyclic convolution;
  * basis conversion and ModDown by their CRT formulas on Python ints;
  * Philox4x32-10 re-implemented from the published round function.

The float64 encode/decode FFT is restated with the same operation order as
the contract (Python floats are IEEE binary64 without FMA), so it is
bit-exact with the C oracle and the GPU.
"""

from __future__ import annotations

import math

M0, M1, W0, W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85
MASK32 = 0xFFFFFFFF
DOM_SK, DOM_ENC_A, DOM_ENC_E, DOM_KSK_A, DOM_KSK_E = 1, 2, 3, 4, 5


def philox(ctr, key):
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for _ in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & MASK32, p1 & MASK32, ((p0 >> 32) ^ c3 ^ k1) & MASK32, p0 & MASK32
        k0 = (k0 + W0) & MASK32
        k1 = (k1 + W1) & MASK32
    return [c0, c1, c2, c3]


def is_prime(n):
    if n < 2:
        return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def gen_moduli(N, bits_list):
    out = []
    for bits in bits_list:
        k = 1
        while True:
            cand = (1 << bits) - k * 2 * N + 1
            k += 1
            if cand not in out and is_prime(cand):
                out.append(cand)
                break
    return out


def find_psi(q, N):
    e = (q - 1) // (2 * N)
    g = 2
    while True:
        psi = pow(g, e, q)
        if pow(psi, N, q) == q - 1:
            return psi
        g += 1


def brv(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


def centered(x, q):
    x %= q
    return x - q if x > (q - 1) // 2 else x


class PyRef:
    def __init__(self, log_n, q_bits, p_bits, alpha, seed=0, scale=2.0 ** 40):
        self.logN, self.N, self.n = log_n, 1 << log_n, 1 << (log_n - 1)
        self.L, self.K, self.alpha = len(q_bits), len(p_bits), alpha
        self.dnum = -(-self.L // alpha)
        self.seed, self.scale = seed, scale
        self.mod = gen_moduli(self.N, list(q_bits) + list(p_bits))
        self.psi = [find_psi(q, self.N) for q in self.mod]
        N = self.N
        self.s = [self._rnd(DOM_SK, 0, 0, j >> 2)[j & 3] % 3 - 1 for j in range(N)]
        n = self.n
        self.wr = [math.cos(2.0 * math.pi * k / n) for k in range(n)]
        self.wi = [math.sin(2.0 * math.pi * k / n) for k in range(n)]
        self.zr = [math.cos(math.pi * k / N) for k in range(n)]
        self.zi = [math.sin(math.pi * k / N) for k in range(n)]
        self.pos, g = [], 1
        for _ in range(n):
            self.pos.append((g - 1) // 4)
            g = g * 5 % (2 * N)

    # -- randomness
    def _rnd(self, dom, obj, limb, idx):
        return philox([idx & MASK32, limb, obj & MASK32, dom], [self.seed & MASK32, self.seed >> 32])

    def cbd(self, dom, obj):
        out = []
        for j in range(self.N):
            r = self._rnd(dom, obj, 0, j)
            out.append(bin(r[0] & 0x1FFFFF).count("1") - bin(r[1] & 0x1FFFFF).count("1"))
        return out

    def uniform(self, dom, obj, limb, q):
        # one Philox block per pair of indices differing in bit 4; accept x < q*floor(2^64/q), else
        # redraw from block (k, limb, obj, dom + 16 t); the value is x mod q (exactly uniform)
        T = ((1 << 64) // q) * q
        out = []
        for k in range(self.N):
            r = self._rnd(dom, obj, limb, ((k >> 5) << 4) | (k & 15))
            x = (r[2] | r[3] << 32) if k & 16 else (r[0] | r[1] << 32)
            t = 0
            while x >= T:
                t += 1
                r = self._rnd(dom + 16 * t, obj, limb, k)
                x = r[0] | r[1] << 32
            out.append(x % q)
        return out

    # -- transforms by definition
    def ntt(self, a, m):
        q, psi, N = self.mod[m], self.psi[m], self.N
        out = []
        for k in range(N):
            x = pow(psi, 2 * brv(k, self.logN) + 1, q)
            acc, p = 0, 1
            for c in a:
                acc += c * p
                p = p * x % q
            out.append(acc % q)
        return out

    def intt(self, A, m):
        """solve the evaluation system: a_j = N^-1 sum_k A_k x_k^-j"""
        q, psi, N = self.mod[m], self.psi[m], self.N
        ninv = pow(N, q - 2, q)
        xs = [pow(psi, 2 * brv(k, self.logN) + 1, q) for k in range(N)]
        out = []
        for j in range(N):
            acc = 0
            for k in range(N):
                acc += A[k] * pow(xs[k], (2 * N - j) % (2 * N), q)
            out.append(acc * ninv % q)
        return out

    def negacyclic(self, a, b, q):
        N = self.N
        out = [0] * N
        for i in range(N):
            for j in range(N):
                if i + j < N:
                    out[i + j] += a[i] * b[j]
                else:
                    out[i + j - N] -= a[i] * b[j]
        return [x % q for x in out]

    # -- FFT (same operation order as the contract)
    def _fft(self, re, im, sign):
        n, bits = self.n, self.logN - 1
        for i in range(n):
            r = brv(i, bits)
            if r > i:
                re[i], re[r] = re[r], re[i]
                im[i], im[r] = im[r], im[i]
        length = 2
        while length <= n:
            half, step = length // 2, n // length
            for s in range(0, n, length):
                for k in range(half):
                    wr = self.wr[k * step]
                    wi = -self.wi[k * step] if sign < 0 else self.wi[k * step]
                    vr0, vi0 = re[s + k + half], im[s + k + half]
                    vr = vr0 * wr - vi0 * wi
                    vi = vr0 * wi + vi0 * wr
                    ur, ui = re[s + k], im[s + k]
                    re[s + k], im[s + k] = ur + vr, ui + vi
                    re[s + k + half], im[s + k + half] = ur - vr, ui - vi
            length *= 2

    def encode(self, vals, scale):
        n = self.n
        re, im = [0.0] * n, [0.0] * n
        for i, v in enumerate(vals):
            re[self.pos[i]] = float(v)
        self._fft(re, im, -1)
        m = [0] * self.N
        for j in range(n):
            vr, vi = re[j] * (1.0 / n), im[j] * (1.0 / n)
            ur = vr * self.zr[j] + vi * self.zi[j]
            ui = vi * self.zr[j] - vr * self.zi[j]
            m[j] = int(round(ur * scale))  # Python round() is half-to-even, like rint
            m[j + n] = int(round(ui * scale))
        return m

    def decode(self, coeffs, scale):
        n = self.n
        re, im = [0.0] * n, [0.0] * n
        for j in range(n):
            ur, ui = coeffs[j] / scale, coeffs[j + n] / scale
            re[j] = ur * self.zr[j] - ui * self.zi[j]
            im[j] = ur * self.zi[j] + ui * self.zr[j]
        self._fft(re, im, +1)
        return [re[self.pos[i]] for i in range(n)]

    # -- keys, encryption
    def sk_ntt(self, m):
        return self.ntt([x % self.mod[m] for x in self.s], m)

    def encrypt(self, vals, ct_index, scale=None):
        m = self.encode(vals, scale or self.scale)
        e = self.cbd(DOM_ENC_E, ct_index)
        c0, c1 = [], []
        for i in range(self.L):
            q = self.mod[i]
            p0 = self.ntt([(a + b) % q for a, b in zip(m, e)], i)
            a = self.uniform(DOM_ENC_A, ct_index, i, q)
            s = self.sk_ntt(i)
            c0.append([(x - y * z) % q for x, y, z in zip(p0, a, s)])
            c1.append(a)
        return [c0, c1]

    def switch_key(self, g=0):
        L, K, N = self.L, self.K, self.N
        P = 1
        for p in self.mod[L:]:
            P *= p
        key = []
        for j in range(self.dnum):
            obj = g * 64 + j
            e = self.cbd(DOM_KSK_E, obj)
            B, A = [], []
            for m in range(L + K):
                q = self.mod[m]
                s = self.sk_ntt(m)
                a = self.uniform(DOM_KSK_A, obj, m, q)
                en = self.ntt([x % q for x in e], m)
                b = [(x - y * z) % q for x, y, z in zip(en, a, s)]
                if m < L and j * self.alpha <= m < (j + 1) * self.alpha:
                    if g % 2 == 0:  # s^2 (g = 0) or the power key s^(g/2+2)
                        pw = 2 if g == 0 else g // 2 + 2
                        sp = [pow(x, pw, q) for x in s]
                    else:
                        sp = self.automorphism(s, g)
                    b = [(x + P * y) % q for x, y in zip(b, sp)]
                B.append(b)
                A.append(a)
            key.append([B, A])
        return key

    def automorphism(self, poly, g):
        N, logN = self.N, self.logN
        out = []
        for k in range(N):
            e = 2 * brv(k, logN) + 1
            e2 = e * g % (2 * N)
            out.append(poly[brv((e2 - 1) // 2, logN)])
        return out

    # -- key switching by the CRT definitions
    def keyswitch(self, d, key, ell):
        """d: ell limbs (NTT).  Returns (o0, o1) each ell limbs (NTT)."""
        L, K = self.L, self.K
        mods = self.mod[:ell] + self.mod[L:]
        midx = list(range(ell)) + list(range(L, L + K))
        dc = [self.intt(d[i], i) for i in range(ell)]
        beta = -(-ell // self.alpha)
        acc = [[[0] * self.N for _ in mods] for _ in range(2)]
        for j in range(beta):
            S = list(range(j * self.alpha, min((j + 1) * self.alpha, ell)))
            QS = 1
            for s in S:
                QS *= self.mod[s]
            for t, m in enumerate(midx):
                q = self.mod[m]
                if t in S:
                    ext = d[t]
                else:
                    vals = []
                    for k in range(self.N):
                        y = 0
                        for s in S:
                            qs = self.mod[s]
                            qh = QS // qs
                            y += (dc[s][k] * pow(qh % qs, -1, qs) % qs) * qh
                        vals.append(y % q)
                    ext = self.ntt(vals, m)
                for c in range(2):
                    kk = key[j][c][m]
                    acc[c][t] = [(x + y * z) % q for x, y, z in zip(acc[c][t], ext, kk)]
        P = 1
        for p in self.mod[L:]:
            P *= p
        outs = []
        for c in range(2):
            xp = [self.intt(acc[c][ell + k], L + k) for k in range(K)]
            o = []
            for i in range(ell):
                q = self.mod[i]
                vals = []
                for k in range(self.N):
                    y = 0
                    for kk in range(K):
                        pk = self.mod[L + kk]
                        ph = P // pk
                        y += (xp[kk][k] * pow(ph % pk, -1, pk) % pk) * ph
                    vals.append(y % q)
                conv = self.ntt(vals, i)
                pinv = pow(P % q, -1, q)
                o.append([(x - y) * pinv % q for x, y in zip(acc[c][i], conv)])
            outs.append(o)
        return outs[0], outs[1]

    def rescale(self, ct):
        """ct: list of components, each a list of ell limbs (NTT)."""
        ell = len(ct[0])
        l = ell - 1
        ql = self.mod[l]
        out = []
        for comp in ct:
            r = [centered(x, ql) for x in self.intt(comp[l], l)]
            o = []
            for i in range(l):
                q = self.mod[i]
                t = self.ntt([x % q for x in r], i)
                inv = pow(ql, -1, q)
                o.append([(x - y) * inv % q for x, y in zip(comp[i], t)])
            out.append(o)
        return out

    def decrypt_coeffs(self, ct):
        ell = len(ct[0])
        D = min(ell, 2)
        xs = []
        for i in range(D):
            q = self.mod[i]
            s = self.sk_ntt(i)
            xs.append(self.intt([(a + b * c) % q for a, b, c in zip(ct[0][i], ct[1][i], s)], i))
        Q = 1
        for i in range(D):
            Q *= self.mod[i]
        out = []
        for k in range(self.N):
            v = 0
            for i in range(D):
                qi = self.mod[i]
                qh = Q // qi
                v += xs[i][k] * pow(qh % qi, -1, qi) * qh
            out.append(centered(v, Q))
        return out
