"""ctypes wrapper over the C oracle (oracle/ckks_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_2604_16834_b200) never imports this module.

Every method takes and returns numpy uint64 arrays in the layout of the
product ABI: a ciphertext is [n_comp][ell][N] in the NTT domain.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libckks_oracle.so")


class OcParams(C.Structure):
    _fields_ = [
        ("log_n", C.c_int32),
        ("n_q", C.c_int32),
        ("n_p", C.c_int32),
        ("alpha", C.c_int32),
        ("q_bits", C.c_int32 * 48),
        ("p_bits", C.c_int32 * 16),
        ("seed", C.c_uint64),
        ("scale", C.c_double),
        ("sk_hamming", C.c_int32),
        ("reserved", C.c_int32),
    ]


def build() -> str:
    """Compile the oracle (make -C oracle); returns the .so path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        vp, u64p, i64p, dp = C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_int64), C.POINTER(C.c_double)
        L.oc_create.restype = vp
        L.oc_create.argtypes = [C.POINTER(OcParams)]
        L.oc_destroy.argtypes = [vp]
        L.oc_coeff_view.restype = vp
        L.oc_coeff_view.argtypes = [vp, C.c_int]
        L.oc_moduli.argtypes = [vp, u64p, u64p]
        L.oc_philox.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.oc_ntt.argtypes = [vp, u64p, C.c_int]
        L.oc_intt.argtypes = [vp, u64p, C.c_int]
        L.oc_encode.argtypes = [vp, dp, C.c_int, C.c_double, i64p]
        L.oc_encode_c.argtypes = [vp, dp, dp, C.c_int, C.c_double, i64p]
        L.oc_decode.argtypes = [vp, dp, C.c_double, dp]
        L.oc_secret_key.argtypes = [vp, u64p]
        L.oc_gen_switch_key.argtypes = [vp, C.c_uint32, u64p]
        L.oc_encrypt.argtypes = [vp, dp, C.c_int, C.c_double, C.c_uint32, u64p]
        L.oc_decrypt.argtypes = [vp, u64p, C.c_int, C.c_double, dp]
        L.oc_decrypt_coeffs.argtypes = [vp, u64p, C.c_int, dp]
        for name in ("oc_add", "oc_sub"):
            getattr(L, name).argtypes = [vp, u64p, u64p, u64p, C.c_int, C.c_int]
        L.oc_add_const.argtypes = [vp, u64p, u64p, u64p, C.c_int]
        L.oc_mul_const.argtypes = [vp, u64p, u64p, u64p, C.c_int, C.c_int]
        L.oc_mul_plain.argtypes = [vp, u64p, u64p, u64p, C.c_int, C.c_int]
        L.oc_tensor.argtypes = [vp, u64p, u64p, u64p, C.c_int]
        L.oc_keyswitch.argtypes = [vp, u64p, u64p, C.c_int, u64p, u64p]
        L.oc_relin.argtypes = [vp, u64p, u64p, u64p, C.c_int]
        L.oc_relin_rescale.argtypes = [vp, u64p, u64p, u64p, C.c_int, C.c_int]
        L.oc_relin_rescale_n.argtypes = [vp, u64p, C.c_int, C.POINTER(vp), u64p, C.c_int, C.c_int]
        L.oc_tensor_sq.argtypes = [vp, u64p, C.c_int, u64p, C.c_int]
        L.oc_rescale.argtypes = [vp, u64p, u64p, C.c_int, C.c_int]
        L.oc_automorphism.argtypes = [vp, u64p, C.c_uint32, u64p, C.c_int]
        L.oc_rotate.argtypes = [vp, u64p, C.c_uint32, u64p, u64p, C.c_int]
        L.oc_hoist_key.argtypes = [vp, u64p, C.c_uint32, u64p]
        L.oc_rotate_hoisted.argtypes = [vp, u64p, C.c_uint32, u64p, u64p, C.c_int]
        L.oc_mult_ct.argtypes = [vp, u64p, u64p, u64p, u64p, C.c_int]
        L.oc_plain_to_ntt.argtypes = [vp, i64p, u64p, C.c_int]
        L.oc_lincomb.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.c_int, C.POINTER(C.c_int32),
                                 C.POINTER(C.c_int32), i64p, C.c_int, C.c_int, C.c_int]
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _u64(a):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return _p(a, C.c_uint64)


def philox(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().oc_philox(c, k, o)
    return list(o)


def make_params(log_n, q_bits, p_bits, alpha, seed, scale, sk_hamming=0):
    p = OcParams()
    p.sk_hamming = sk_hamming
    p.log_n = log_n
    p.n_q = len(q_bits)
    p.n_p = len(p_bits)
    p.alpha = alpha
    for i, b in enumerate(q_bits):
        p.q_bits[i] = b
    for i, b in enumerate(p_bits):
        p.p_bits[i] = b
    p.seed = seed
    p.scale = scale
    return p


class Oracle:
    """One oracle context: moduli, twiddles, secret key (from params.seed)."""

    def __init__(self, log_n, q_bits, p_bits, alpha, seed=0, scale=2.0 ** 40, sk_hamming=0):
        self.params = make_params(log_n, q_bits, p_bits, alpha, seed, scale, sk_hamming)
        self.sk_hamming = sk_hamming
        self.N = 1 << log_n
        self.n = self.N // 2
        self.L = len(q_bits)
        self.K = len(p_bits)
        self.alpha = alpha
        self.dnum = (self.L + alpha - 1) // alpha
        self.scale = scale
        self._h = lib().oc_create(C.byref(self.params))
        mods = np.zeros(self.L + self.K, np.uint64)
        psi = np.zeros(self.L + self.K, np.uint64)
        lib().oc_moduli(self._h, _u64(mods), _u64(psi))
        self.moduli = [int(x) for x in mods]
        self.psi = [int(x) for x in psi]

    def coeff_view(self, n):
        """Element-wise-only oracle over n sampled evaluation points (oc_coeff_view):
        add/sub/add_const/mul_const/mul_plain/tensor/tensor_sq/lincomb on
        [nc][ell][n] arrays give exactly those points of the full-ring results.
        Pack a ciphertext's sampled points with ``ct[..., idx]``."""
        return CoeffView(self, n)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().oc_destroy(h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self._h = None

    # -- transforms
    def ntt(self, poly, mod_idx):
        a = np.ascontiguousarray(poly, dtype=np.uint64).copy()
        lib().oc_ntt(self._h, _u64(a), mod_idx)
        return a

    def intt(self, poly, mod_idx):
        a = np.ascontiguousarray(poly, dtype=np.uint64).copy()
        lib().oc_intt(self._h, _u64(a), mod_idx)
        return a

    def encode(self, vals, scale=None):
        v = np.ascontiguousarray(vals, dtype=np.float64)
        m = np.zeros(self.N, np.int64)
        lib().oc_encode(self._h, _p(v, C.c_double), v.size, scale or self.scale, _p(m, C.c_int64))
        return m

    def encode_complex(self, vals, scale=None):
        """Complex slot vector -> plaintext coefficients (oc_encode_c)."""
        v = np.asarray(vals, dtype=np.complex128)
        re, im = np.ascontiguousarray(v.real), np.ascontiguousarray(v.imag)
        m = np.zeros(self.N, np.int64)
        lib().oc_encode_c(self._h, _p(re, C.c_double), _p(im, C.c_double), v.size, scale or self.scale,
                          _p(m, C.c_int64))
        return m

    def mod_raise(self, ct, ell_out):
        """ModRaise (bootstrapping's first step): limb 0 of each component, INTT,
        centred lift mod q_0, then every limb of the chain q_0..q_{ell_out-1}, NTT."""
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        q0 = self.moduli[0]
        out = np.zeros((ct.shape[0], ell_out, self.N), np.uint64)
        for comp in range(ct.shape[0]):
            v = self.intt(ct[comp, 0], 0)
            cv = np.where(v > np.uint64(q0 // 2), v.astype(np.int64) - np.int64(q0), v.astype(np.int64))
            for l in range(ell_out):
                out[comp, l] = self.ntt(np.mod(cv, np.int64(self.moduli[l])).astype(np.uint64), l)
        return out

    def decode(self, coeffs, scale):
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.zeros(self.n, np.float64)
        lib().oc_decode(self._h, _p(c, C.c_double), scale, _p(out, C.c_double))
        return out

    # -- keys
    def secret_key(self):
        sk = np.zeros((self.L + self.K, self.N), np.uint64)
        lib().oc_secret_key(self._h, _u64(sk))
        return sk

    def switch_key(self, galois_elt=0):
        k = np.zeros((self.dnum, 2, self.L + self.K, self.N), np.uint64)
        lib().oc_gen_switch_key(self._h, galois_elt, _u64(k))
        return k

    # -- enc / dec
    def encrypt(self, vals, ct_index, scale=None):
        v = np.ascontiguousarray(vals, dtype=np.float64)
        ct = np.zeros((2, self.L, self.N), np.uint64)
        lib().oc_encrypt(self._h, _p(v, C.c_double), v.size, scale or self.scale, ct_index, _u64(ct))
        return ct

    def decrypt(self, ct, scale):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        ell = ct.shape[1]
        out = np.zeros(self.n, np.float64)
        lib().oc_decrypt(self._h, _u64(ct), ell, scale, _p(out, C.c_double))
        return out

    def decrypt_coeffs(self, ct):
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        out = np.zeros(self.N, np.float64)
        lib().oc_decrypt_coeffs(self._h, _u64(ct), ct.shape[1], _p(out, C.c_double))
        return out

    # -- arithmetic
    def add(self, a, b):
        out = np.zeros_like(a)
        lib().oc_add(self._h, _u64(a), _u64(b), _u64(out), a.shape[1], a.shape[0])
        return out

    def sub(self, a, b):
        out = np.zeros_like(a)
        lib().oc_sub(self._h, _u64(a), _u64(b), _u64(out), a.shape[1], a.shape[0])
        return out

    def add_const(self, ct, residues):
        r = np.ascontiguousarray(residues, dtype=np.uint64)
        out = np.zeros_like(ct)
        lib().oc_add_const(self._h, _u64(ct), _u64(r), _u64(out), ct.shape[1])
        return out

    def mul_const(self, ct, residues):
        r = np.ascontiguousarray(residues, dtype=np.uint64)
        out = np.zeros_like(ct)
        lib().oc_mul_const(self._h, _u64(ct), _u64(r), _u64(out), ct.shape[1], ct.shape[0])
        return out

    def mul_plain(self, ct, pt):
        out = np.zeros_like(ct)
        lib().oc_mul_plain(self._h, _u64(ct), _u64(np.ascontiguousarray(pt)), _u64(out), ct.shape[1], ct.shape[0])
        return out

    def plain_to_ntt(self, m, ell):
        m = np.ascontiguousarray(m, dtype=np.int64)
        pt = np.zeros((ell, self.N), np.uint64)
        lib().oc_plain_to_ntt(self._h, _p(m, C.c_int64), _u64(pt), ell)
        return pt

    def tensor(self, a, b):
        ell = a.shape[1]
        out = np.zeros((3, ell, self.N), np.uint64)
        lib().oc_tensor(self._h, _u64(a), _u64(b), _u64(out), ell)
        return out

    def keyswitch(self, d, key):
        ell = d.shape[0]
        o0 = np.zeros((ell, self.N), np.uint64)
        o1 = np.zeros((ell, self.N), np.uint64)
        lib().oc_keyswitch(self._h, _u64(np.ascontiguousarray(d)), _u64(key), ell, _u64(o0), _u64(o1))
        return o0, o1

    def relin(self, d3, key):
        ell = d3.shape[1]
        out = np.zeros((2, ell, self.N), np.uint64)
        lib().oc_relin(self._h, _u64(d3), _u64(key), _u64(out), ell)
        return out

    def relin_rescale(self, d3, key, extra):
        """relinearise + `extra` rescales as one joint ModDown (oc_relin_rescale)."""
        ell = d3.shape[1]
        out = np.zeros((2, ell - extra, self.N), np.uint64)
        lib().oc_relin_rescale(self._h, _u64(np.ascontiguousarray(d3)), _u64(key), _u64(out), ell, extra)
        return out

    def relin_rescale_n(self, d, keys, extra):
        """nc-component relinearisation (keys[k-2] = switch_key(power code of s^k), see
        power_key_elt) + `extra` rescales as one joint ModDown (oc_relin_rescale_n)."""
        d = np.ascontiguousarray(d, dtype=np.uint64)
        nc, ell = d.shape[0], d.shape[1]
        assert len(keys) == nc - 2
        kp = (C.c_void_p * len(keys))(*[k.ctypes.data for k in keys])
        out = np.zeros((2, ell - extra, self.N), np.uint64)
        lib().oc_relin_rescale_n(self._h, _u64(d), nc, kp, _u64(out), ell, extra)
        return out

    def tensor_sq(self, a):
        """square of an nc-component ciphertext: 2nc-1 components (oc_tensor_sq)."""
        a = np.ascontiguousarray(a, dtype=np.uint64)
        nc, ell = a.shape[0], a.shape[1]
        out = np.zeros((2 * nc - 1, ell, self.N), np.uint64)
        lib().oc_tensor_sq(self._h, _u64(a), nc, _u64(out), ell)
        return out

    def rescale(self, ct):
        nc, ell = ct.shape[0], ct.shape[1]
        out = np.zeros((nc, ell - 1, self.N), np.uint64)
        lib().oc_rescale(self._h, _u64(np.ascontiguousarray(ct)), _u64(out), ell, nc)
        return out

    def automorphism(self, polys, g):
        polys = np.ascontiguousarray(polys, dtype=np.uint64)
        out = np.zeros_like(polys)
        lib().oc_automorphism(self._h, _u64(polys), g, _u64(out), polys.size // self.N)
        return out

    def hoist_key(self, key, g):
        """sigma_{g^-1} applied to every polynomial of switch key `key` (oc_hoist_key)."""
        key = np.ascontiguousarray(key, dtype=np.uint64)
        out = np.zeros_like(key)
        lib().oc_hoist_key(self._h, _u64(key), g, _u64(out))
        return out

    def rotate_hoisted(self, ct, g, hkey):
        """Hoisted rotation (oc_rotate_hoisted): KS of the unrotated c1 with the
        hoisting key, + c0, then sigma_g on both components."""
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        out = np.zeros_like(ct)
        lib().oc_rotate_hoisted(self._h, _u64(ct), g, _u64(hkey), _u64(out), ct.shape[1])
        return out

    def rotate(self, ct, g, key):
        out = np.zeros_like(ct)
        lib().oc_rotate(self._h, _u64(ct), g, _u64(key), _u64(out), ct.shape[1])
        return out

    def mult_ct(self, a, b, relin_key):
        ell = a.shape[1]
        out = np.zeros((2, ell - 1, self.N), np.uint64)
        lib().oc_mult_ct(self._h, _u64(a), _u64(b), _u64(relin_key), _u64(out), ell)
        return out

    def lincomb(self, ins, row_ptr, col, w, n_threads=0):
        """ins: list of cts (same shape); returns list of len(row_ptr)-1 cts."""
        nc, ell = ins[0].shape[0], ins[0].shape[1]
        n_out = len(row_ptr) - 1
        outs = [np.zeros((nc, ell, self.N), np.uint64) for _ in range(n_out)]
        in_p = (C.c_void_p * len(ins))(*[a.ctypes.data for a in ins])
        out_p = (C.c_void_p * n_out)(*[a.ctypes.data for a in outs])
        rp = np.ascontiguousarray(row_ptr, np.int32)
        cl = np.ascontiguousarray(col, np.int32)
        ww = np.ascontiguousarray(w, np.int64)
        lib().oc_lincomb(self._h, in_p, out_p, n_out, _p(rp, C.c_int32), _p(cl, C.c_int32),
                         _p(ww, C.c_int64), ell, nc, n_threads)
        return outs


class CoeffView(Oracle):
    """Oracle.coeff_view: same moduli, N = n sampled points, element-wise ops only."""

    _ELEMENTWISE = {"add", "sub", "add_const", "mul_const", "mul_plain", "tensor", "tensor_sq", "lincomb"}

    def __init__(self, parent, n):  # noqa: D107 -- no oc_create: the tables stay with the parent
        self.params = parent.params
        self.N = n
        self.n = 0
        self.L, self.K, self.alpha, self.dnum = parent.L, parent.K, parent.alpha, parent.dnum
        self.scale = parent.scale
        self.moduli, self.psi = parent.moduli, parent.psi
        self._parent = parent
        self._h = lib().oc_coeff_view(parent._h, n)

    def __getattribute__(self, name):
        if (not name.startswith("_") and name not in CoeffView._ELEMENTWISE and callable(getattr(Oracle, name, None))
                and name not in ("coeff_view",)):
            raise TypeError(f"CoeffView supports element-wise operations only, not {name}")
        return object.__getattribute__(self, name)


def power_key_elt(power: int) -> int:
    """Key code of the s^power switching key: 0 for s^2 (relinearisation), the even
    code 2 (power - 2) for s^3, s^4 (never a Galois element, which is odd)."""
    return 0 if power == 2 else 2 * (power - 2)


def galois_elt(k: int, N: int) -> int:
    """Galois element for a left rotation by k slots: 5^k mod 2N (engine.py:13-15)."""
    n = N // 2
    return pow(5, k % n, 2 * N)
