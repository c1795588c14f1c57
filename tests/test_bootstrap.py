"""CKKS bootstrapping circuit on the CPU oracle.

The reference's bootstrap (/root/reference/pkg/src/hebatch/engine.py:315-319)
resets the level to max_level - bootstrap_reserve and keeps the slots; the
circuit here (paper_2604_16834_b200/bootstrap.py) does that for real.  These
CPU tests pin the circuit's algebra: the DFT diagonals against the oracle's
own encoder, the BSGS decomposition, and a full bootstrap of an oracle
ciphertext on a 64-point ring (decrypts to the input slots).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from helpers import oracle_for
from oracle_boot import OCt, OracleBootOps
from paper_2604_16834_b200.bootstrap import (BootPlan, Bootstrapper, bsgs_plains, cts_diagonals, secret_bound,
                                             stc_diagonals)


def _dense(diags):
    n = diags.shape[1]
    M = np.zeros((n, n), np.complex128)
    for k in range(n):
        for i in range(n):
            M[i, (i + k) % n] = diags[k, i]
    return M


def test_dft_diagonals_match_the_encoder():
    """V (from stc_diagonals) maps u_j = m_j + i m_{j+n} to the slots the oracle decodes."""
    orc = oracle_for("boot6")
    N, n = orc.N, orc.n
    rng = np.random.default_rng(3)
    m = rng.integers(-1000, 1000, N).astype(np.float64)
    u = m[:n] + 1j * m[n:]
    V = _dense(stc_diagonals(N))
    slots = V @ u
    assert np.allclose(orc.decode(m, 1.0), slots.real, atol=1e-6)
    Vi = _dense(cts_diagonals(N))
    assert np.allclose(Vi @ V, np.eye(n), atol=1e-9)
    # the complex encoder inverts V: encode(z) = round(scale * V^-1 z) as (re, im) halves
    z = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    enc = orc.encode_complex(z, 2.0 ** 30)
    uu = Vi @ z * 2.0 ** 30
    assert np.max(np.abs(enc[:n] - uu.real)) <= 0.5 + 1e-6
    assert np.max(np.abs(enc[n:] - uu.imag)) <= 0.5 + 1e-6


def test_bsgs_decomposition():
    rng = np.random.default_rng(4)
    n, b, G = 32, 8, 4
    d = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    z = rng.normal(size=n) + 1j * rng.normal(size=n)
    p = bsgs_plains(d, b, G)
    out = np.zeros(n, np.complex128)
    for g in range(G):
        inner = sum(p[g, j] * np.roll(z, -j) for j in range(b))
        out += np.roll(inner, -b * g)
    assert np.allclose(out, _dense(d) @ z)


def test_plan_parameters():
    p = BootPlan(N=1 << 12, q0=(1 << 60) - 1)
    assert p.r == 9 and p.depth == 18 and p.baby * p.giant == p.n
    assert 2 * math.pi * (secret_bound(1 << 12) + 0.25) / (1 << p.r) <= 1.25
    p6 = BootPlan(N=64, q0=(1 << 60) - 1)
    assert p6.r == 6 and p6.depth == 15


def test_bootstrap_circuit_on_the_oracle():
    """Encrypt at the top level, drop to level 0, bootstrap: the slots come back."""
    orc = oracle_for("boot6")
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, orc.n)
    ct = orc.encrypt(x, 0)
    low = OCt(ct[:, :1], orc.scale)
    assert np.max(np.abs(orc.decrypt(low.data, low.scale) - x)) < 1e-9
    ops = OracleBootOps(orc)
    plan = BootPlan(N=orc.N, q0=orc.moduli[0])
    out = Bootstrapper(ops, plan).run(low, orc.L)
    assert out.level == orc.L - 1 - plan.depth
    err = np.max(np.abs(orc.decrypt(out.data, out.scale) - x))
    assert err < 1e-4, err
