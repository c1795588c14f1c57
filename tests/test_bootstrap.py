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
from paper_2604_16834_b200.bootstrap import (BootPlan, Bootstrapper, BsgsStage, apply_map, butterfly_stages,
                                             dft_groups, secret_bound)


def _vmat(N):
    n = N // 2
    p5 = np.array([pow(5, i, 2 * N) for i in range(n)], np.int64)
    return np.exp(1j * np.pi * (np.outer(p5, np.arange(n)) % (2 * N)) / N)


def _bitrev(n):
    m = n.bit_length() - 1
    return np.array([int(format(i, f"0{m}b")[::-1], 2) for i in range(n)])


def test_v_matches_the_encoder():
    """V[i][j] = zeta^(5^i j) maps u_j = m_j + i m_{j+n} to the slots the oracle decodes."""
    orc = oracle_for("boot6")
    N, n = orc.N, orc.n
    rng = np.random.default_rng(3)
    m = rng.integers(-1000, 1000, N).astype(np.float64)
    assert np.allclose(orc.decode(m, 1.0), (_vmat(N) @ (m[:n] + 1j * m[n:])).real, atol=1e-6)
    # the complex encoder inverts V: encode(z) = round(scale V^-1 z) as (re, im) halves
    z = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    enc = orc.encode_complex(z, 2.0 ** 30)
    uu = np.linalg.solve(_vmat(N), z) * 2.0 ** 30
    assert np.max(np.abs(enc[:n] - uu.real)) <= 0.5 + 1e-6
    assert np.max(np.abs(enc[n:] - uu.imag)) <= 0.5 + 1e-6


@pytest.mark.parametrize("N", [16, 64, 512, 4096])
def test_factored_dft(N):
    """V = B_m .. B_1 R and R V^-1 = B_1^-1 .. B_m^-1, stage by stage and merged into levels."""
    n = N // 2
    rng = np.random.default_rng(N)
    u = rng.normal(size=n) + 1j * rng.normal(size=n)
    R = _bitrev(n)
    z = _vmat(N) @ u
    x = u[R]
    for D in butterfly_stages(N):
        x = apply_map(D, x)
    assert np.allclose(x, z, atol=1e-9 * n)
    y = z
    for D in reversed(butterfly_stages(N, inverse=True)):
        y = apply_map(D, y)
    assert np.allclose(y, u[R], atol=1e-9 * n)
    for levels in (1, 2, 3):
        x, y = u[R], z
        for h0, D in dft_groups(N, levels, inverse=False):
            assert all(o % h0 == 0 for o in D)
            x = apply_map(D, x)
        for h0, D in dft_groups(N, levels, inverse=True):
            y = apply_map(D, y)
        assert np.allclose(x, z, atol=1e-9 * n) and np.allclose(y, u[R], atol=1e-9 * n)


@pytest.mark.parametrize("levels", [1, 2, 3])
def test_bsgs_stage_reproduces_the_level(levels):
    N, n = 256, 128
    rng = np.random.default_rng(levels)
    x = rng.normal(size=n) + 1j * rng.normal(size=n)
    for h0, D in dft_groups(N, levels, inverse=True):
        st = BsgsStage.build(h0, D, n)
        out = np.zeros(n, np.complex128)
        for g in range(st.giant):
            inner = sum(st.plains[g, j] * np.roll(x, -j * h0) for j in range(st.baby))
            out += np.roll(inner, -((st.base + g * st.baby) * h0) % n)
        assert np.allclose(out, apply_map(D, x))
        assert st.baby * st.giant < 2 * len(D) + 2 * st.baby


def test_plan_parameters():
    p = BootPlan(N=1 << 12, q0=(1 << 60) - 1)
    assert p.r == 9 and p.dft_levels == 2 and p.depth == 20
    assert 2 * math.pi * (secret_bound(1 << 12) + 0.25) / (1 << p.r) <= 1.25
    p6 = BootPlan(N=64, q0=(1 << 60) - 1)
    assert p6.r == 6 and p6.depth == 15
    ps = BootPlan(N=1 << 16, q0=(1 << 60) - 1, hamming=128)
    assert ps.r == 7 and ps.dft_levels == 3 and ps.depth == 20


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
    out = Bootstrapper(ops, plan, low.scale).run([low], orc.L)[0]
    assert out.level == orc.L - 1 - plan.depth
    err = np.max(np.abs(orc.decrypt(out.data, out.scale) - x))
    assert err < 1e-4, err


def test_sparse_secret_on_the_oracle():
    """sk_hamming = h: ternary coefficients, about h of them nonzero (bootstrapping's K bound)."""
    import oracle as O

    o = O.Oracle(11, [60, 50, 50], [60], 1, seed=9, scale=2.0 ** 50, sk_hamming=64)
    q = o.moduli[0]
    c = o.intt(o.secret_key()[0], 0)
    v = np.where(c > q // 2, c.astype(np.int64) - np.int64(q), c.astype(np.int64))
    assert set(np.unique(v)) <= {-1, 0, 1}
    assert 64 - 4 * 8 <= np.count_nonzero(v) <= 64 + 4 * 8
    # every limb holds the same small polynomial
    c1 = o.intt(o.secret_key()[1], 1)
    q1 = o.moduli[1]
    v1 = np.where(c1 > q1 // 2, c1.astype(np.int64) - np.int64(q1), c1.astype(np.int64))
    assert np.array_equal(v, v1)
