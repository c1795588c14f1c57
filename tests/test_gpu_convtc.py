"""The tcgen05 fused conv kernels (csrc/convtc.cu) on the B200.

Two levels of evidence, both bit-exact:
  * against the CPU oracle's conv -> tensor square -> add_const -> window-sum
    chain (tests/test_gpu_parity._oracle_conv_square_sum) on config 3's prime
    sizes at N = 2^12 (ring "cfg3s"), at the image widths the kernels tile
    (16 and 32 pixels), every weight-digit count and ring-wrap position;
  * against the mma.sync kernels (themselves pinned to the oracle by
    test_gpu_parity) on the config-3 ring at N = 2^16 and 9 limbs, the exact
    launch shapes run_cnn / bench.py issue.
"""

from __future__ import annotations

import numpy as np
import pytest

from helpers import engine_context, from_np, oracle_for, rand_residues, to_np
from test_gpu_parity import _oracle_conv_square_sum

pytestmark = pytest.mark.gpu


_KEEP = []  # pointer arrays passed as `_ptrs(x).ctypes.data` must outlive the call


def _ptrs(ts):
    a = np.array([t.data_ptr() for t in ts], np.uint64)
    _KEEP.append(a)
    del _KEEP[:-16]
    return a


@pytest.fixture(scope="module")
def small():
    from paper_2604_16834_b200.engine import GpuEngine

    return GpuEngine(engine_context("cfg3s")), oracle_for("cfg3s")


def _run(eng, fn, ins, nci, p, H, W, M, pool, y0, y1, wi, bres, cst, ell):
    import torch

    nwin = ((y1 - y0) // 2) * (W // 2) if pool else 1
    outs = [torch.zeros((2 * nci - 1, ell, eng.N), dtype=torch.int64, device=eng.device) for _ in range(M * nwin)]
    pi, po = _ptrs(ins), _ptrs(outs)
    rc = fn(eng._h, pi.ctypes.data, nci, p, H, W, po.ctypes.data, M, pool, y0, y1, wi.ctypes.data,
            bres.ctypes.data if bres is not None else None, cst.ctypes.data if cst is not None else None, ell, None)
    assert rc == 0, eng._L.he_last_error()
    return outs


@pytest.mark.parametrize("W,H,rows,wbits,p,M", [(16, 4, (0, 4), 20, 3, 16), (32, 4, (2, 4), 14, 3, 16),
                                                (16, 8, (2, 8), 7, 2, 11), (32, 2, (0, 2), 20, 1, 16)])
def test_convtc_pool_vs_oracle(small, W, H, rows, wbits, p, M):
    """conv1 shape class (2-component inputs, p <= 3, 2x2 pool) vs the oracle chain."""
    eng, orc = small
    rng = np.random.default_rng(100 + W + H + wbits)
    ell = 3
    mods = eng.moduli[:ell]
    x = rand_residues(rng, mods, (p * H * W, 2), eng.N)
    ins = [from_np(x[i], eng.device) for i in range(p * H * W)]
    lim = 1 << wbits
    wi = rng.integers(-lim, lim, size=(M, 9 * p), dtype=np.int64)
    bres = np.array([[int(rng.integers(0, q)) for q in mods] for _ in range(M)], np.uint64)
    cst = np.array([int(rng.integers(0, q)) for q in mods], np.uint64)
    y0, y1 = rows
    got = _run(eng, eng._L.he_conv_square_sum_tc, ins, 2, p, H, W, M, 1, y0, y1, wi, bres, cst, ell)
    ref = _oracle_conv_square_sum(orc, [x[i] for i in range(p * H * W)], p, H, W, wi, bres, cst, 1, y0, y1)
    for k, (o, r) in enumerate(zip(got, ref)):
        assert np.array_equal(to_np(o), r), k


@pytest.mark.parametrize("H,rows,wbits,M", [(2, (0, 2), 14, 18), (4, (1, 3), 9, 32)])
def test_convtc_gap_vs_oracle(small, H, rows, wbits, M):
    """conv2 shape class (3-component carried inputs, 16 -> M channels, 16 wide, global sum)
    vs the oracle chain: 5-component window sums, both channel halves."""
    eng, orc = small
    rng = np.random.default_rng(200 + H + wbits)
    ell, p, W = 3, 16, 16
    mods = eng.moduli[:ell]
    x = rand_residues(rng, mods, (p * H * W, 3), eng.N)
    ins = [from_np(x[i], eng.device) for i in range(p * H * W)]
    lim = 1 << wbits
    wi = rng.integers(-lim, lim, size=(M, 9 * p), dtype=np.int64)
    bres = np.array([[int(rng.integers(0, q)) for q in mods] for _ in range(M)], np.uint64)
    cst = np.array([int(rng.integers(0, q)) for q in mods], np.uint64)
    y0, y1 = rows
    got = _run(eng, eng._L.he_conv_square_sum_tc, ins, 3, p, H, W, M, 0, y0, y1, wi, bres, cst, ell)
    ref = _oracle_conv_square_sum(orc, [x[i] for i in range(p * H * W)], p, H, W, wi, bres, cst, 0, y0, y1)
    for k, (o, r) in enumerate(zip(got, ref)):
        assert np.array_equal(to_np(o), r), k


@pytest.mark.parametrize("shape", ["conv1", "conv2"])
def test_convtc_extreme_values_vs_oracle(small, shape):
    """The 32-/64-bit shift-sum bounds of the integer recombination: inputs whose residues are all
    q - 1 or 2^40 - 2^32 - 1 patterns (every byte plane at or near 255) with the heaviest weights
    the launcher accepts (same sign, every digit large), against the oracle chain; heavier weights
    are refused (HE_EINVAL, nothing enqueued) so the caller falls back to the mma.sync kernels."""
    eng, orc = small
    ell = 3
    mods = eng.moduli[:ell]
    if shape == "conv1":
        nci, p, H, W, M, pool, rows = 2, 3, 2, 16, 16, 1, (0, 2)
        heavy = (127 << 16) + (127 << 8) + 127       # three digits of 127: 255 * 27 * 381 < 2^22.5
        too_heavy = None                              # 27 taps cannot exceed the bound with three digits
    else:
        nci, p, H, W, M, pool, rows = 3, 16, 2, 16, 32, 0, (0, 2)
        heavy = (30 << 8) + 127                       # 255 * 144 * 157 = 5.77e6 < 2^22.5 = 5.93e6
        too_heavy = (127 << 8) + 127
    n_in = p * H * W
    x = np.empty((n_in, nci, ell, eng.N), np.uint64)
    for l, q in enumerate(mods):
        x[:, :, l, 0::2] = q - 1
        x[:, :, l, 1::2] = (1 << 40) - (1 << 32) - 1 if (1 << 40) - (1 << 32) - 1 < q else q - 2
    ins = [from_np(x[i], eng.device) for i in range(n_in)]
    wi = np.full((M, 9 * p), heavy, np.int64)
    wi[1::2] *= -1
    bres = np.array([[q - 1 for q in mods] for _ in range(M)], np.uint64)
    cst = np.array([q - 1 for q in mods], np.uint64)
    y0, y1 = rows
    got = _run(eng, eng._L.he_conv_square_sum_tc, ins, nci, p, H, W, M, pool, y0, y1, wi, bres, cst, ell)
    ref = _oracle_conv_square_sum(orc, [x[i] for i in range(n_in)], p, H, W, wi, bres, cst, pool, y0, y1)
    for k, (o, r) in enumerate(zip(got, ref)):
        assert np.array_equal(to_np(o), r), k
    if too_heavy is not None:
        import torch

        w2 = np.full((M, 9 * p), too_heavy, np.int64)
        outs = [torch.zeros((2 * nci - 1, ell, eng.N), dtype=torch.int64, device=eng.device) for _ in range(M)]
        pi, po = _ptrs(ins), _ptrs(outs)
        rc = eng._L.he_conv_square_sum_tc(eng._h, pi.ctypes.data, nci, p, H, W, po.ctypes.data, M, pool, y0, y1,
                                          w2.ctypes.data, None, None, ell, None)
        assert rc != 0 and b"too heavy" in eng._L.he_last_error()


def _rand_dev(eng, count, nci, ell, seed):
    import torch

    g = torch.Generator(device=eng.device)
    g.manual_seed(seed)
    out = torch.empty((count, nci, ell, eng.N), dtype=torch.int64, device=eng.device)
    for l, q in enumerate(eng.moduli[:ell]):
        out[:, :, l] = torch.randint(0, int(q), (count, nci, eng.N), generator=g, device=eng.device,
                                     dtype=torch.int64)
    return out


def test_convtc_conv1_shape_vs_mma_sync():
    """config 3's conv1 launch (p=3 -> 16, 32 wide, 9 limbs, N = 2^16, 20-bit weights) on a
    reduced 8-row image: tcgen05 kernel == mma.sync kernel, every output limb."""
    import torch

    from paper_2604_16834_b200.engine import GpuEngine

    eng = GpuEngine(engine_context("cfg3"))
    L = eng._L
    p, H, W, M, ell = 3, 8, 32, 16, 9
    x = _rand_dev(eng, p * H * W, 2, ell, 5)
    ins = [x[i] for i in range(p * H * W)]
    rng = np.random.default_rng(7)
    wi = rng.integers(-(1 << 20), 1 << 20, size=(M, 27), dtype=np.int64)
    bres = np.array([[int(rng.integers(0, q)) for q in eng.moduli[:ell]] for _ in range(M)], np.uint64)
    cst = np.array([int(rng.integers(0, q)) for q in eng.moduli[:ell]], np.uint64)
    for y0, y1 in ((0, 8), (2, 6)):
        got = _run(eng, L.he_conv_square_sum_tc, ins, 2, p, H, W, M, 1, y0, y1, wi, bres, cst, ell)
        old = L.he_set_conv_tc(0)
        try:
            ref = _run(eng, L.he_conv_square_sum_n, ins, 2, p, H, W, M, 1, y0, y1, wi, bres, cst, ell)
        finally:
            L.he_set_conv_tc(old)
        torch.cuda.synchronize()
        for k, (o, r) in enumerate(zip(got, ref)):
            assert torch.equal(o, r), (y0, y1, k)


def test_convtc_conv2_shape_vs_mma_sync():
    """config 3's conv2 launch (carried 3-component inputs, 16 -> 32, 16 wide, 9 limbs, N = 2^16,
    14-bit weights, global sum) on an 8-row image: tcgen05 kernel == mma.sync kernel."""
    import torch

    from paper_2604_16834_b200.engine import GpuEngine

    eng = GpuEngine(engine_context("cfg3"))
    L = eng._L
    p, H, W, M, ell = 16, 8, 16, 32, 9
    x = _rand_dev(eng, p * H * W, 3, ell, 6)
    ins = [x[i] for i in range(p * H * W)]
    rng = np.random.default_rng(9)
    wi = rng.integers(-(1 << 14), 1 << 14, size=(M, 9 * p), dtype=np.int64)
    bres = np.array([[int(rng.integers(0, q)) for q in eng.moduli[:ell]] for _ in range(M)], np.uint64)
    cst = np.array([int(rng.integers(0, q)) for q in eng.moduli[:ell]], np.uint64)
    for y0, y1 in ((0, 8), (2, 6)):
        got = _run(eng, L.he_conv_square_sum_tc, ins, 3, p, H, W, M, 0, y0, y1, wi, bres, cst, ell)
        old = L.he_set_conv_tc(0)
        try:
            ref = _run(eng, L.he_conv_square_sum_n, ins, 3, p, H, W, M, 0, y0, y1, wi, bres, cst, ell)
        finally:
            L.he_set_conv_tc(old)
        torch.cuda.synchronize()
        for k, (o, r) in enumerate(zip(got, ref)):
            assert torch.equal(o, r), (y0, y1, k)


def _planar(eng, C, H, W, ell):
    import torch

    return torch.zeros(ell * (eng.N // 8) * H * W * 1920, dtype=torch.uint8, device=eng.device)


def test_planar_pack_roundtrip(small):
    import torch

    eng, _ = small
    rng = np.random.default_rng(5)
    C, H, W, ell = 16, 3, 5, 3
    x = rand_residues(rng, eng.moduli[:ell], (C * H * W, 3), eng.N)
    ins = [from_np(x[i], eng.device) for i in range(C * H * W)]
    pl = _planar(eng, C, H, W, ell)
    assert eng._L.he_planar_pack(eng._h, _ptrs(ins).ctypes.data, C, H, W, ell, pl.data_ptr(), None) == 0
    outs = [torch.zeros_like(t) for t in ins]
    assert eng._L.he_planar_unpack(eng._h, pl.data_ptr(), C, H, W, ell, _ptrs(outs).ctypes.data, None) == 0
    for a, b in zip(ins, outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("ring", ["cfg3s", "cfg3"])
def test_planar_carry_conv2_equals_pointer_path(small, ring):
    """conv2 reading the planar carry (one bulk copy per row) == conv2 reading ciphertexts."""
    import torch

    from paper_2604_16834_b200.engine import GpuEngine

    eng = small[0] if ring == "cfg3s" else GpuEngine(engine_context("cfg3"))
    L = eng._L
    p, H, W, M = 16, 6, 16, 32
    ell = 3 if ring == "cfg3s" else 9
    x = _rand_dev(eng, p * H * W, 3, ell, 11)
    ins = [x[i] for i in range(p * H * W)]
    rng = np.random.default_rng(12)
    wi = rng.integers(-(1 << 14), 1 << 14, size=(M, 9 * p), dtype=np.int64)
    bres = np.array([[int(rng.integers(0, q)) for q in eng.moduli[:ell]] for _ in range(M)], np.uint64)
    cst = np.array([int(rng.integers(0, q)) for q in eng.moduli[:ell]], np.uint64)
    pl = _planar(eng, p, H, W, ell)
    assert L.he_planar_pack(eng._h, _ptrs(ins).ctypes.data, p, H, W, ell, pl.data_ptr(), None) == 0
    for y0, y1 in ((0, 6), (1, 4)):
        ref = _run(eng, L.he_conv_square_sum_tc, ins, 3, p, H, W, M, 0, y0, y1, wi, bres, cst, ell)
        got = [torch.zeros_like(t) for t in ref]
        rc = L.he_conv_square_sum_pl(eng._h, None, 3, p, H, W, _ptrs(got).ctypes.data, M, 0, y0, y1,
                                     wi.ctypes.data, bres.ctypes.data, cst.ctypes.data, ell, pl.data_ptr(), None,
                                     None)
        assert rc == 0, L.he_last_error()
        torch.cuda.synchronize()
        for k, (o, r) in enumerate(zip(got, ref)):
            assert torch.equal(o, r), (y0, y1, k)


@pytest.mark.parametrize("ring", ["cfg3s", "cfg3"])
def test_planar_carry_conv1_equals_pointer_path(small, ring):
    """conv1 writing the planar carry == conv1's pooled ciphertexts, packed."""
    import torch

    from paper_2604_16834_b200.engine import GpuEngine

    eng = small[0] if ring == "cfg3s" else GpuEngine(engine_context("cfg3"))
    L = eng._L
    p, H, W, M = 3, 8, 32, 16
    ell = 3 if ring == "cfg3s" else 9
    x = _rand_dev(eng, p * H * W, 2, ell, 13)
    ins = [x[i] for i in range(p * H * W)]
    rng = np.random.default_rng(14)
    wi = rng.integers(-(1 << 20), 1 << 20, size=(M, 27), dtype=np.int64)
    bres = np.array([[int(rng.integers(0, q)) for q in eng.moduli[:ell]] for _ in range(M)], np.uint64)
    cst = np.array([int(rng.integers(0, q)) for q in eng.moduli[:ell]], np.uint64)
    H2, W2 = H // 2, W // 2
    pl = _planar(eng, M, H2, W2, ell)
    for y0, y1 in ((0, 4), (4, 8)):  # two tiles filling the map
        rc = L.he_conv_square_sum_pl(eng._h, _ptrs(ins).ctypes.data, 2, p, H, W, None, M, 1, y0, y1,
                                     wi.ctypes.data, bres.ctypes.data, cst.ctypes.data, ell, None, pl.data_ptr(),
                                     None)
        assert rc == 0, L.he_last_error()
    ref = _run(eng, L.he_conv_square_sum_tc, ins, 2, p, H, W, M, 1, 0, H, wi, bres, cst, ell)  # [m][y2][x2]
    got = [torch.zeros_like(t) for t in ref]
    assert L.he_planar_unpack(eng._h, pl.data_ptr(), M, H2, W2, ell, _ptrs(got).ctypes.data, None) == 0
    torch.cuda.synchronize()
    for k, (o, r) in enumerate(zip(got, ref)):
        assert torch.equal(o, r), k
