"""tcgen05 (5th-generation tensor core) building blocks on the B200.

The fused conv kernels of csrc/convtc.cu run their exact int8 digit GEMMs
through tcgen05.mma kind::i8 with accumulators in TMEM.  This test pins the
shared-memory descriptor and instruction-descriptor encodings they rely on:
D = A x B for a deterministic u8 A and s8 B, compared exactly with numpy, for
both operand layouts and every N the kernels use.
"""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _hash(x):
    x = x.astype(np.uint32)
    x ^= x >> np.uint32(16)
    x = (x * np.uint32(0x7FEB352D)).astype(np.uint32)
    x ^= x >> np.uint32(15)
    x = (x * np.uint32(0x846CA68B)).astype(np.uint32)
    x ^= x >> np.uint32(16)
    return x


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("n", [16, 32, 64, 112, 128, 192, 256])
def test_tc5_mma_i8_exact(n, layout):
    import torch

    from paper_2604_16834_b200 import _lib

    lib = _lib.load()
    out = torch.zeros((128, n), dtype=torch.int32, device="cuda")
    _lib.check(lib.he_tc5_selftest(0, n, layout, out.data_ptr()), "he_tc5_selftest")
    a = (_hash(np.arange(128 * 64, dtype=np.uint64)) & 0xFF).astype(np.int64).reshape(128, 64)
    b = (_hash(np.uint32(0x9E3779B9) + np.arange(n * 64, dtype=np.uint32)) & 0xFF).astype(np.uint8)
    b = b.view(np.int8).astype(np.int64).reshape(n, 64)
    ref = a @ b.T
    assert np.array_equal(out.cpu().numpy().astype(np.int64), ref)


def test_tc5_rate_report():
    from paper_2604_16834_b200 import _lib

    lib = _lib.load()
    for n in (16, 32, 64, 112, 128, 256):
        r = np.zeros(2)
        _lib.check(lib.he_microbench_tc5(0, n, r.ctypes.data), "he_microbench_tc5")
        print(f"tcgen05 kind::i8 M=128 N={n}: {r[0] / 1e12:.1f} TMAC/s, {r[1]:.1f} cycles/MMA")
        assert r[0] > 0
        for nd in (2, 4, 8):
            if nd * n <= 256:
                _lib.check(lib.he_microbench_tc5_indep(0, n, nd, r.ctypes.data), "he_microbench_tc5_indep")
                print(f"  {nd} independent accumulators: {r[0] / 1e12:.1f} TMAC/s, {r[1]:.1f} cycles/MMA")


def test_tmem_read_rate_report():
    from paper_2604_16834_b200 import _lib

    lib = _lib.load()
    for warps in (4, 8, 16, 32):
        for cols in (4, 8, 16):
            r = np.zeros(2)
            _lib.check(lib.he_microbench_tmem_ld(0, warps, cols, r.ctypes.data), "he_microbench_tmem_ld")
            print(f"TMEM read {warps} warps 32x32b.x{cols}: {r[0]:.1f} B/cycle/SM")
            assert r[0] > 0
