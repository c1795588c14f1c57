"""CKKS bootstrapping on the B200 engine vs the CPU oracle.

Reference contract (/root/reference/pkg/src/hebatch/engine.py:315-327,
SPEC.md:94-98): bootstrap keeps the slots, resets the level to
max_level - bootstrap_reserve and advances only the ``bootstraps`` counter;
ensure_level bootstraps (and releases) a ciphertext below the needed level.

Parity: the two new kernels (complex plaintext encoding, ModRaise) are
compared with the oracle bit for bit, and the whole GPU bootstrap is compared
limb for limb with the same circuit (paper_2604_16834_b200/bootstrap.py) run
on the oracle backend (tests/oracle_boot.py: every op an oracle call).
"""

from __future__ import annotations

import time

import numpy as np
import pytest

from helpers import engine_context, from_np, oracle_for, rand_residues, to_np

pytestmark = pytest.mark.gpu


def _depth(name):
    """The circuit's depth on ring `name` (= the bootstrap_reserve the tests use)."""
    from helpers import PARAMS
    from paper_2604_16834_b200.bootstrap import BootPlan

    spec = PARAMS[name]
    return BootPlan(N=1 << spec[0], q0=1, hamming=spec[5] if len(spec) > 5 else 0).depth


def _engine(name, reserve=1):
    from paper_2604_16834_b200.engine import GpuEngine

    return GpuEngine(engine_context(name, bootstrap_reserve=reserve))


def _boot_engine(name):
    return _engine(name, _depth(name))


@pytest.mark.parametrize("name", ["cfg1", "boot11"])
def test_encode_plain_complex_bit_exact(name):
    import torch

    eng, orc = _engine(name), oracle_for(name)
    rng = np.random.default_rng(71)
    n, L = eng.context.n, eng.context.n_q
    z = rng.uniform(-1, 1, (3, n)) + 1j * rng.uniform(-1, 1, (3, n))
    scale = float(eng.moduli[L - 1]) * 2.0 ** 7
    re = torch.as_tensor(np.ascontiguousarray(z.real), device=eng.device)
    im = torch.as_tensor(np.ascontiguousarray(z.imag), device=eng.device)
    pt = torch.empty((3, L, eng.N), dtype=torch.int64, device=eng.device)
    assert eng._L.he_encode_plain_batch_c(eng._h, re.data_ptr(), im.data_ptr(), 3, n, scale, L, pt.data_ptr(),
                                          None) == 0
    torch.cuda.synchronize()
    got = to_np(pt)
    for i in range(3):
        assert np.array_equal(got[i], orc.plain_to_ntt(orc.encode_complex(z[i], scale), L)), i


@pytest.mark.parametrize("name", ["cfg1", "boot11", "cfg3"])
def test_mod_raise_bit_exact(name):
    import torch

    from paper_2604_16834_b200 import _lib

    eng, orc = _engine(name), oracle_for(name)
    rng = np.random.default_rng(72)
    L = eng.context.n_q
    ell_in = min(3, L)
    x = rand_residues(rng, eng.moduli[:ell_in], (2, 2), eng.N)              # [ct][comp][limb][N]
    ins = [from_np(x[i], eng.device) for i in range(2)]
    outs = [torch.zeros((2, L, eng.N), dtype=torch.int64, device=eng.device) for _ in range(2)]
    pi = _lib.ptr_array([t.data_ptr() for t in ins])
    po = _lib.ptr_array([t.data_ptr() for t in outs])
    assert eng._L.he_mod_raise(eng._h, _lib.addr(pi), ell_in, _lib.addr(po), 2, L, None) == 0, eng._L.he_last_error()
    torch.cuda.synchronize()
    for i in range(2):
        assert np.array_equal(to_np(outs[i]), orc.mod_raise(x[i], L)), i


@pytest.mark.parametrize("name", ["boot11", "boot11s"])
def test_bootstrap_bit_exact_vs_oracle_circuit_and_contract(name):
    from oracle_boot import OCt, OracleBootOps
    from paper_2604_16834_b200.bootstrap import Bootstrapper

    eng, orc = _boot_engine(name), oracle_for(name)
    rng = np.random.default_rng(73)
    x = rng.uniform(-1, 1, eng.context.n)
    ct = eng.encrypt_batch(x[None])[0]
    before, live = eng.snapshot_counters(), eng.live_ciphertexts
    out = eng.bootstrap(ct)
    after = eng.snapshot_counters()
    # the reference's contract (engine.py:315-319)
    assert out.level == eng.context.max_level - eng.context.bootstrap_reserve
    assert after.bootstraps == before.bootstraps + 1
    for f in ("rotations", "plain_mults", "ct_mults", "adds", "key_loads"):
        assert getattr(after, f) == getattr(before, f), f
    assert eng.live_ciphertexts == live + 1
    err = np.max(np.abs(eng.decrypt(out) - x))
    assert err < 1e-4, err
    # limb for limb against the same circuit on the oracle
    plan = eng.boot_plan()
    src = to_np(ct.data)
    ref = Bootstrapper(OracleBootOps(orc), plan, ct.scale).run([OCt(src[:, :1], ct.scale)], eng.context.n_q)[0]
    assert ref.level == out.level and ref.scale == out.scale
    assert np.array_equal(to_np(out.data), ref.data)


@pytest.mark.parametrize("name", ["boot12", "boot16s"])
def test_bootstrap_precision_ensure_level_and_products(name):
    eng = _boot_engine(name)
    reserve = eng.context.bootstrap_reserve
    rng = np.random.default_rng(74)
    x = rng.uniform(-1, 1, eng.context.n)
    ct = eng.encrypt_batch(x[None])[0]
    low = eng.drop_level_batch([ct], 0)[0]
    t0 = time.perf_counter()
    eng.bootstrap(low)  # keys, DFT plans
    eng.synchronize()
    first = (time.perf_counter() - t0) * 1e3
    reps = 3
    t0 = time.perf_counter()
    for _ in range(reps):
        out = eng.bootstrap(low)
    eng.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / reps
    err = np.max(np.abs(eng.decrypt(out) - x))
    plan = eng.boot_plan()
    print(f"\nbootstrap N=2^{eng.context.log_n} ({eng.context.n} slots, {eng.context.n_q} limbs, h={plan.hamming}, "
          f"depth {plan.depth}, r={plan.r}, {len(plan.rotation_offsets())} rotation keys): {ms:.1f} ms "
          f"(first call {first:.0f} ms incl. keygen), max|err| = {err:.2e}")
    assert err < 1e-4, err
    # the refreshed ciphertext computes: x^2 at the restored level
    sq = eng.mult_ct(out, out)
    assert np.max(np.abs(eng.decrypt(sq) - x * x)) < 2e-4
    # ensure_level: bootstraps (and releases) only below the needed level
    n0 = eng.snapshot_counters().bootstraps
    same = eng.ensure_level(out, out.level)
    assert same is out and eng.snapshot_counters().bootstraps == n0
    fresh = eng.ensure_level(low, 1)
    assert fresh.level == eng.context.max_level - reserve
    assert eng.snapshot_counters().bootstraps == n0 + 1
    assert np.max(np.abs(eng.decrypt(fresh) - x)) < 1e-4


def test_bootstrap_batch_equals_single_bootstraps():
    """bootstrap_batch: one launch sequence for several ciphertexts, each result
    bit-identical to its own bootstrap (N = 2^11, sparse secret)."""
    name = "boot11s"
    eng = _boot_engine(name)
    rng = np.random.default_rng(75)
    xs = rng.uniform(-1, 1, (3, eng.context.n))
    cts = eng.encrypt_batch(xs)
    n0 = eng.snapshot_counters().bootstraps
    outs = eng.bootstrap_batch(cts)
    assert eng.snapshot_counters().bootstraps == n0 + 3
    for i, c in enumerate(cts):
        single = eng.bootstrap(c)
        assert np.array_equal(to_np(outs[i].data), to_np(single.data)) and outs[i].scale == single.scale
        assert np.max(np.abs(eng.decrypt(outs[i]) - xs[i])) < 1e-4
