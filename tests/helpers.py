"""Shared test helpers: parameter sets and GPU<->oracle plumbing."""

from __future__ import annotations

import numpy as np

# name -> (log_n, q_bits, p_bits, alpha, scale_bits)
PARAMS = {
    "tiny": (5, (60, 40, 40, 40), (60, 60), 2, 40),
    "cfg1": (12, (60, 40, 40, 40, 40), (60,), 1, 40),
    "cfg2": (16, (50,) * 24, (50,) * 4, 4, 50),
    "cfg3": (16, (40,) * 14, (42,) * 3, 3, 40),
    "cfg4": (16, (50,) * 24, (50,) * 4, 4, 50),
    # config 4's prime sizes on a small ring (degree-3 CNN tests on one GPU)
    "cfg4s": (12, (50,) * 10, (50,) * 2, 2, 50),
    # config 3's prime sizes on a small ring (tcgen05 conv kernels vs the oracle)
    "cfg3s": (12, (40,) * 6, (42,) * 2, 3, 40),
    # the paper's pipeline-1 ring degree (N = 2^15, 46-bit rescale primes): the split
    # global-stage + shared-memory NTT (ntt.cu ntt_big) and the generic key switch
    "p15": (15, (60, 46, 46, 46, 46, 46), (60, 60), 2, 46),
    # config 3's 9-limb carry plan (inputs at 9 of 14 limbs) on a 64-point ring (CPU tests)
    "carry9": (6, (40,) * 9, (42,) * 3, 3, 40),
    # bootstrapping rings (bootstrap.py): q_0 of 60 bits over 50-bit rescale primes at
    # scale 2^50 (q_0 / scale = 2^10); depth 15 at N = 64, 18 at N = 2^11 / 2^12
    "boot6": (6, (60,) + (50,) * 16, (60,) * 3, 3, 50),
    "boot11": (11, (60,) + (50,) * 22, (60,) * 3, 3, 50),
    "boot12": (12, (60,) + (50,) * 22, (60,) * 3, 3, 50),
    # sparse secret (expected Hamming weight 64, 6th field): K ~ 18, r = 7
    "boot11s": (11, (60,) + (50,) * 22, (60,) * 3, 3, 50, 64),
    # the config-2/4 ring degree with a sparse secret (h = 128): depth 20 of 25 levels
    "boot16s": (16, (60,) + (50,) * 25, (60,) * 4, 4, 50, 128),
}


def engine_context(name, seed=1, bootstrap_reserve=1):
    from paper_2604_16834_b200.engine import EngineContext

    log_n, qb, pb, alpha, sb, *rest = PARAMS[name]
    L = len(qb)
    return EngineContext(secret_hamming=rest[0] if rest else 0, n=1 << (log_n - 1), max_level=L - 1, bootstrap_reserve=bootstrap_reserve,
                         first_modulus_bits=qb[0],
                         rescale_bits=qb[-1] if L > 1 else qb[0], key_switch_digits=-(-L // alpha),
                         noise_seed=seed, special_prime_bits=tuple(pb), scale_bits=sb, q_bits=tuple(qb))


def oracle_for(name, seed=1):
    import oracle as O

    log_n, qb, pb, alpha, sb, *rest = PARAMS[name]
    return O.Oracle(log_n, list(qb), list(pb), alpha, seed=seed, scale=2.0 ** sb, sk_hamming=rest[0] if rest else 0)


def to_np(t):
    """torch int64 cuda tensor -> numpy uint64 (same bits)."""
    return t.detach().cpu().numpy().view(np.uint64)


def from_np(a, device):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(device)


def rand_residues(rng, moduli, shape_prefix, N):
    """uniform residues: array [*shape_prefix, len(moduli), N]"""
    out = np.empty(tuple(shape_prefix) + (len(moduli), N), np.uint64)
    for i, q in enumerate(moduli):
        out[..., i, :] = rng.integers(0, q, size=tuple(shape_prefix) + (N,), dtype=np.uint64)
    return out
