"""The five BASELINE.json configurations as engine contexts + workloads.

Appendix decisions of SURVEY.md (recorded in DESIGN.md section 3):
  * config 1: Q = 60 + 4x40 bits, P = 1x60, key_switch_digits 5 (alpha = 1),
    bootstrap_reserve = 1 (the reference default 10 violates 0 < r < max_level).
  * config 3: Q = 14x40, P = 3x42, digits 5 (alpha = 3), scale 2^40: every prime
    below 2^42, so every NTT / BConv / inner product runs on the FP64 path
    (DESIGN.md section 3); P = 2^126 exceeds every 3-limb digit (2^120).
  * configs 2 and 4: Q = 24x50, P = 4x50, digits 6 (alpha = 4), scale 2^50.
  * config 4 head: GAP then dense 64 -> 10.  Biases: zero everywhere.
"""

from __future__ import annotations

from .engine import EngineContext
from .featuremajor import Activation, CnnSpec, MlpSpec


def context(cfg: int, seed: int = 0, device: int = 0) -> EngineContext:
    if cfg == 1:
        return EngineContext(n=2048, max_level=4, bootstrap_reserve=1, first_modulus_bits=60, rescale_bits=40,
                             key_switch_digits=5, noise_seed=seed, special_prime_bits=(60,), scale_bits=40,
                             device=device)
    if cfg in (2, 4):
        return EngineContext(n=32768, max_level=23, bootstrap_reserve=1, first_modulus_bits=50, rescale_bits=50,
                             key_switch_digits=6, noise_seed=seed, special_prime_bits=(50,) * 4, scale_bits=50,
                             device=device)
    if cfg in (3, 5):
        return EngineContext(n=32768, max_level=13, bootstrap_reserve=1, first_modulus_bits=40, rescale_bits=40,
                             key_switch_digits=5, noise_seed=seed, special_prime_bits=(42,) * 3, scale_bits=40,
                             device=device)
    raise ValueError(f"unknown config {cfg}")


def boot_context(seed: int = 0, device: int = 0) -> EngineContext:
    """The bootstrapping ring (no BASELINE config bootstraps; engine.bootstrap,
    bootstrap.py): N = 2^16, q_0 of 60 bits + 25 x 50-bit rescale primes at scale
    2^50, 4 x 60-bit special primes (dnum 7), sparse secret of expected Hamming
    weight 128.  The circuit takes 20 levels (bootstrap_reserve), leaving 5."""
    return EngineContext(n=32768, max_level=25, bootstrap_reserve=20, first_modulus_bits=60, rescale_bits=50,
                         key_switch_digits=7, noise_seed=seed, special_prime_bits=(60,) * 4, scale_bits=50,
                         secret_hamming=128, device=device)


MLP1 = MlpSpec(sizes=(64, 32, 10), act=Activation((0.0, 0.0, 1.0)))
CNN3 = CnnSpec(channels=(3, 16, 32), H=32, W=32, act=Activation((0.25, 0.5, 0.125)), pool_after=(0,))
CNN4 = CnnSpec(channels=(3, 16, 32, 64, 64), H=32, W=32, act=Activation((0.5, 0.5, 0.0, 0.0625)),
               pool_after=(1, 3))

SAMPLES = {1: 2048, 3: 32768, 4: 32768, 5: 8 * 32768}
