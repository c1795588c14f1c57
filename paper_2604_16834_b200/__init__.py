"""B200-native batched RNS-CKKS engine for encrypted inference (arXiv 2604.16834).

Drop-in for the hot path of the reference package ``hebatch``: the same
``EngineContext`` / ``VectorEngine`` / ``pack_inputs`` / ``conv_forward`` /
``unpack_outputs`` API, backed by hand-written sm_100a CUDA kernels in
``libhe_sm100.so`` (C-ABI: include/he_sm100.h) instead of float64 slot
simulation.  See DESIGN.md.
"""

import os as _os
import sys as _sys

# Ciphertext tensors come from torch; kernel scratch comes from cudaMallocAsync
# inside libhe_sm100.so.  Both must draw on the SAME stream-ordered pool, or
# memory freed by one is invisible to the other (config 3 peaks at ~135 GB).
# torch fixes its allocator backend when it is imported, so this only takes
# effect if the package is imported first (bench.py / conftest set it too).
if "torch" not in _sys.modules:
    _os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")

from .errors import HebatchError  # noqa: E402,F401

__version__ = "0.1.0"


def __getattr__(name):
    # lazy: importing the package must not require torch / a GPU (CPU tests)
    if name in ("EngineContext", "GpuEngine", "CipherVec", "PlainVec", "OpCounters", "RotationKeySet",
                "VectorEngine"):
        from . import engine

        return getattr(engine, name)
    raise AttributeError(name)
