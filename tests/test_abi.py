"""The C-ABI library loads (no GPU needed) and exports exactly what
include/he_sm100.h declares; the product path refuses to run without it."""

from __future__ import annotations

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "he_sm100.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(he_[a-z0-9_]+)\s*\(", src))


def test_header_and_binding_list_agree():
    from paper_2604_16834_b200 import _lib

    assert _declared() == set(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    from paper_2604_16834_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libhe_sm100.so not built (run __graft_entry__.build())")
    lib = _lib.load()
    for name in _lib.EXPORTS:
        assert hasattr(lib, name), name
    assert lib.he_abi_version() == 2
    assert lib.he_launch_count() >= 0


def test_bad_arguments_fail_before_any_device_work():
    """Argument validation is host-side and returns typed codes (no GPU used)."""
    from paper_2604_16834_b200 import _lib
    from paper_2604_16834_b200.errors import HebatchError

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = _lib.load()
    assert lib.he_ntt(None, None, 1, 1, 0, None) == _lib.HE_EINVAL
    with pytest.raises(HebatchError):
        _lib.check(lib.he_add(None, None, None, None, 1, 1, 2, None), "add")


def test_engine_fails_loudly_without_gpu():
    import torch

    from paper_2604_16834_b200 import configs
    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.errors import HebatchError

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(HebatchError):
        GpuEngine(configs.context(1))
