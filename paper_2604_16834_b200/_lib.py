"""ctypes binding of libhe_sm100.so (the C-ABI declared in include/he_sm100.h).

There is no CPU fallback: if the shared library is missing or cannot be
loaded, every entry point raises.  Build it with ``make -C
paper_2604_16834_b200/csrc`` or ``python -c "import __graft_entry__ as g;
g.build()"``.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import (
    ContextMismatch,
    HebatchError,
    LengthExceedsSlots,
    LevelExhausted,
    MissingRotationKey,
)

LIB_PATH = os.environ.get("HE_SM100_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhe_sm100.so")

HE_OK, HE_EINVAL, HE_ECUDA, HE_ENOKEY, HE_ELEVEL, HE_ENOMEM, HE_ECONTEXT, HE_ELENGTH = 0, -1, -2, -3, -4, -5, -6, -7

# every symbol include/he_sm100.h declares (tests check the .so exports them all)
EXPORTS = [
    "he_last_error", "he_abi_version", "he_ctx_create", "he_ctx_destroy", "he_ctx_moduli",
    "he_gen_switch_key", "he_drop_switch_key", "he_has_switch_key", "he_export_secret_key",
    "he_export_switch_key", "he_import_switch_key", "he_lincomb_plain", "he_encode_plain_batch", "he_encode_plain_batch_c", "he_mod_raise", "he_ntt", "he_encrypt", "he_encrypt_level", "he_decrypt", "he_decrypt_coeffs",
    "he_encode_plain", "he_add", "he_sub", "he_add_const", "he_mul_const", "he_mul_plain",
    "he_drop_limbs", "he_tensor", "he_relin", "he_keyswitch", "he_rescale", "he_mult_ct",
    "he_automorphism", "he_rotate", "he_lincomb", "he_sync", "he_launch_count", "he_lincomb_grouped",
    "he_microbench_intpipe", "he_square_sum", "he_conv_mma", "he_relin_rescale", "he_relin_rescale_n", "he_conv_square_sum", "he_conv_square_sum_n",
    "he_microbench_fp64",
    "he_microbench_imma",
    "he_tc5_selftest",
    "he_microbench_tc5",
    "he_microbench_tc5_strided",
    "he_microbench_tc5_indep",
    "he_microbench_tmem_ld",
    "he_conv_square_sum_tc",
    "he_set_conv_tc",
    "he_convtc_profile",
    "he_conv_square_sum_pl",
    "he_planar_pack",
    "he_planar_unpack",
    "he_rotate_hoisted",
    "he_gen_hoist_key",
]


class HeParams(C.Structure):
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


class HeCudaError(HebatchError):
    """A CUDA runtime or allocation failure inside libhe_sm100.so."""


_lib = None


def load():
    """Load the library (raises OSError/HebatchError if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise HebatchError(
            f"{LIB_PATH} is missing: the sm_100a engine has no CPU fallback. "
            "Build it with `make -C paper_2604_16834_b200/csrc`."
        )
    L = C.CDLL(LIB_PATH)
    vp, i, u32, u64, dbl = C.c_void_p, C.c_int, C.c_uint32, C.c_uint64, C.c_double
    pp = C.c_void_p  # host array of device pointers (passed as address)
    sig = {
        "he_last_error": (C.c_char_p, []),
        "he_abi_version": (i, []),
        "he_ctx_create": (i, [C.POINTER(HeParams), i, C.POINTER(vp)]),
        "he_ctx_destroy": (i, [vp]),
        "he_ctx_moduli": (i, [vp, vp, vp]),
        "he_gen_switch_key": (i, [vp, u32, vp]),
        "he_drop_switch_key": (i, [vp, u32]),
        "he_has_switch_key": (i, [vp, u32]),
        "he_export_secret_key": (i, [vp, vp, vp]),
        "he_export_switch_key": (i, [vp, u32, vp, vp]),
        "he_import_switch_key": (i, [vp, u32, vp, vp]),
        "he_lincomb_plain": (i, [vp, vp, i, vp, vp, i, i, vp]),
        "he_encode_plain_batch": (i, [vp, vp, i, i, dbl, i, vp, vp]),
        "he_encode_plain_batch_c": (i, [vp, vp, vp, i, i, dbl, i, vp, vp]),
        "he_mod_raise": (i, [vp, pp, i, pp, i, i, vp]),
        "he_ntt": (i, [vp, vp, i, i, i, vp]),
        "he_encrypt": (i, [vp, vp, i, i, dbl, u32, pp, vp]),
        "he_encrypt_level": (i, [vp, vp, i, i, dbl, u32, i, pp, vp]),
        "he_decrypt": (i, [vp, pp, i, i, vp, vp, vp]),
        "he_decrypt_coeffs": (i, [vp, pp, i, i, vp, vp]),
        "he_encode_plain": (i, [vp, vp, i, dbl, i, vp, vp]),
        "he_add": (i, [vp, pp, pp, pp, i, i, i, vp]),
        "he_sub": (i, [vp, pp, pp, pp, i, i, i, vp]),
        "he_add_const": (i, [vp, pp, pp, i, i, i, vp, vp]),
        "he_mul_const": (i, [vp, pp, pp, i, i, i, vp, vp]),
        "he_mul_plain": (i, [vp, pp, vp, pp, i, i, i, vp]),
        "he_drop_limbs": (i, [vp, pp, pp, i, i, i, i, vp]),
        "he_tensor": (i, [vp, pp, pp, pp, i, i, vp]),
        "he_relin": (i, [vp, pp, pp, i, i, vp]),
        "he_relin_rescale": (i, [vp, pp, pp, i, i, i, vp]),
        "he_relin_rescale_n": (i, [vp, pp, pp, i, i, i, i, vp]),
        "he_keyswitch": (i, [vp, u32, pp, pp, pp, i, i, vp]),
        "he_rescale": (i, [vp, pp, pp, i, i, i, vp]),
        "he_mult_ct": (i, [vp, pp, pp, pp, i, i, vp]),
        "he_automorphism": (i, [vp, u32, pp, pp, i, i, i, vp]),
        "he_rotate": (i, [vp, u32, pp, pp, i, i, vp]),
        "he_lincomb": (i, [vp, pp, i, pp, i, vp, vp, vp, i, i, vp]),
        "he_sync": (i, [vp]),
        "he_launch_count": (C.c_ulonglong, []),
        "he_lincomb_grouped": (i, [vp, pp, i, pp, i, i, vp, vp, vp, vp, i, i, i, vp, vp, i, i, vp]),
        "he_microbench_intpipe": (i, [i, vp]),
        "he_microbench_fp64": (i, [i, vp]),
        "he_microbench_imma": (i, [i, vp]),
        "he_tc5_selftest": (i, [i, i, i, vp]),
        "he_microbench_tc5": (i, [i, i, vp]),
        "he_microbench_tc5_strided": (i, [i, i, i, i, vp]),
        "he_microbench_tc5_indep": (i, [i, i, i, vp]),
        "he_microbench_tmem_ld": (i, [i, i, i, vp]),
        "he_conv_square_sum_tc": (i, [vp, vp, i, i, i, i, vp, i, i, i, i, vp, vp, vp, i, vp]),
        "he_set_conv_tc": (i, [i]),
        "he_convtc_profile": (i, [i, vp]),
        "he_conv_square_sum_pl": (i, [vp, vp, i, i, i, i, vp, i, i, i, i, vp, vp, vp, i, vp, vp, vp]),
        "he_planar_pack": (i, [vp, vp, i, i, i, i, vp, vp]),
        "he_planar_unpack": (i, [vp, vp, i, i, i, i, vp, vp]),
        "he_rotate_hoisted": (i, [vp, vp, i, pp, pp, i, i, vp]),
        "he_gen_hoist_key": (i, [vp, u32, vp]),
        "he_square_sum": (i, [vp, pp, i, pp, i, vp, vp, vp, i, vp]),
        "he_conv_mma": (i, [vp, pp, i, pp, i, i, vp, vp, i, i, i, vp, vp, i, i, vp]),
        "he_conv_square_sum": (i, [vp, pp, i, i, i, pp, i, i, i, i, vp, vp, vp, i, vp]),
        "he_conv_square_sum_n": (i, [vp, pp, i, i, i, i, pp, i, i, i, i, vp, vp, vp, i, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    if L.he_abi_version() != 2:  # 2: he_params.sk_hamming
        raise HebatchError("libhe_sm100.so ABI version mismatch")
    _lib = L
    return L


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI status code onto the reference's exception classes."""
    if rc == HE_OK:
        return
    msg = (load().he_last_error() or b"").decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == HE_ENOKEY:
        raise MissingRotationKey(-1) if not msg else _missing(msg)
    if rc == HE_ELEVEL:
        raise LevelExhausted(msg)
    if rc == HE_ECONTEXT:
        raise ContextMismatch(msg)
    if rc == HE_ELENGTH:
        raise LengthExceedsSlots(msg)
    if rc in (HE_ECUDA, HE_ENOMEM):
        raise HeCudaError(msg)
    raise HebatchError(msg)


def _missing(msg: str) -> HebatchError:
    e = MissingRotationKey(-1)
    e.args = (msg,)
    return e


def ptr_array(ptrs) -> np.ndarray:
    """Host uint64 array of device addresses (keep it alive across the call)."""
    return np.ascontiguousarray(np.asarray(ptrs, dtype=np.uint64))


def addr(a: np.ndarray) -> int:
    return a.ctypes.data
