"""Loader for the sm_100a evaluator library (libhelr_ckks.so, C ABI in
include/helr_ckks.h).

There is no CPU fallback: if the shared library is missing or cannot be
loaded, every evaluator entry point raises ``NativeLibraryError``.  Build it
with ``python -m paper_2406_13221_b200.build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
# HELR_LIB: developer knob for A/B runs of differently built variants of the
# same library (tools/build_variant.sh); never a different implementation
LIB_PATH = Path(os.environ.get("HELR_LIB") or PKG / "libhelr_ckks.so")


class NativeLibraryError(RuntimeError):
    pass


class HelrError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


_u64p = ctypes.c_void_p  # device pointers travel as integers
_vp = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64

# name -> argtypes (all return int status)
SIGNATURES = {
    "helr_ctx_create": [ctypes.POINTER(_vp), _i, _i, _i, _i, ctypes.POINTER(ctypes.c_uint64),
                        ctypes.POINTER(ctypes.c_uint64), _i, _i],
    "helr_ctx_destroy": [_vp],
    "helr_ntt_fwd": [_vp, _u64p, _i, _i, _i, _i64, _vp],
    "helr_ntt_inv": [_vp, _u64p, _i, _i, _i, _i64, _vp],
    "helr_keygen_secret": [_vp, _u64p, _u64, _vp],
    "helr_keygen_secret_hw": [_vp, _u64p, _u64, _i, _vp],
    "helr_keygen_switch": [_vp, _u64p, _i64, _u64p, _u64, _u64, _vp],
    "helr_encrypt": [_vp, _u64p, _u64p, _u64p, _i, _i, _u64, _u64, _vp],
    "helr_decrypt": [_vp, _u64p, _u64p, _i, _i, _u64p, _vp],
    "helr_encode_plain": [_vp, _u64p, _u64p, _i, _i, _vp],
    "helr_encode": [_vp, _vp, _vp, _i64, _i, ctypes.c_double, _vp, _vp],
    "helr_decode": [_vp, _vp, _i, ctypes.c_double, _vp, _vp, _i64, _vp],
    "helr_add": [_vp, _u64p, _u64p, _u64p, _i, _i, _vp],
    "helr_sub": [_vp, _u64p, _u64p, _u64p, _i, _i, _vp],
    "helr_add_const": [_vp, _u64p, _u64p, _u64p, _i, _i, _vp],
    "helr_add_plain": [_vp, _u64p, _u64p, _u64p, _i, _i, _vp],
    "helr_mul_const": [_vp, _u64p, _u64p, _u64p, _i, _i, _vp],
    "helr_mul_plain": [_vp, _u64p, _u64p, _u64p, _i, _i, _vp],
    "helr_reduce": [_vp, _u64p, _u64p, _i, _i, _vp],
    "helr_metrics": [_vp, _vp, _vp, _vp, _i, _i, _vp, ctypes.POINTER(ctypes.c_double), _vp],
    "helr_metrics_scratch": None,  # returns size_t (bound in metrics.py)
    "helr_rescale": [_vp, _u64p, _u64p, _i, _i, _vp],
    "helr_mod_raise": [_vp, _u64p, _u64p, _i, _i, _vp],
    "helr_mul_relin": [_vp, _u64p, _u64p, _u64p, _u64p, _i, _i, _vp],
    "helr_mul_relin_rescale": [_vp, _u64p, _u64p, _u64p, _u64p, _i, _i, _vp],
    "helr_imul": [_vp, _u64p, _u64p, _i, _i, _vp],
    "helr_rotate": [_vp, _u64p, _i64, _u64p, _u64p, _i, _i, _i, _vp],
    "helr_refresh": [_vp, _u64p, _u64p, _i, ctypes.c_double, _u64p, _i, _i, _u64, _u64, _vp],
    "helr_rotsum_groups": [_i, _i, ctypes.POINTER(ctypes.c_int)],
    "helr_rotsum": [_vp, _u64p, _i, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_void_p), _u64p, _i, _i, _i,
                    _vp],
    "helr_nag_iteration": None,  # bound lazily by driver.py (struct argument)
    "helr_last_error": [ctypes.c_char_p, ctypes.c_size_t],
    "helr_version": [],
}

_lib = None


def load():
    """The loaded library; raises NativeLibraryError when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryError(
            f"{LIB_PATH} is missing: build the sm_100a library first "
            "(python -m paper_2406_13221_b200.build); there is no CPU fallback")
    try:
        lib = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = ctypes.c_int
        if args is not None:
            fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    load().helr_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


def check(status: int, what: str) -> None:
    if status != 0:
        raise HelrError(f"{what} failed ({status}): {last_error()}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
