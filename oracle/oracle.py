"""ctypes binding of the CPU RNS-CKKS oracle (ckks_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs use it as the checker / CPU baseline.  The product package
never imports this module.

All buffers are numpy uint64 arrays in the layouts documented in
include/helr_ckks.h (ciphertext u64[2][L][N], key u64[beta][2][L+K][N]).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libckks_oracle.so"

_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_intp = ctypes.POINTER(ctypes.c_int)


def build(force: bool = False) -> Path:
    src = HERE / "ckks_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        vp = ctypes.c_void_p
        sig = {
            "oc_create": (vp, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _u64p, _u64p, ctypes.c_int]),
            "oc_destroy": (None, [vp]),
            "oc_beta": (ctypes.c_int, [vp]),
            "oc_alpha": (ctypes.c_int, [vp]),
            "oc_prng": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]),
            "oc_ntt": (None, [vp, _u64p, ctypes.c_int]),
            "oc_intt": (None, [vp, _u64p, ctypes.c_int]),
            "oc_ntt_batch": (None, [vp, _u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int]),
            "oc_keygen_secret": (None, [vp, ctypes.c_uint64, _u64p]),
            "oc_keygen_secret_hw": (None, [vp, ctypes.c_uint64, ctypes.c_int, _u64p]),
            "oc_secret_coeffs": (None, [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, _i64p]),
            "oc_keygen_switch": (None, [vp, _u64p, ctypes.c_int64, _u64p, ctypes.c_uint64, ctypes.c_uint64]),
            "oc_encrypt": (None, [vp, _u64p, _i64p, _u64p, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64]),
            "oc_decrypt": (None, [vp, _u64p, _u64p, ctypes.c_int, ctypes.c_int, _i64p]),
            "oc_encode_plain": (None, [vp, _i64p, _u64p, ctypes.c_int, ctypes.c_int]),
            "oc_add": (None, [vp, _u64p, _u64p, _u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
            "oc_add_const": (None, [vp, _u64p, _u64p, _u64p, ctypes.c_int, ctypes.c_int]),
            "oc_add_plain": (None, [vp, _u64p, _u64p, _u64p, ctypes.c_int, ctypes.c_int]),
            "oc_mul_const": (None, [vp, _u64p, _u64p, _u64p, ctypes.c_int, ctypes.c_int]),
            "oc_mul_plain": (None, [vp, _u64p, _u64p, _u64p, ctypes.c_int, ctypes.c_int]),
            "oc_imul": (None, [vp, _u64p, _u64p, ctypes.c_int, ctypes.c_int]),
            "oc_rescale": (None, [vp, _u64p, _u64p, ctypes.c_int, ctypes.c_int]),
            "oc_basis_convert": (None, [vp, _u64p, _intp, ctypes.c_int, _u64p, _intp, ctypes.c_int]),
            "oc_keyswitch": (None, [vp, _u64p, _u64p, ctypes.c_int, _u64p, _u64p]),
            "oc_rotsum": (None, [vp, _u64p, ctypes.c_int, _i64p, ctypes.POINTER(_u64p), _u64p, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_int]),
            "oc_relin_rescale_tensor": (None, [vp, _u64p, _u64p, _u64p, ctypes.c_int]),
            "oc_mul_relin_rescale": (None, [vp, _u64p, _u64p, _u64p, _u64p, ctypes.c_int, ctypes.c_int]),
            "oc_tensor": (None, [vp, _u64p, _u64p, _u64p, ctypes.c_int]),
            "oc_mul_relin": (None, [vp, _u64p, _u64p, _u64p, _u64p, ctypes.c_int, ctypes.c_int]),
            "oc_automorph": (None, [vp, _u64p, _u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int64]),
            "oc_rotate": (None, [vp, _u64p, ctypes.c_int64, _u64p, _u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
            "oc_mod_raise": (None, [vp, _u64p, _u64p, ctypes.c_int, ctypes.c_int]),
            "oc_refresh": (None, [vp, _u64p, _u64p, ctypes.c_int, ctypes.c_double, _u64p, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle buffers must be C-contiguous"
    if a.dtype == np.uint64:
        return a.ctypes.data_as(_u64p)
    if a.dtype == np.int64:
        return a.ctypes.data_as(_i64p)
    if a.dtype == np.intc:
        return a.ctypes.data_as(_intp)
    raise TypeError(a.dtype)


def prng(seed: int, stream: int, ctr: int) -> int:
    return int(lib().oc_prng(seed, stream, ctr))


class Oracle:
    """CPU evaluator over the same ring as the device library."""

    def __init__(self, params, threads: int | None = None):
        if threads is not None:
            os.environ["OMP_NUM_THREADS"] = str(threads)
        self.params = params
        self.N = params.n
        self.L = params.L
        self.K = params.K
        pr = np.array(params.primes, dtype=np.uint64)
        ps = np.array(params.psi, dtype=np.uint64)
        self._h = lib().oc_create(params.log_n, params.L, params.K, params.dnum, _p(pr), _p(ps), params.cbd_eta)
        if not self._h:
            raise ValueError("oracle context creation failed")
        self.beta = lib().oc_beta(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.oc_destroy(h)
            self._h = None

    # shapes
    def ct_zeros(self, count: int = 1) -> np.ndarray:
        return np.zeros((count, 2, self.L, self.N), dtype=np.uint64)

    def key_zeros(self) -> np.ndarray:
        return np.zeros((self.beta, 2, self.L + self.K, self.N), dtype=np.uint64)

    # ring
    def ntt(self, a: np.ndarray, prime: int, inverse: bool = False) -> np.ndarray:
        out = np.ascontiguousarray(a, dtype=np.uint64).copy()
        (lib().oc_intt if inverse else lib().oc_ntt)(self._h, _p(out), prime)
        return out

    def ntt_batch(self, data: np.ndarray, first: int, n_limbs: int, inverse: bool = False) -> np.ndarray:
        out = np.ascontiguousarray(data, dtype=np.uint64).copy()
        count = out.shape[0]
        stride = out[0].size
        lib().oc_ntt_batch(self._h, _p(out), first, n_limbs, count, stride, 1 if inverse else 0)
        return out

    # keys
    def keygen_secret(self, seed: int, hw: int = 0) -> np.ndarray:
        """NTT-form secret over every prime; hw = 0 uniform ternary, else
        exactly hw nonzero +-1 coefficients."""
        sk = np.zeros((self.L + self.K, self.N), dtype=np.uint64)
        lib().oc_keygen_secret_hw(self._h, seed, hw, _p(sk))
        return sk

    def secret_coeffs(self, seed: int, hw: int = 0) -> np.ndarray:
        s = np.zeros(self.N, dtype=np.int64)
        lib().oc_secret_coeffs(seed, self.N, hw, _p(s))
        return s

    def keygen_switch(self, sk, galois: int, seed: int, key_id: int) -> np.ndarray:
        evk = self.key_zeros()
        lib().oc_keygen_switch(self._h, _p(sk), galois, _p(evk), seed, key_id)
        return evk

    # encryption
    def encrypt(self, sk, msg: np.ndarray, level: int, seed: int, first_id: int) -> np.ndarray:
        msg = np.ascontiguousarray(np.atleast_2d(msg), dtype=np.int64)
        ct = self.ct_zeros(msg.shape[0])
        lib().oc_encrypt(self._h, _p(sk), _p(msg), _p(ct), msg.shape[0], level, seed, first_id)
        return ct

    def decrypt(self, sk, ct: np.ndarray, level: int) -> np.ndarray:
        ct = np.ascontiguousarray(ct.reshape(-1, 2, self.L, self.N))
        out = np.zeros((ct.shape[0], self.N), dtype=np.int64)
        lib().oc_decrypt(self._h, _p(sk), _p(ct), ct.shape[0], level, _p(out))
        return out

    def encode_plain(self, msg: np.ndarray, level: int) -> np.ndarray:
        msg = np.ascontiguousarray(np.atleast_2d(msg), dtype=np.int64)
        pt = np.zeros((msg.shape[0], self.L, self.N), dtype=np.uint64)
        lib().oc_encode_plain(self._h, _p(msg), _p(pt), msg.shape[0], level)
        return pt

    # arithmetic; all take/return u64[count][2][L][N]
    def _out(self, a):
        return np.zeros_like(a)

    def add(self, a, b, level, sub=False):
        out = self._out(a)
        lib().oc_add(self._h, _p(a), _p(b), _p(out), a.shape[0], level, 1 if sub else 0)
        return out

    def add_const(self, a, c, level):
        out = self._out(a)
        lib().oc_add_const(self._h, _p(a), _p(np.ascontiguousarray(c, dtype=np.uint64)), _p(out), a.shape[0], level)
        return out

    def add_plain(self, a, pt, level):
        out = self._out(a)
        lib().oc_add_plain(self._h, _p(a), _p(np.ascontiguousarray(pt)), _p(out), a.shape[0], level)
        return out

    def mul_const(self, a, c, level):
        out = self._out(a)
        lib().oc_mul_const(self._h, _p(a), _p(np.ascontiguousarray(c, dtype=np.uint64)), _p(out), a.shape[0], level)
        return out

    def mul_plain(self, a, pt, level):
        out = self._out(a)
        lib().oc_mul_plain(self._h, _p(a), _p(np.ascontiguousarray(pt)), _p(out), a.shape[0], level)
        return out

    def imul(self, a, level):
        out = self._out(a)
        lib().oc_imul(self._h, _p(a), _p(out), a.shape[0], level)
        return out

    def rescale(self, a, level):
        out = self._out(a)
        lib().oc_rescale(self._h, _p(a), _p(out), a.shape[0], level)
        return out

    def basis_convert(self, coef: np.ndarray, src, dst) -> np.ndarray:
        src_a = np.ascontiguousarray(src, dtype=np.intc)
        dst_a = np.ascontiguousarray(dst, dtype=np.intc)
        out = np.zeros((len(dst), self.N), dtype=np.uint64)
        lib().oc_basis_convert(self._h, _p(np.ascontiguousarray(coef, dtype=np.uint64)), _p(src_a), len(src),
                               _p(out), _p(dst_a), len(dst))
        return out

    def keyswitch(self, d: np.ndarray, evk, level):
        d = np.ascontiguousarray(d, dtype=np.uint64)
        k0 = np.zeros((level + 1, self.N), dtype=np.uint64)
        k1 = np.zeros_like(k0)
        lib().oc_keyswitch(self._h, _p(d), _p(evk), level, _p(k0), _p(k1))
        return k0, k1

    def tensor(self, a, b, level):
        """[d0, d1, d2] of one ciphertext pair, u64[3][L][N]."""
        d = np.zeros((3, self.L, self.N), dtype=np.uint64)
        lib().oc_tensor(self._h, _p(np.ascontiguousarray(a)), _p(np.ascontiguousarray(b)), _p(d), level)
        return d

    def mul_relin(self, a, b, rlk, level):
        out = self._out(a)
        lib().oc_mul_relin(self._h, _p(a), _p(b), _p(rlk), _p(out), a.shape[0], level)
        return out

    def mul_relin_rescale(self, a, b, rlk, level):
        """rescale(relin(a*b)) with the rescale merged into ModDown (level-1 out)."""
        out = self._out(a)
        lib().oc_mul_relin_rescale(self._h, _p(np.ascontiguousarray(a)), _p(np.ascontiguousarray(b)), _p(rlk),
                                   _p(out), a.shape[0], level)
        return out

    def relin_rescale_tensor(self, d, rlk, level):
        """d = [d0, d1, d2] (u64[3][L][N]) -> one ciphertext at level-1."""
        out = np.zeros((1, 2, self.L, self.N), dtype=np.uint64)
        lib().oc_relin_rescale_tensor(self._h, _p(np.ascontiguousarray(d)), _p(rlk), _p(out), level)
        return out

    def automorph(self, a, level, galois):
        out = self._out(a)
        lib().oc_automorph(self._h, _p(a), _p(out), a.shape[0], level, galois)
        return out

    def rotate(self, a, galois, gk, level, accumulate=False):
        out = self._out(a)
        lib().oc_rotate(self._h, _p(a), galois, _p(gk), _p(out), a.shape[0], level, 1 if accumulate else 0)
        return out

    def rotsum(self, a, gals, keys, level, include_identity=True):
        """[a +] sum_t rot_{gals[t]}(a) with one hoisted key switch."""
        a = np.ascontiguousarray(a)
        out = self._out(a)
        g = np.ascontiguousarray(np.array(gals, dtype=np.int64))
        ks = [np.ascontiguousarray(k) for k in keys]
        arr = (_u64p * len(ks))(*[_p(k) for k in ks])
        lib().oc_rotsum(self._h, _p(a), len(ks), _p(g), arr, _p(out), a.shape[0], level, 1 if include_identity else 0)
        return out

    def mod_raise(self, a, level_out):
        a = np.ascontiguousarray(a)
        out = self._out(a)
        lib().oc_mod_raise(self._h, _p(a), _p(out), a.shape[0], level_out)
        return out

    def refresh(self, sk, a, in_level, ratio, out_level, seed, first_id):
        out = self._out(a)
        lib().oc_refresh(self._h, _p(sk), _p(a), in_level, float(ratio), _p(out), out_level, a.shape[0],
                         seed, first_id)
        return out
