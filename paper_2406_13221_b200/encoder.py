"""Host-side CKKS encoding: slot vectors <-> integer polynomials (fp64).

The reference's ``SimContext.enc`` zero-pads a message to N/2 complex slots
(hesim.py:146-158) and ``dec`` returns them (hesim.py:160-162).  Here a slot
vector z in C^(N/2) becomes the real polynomial m(X) in R[X]/(X^N + 1) with
m(zeta^(5^j)) = z_j and m(zeta^(-5^j)) = conj(z_j), zeta = exp(i*pi/N), and
is scaled and rounded to integers.  Slot j <-> root zeta^(5^j), so the
Galois map X -> X^(5^k) is the reference's left rotation by k
(``np.roll(slots, -k)``, hesim.py:222).

The transform is one length-N complex FFT: with b_i = m_i * zeta^i,
m(zeta^(2t+1)) = sum_i b_i exp(2 pi i t i / N), i.e. the evaluations are
N * ifft(b).  Encoding and decoding stay on the host in fp64 (the device
never sees floating point except in the refresh stand-in's ratio), so the
device library and any CPU checker are fed identical integers.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

__all__ = ["Encoder"]

_INT_LIMIT = float(2 ** 62)


@lru_cache(maxsize=16)
def _tables(log_n: int):
    n = 1 << log_n
    s = n >> 1
    two_n = 2 * n
    pw = np.empty(s, dtype=np.int64)
    acc = 1
    for j in range(s):
        pw[j] = acc
        acc = (acc * 5) % two_n
    t_pos = (pw - 1) // 2                 # zeta^(5^j)   = zeta^(2t+1)
    t_neg = (two_n - pw - 1) // 2         # zeta^(-5^j)
    i = np.arange(n)
    twist = np.exp(1j * np.pi * i / n)    # zeta^i
    return t_pos, t_neg, twist, np.conj(twist)


class Encoder:
    """Slot <-> coefficient maps for one ring degree N = 2**log_n."""

    def __init__(self, log_n: int):
        self.log_n = log_n
        self.n = 1 << log_n
        self.slots = self.n >> 1
        self._t_pos, self._t_neg, self._twist, self._untwist = _tables(log_n)

    def coefficients(self, z) -> np.ndarray:
        """Real coefficients of the polynomial whose slots are ``z`` (batched on axis 0)."""
        z = np.asarray(z, dtype=np.complex128)
        single = z.ndim == 1
        z = np.atleast_2d(z)
        if z.shape[-1] > self.slots:
            raise ValueError(f"message has {z.shape[-1]} slots, maximum is {self.slots}")
        full = np.zeros((z.shape[0], self.slots), dtype=np.complex128)
        full[:, : z.shape[-1]] = z
        ev = np.zeros((z.shape[0], self.n), dtype=np.complex128)
        ev[:, self._t_pos] = full
        ev[:, self._t_neg] = np.conj(full)
        b = np.fft.fft(ev, axis=-1) / self.n
        m = np.real(b * self._untwist)
        return m[0] if single else m

    def encode(self, z, scale: float) -> np.ndarray:
        """round(scale * m) as int64 coefficients."""
        m = self.coefficients(z) * float(scale)
        if np.max(np.abs(m), initial=0.0) >= _INT_LIMIT:
            raise ValueError("encoded coefficient exceeds 2**62; lower the scale or the values")
        return np.rint(m).astype(np.int64)

    def encode_constant(self, c: float, scale: float) -> int:
        """A real constant in every slot is the constant polynomial c."""
        v = float(c) * float(scale)
        if abs(v) >= _INT_LIMIT:
            raise ValueError("encoded constant exceeds 2**62")
        return int(np.rint(v))

    def decode(self, coef, scale: float) -> np.ndarray:
        """Slots of the integer polynomial ``coef`` divided by ``scale``."""
        c = np.asarray(coef)
        single = c.ndim == 1
        c = np.atleast_2d(c).astype(np.float64)
        ev = np.fft.ifft(c * self._twist, axis=-1) * self.n
        z = ev[:, self._t_pos] / float(scale)
        return z[0] if single else z
