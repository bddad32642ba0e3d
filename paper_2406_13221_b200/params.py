"""Scheme parameters: the reference's ``HeParams`` surface plus the RNS-CKKS
ring the reference only models.

``HeParams`` mirrors ``helr.hesim.HeParams`` (hesim.py:41-84): the same
fields, validation messages and ``from_file`` JSON keys, because the driver
(``enctrain.py:253``, ``enctrain.py:387``) and the layout planner
(``encoding.py:73``) read exactly ``log_q``, ``log_delta`` and ``slots``.

``CkksParams`` is new.  It fixes the real ring: N = 2**log_n, a modulus
chain q_0 (about 2**60) and q_1..q_{L-1} (about 2**log_scale, alternately
just above and below so the per-level scale stays close to 2**log_scale),
K special primes p_k (about 2**40 by default, or 2**61) for hybrid key
switching with ``dnum`` digits of ``alpha`` limbs, and one primitive 2N-th
root of unity per prime.
All primes are below 2**61 so the lazy [0, 8q) NTT butterflies (approximate
Shoup quotients) and the 128-bit key-product accumulators never overflow.  Everything here is plain integer arithmetic and
deterministic, so the device library and any CPU checker are handed the
identical chain and roots.

Level accounting for the drop-in surface: a ciphertext whose top active
limb is ``ell`` reports ``level_bits = log_delta * (ell + 1)``; a fresh
ciphertext reports ``log_q = log_delta * L``.  Every rescale (ct x ct or
constant product) drops exactly one limb, i.e. ``log_delta`` bits, which
reproduces the reference's bookkeeping (hesim.py:136-142) with
``log_delta_c == log_delta``.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from functools import cached_property

__all__ = [
    "HeParams",
    "CkksParams",
    "ciphertext_size_mb",
    "is_prime",
    "ntt_primes",
]


@dataclass(frozen=True)
class HeParams:
    """Reference parameter surface (hesim.py:41-84), same defaults and checks."""

    log_n: int = 16
    log_q: int = 275
    log_delta: int = 30
    log_delta_c: int = 20
    noise_sigma: float = 0.0
    seed: int = 0

    def __post_init__(self):
        if self.log_n < 2:
            raise ValueError(f"log_n must be >= 2, got {self.log_n}")
        if self.log_q <= self.log_delta:
            raise ValueError(f"log_q ({self.log_q}) must exceed log_delta ({self.log_delta})")
        if self.log_delta < 1 or self.log_delta_c < 1:
            raise ValueError("rescale amounts must be positive")
        if self.noise_sigma < 0:
            raise ValueError(f"noise_sigma must be >= 0, got {self.noise_sigma}")

    @property
    def slots(self) -> int:
        return 1 << (self.log_n - 1)

    @classmethod
    def from_file(cls, path) -> "HeParams":
        """JSON keys logN, logQ, logDelta, logDeltaC, noise, seed (hesim.py:72-84)."""
        with open(path, "r", encoding="utf-8") as fh:
            raw = json.load(fh)
        return cls(
            log_n=int(raw.get("logN", cls.log_n)),
            log_q=int(raw.get("logQ", cls.log_q)),
            log_delta=int(raw.get("logDelta", cls.log_delta)),
            log_delta_c=int(raw.get("logDeltaC", cls.log_delta_c)),
            noise_sigma=float(raw.get("noise", 0.0)),
            seed=int(raw.get("seed", 0)),
        )


def ciphertext_size_mb(params) -> float:
    """Nominal fresh-ciphertext size 2 * N * log_q bits (hesim.py:87-90)."""
    return 2 * (1 << params.log_n) * params.log_q / 8 / 1e6


# ---------------------------------------------------------------------------
# primes and roots

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (covers every 64-bit word)."""
    if n < 2:
        return False
    for p in _MR_BASES:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _MR_BASES:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def ntt_primes(log_n: int, bits: int, count: int, *, mode: str = "below",
               exclude: tuple = ()) -> list[int]:
    """``count`` primes q = 1 (mod 2N) near 2**bits.

    mode "below": descending from 2**bits.  mode "closest": alternately the
    nearest unused prime above and below 2**bits (keeps rescaled scales
    near 2**bits).
    """
    m = 2 << log_n  # 2N
    target = 1 << bits
    found: list[int] = []
    taken = set(exclude)
    if mode == "below":
        c = (target - 1) // m * m + 1
        while len(found) < count:
            if c < 3:
                raise ValueError(f"ran out of {bits}-bit primes = 1 mod {m}")
            if c not in taken and is_prime(c):
                found.append(c)
                taken.add(c)
            c -= m
        return found
    if mode != "closest":
        raise ValueError(f"unknown prime search mode {mode!r}")
    up = (target // m + 1) * m + 1
    dn = (target - 1) // m * m + 1
    want_up = True
    while len(found) < count:
        if want_up:
            while up in taken or not is_prime(up):
                up += m
            found.append(up)
            taken.add(up)
            up += m
        else:
            while dn in taken or not is_prime(dn):
                dn -= m
            found.append(dn)
            taken.add(dn)
            dn -= m
        want_up = not want_up
    return found


def primitive_2n_root(q: int, log_n: int) -> int:
    """Smallest x**((q-1)/2N) over x = 2, 3, ... that has exact order 2N."""
    n2 = 2 << log_n
    if (q - 1) % n2:
        raise ValueError(f"{q} is not 1 mod {n2}")
    e = (q - 1) // n2
    x = 2
    while True:
        psi = pow(x, e, q)
        if pow(psi, n2 >> 1, q) == q - 1:
            return psi
        x += 1


@dataclass(frozen=True)
class CkksParams:
    """A concrete RNS-CKKS ring.

    q: the L ciphertext primes (q[0] is the decryption prime, q[1:] are
    rescaling primes); p: the K special primes (product P well above the
    largest key-switching digit modulus); dnum: number of
    key-switching digits at the top level.  ``scale_bits`` is the nominal
    log2 of the fresh encoding scale.  ``cbd_eta`` is the centred-binomial
    error parameter (variance eta/2; 21 gives sigma ~ 3.24).
    """

    log_n: int
    q: tuple
    p: tuple
    dnum: int
    scale_bits: int = 40
    cbd_eta: int = 21
    secret_hw: int = 64
    psi: tuple = field(default=(), compare=False)
    # bootstrappable chains (bootstrap.bootstrap_ring): number of working
    # levels below the bootstrapping levels; 0 = the whole chain is working levels
    work_levels: int = 0

    def __post_init__(self):
        if not 2 <= self.log_n <= 17:
            raise ValueError(f"log_n must be in [2, 17], got {self.log_n}")
        if len(self.q) < 2:
            raise ValueError("need at least two ciphertext primes")
        if self.dnum < 1 or self.dnum > len(self.q):
            raise ValueError(f"dnum must be in [1, {len(self.q)}], got {self.dnum}")
        if len(self.p) < 1 or len(self.q) + len(self.p) > 64:
            raise ValueError(f"need 1..{64 - len(self.q)} special primes, got {len(self.p)}")
        m = 2 << self.log_n
        for x in tuple(self.q) + tuple(self.p):
            if x >= (1 << 61) or (x - 1) % m or not is_prime(x):
                raise ValueError(f"{x} is not an NTT-friendly prime < 2**61 for N=2**{self.log_n}")
        if len(set(self.q) | set(self.p)) != len(self.q) + len(self.p):
            raise ValueError("primes must be distinct")
        if not 0 <= self.work_levels < len(self.q):
            raise ValueError(f"work_levels must be in [0, {len(self.q)}), got {self.work_levels}")
        if not 0 < self.cbd_eta <= 32:
            raise ValueError(f"cbd_eta must be in [1, 32], got {self.cbd_eta}")
        if not self.psi:
            roots = tuple(primitive_2n_root(x, self.log_n) for x in tuple(self.q) + tuple(self.p))
            object.__setattr__(self, "psi", roots)

    # -- construction ------------------------------------------------------

    @classmethod
    def generate(cls, log_n: int, n_q: int, dnum: int = 3, scale_bits: int = 40,
                 q0_bits: int = 60, p_bits: int = 40, cbd_eta: int = 21, secret_hw: int = 64,
                 n_special: int = None, ks_margin_bits: int = 20) -> "CkksParams":
        """Special primes: ``n_special`` of ``p_bits`` bits, by default the
        fewest whose product exceeds the largest digit modulus (the one
        holding q_0) by ``ks_margin_bits`` — alpha primes of 61 bits, or
        alpha + 1 of 40 bits.  40-bit specials (the default) let every limb
        but q_0 take the fp64 NTT path (primes < 2^41)."""
        alpha = -(-n_q // dnum)
        if n_special is None:
            digit_bits = q0_bits + (min(alpha, n_q) - 1) * scale_bits
            n_special = -(-(digit_bits + ks_margin_bits) // p_bits)
        q0 = ntt_primes(log_n, q0_bits, 1, mode="below")
        scaling = ntt_primes(log_n, scale_bits, n_q - 1, mode="closest", exclude=tuple(q0))
        special = ntt_primes(log_n, p_bits, n_special, mode="below", exclude=tuple(q0 + scaling))
        return cls(log_n=log_n, q=tuple(q0 + scaling), p=tuple(special), dnum=dnum,
                   scale_bits=scale_bits, cbd_eta=cbd_eta, secret_hw=secret_hw)

    # -- derived -------------------------------------------------------------

    @property
    def n(self) -> int:
        return 1 << self.log_n

    @property
    def slots(self) -> int:
        return 1 << (self.log_n - 1)

    @property
    def hw(self) -> int:
        """Effective secret Hamming weight (0 = uniform ternary); capped at N/2
        for tiny test rings."""
        return min(self.secret_hw, self.n // 2) if self.secret_hw > 0 else 0

    @property
    def L(self) -> int:
        return len(self.q)

    @property
    def K(self) -> int:
        return len(self.p)

    @property
    def alpha(self) -> int:
        return -(-len(self.q) // self.dnum)

    @property
    def primes(self) -> tuple:
        return tuple(self.q) + tuple(self.p)

    @property
    def top_level(self) -> int:
        """The working top: the level of fresh encryptions and of refreshed
        ciphertexts.  Equal to L - 1 unless the chain reserves bootstrapping
        levels above it (``work_levels``)."""
        return self.work_levels if self.work_levels else self.L - 1

    def digits(self, level: int) -> int:
        """Number of key-switching digits in use at ``level`` (level+1 limbs)."""
        return -(-(level + 1) // self.alpha)

    @cached_property
    def level_scales(self) -> tuple:
        """Canonical scale per level: Delta_top = 2**scale_bits,
        Delta_{l-1} = Delta_l**2 / q_l (so ct x ct products of canonical
        operands land exactly on the next canonical scale)."""
        s = [0.0] * self.L
        top = self.top_level
        s[top] = float(2 ** self.scale_bits)
        for lvl in range(top, 0, -1):
            s[lvl - 1] = s[lvl] * s[lvl] / float(self.q[lvl])
        # bootstrapping levels (above the working top) have no canonical
        # scale: bootstrap.Bootstrapper tracks its own labels there
        return tuple(s)

    def he_params(self, noise_sigma: float = 1e-7, seed: int = 0) -> HeParams:
        """The reference-facing view: one limb = ``scale_bits`` bits of level.

        ``noise_sigma`` > 0 tells the reference driver that decryptions are
        approximate (it disables the exact replication check,
        enctrain.py:337); it is a nominal figure, the real noise is the
        CKKS error.
        """
        return HeParams(log_n=self.log_n, log_q=self.scale_bits * (self.top_level + 1),
                        log_delta=self.scale_bits, log_delta_c=self.scale_bits,
                        noise_sigma=noise_sigma, seed=seed)

    def level_bits(self, level: int) -> int:
        return self.scale_bits * (level + 1)

    def level_of_bits(self, bits: int) -> int:
        return bits // self.scale_bits - 1

    def log2_q_total(self) -> float:
        return sum(math.log2(x) for x in self.q)
