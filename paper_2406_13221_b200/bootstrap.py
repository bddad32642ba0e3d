"""Real CKKS bootstrapping over the ring primitives.

The reference only *models* a bootstrap: ``SimContext.bootstrap`` restores
the level and bumps a counter (hesim.py:228-236); the paper's own runs spend
~38 of 45 s per iteration in it.  This module is the real
thing, composed from the evaluator primitives of ``include/helr_ckks.h``
(every step is a hand-written sm_100a kernel; nothing here touches the
secret key):

1. **ModRaise** (``helr_mod_raise``): the exhausted ciphertext is read modulo
   q_0 and re-interpreted modulo the full chain Q_top; it now encrypts
   t = m + q_0 I with a small integer polynomial I (|I| <= K for a sparse
   secret of Hamming weight h: I is a sum of h + 1 roundings).
2. **CoeffToSlot**: the inverse of the encoding map, evaluated homomorphically
   as G_c sparse-diagonal factors of the special FFT (HEAAN's
   ``fftSpecialInv`` butterflies, grouped radix-2^k, each applied with
   baby-step/giant-step rotations), so the slots hold the coefficients
   t_i / (q_0 K); one conjugation splits them into two real ciphertexts.
3. **EvalMod**: t mod q_0 through the scaled sine: a Chebyshev interpolant of
   cos(2 pi (K u - 1/4) / 2^r) (Paterson-Stockmeyer over the T_k basis,
   depth log2(d + 1) + 1) followed by r double-angle steps
   cos 2x = 2 cos^2 x - 1, which yields sin(2 pi t / q_0) ~ 2 pi m / q_0.
4. **SlotToCoeff**: the forward special FFT in G_s grouped factors back to
   coefficients, landing on the working top level at the canonical scale.

Scales are tracked exactly (fp64 labels): multiplying every slot by a
constant is a re-labelling of the scale, plaintext diagonals are encoded at
whatever scale makes the product land on the level's canonical scale, and
ciphertexts only meet in additions at equal scales.

The circuit is written against a small evaluator protocol (``GpuRing`` below
is the product's implementation; the parity tests drive the same circuit
with the CPU ring oracle and compare every residue).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from .encoder import Encoder
from .params import CkksParams, ntt_primes

__all__ = ["BootstrapConfig", "Bootstrapper", "GpuRing", "bootstrap_ring", "dft_stage", "compose",
           "grouped_dft_factors", "chebyshev_coefficients"]


# ---------------------------------------------------------------------------
# special-FFT factors in diagonal form
#
# A matrix M acting on the slot vector z is stored as {d: diag_d} with
# (M z)[k] = sum_d diag_d[k] * z[(k + d) mod n]  (rot(z, d)[k] = z[k + d] is the
# evaluator's left rotation by d slots, hesim.py:222).

def _bitrev(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    idx = np.arange(n)
    out = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        out |= ((idx >> b) & 1) << (bits - 1 - b)
    return out


def dft_stage(log_n: int, length: int, inverse: bool) -> Dict[int, np.ndarray]:
    """One butterfly stage of the special FFT on n = N/2 slots.

    Forward (block length ``length``, half h): out[i+j] = a + w_j b,
    out[i+j+h] = a - w_j b with w_j = exp(2 pi i (5^j mod 4 length) / (4 length)).
    Inverse (un-normalised, i.e. 2x the true inverse): a = u + l,
    b = conj(w_j) (u - l).  The product of the forward stages, applied to the
    bit-reversed coefficient vector, is the encoding matrix U0[j][i] =
    zeta^(5^j i); the un-normalised inverse stages compose to n U0^-1.
    """
    n = 1 << (log_n - 1)
    h = length >> 1
    k = np.arange(n)
    j = k % length
    upper = j < h
    jj = np.where(upper, j, j - h)
    pw = np.array([pow(5, int(x), 4 * length) for x in range(h)], dtype=np.float64)
    w = np.exp(2j * np.pi * pw[jj] / (4 * length))
    zero = np.zeros(n, dtype=np.complex128)
    d0, dp, dm = zero.copy(), zero.copy(), zero.copy()
    if not inverse:
        d0[upper] = 1.0
        dp[upper] = w[upper]
        d0[~upper] = -w[~upper]
        dm[~upper] = 1.0
    else:
        d0[upper] = 1.0
        dp[upper] = 1.0
        d0[~upper] = -np.conj(w[~upper])
        dm[~upper] = np.conj(w[~upper])
    out: Dict[int, np.ndarray] = {}
    for off, d in ((0, d0), (h % n, dp), ((-h) % n, dm)):
        if np.any(d != 0):
            out[off] = out.get(off, 0) + d
    return out


def compose(a: Dict[int, np.ndarray], b: Dict[int, np.ndarray], n: int) -> Dict[int, np.ndarray]:
    """Diagonal form of the matrix product A B (B applied first)."""
    out: Dict[int, np.ndarray] = {}
    for da, va in a.items():
        for db, vb in b.items():
            d = (da + db) % n
            term = va * np.roll(vb, -da)
            out[d] = out[d] + term if d in out else term
    return {d: v for d, v in out.items() if np.any(np.abs(v) > 0)}


def apply_diagonals(m: Dict[int, np.ndarray], z: np.ndarray) -> np.ndarray:
    out = np.zeros_like(z, dtype=np.complex128)
    for d, v in m.items():
        out = out + v * np.roll(z, -d)
    return out


def _split_levels(total: int, groups: int) -> List[int]:
    base, extra = divmod(total, groups)
    return [base + (1 if i < extra else 0) for i in range(groups)]


def grouped_dft_factors(log_n: int, groups: int, inverse: bool) -> List[Dict[int, np.ndarray]]:
    """The log2(n) butterfly stages merged into ``groups`` matrices, in the
    order they are applied.  Forward: stage lengths 2, 4, ..., n (input in
    bit-reversed order).  Inverse: n, ..., 4, 2 (output in bit-reversed order)."""
    n = 1 << (log_n - 1)
    stages = log_n - 1
    groups = max(1, min(groups, stages))
    lens = [2 << s for s in range(stages)]
    if inverse:
        lens = lens[::-1]
    out = []
    pos = 0
    for cnt in _split_levels(stages, groups):
        m = None
        for length in lens[pos:pos + cnt]:
            st = dft_stage(log_n, length, inverse)
            m = st if m is None else compose(st, m, n)
        out.append(m)
        pos += cnt
    return out


def chebyshev_coefficients(k_range: int, double_angles: int, degree: int) -> np.ndarray:
    """Chebyshev interpolant (first-kind nodes) of
    f(u) = cos(2 pi (K u - 1/4) / 2^r) on [-1, 1]."""
    from numpy.polynomial import chebyshev as C

    def f(u):
        return np.cos(2.0 * np.pi * (k_range * u - 0.25) / (1 << double_angles))

    return C.chebinterpolate(f, degree)


# ---------------------------------------------------------------------------
# parameters

@dataclass(frozen=True)
class BootstrapConfig:
    """Shape of the bootstrapping circuit.

    ``k_range``: bound K on |I| (t = m + q_0 I); 16 covers a Hamming-weight-64
    secret at 6.9 sigma.  ``degree`` must be 2^k - 1 (>= 15).  Levels consumed:
    c2s_groups + (log2(degree + 1) + 1) + double_angles + s2c_groups."""

    c2s_groups: int = 3
    s2c_groups: int = 3
    k_range: int = 16
    double_angles: int = 3
    degree: int = 63
    baby_log: int = 3          # Paterson-Stockmeyer baby step 2^baby_log
    boot_bits: int = 59        # EvalMod working scale: its rescale noise, amplified by K q_0 / scale_in, sets the precision
    min_ratio_bits: float = 11.5  # refuse inputs with q_0 / scale below 2^this (sine linearity)

    def __post_init__(self):
        if self.degree + 1 < (2 << self.baby_log) or (self.degree + 1) & self.degree:
            raise ValueError("degree must be 2^k - 1 with 2^k >= 2 * baby step")

    @property
    def poly_depth(self) -> int:
        return (self.degree + 1).bit_length() - 1 + 1

    @property
    def depth(self) -> int:
        return self.c2s_groups + self.poly_depth + self.double_angles + self.s2c_groups


def bootstrap_ring(log_n: int, work_levels: int = 7, scale_bits: int = 40, cfg: Optional[BootstrapConfig] = None,
                   dnum: Optional[int] = None, q0_bits: int = 60, s2c_bits: int = 45, c2s_bits: int = 58,
                   secret_hw: int = 64, cbd_eta: int = 21, p_bits: int = 60) -> CkksParams:
    """A modulus chain with room for one bootstrap above ``work_levels``
    working levels: q_0 | work_levels primes of ``scale_bits`` | s2c_groups of
    ``s2c_bits`` | EvalMod primes of ``cfg.boot_bits`` | c2s_groups of
    ``c2s_bits``.  ``CkksParams.work_levels`` marks the working top: fresh
    encryptions and bootstrap outputs live there, the levels above are only
    visited inside ``Bootstrapper.bootstrap``."""
    cfg = cfg or BootstrapConfig()
    taken: List[int] = []

    def take(bits, count, mode="closest"):
        got = ntt_primes(log_n, bits, count, mode=mode, exclude=tuple(taken))
        taken.extend(got)
        return got

    q = take(q0_bits, 1, "below")
    q += take(scale_bits, work_levels)
    q += take(s2c_bits, cfg.s2c_groups)
    q += take(cfg.boot_bits, cfg.poly_depth + cfg.double_angles)
    q += take(c2s_bits, cfg.c2s_groups)
    n_q = len(q)
    if dnum is None:
        dnum = -(-n_q // 4)
    alpha = -(-n_q // dnum)
    digit_bits = max(sum(math.log2(x) for x in q[j * alpha:(j + 1) * alpha]) for j in range(dnum))
    n_special = int(-(-(digit_bits + 20) // p_bits))
    p = take(p_bits, n_special, "below")
    return CkksParams(log_n=log_n, q=tuple(q), p=tuple(p), dnum=dnum, scale_bits=scale_bits, cbd_eta=cbd_eta,
                      secret_hw=secret_hw, work_levels=work_levels)


# ---------------------------------------------------------------------------
# ciphertext bookkeeping inside the circuit

@dataclass
class _Ct:
    buf: object      # evaluator buffer: [count][2][L][N]
    level: int
    scale: float


@dataclass
class _Transform:
    """One grouped DFT factor prepared for baby-step/giant-step evaluation."""
    diagonals: Dict[int, np.ndarray]
    step: int = 1
    baby: int = 1
    giants: List[int] = field(default_factory=list)   # giant indices i (offset g*i*step)
    terms: Dict[int, List[int]] = field(default_factory=dict)  # giant i -> baby j list
    signed: Dict[int, int] = field(default_factory=dict)       # (g*i + j) -> offset mod n

    @classmethod
    def plan(cls, diagonals: Dict[int, np.ndarray], n: int) -> "_Transform":
        offs = sorted(diagonals)
        step = n
        for d in offs:
            step = math.gcd(step, d) if d else step
        step = max(step, 1) if any(offs) else 1
        m = n // step
        ks = {}
        for d in offs:
            k = (d // step) % m
            if k >= (m + 1) // 2 and m > 2:
                k -= m      # signed representative: lower groups have offsets +-
            ks[k] = d
        lo, hi = min(ks), max(ks)
        span = hi - lo + 1
        g = 1
        while g * g < span:
            g <<= 1
        t = cls(diagonals=diagonals, step=step, baby=g)
        for k, d in sorted(ks.items()):
            i, j = k // g, k % g   # Python floor division: j in [0, g)
            t.terms.setdefault(i, []).append(j)
            t.signed[g * i + j] = d
        t.giants = sorted(t.terms)
        return t

    def rotations(self, n: int) -> List[int]:
        """Slot rotations (mod n) this transform needs keys for."""
        out = set()
        for i, js in self.terms.items():
            if (self.baby * i * self.step) % n:
                out.add((self.baby * i * self.step) % n)
            for j in js:
                if (j * self.step) % n:
                    out.add((j * self.step) % n)
        return sorted(out)


class Bootstrapper:
    """Plans and runs one bootstrap on ``ring`` (see module docstring).

    ``ring`` supplies the primitives (names as in the C ABI): ``add``, ``sub``,
    ``add_const``, ``mul_const``, ``mul_plain``, ``encode_plain``,
    ``rescale``, ``mul`` (relinearise + rescale), ``rotate`` (by Galois
    element), ``imul``, ``mod_raise``, ``cat``, ``split``; buffers are opaque.
    """

    def __init__(self, ring, cfg: Optional[BootstrapConfig] = None):
        self.ring = ring
        self.ck: CkksParams = ring.params
        self.cfg = cfg or BootstrapConfig()
        ck, cfg = self.ck, self.cfg
        self.n = ck.slots
        self.top = ck.L - 1
        self.out_level = self.top - cfg.depth
        if self.out_level < 1:
            raise ValueError(f"bootstrapping needs {cfg.depth} levels above the working top; the chain has {ck.L} limbs")
        self.encoder = Encoder(ck.log_n)
        self.c2s = [_Transform.plan(m, self.n) for m in grouped_dft_factors(ck.log_n, cfg.c2s_groups, True)]
        self.s2c = [_Transform.plan(m, self.n) for m in grouped_dft_factors(ck.log_n, cfg.s2c_groups, False)]
        self.cheb = chebyshev_coefficients(cfg.k_range, cfg.double_angles, cfg.degree)
        # EvalMod canonical scales: S at the EvalMod input level, then S^2 / q down the chain
        self.eval_top = self.top - len(self.c2s)
        self.eval_bottom = self.eval_top - cfg.poly_depth - cfg.double_angles
        self.S = {self.eval_top: float(2 ** cfg.boot_bits)}
        for lvl in range(self.eval_top, self.eval_bottom, -1):
            self.S[lvl - 1] = self.S[lvl] * self.S[lvl] / float(ck.q[lvl])
        self.out_scale = float(ck.level_scales[self.out_level])
        self._pt_cache: dict = {}
        self.pt_variants = 4
        self.conj_galois = 2 * ck.n - 1

    # -- what the evaluator has to prepare -----------------------------------
    def galois_elements(self) -> List[int]:
        two_n = 2 * self.ck.n
        rots = set()
        for t in self.c2s + self.s2c:
            rots.update(t.rotations(self.n))
        return sorted({pow(5, r, two_n) for r in rots} | {self.conj_galois})

    # -- primitives with bookkeeping -----------------------------------------
    def _const(self, value: float) -> int:
        # constants are reduced per limb by the evaluator, so they may exceed a
        # machine word (additive constants before a rescale sit at scale^2)
        v = float(value)
        if not math.isfinite(v):
            raise ValueError("non-finite constant")
        return int(np.rint(v)) if abs(v) < 2.0 ** 62 else int(v)

    def _to_level(self, x: _Ct, level: int, scale: float) -> _Ct:
        """Bring x down to ``level`` landing on ``scale``: drop limbs to
        level + 1, then one integer constant product and one rescale."""
        if x.level == level:
            if abs(x.scale / scale - 1.0) > 1e-9:
                raise ValueError(f"scale mismatch at level {level}: {x.scale} vs {scale}")
            return x
        if x.level < level:
            raise ValueError("cannot move a ciphertext up")
        top = level + 1
        c = self._const(scale * float(self.ck.q[top]) / x.scale)
        buf = self.ring.rescale(self.ring.mul_const(x.buf, c, top), top)
        return _Ct(buf, level, x.scale * c / float(self.ck.q[top]))

    def _mul(self, a: _Ct, b: _Ct) -> _Ct:
        lvl = min(a.level, b.level)
        a = self._to_level(a, lvl, self.S[lvl])
        b = self._to_level(b, lvl, self.S[lvl])
        return _Ct(self.ring.mul(a.buf, b.buf, lvl), lvl - 1, a.scale * b.scale / float(self.ck.q[lvl]))

    def _add(self, a: _Ct, b: _Ct, sub: bool = False) -> _Ct:
        lvl = min(a.level, b.level)
        a = self._to_level(a, lvl, self.S[lvl])
        b = self._to_level(b, lvl, self.S[lvl])
        if abs(a.scale / b.scale - 1.0) > 1e-9:
            raise ValueError(f"scale mismatch in add at level {lvl}: {a.scale} vs {b.scale}")
        f = self.ring.sub if sub else self.ring.add
        return _Ct(f(a.buf, b.buf, lvl), lvl, a.scale)

    def _add_scalar(self, a: _Ct, value: float) -> _Ct:
        return _Ct(self.ring.add_const(a.buf, self._const(value * a.scale), a.level), a.level, a.scale)

    def _double_minus_one(self, sq: _Ct) -> _Ct:
        """2 x - 1 (x a fresh product)."""
        d = _Ct(self.ring.add(sq.buf, sq.buf, sq.level), sq.level, sq.scale)
        return self._add_scalar(d, -1.0)

    # -- linear transforms ------------------------------------------------------
    def _plaintexts(self, key, t: _Transform, level: int, pt_scale: float):
        """Encoded diagonals of one factor, cached per (factor, level, scale).
        CoeffToSlot scales are fixed by the chain; SlotToCoeff scales follow
        the input's scale label (W and V of the per-op driver arrive at two
        different bottom scales), so a few variants per factor are kept
        (least recently used dropped beyond ``pt_variants``)."""
        ck = (key, level, float(pt_scale))
        if ck in self._pt_cache:
            self._pt_cache[ck] = self._pt_cache.pop(ck)     # most recently used last
            return self._pt_cache[ck][0]
        pts = {}
        g, st, n = t.baby, t.step, self.n
        for i, js in t.terms.items():
            for j in js:
                d = t.signed[g * i + j]
                vec = np.roll(t.diagonals[d], (g * i * st) % n)   # rot(diag, -g i step)
                pts[(i, j)] = self.ring.encode_plain(self.encoder.encode(vec, pt_scale), level)
        same = [k for k in self._pt_cache if k[0] == key and k[1] == level]
        while len(same) >= self.pt_variants:
            del self._pt_cache[same.pop(0)]
        self._pt_cache[ck] = (pts, pt_scale)
        return pts

    def _linear(self, key, t: _Transform, x: _Ct, target_scale: float) -> _Ct:
        """x -> rescale(M x), landing on ``target_scale`` at level - 1."""
        lvl, n, two_n = x.level, self.n, 2 * self.ck.n
        pt_scale = target_scale * float(self.ck.q[lvl]) / x.scale
        pts = self._plaintexts(key, t, lvl, pt_scale)
        g, st = t.baby, t.step
        babies = {0: x.buf}
        for j in sorted({j for js in t.terms.values() for j in js}):
            if j and j not in babies:
                babies[j] = self.ring.rotate(x.buf, pow(5, (j * st) % n, two_n), lvl)
        acc = None
        for i in t.giants:
            inner = None
            for j in t.terms[i]:
                term = self.ring.mul_plain(babies[j], pts[(i, j)], lvl)
                inner = term if inner is None else self.ring.add(inner, term, lvl)
            r = (g * i * st) % n
            if r:
                inner = self.ring.rotate(inner, pow(5, r, two_n), lvl)
            acc = inner if acc is None else self.ring.add(acc, inner, lvl)
        out = self.ring.rescale(acc, lvl)
        return _Ct(out, lvl - 1, x.scale * pt_scale / float(self.ck.q[lvl]))

    # -- EvalMod ------------------------------------------------------------------
    def _chebyshev(self, u: _Ct) -> _Ct:
        """sum_k c_k T_k(u), Paterson-Stockmeyer over the Chebyshev basis."""
        cfg = self.cfg
        b = 1 << cfg.baby_log
        T: Dict[int, _Ct] = {1: u}

        def get(k: int) -> _Ct:
            if k in T:
                return T[k]
            if k % 2 == 0:
                h = get(k // 2)
                T[k] = self._double_minus_one(self._mul(h, h))
            else:
                a, c = get((k + 1) // 2), get(k // 2)
                p = self._mul(a, c)
                d = _Ct(self.ring.add(p.buf, p.buf, p.level), p.level, p.scale)
                T[k] = self._add(d, get(1), sub=True)     # T_{a+c} = 2 T_a T_c - T_{|a-c|}, |a - c| = 1
            return T[k]

        for k in range(2, b + 1):
            get(k)
        giant = b
        while 2 * giant <= cfg.degree:
            giant *= 2
            get(giant)
        base_level = min(T[k].level for k in range(1, b))
        base = {k: self._to_level(T[k], base_level, self.S[base_level]) for k in range(1, b)}

        def baby_poly(c: np.ndarray) -> _Ct:
            # sum_{k<b} c_k T_k: integer constant products at a common factor, one rescale
            lvl = base_level
            factor = self.S[lvl - 1] * float(self.ck.q[lvl]) / self.S[lvl]
            acc = None
            for k in range(1, b):
                if k >= len(c) or c[k] == 0.0:
                    continue
                term = self.ring.mul_const(base[k].buf, self._const(c[k] * factor), lvl)
                acc = term if acc is None else self.ring.add(acc, term, lvl)
            if acc is None:
                raise ValueError("degenerate Chebyshev block (all-zero coefficients)")
            s = self.S[lvl] * factor
            acc = self.ring.add_const(acc, self._const(c[0] * s), lvl)
            return _Ct(self.ring.rescale(acc, lvl), lvl - 1, s / float(self.ck.q[lvl]))

        def evaluate(c: np.ndarray) -> _Ct:
            if len(c) <= b:
                return baby_poly(c)
            h = b
            while 2 * h < len(c):
                h *= 2
            # Chebyshev split at T_h: c_{h+j} T_{h+j} = 2 c_{h+j} T_h T_j - c_{h+j} T_{h-j}
            quo = np.zeros(len(c) - h)
            rem = np.array(c[:h], dtype=np.float64)
            quo[0] = c[h]
            for j in range(1, len(c) - h):
                quo[j] = 2.0 * c[h + j]
                rem[h - j] -= c[h + j]
            return self._add(self._mul(evaluate(quo), T[h]), evaluate(rem))

        return evaluate(np.asarray(self.cheb, dtype=np.float64))

    def _eval_mod(self, u: _Ct) -> _Ct:
        c = self._chebyshev(u)
        for _ in range(self.cfg.double_angles):
            c = self._double_minus_one(self._mul(c, c))
        return c

    # -- the bootstrap ---------------------------------------------------------------
    def bootstrap(self, buf, level: int, scale: float):
        """One ciphertext (buffer [1][2][L][N]) at any level with scale label
        ``scale`` -> (buffer, out_level, out_scale) encrypting the same slots."""
        ck, cfg, ring = self.ck, self.cfg, self.ring
        q0 = float(ck.q[0])
        if math.log2(q0 / scale) < cfg.min_ratio_bits:
            raise ValueError(f"bootstrap input scale 2^{math.log2(scale):.1f} is too close to q_0 = 2^{math.log2(q0):.1f}")
        # (1) read modulo q_0, re-interpret modulo Q_top; the slots now hold
        # t(zeta_j) with t = m + q_0 I.  Label the scale so that the
        # un-normalised inverse DFT and the conjugate sum below leave t_i / (q_0 K).
        x = _Ct(ring.mod_raise(buf, self.top), self.top, q0 * cfg.k_range * 2.0 * self.n)
        # (2) CoeffToSlot: glide the scale label geometrically down to the EvalMod scale
        s_in, s_out = x.scale, self.S[self.eval_top]
        for gi, t in enumerate(self.c2s):
            target = s_in * (s_out / s_in) ** ((gi + 1) / len(self.c2s))
            if gi == len(self.c2s) - 1:
                target = s_out
            x = self._linear(("c2s", gi), t, x, target)
        cj = ring.rotate(x.buf, self.conj_galois, x.level)
        re2 = ring.add(x.buf, cj, x.level)                       # w + conj(w) = 2 Re w
        im2 = ring.imul(ring.sub(cj, x.buf, x.level), x.level)   # i (conj(w) - w) = 2 Im w
        u = _Ct(ring.cat([re2, im2]), x.level, x.scale)
        # (3) EvalMod on both halves at once
        v = self._eval_mod(u)
        # sin(2 pi t / q_0) ~ 2 pi m / q_0: re-label so the value is m / scale
        v = _Ct(v.buf, v.level, v.scale * 2.0 * np.pi * scale / q0)
        v_re, v_im = ring.split(v.buf, 2)
        w = ring.add(v_re, ring.imul(v_im, v.level), v.level)
        y = _Ct(w, v.level, v.scale)
        # (4) SlotToCoeff, landing on the canonical scale of the working top
        s_in, s_out = y.scale, self.out_scale
        for gi, t in enumerate(self.s2c):
            target = s_in * (s_out / s_in) ** ((gi + 1) / len(self.s2c))
            if gi == len(self.s2c) - 1:
                target = s_out
            y = self._linear(("s2c", gi), t, y, target)
        return y.buf, y.level, y.scale


# ---------------------------------------------------------------------------
# the product's evaluator for the circuit: thin calls into libhelr_ckks.so

class GpuRing:
    """Primitive evaluator over a ``GpuContext`` (device buffers int64[count][2][L][N])."""

    def __init__(self, ctx):
        import torch

        self._torch = torch
        self.ctx = ctx
        self.params: CkksParams = ctx.ckks

    def _stream(self):
        return self._torch.cuda.current_stream().cuda_stream

    def _out(self, a):
        return self._torch.empty_like(a)

    def _res(self, value: int, level: int):
        return self.ctx._residues(int(value), level)

    def _bin(self, name, a, b, level):
        out = self._out(a)
        self.ctx._call(name, a.data_ptr(), b.data_ptr(), out.data_ptr(), a.shape[0], level, self._stream())
        return out

    def add(self, a, b, level):
        return self._bin("helr_add", a, b, level)

    def sub(self, a, b, level):
        return self._bin("helr_sub", a, b, level)

    def add_const(self, a, value: int, level):
        return self._bin("helr_add_const", a, self._res(value, level), level)

    def mul_const(self, a, value: int, level):
        return self._bin("helr_mul_const", a, self._res(value, level), level)

    def mul_plain(self, a, pt, level):
        return self._bin("helr_mul_plain", a, pt, level)

    def encode_plain(self, coef: np.ndarray, level: int):
        return self.ctx._plain(coef, level)

    def rescale(self, a, level):
        out = self._out(a)
        self.ctx._call("helr_rescale", a.data_ptr(), out.data_ptr(), a.shape[0], level, self._stream())
        return out

    def mul(self, a, b, level):
        out = self._out(a)
        self.ctx._call("helr_mul_relin_rescale", a.data_ptr(), b.data_ptr(), self.ctx.rlk.data_ptr(), out.data_ptr(),
                       a.shape[0], level, self._stream())
        return out

    def rotate(self, a, galois: int, level):
        out = self._out(a)
        self.ctx._call("helr_rotate", a.data_ptr(), int(galois), self.ctx.galois_key(galois).data_ptr(), out.data_ptr(),
                       a.shape[0], level, 0, self._stream())
        return out

    def imul(self, a, level):
        out = self._out(a)
        self.ctx._call("helr_imul", a.data_ptr(), out.data_ptr(), a.shape[0], level, self._stream())
        return out

    def mod_raise(self, a, level_out: int):
        out = self._out(a)
        self.ctx._call("helr_mod_raise", a.data_ptr(), out.data_ptr(), a.shape[0], level_out, self._stream())
        return out

    def cat(self, bufs):
        return self._torch.cat(list(bufs), dim=0).contiguous()

    def split(self, buf, parts: int):
        return [c.contiguous() for c in self._torch.chunk(buf, parts, dim=0)]
