"""Plaintext side of the training path: the quadratic-gradient scales B̄,
the degree-3 sigmoid stand-ins, the step schedules and the NAG scalars,
plus the result metrics.  Semantics follow the reference modules cited per
symbol; the code is written independently.

- B̄ (``helr.quadgrad``): b_j = 1 / (eps + sum_k |(X'X/4)_jk|)
  (quadgrad.py:53-73), harmonic merge across batches (quadgrad.py:76-92).
- ``PolyApprox`` / ``G8`` / ``G16`` / ``complement`` (sigmoid.py:43-81), and
  ``BASELINE_CUBIC`` = 0.5 + 0.15012 x - 0.001593 x^3 (BASELINE.json configs).
- ``LrSchedule`` / ``f2`` (optim.py:53-83) and ``ExpDecay`` = 1 + 10 e^-t
  (BASELINE.json; not expressible by f2).
- ``TrainConfig`` (optim.py:157-178), ``next_alpha`` (optim.py:97-98),
  ``predict`` / ``accuracy`` / ``auroc`` / ``log_likelihood`` /
  ``gradient`` (optim.py:123-136, 200-229).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

DEFAULT_EPSILON = 1e-8
ALPHA0_INIT = 0.01
SIGMOID_CHOICES = ("exact", "g8", "g16")


# ----------------------------------------------------------------- B̄ scales
@dataclass(frozen=True, eq=False)
class QuadScaler:
    b: np.ndarray
    epsilon: float = DEFAULT_EPSILON

    def __post_init__(self):
        b = np.asarray(self.b, dtype=np.float64)
        object.__setattr__(self, "b", b)
        if b.ndim != 1:
            raise ValueError(f"scale vector must be 1-D, got shape {b.shape}")
        if not np.all(b > 0):
            raise ValueError("all scales must be strictly positive")
        if self.epsilon <= 0:
            raise ValueError(f"epsilon must be positive, got {self.epsilon}")

    def __len__(self) -> int:
        return int(self.b.shape[0])


def hessian_bound(X) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2:
        raise ValueError(f"design matrix must be 2-D, got shape {X.shape}")
    return (X.T @ X) / 4.0


def build_bbar(H, epsilon: float = DEFAULT_EPSILON) -> QuadScaler:
    H = np.asarray(H, dtype=np.float64)
    if H.ndim != 2 or H.shape[0] != H.shape[1]:
        raise ValueError(f"Hessian must be square, got shape {H.shape}")
    if epsilon <= 0:
        raise ValueError(f"epsilon must be positive, got {epsilon}")
    return QuadScaler(1.0 / (np.abs(H).sum(axis=1) + epsilon), epsilon)


def scaler_for(X, epsilon: float = DEFAULT_EPSILON) -> QuadScaler:
    return build_bbar(hessian_bound(X), epsilon)


def merge_bbar(scalers: Sequence[QuadScaler]) -> QuadScaler:
    if not scalers:
        raise ValueError("need at least one scaler to merge")
    dim = len(scalers[0])
    total = np.zeros(dim)
    for idx, s in enumerate(scalers):
        if len(s) != dim:
            raise ValueError(f"scaler {idx} has length {len(s)}, expected {dim}")
        total += 1.0 / s.b
    return QuadScaler(1.0 / total, max(s.epsilon for s in scalers))


def per_batch_scalers(X, batch_size: int, epsilon: float = DEFAULT_EPSILON) -> list:
    if batch_size < 1:
        raise ValueError(f"batch_size must be >= 1, got {batch_size}")
    X = np.asarray(X, dtype=np.float64)
    return [scaler_for(X[k:k + batch_size], epsilon) for k in range(0, X.shape[0], batch_size)]


def quad_gradient(scaler: QuadScaler, g) -> np.ndarray:
    g = np.asarray(g, dtype=np.float64)
    if g.shape != scaler.b.shape:
        raise ValueError(f"length mismatch: gradient {g.shape} vs scales {scaler.b.shape}")
    return scaler.b * g


# ----------------------------------------------------------------- sigmoid
def sigmoid(x):
    x = np.asarray(x, dtype=np.float64)
    out = np.where(x >= 0, 1.0 / (1.0 + np.exp(-np.abs(x))), np.exp(-np.abs(x)) / (1.0 + np.exp(-np.abs(x))))
    return float(out) if out.ndim == 0 else out


@dataclass(frozen=True, eq=False)
class PolyApprox:
    coefficients: tuple
    interval: tuple

    def __post_init__(self):
        lo, hi = self.interval
        if not lo < hi:
            raise ValueError(f"interval must satisfy lo < hi, got ({lo}, {hi})")
        if len(self.coefficients) == 0:
            raise ValueError("need at least one coefficient")
        if not all(np.isfinite(c) for c in self.coefficients):
            raise ValueError("coefficients must be finite")

    @property
    def degree(self) -> int:
        return len(self.coefficients) - 1

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64)
        acc = np.zeros_like(x) + self.coefficients[-1]
        for c in reversed(self.coefficients[:-1]):
            acc = acc * x + c
        return acc

    def complement(self) -> "PolyApprox":
        """1 - p(x), the polynomial on the gradient path (sigmoid.py:72-76)."""
        c = [-v for v in self.coefficients]
        c[0] += 1.0
        return PolyApprox(tuple(c), self.interval)

    def padded(self, degree: int = 3) -> tuple:
        if self.degree > degree:
            raise ValueError(f"circuit supports degree <= {degree}, got degree {self.degree}")
        return tuple(self.coefficients) + (0.0,) * (degree + 1 - len(self.coefficients))


G8 = PolyApprox((0.5, 0.15, 0.0, -0.0015), (-8.0, 8.0))
G16 = PolyApprox((0.5, 0.0843, 0.0, -0.0002), (-16.0, 16.0))
BASELINE_CUBIC = PolyApprox((0.5, 0.15012, 0.0, -0.001593), (-8.0, 8.0))


def poly_for(name: str) -> PolyApprox:
    table = {"g8": G8, "g16": G16, "baseline": BASELINE_CUBIC}
    if name not in table:
        raise ValueError(f"no polynomial form for sigmoid {name!r}")
    return table[name]


# ----------------------------------------------------------------- schedules
@dataclass(frozen=True)
class LrSchedule:
    """max - (max - min) (t/T)^gamma, clamped past T (optim.py:53-76)."""

    max: float
    min: float
    T: int
    gamma: float

    def __post_init__(self):
        if self.max < self.min:
            raise ValueError(f"need max >= min, got {self.max} < {self.min}")
        if self.T < 1:
            raise ValueError(f"need T >= 1, got {self.T}")
        if self.gamma <= 0:
            raise ValueError(f"need gamma > 0, got {self.gamma}")

    @classmethod
    def constant(cls, value: float) -> "LrSchedule":
        return cls(max=value, min=value, T=1, gamma=1.0)

    def __call__(self, t: int) -> float:
        return f2(self, t)


def f2(schedule: LrSchedule, t: int) -> float:
    if t < 0:
        raise ValueError(f"iteration count must be >= 0, got {t}")
    frac = min(t, schedule.T) / schedule.T
    return schedule.max - (schedule.max - schedule.min) * frac ** schedule.gamma


@dataclass(frozen=True)
class ExpDecay:
    """lr(t) = base + amp * exp(-t) with t the 0-based NAG step (BASELINE.json)."""

    base: float = 1.0
    amp: float = 10.0

    def __call__(self, t: int) -> float:
        if t < 0:
            raise ValueError(f"iteration count must be >= 0, got {t}")
        return self.base + self.amp * math.exp(-t)


def lr_at(schedule, t: int) -> float:
    return f2(schedule, t) if isinstance(schedule, LrSchedule) else float(schedule(t))


def next_alpha(alpha: float) -> float:
    return 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * alpha * alpha))


@dataclass(frozen=True)
class TrainConfig:
    """Same fields and checks as optim.py:157-178."""

    mode: str = "full_batch"
    batch_size: int = 1024
    epochs: Optional[int] = None
    max_iterations: int = 26
    schedule: object = field(default_factory=lambda: LrSchedule(2.0, 1.0, 36, 2.5))
    sigmoid: str = "exact"
    shuffle: bool = False
    seed: int = 0

    def __post_init__(self):
        if self.mode not in ("full_batch", "mini_batch"):
            raise ValueError(f"mode must be full_batch or mini_batch, got {self.mode!r}")
        if self.batch_size < 1:
            raise ValueError(f"batch_size must be >= 1, got {self.batch_size}")
        if self.max_iterations < 0:
            raise ValueError(f"max_iterations must be >= 0, got {self.max_iterations}")
        if self.sigmoid not in SIGMOID_CHOICES + ("baseline",):
            raise ValueError(f"sigmoid must be one of {SIGMOID_CHOICES}, got {self.sigmoid!r}")
        if self.epochs is not None and self.epochs < 1:
            raise ValueError(f"epochs must be >= 1, got {self.epochs}")


# ----------------------------------------------------------------- metrics
def log_likelihood(Z, w) -> float:
    u = np.asarray(Z) @ np.asarray(w)
    return float(-np.mean(np.logaddexp(0.0, -u)))


def gradient(Z, w, sig=sigmoid) -> np.ndarray:
    Z = np.asarray(Z)
    return Z.T @ (1.0 - np.asarray(sig(Z @ np.asarray(w))))


def predict(w, X) -> np.ndarray:
    return np.where(np.asarray(X) @ np.asarray(w) >= 0.0, 1.0, -1.0)


def accuracy(y_true, y_pred) -> float:
    return float(np.mean(np.asarray(y_true) == np.asarray(y_pred)))


def auroc(y_true, scores) -> float:
    """Midrank (tie-averaged) rank-sum AUROC (optim.py:209-229)."""
    y = np.asarray(y_true)
    s = np.asarray(scores, dtype=np.float64)
    pos = y > 0
    n_pos = int(pos.sum())
    n_neg = s.shape[0] - n_pos
    if n_pos == 0 or n_neg == 0:
        raise ValueError("AUROC undefined: only one class present")
    order = np.argsort(s, kind="mergesort")
    ss = s[order]
    # group equal scores; each group gets the mean of its 1-based ranks
    starts = np.flatnonzero(np.r_[True, ss[1:] != ss[:-1]])
    ends = np.r_[starts[1:], ss.shape[0]]
    ranks_sorted = np.repeat(0.5 * (starts + ends - 1) + 1.0, ends - starts)
    ranks = np.empty_like(ranks_sorted)
    ranks[order] = ranks_sorted
    return (float(ranks[pos].sum()) - n_pos * (n_pos + 1) / 2.0) / (n_pos * n_neg)
