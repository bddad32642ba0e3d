"""Training inputs: ``Dataset`` / ``make_dataset`` / ``build_z`` with the
reference's invariants (data.py:49-131), and the seeded synthetic workloads
of BASELINE.json (Toy, Medium, Paper shape), which stand in for the paper's
private financial data and for MNIST (not vendored).

Synthetic recipes:
- Toy: n=1,024, 15 features iid U[-1,1] + bias; beta* ~ N(0, 1/16) over the
  16 coefficients; y = +1 w.p. sigmoid(x . beta*) else -1; data seed 0.
- Medium: n=65,536, 63 features N(0, I) mixed by a random orthogonal 63x63
  matrix (QR of a Gaussian, seed 4), min-max to [-1, 1]; beta* ~ N(0, 1/64);
  bias solved by bisection for ~20% positives.
- Paper: n=422,108, 200 features U[-1,1] of which 20 columns (10%) are
  drawn from {-1, 1}; beta* ~ N(0, 1/256); ~20% positives.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["Dataset", "ZMatrix", "make_dataset", "build_z", "toy_dataset", "medium_dataset",
           "paper_dataset", "WORKLOADS"]


@dataclass(frozen=True, eq=False)
class Dataset:
    """Design matrix with an all-ones bias column and labels in {-1, +1}."""

    X: np.ndarray
    y: np.ndarray

    def __post_init__(self):
        X = np.asarray(self.X, dtype=np.float64)
        y = np.asarray(self.y, dtype=np.float64)
        object.__setattr__(self, "X", X)
        object.__setattr__(self, "y", y)
        if X.ndim != 2:
            raise ValueError(f"X must be 2-D, got shape {X.shape}")
        if y.shape != (X.shape[0],):
            raise ValueError(f"y has shape {y.shape}, expected ({X.shape[0]},)")
        if X.shape[0] == 0:
            raise ValueError("dataset is empty")
        if not np.all(np.isfinite(X)):
            raise ValueError("X contains non-finite values")
        if not np.all(X[:, 0] == 1.0):
            raise ValueError("column 0 of X must be the all-ones bias column")
        if not np.all((y == 1.0) | (y == -1.0)):
            raise ValueError("labels must be exactly -1 or +1")

    @property
    def n_samples(self) -> int:
        return int(self.X.shape[0])

    @property
    def n_features(self) -> int:
        return int(self.X.shape[1] - 1)


@dataclass(frozen=True, eq=False)
class ZMatrix:
    Z: np.ndarray


def make_dataset(features, labels) -> Dataset:
    """Prepend the bias column; {0,1} labels become {-1,+1} (data.py:116-127)."""
    feats = np.asarray(features, dtype=np.float64)
    lab = np.asarray(labels, dtype=np.float64)
    if set(np.unique(lab).tolist()) <= {0.0, 1.0}:
        lab = 2.0 * lab - 1.0
    return Dataset(np.column_stack([np.ones(feats.shape[0]), feats]), lab)


def build_z(ds: Dataset) -> ZMatrix:
    """Z[i] = y[i] * X[i] (data.py:130-131)."""
    return ZMatrix(ds.X * ds.y[:, None])


# --------------------------------------------------------------- workloads
def _logistic_labels(rng, X, beta):
    p = 1.0 / (1.0 + np.exp(-(X @ beta)))
    return np.where(rng.random(X.shape[0]) < p, 1.0, -1.0)


def _bias_for_rate(scores, rate):
    """Bias b with mean(sigmoid(scores + b)) == rate, by bisection."""
    lo, hi = -50.0, 50.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if np.mean(1.0 / (1.0 + np.exp(-(scores + mid)))) > rate:
            hi = mid
        else:
            lo = mid
    return 0.5 * (lo + hi)


def toy_dataset(seed: int = 0, n: int = 1024, f: int = 15) -> Dataset:
    rng = np.random.default_rng(seed)
    feats = rng.uniform(-1.0, 1.0, size=(n, f))
    X = np.column_stack([np.ones(n), feats])
    beta = rng.normal(0.0, np.sqrt(1.0 / (f + 1)), size=f + 1)
    return Dataset(X, _logistic_labels(rng, X, beta))


def medium_dataset(seed: int = 0, n: int = 65536, f: int = 63, positive_rate: float = 0.2) -> Dataset:
    rng = np.random.default_rng(seed)
    qr_rng = np.random.default_rng(4)
    Q, _ = np.linalg.qr(qr_rng.normal(size=(f, f)))
    raw = rng.normal(size=(n, f)) @ Q
    lo, hi = raw.min(axis=0), raw.max(axis=0)
    feats = 2.0 * (raw - lo) / (hi - lo) - 1.0
    beta = rng.normal(0.0, np.sqrt(1.0 / (f + 1)), size=f)
    scores = feats @ beta
    bias = _bias_for_rate(scores, positive_rate)
    X = np.column_stack([np.ones(n), feats])
    return Dataset(X, _logistic_labels(rng, X, np.r_[bias, beta]))


def paper_dataset(seed: int = 0, n: int = 422108, f: int = 200, binary_frac: float = 0.1,
                  positive_rate: float = 0.2) -> Dataset:
    rng = np.random.default_rng(seed)
    feats = rng.uniform(-1.0, 1.0, size=(n, f))
    nb = int(round(binary_frac * f))
    bcols = rng.choice(f, size=nb, replace=False)
    feats[:, bcols] = rng.choice([-1.0, 1.0], size=(n, nb))
    beta = rng.normal(0.0, np.sqrt(1.0 / 256.0), size=f)
    scores = feats @ beta
    bias = _bias_for_rate(scores, positive_rate)
    X = np.column_stack([np.ones(n), feats])
    return Dataset(X, _logistic_labels(rng, X, np.r_[bias, beta]))


# name -> (dataset factory, log_n, batch rows per ciphertext block, blocks per batch, iterations)
WORKLOADS = {
    "toy": dict(make=toy_dataset, log_n=13, rows=128, blocks=1, batch=128, epochs=3),
    "medium": dict(make=medium_dataset, log_n=15, rows=1024, blocks=1, batch=1024, epochs=5),
    "paper_mini": dict(make=paper_dataset, log_n=16, rows=128, blocks=8, batch=1024, epochs=3),
    "paper_full": dict(make=paper_dataset, log_n=16, rows=128, blocks=8, batch=1024, iterations=10),
}
