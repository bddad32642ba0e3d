"""Training-harness metrics on the device (helr_metrics, csrc/metrics.cu;
SURVEY.md §8(f) row 4).

The reference computes, every iteration of ``train_encrypted``
(enctrain.py:417-436), the log-likelihood (optim.py:123-126), the
training / validation accuracy (optim.py:200-206) and the midrank AUROC
(optim.py:209-229) on the host — about 51 ms per iteration at the paper
shape.  ``DeviceMetrics`` keeps X and y resident on the GPU and evaluates
all of them in one call (one pass over X, a bitonic sort of the scores, an
exact fp64 midrank sum); the values match ``optimizer.py``'s restatement of
the reference functions (tests/test_gpu_metrics.py).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

__all__ = ["DeviceMetrics"]


class DeviceMetrics:
    """X (n x d, bias column included) and labels y in {-1, +1} resident on
    the device of ``ctx``; ``evaluate(w)`` returns the reference's metrics."""

    def __init__(self, ctx, X, y):
        X = np.ascontiguousarray(X, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64).ravel()
        if X.ndim != 2 or X.shape[0] != y.shape[0] or X.shape[0] < 1:
            raise ValueError("X must be n x d with n labels")
        self.ctx = ctx
        self.n, self.d = X.shape
        self.X = torch.from_numpy(X).to(ctx.device)
        self.y = torch.from_numpy(y).to(ctx.device)
        lib = _lib.load()
        lib.helr_metrics_scratch.restype = ctypes.c_size_t
        lib.helr_metrics_scratch.argtypes = [ctypes.c_int]
        self.scratch = torch.empty(int(lib.helr_metrics_scratch(self.n)), dtype=torch.float64, device=ctx.device)
        self._w = torch.empty(self.d, dtype=torch.float64, device=ctx.device)

    def evaluate(self, w) -> dict:
        w = np.ascontiguousarray(w, dtype=np.float64).ravel()
        if w.shape[0] != self.d:
            raise ValueError(f"weights have {w.shape[0]} entries, X has {self.d} columns")
        self._w.copy_(torch.from_numpy(w))
        out = (ctypes.c_double * 4)()
        self.ctx._call("helr_metrics", self.X.data_ptr(), self.y.data_ptr(), self._w.data_ptr(), self.n, self.d,
                       self.scratch.data_ptr(), out, torch.cuda.current_stream().cuda_stream)
        auc = float(out[2])
        return {"log_likelihood": float(out[0]), "accuracy": float(out[1]), "auroc": None if np.isnan(auc) else auc,
                "n_pos": int(out[3])}

    def auroc(self, w) -> float:
        """Midrank AUROC of X w; raises like the reference with one class."""
        r = self.evaluate(w)["auroc"]
        if r is None:
            raise ValueError("AUROC undefined: only one class present")
        return r
