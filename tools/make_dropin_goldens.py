"""Generate tests/golden/dropin.npz by running the REFERENCE's own
``train_encrypted`` (pkg/src/helr/enctrain.py:303-449, unchanged, over its
SimContext) on small toy problems.  Run in the build container only:

    python tools/make_dropin_goldens.py

tests/test_gpu_dropin.py then runs the product's ``train_encrypted`` with
``ctx=GpuContext`` (real RNS-CKKS on the B200) on the same inputs and
compares weight traces within 1e-6 and ledgers (bootstrap cadence,
consumed bits in units of the context's level cost).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, "/root/reference/pkg/src")

from helr.data import make_dataset  # noqa: E402  (reference)
from helr.enctrain import train_encrypted  # noqa: E402
from helr.hesim import HeParams  # noqa: E402
from helr.optim import LrSchedule, TrainConfig  # noqa: E402

OUT = ROOT / "tests" / "golden" / "dropin.npz"

# name: (n rows, features, mode, sigmoid, enhanced, schedule args, iterations, batch)
CASES = {
    "mini_g8": (6, 3, "mini_batch", "g8", True, (2.0, 1.0, 36, 2.5), 7, 4),
    "full_g16": (6, 3, "full_batch", "g16", True, (2.0, 1.0, 36, 2.5), 7, 4),
    "baseline_g8": (6, 3, "mini_batch", "g8", False, (1.0, 1.0, 36, 2.5), 7, 4),
    "mini_2col": (8, 20, "mini_batch", "g8", True, (2.0, 1.0, 36, 2.5), 6, 4),
}


def main():
    rng = np.random.default_rng(2406)
    out = {}
    for name, (n, f, mode, sig, enh, sched, iters, batch) in CASES.items():
        X = rng.uniform(0.0, 1.0, size=(n, f))
        y = rng.choice([-1.0, 1.0], size=n)
        y[0], y[1] = 1.0, -1.0
        ds = make_dataset(X, y)
        cfg = TrainConfig(mode=mode, batch_size=batch, max_iterations=iters, schedule=LrSchedule(*sched), sigmoid=sig)
        res = train_encrypted(ds, cfg, HeParams(log_n=5, log_q=2000), enhanced=enh, trace_weights=True)
        out[f"{name}_X"] = X
        out[f"{name}_y"] = y
        out[f"{name}_trace"] = np.array(res.weight_trace)
        out[f"{name}_final"] = res.weights
        out[f"{name}_muls"] = np.array([r["muls"] for r in res.ledger])
        out[f"{name}_cmuls"] = np.array([r["cmuls"] for r in res.ledger])
        out[f"{name}_rotations"] = np.array([r["rotations"] for r in res.ledger])
        print(name, res.weights)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
