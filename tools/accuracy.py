#!/usr/bin/env python
"""Long-run value parity of the fused GPU trainer against the reference
goldens (tests/golden): every recorded iteration of a whole run.
    python tools/accuracy.py [toy|medium|paper_mini|paper_full ...]"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2406_13221_b200 import data  # noqa: E402
from paper_2406_13221_b200.ckks import GpuContext  # noqa: E402
from paper_2406_13221_b200.driver import FusedTrainer  # noqa: E402
from paper_2406_13221_b200.optimizer import auroc  # noqa: E402
from paper_2406_13221_b200.params import CkksParams  # noqa: E402

CFG = {
    "toy": (data.toy_dataset, 13, 128, 1, "mini_batch"),
    "medium": (data.medium_dataset, 15, 1024, 1, "mini_batch"),
    "paper_mini": (data.paper_dataset, 16, 128, 8, "mini_batch"),
    "paper_full": (data.paper_dataset, 16, 128, 8, "full_batch"),
}


def run(name, refresh_bits=None, dnum=2):
    make, log_n, rows, blocks, mode = CFG[name]
    gold = np.load(ROOT / "tests" / "golden" / f"{name}.npz")
    ds = make()
    ctx = GpuContext(CkksParams.generate(log_n=log_n, n_q=8, dnum=dnum), seed=2, max_batch=8)
    kw = {} if refresh_bits is None else dict(refresh_bits=refresh_bits)
    tr = FusedTrainer(ctx, ds, rows_per_block=rows, blocks_per_batch=blocks, mode=mode, use_graph=True, **kw)
    refresh_bits = tr.refresh_bits
    its = [int(x) for x in gold["iterations"]]
    worst_w = worst_a = 0.0
    curve = []
    t0 = time.time()
    for t in range(1, its[-1] + 1):
        tr.iterate()
        if t in its:
            k = its.index(t)
            w = tr.weights()
            dw = float(np.max(np.abs(w - gold["weights"][k])))
            da = abs(auroc(ds.y, ds.X @ w) - float(gold["auc"][k]))
            worst_w, worst_a = max(worst_w, dw), max(worst_a, da)
            curve.append((t, dw, da))
    out = dict(workload=name, refresh_bits=refresh_bits, dnum=dnum, iterations=its[-1], max_abs_dw=worst_w, max_abs_dauc=worst_a,
               final_auc=float(gold["auc"][-1]), seconds=time.time() - t0,
               curve=curve if len(curve) < 400 else [c for c in curve if c[0] % 16 == 0])
    print(json.dumps(out), flush=True)
    tr.close()


if __name__ == "__main__":
    # spec: name[:refresh_bits[:dnum]]
    for spec in sys.argv[1:] or ["toy", "medium", "paper_mini"]:
        parts = spec.split(":")
        bits = int(parts[1]) if len(parts) > 1 and parts[1] else None
        dn = int(parts[2]) if len(parts) > 2 else 2
        run(parts[0], bits, dn)
