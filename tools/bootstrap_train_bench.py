#!/usr/bin/env python
"""Paper-shape mini-batch iterations with REAL CKKS bootstrapping of W and V
before every iteration (bootstrap='ckks'), next to the same iterations with
the refresh stand-in: device time per iteration and the weight difference
between the two runs (the stand-in run is the one pinned to the reference
goldens within 1e-6, tests/test_gpu_train.py).

The dataset is the paper generator truncated to `--batches` mini-batches of
1,024 rows x 200 features (the bootstrappable chain has 24 limbs, so the full
413-batch dataset would be 3x the 28 GB of the 8-limb chain).

    python tools/bootstrap_train_bench.py [--batches 16] [--iters 16]
"""
from __future__ import annotations

import argparse
import gc
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2406_13221_b200 import data  # noqa: E402
from paper_2406_13221_b200.bootstrap import bootstrap_ring  # noqa: E402
from paper_2406_13221_b200.ckks import GpuContext  # noqa: E402
from paper_2406_13221_b200.driver import FusedTrainer  # noqa: E402
from paper_2406_13221_b200.params import CkksParams  # noqa: E402


def run(ctx, ds, iters, warm=2):
    tr = FusedTrainer(ctx, ds, rows_per_block=128, blocks_per_batch=8, mode="mini_batch", use_graph=True)
    ws = []
    for _ in range(warm):
        tr.iterate()
        ws.append(tr.weights())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(tr.stream)
    for _ in range(iters):
        tr.iterate()
    e1.record(tr.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    ws.append(tr.weights())
    boots = ctx.counters["bootstrap"]
    tr.close()
    return ms, ws, boots


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=16)
    ap.add_argument("--iters", type=int, default=16)
    ap.add_argument("--work-levels", type=int, default=7, help="7: one iteration per bootstrap; 14: two")
    ap.add_argument("--dnum", type=int, default=None)
    a = ap.parse_args()
    ds = data.paper_dataset(n=1024 * a.batches)
    out = {"rows": ds.n_samples, "features": 200, "iters": a.iters}
    ck = CkksParams.generate(log_n=16, n_q=8, dnum=2)
    ctx = GpuContext(ck, seed=1, max_batch=8)
    ms0, w0, b0 = run(ctx, ds, a.iters)
    out["standin"] = {"ms_per_iteration": round(ms0, 3), "L": ck.L, "K": ck.K, "dnum": ck.dnum}
    del ctx
    gc.collect()
    torch.cuda.empty_cache()
    ckb = bootstrap_ring(16, work_levels=a.work_levels, dnum=a.dnum)
    ctxb = GpuContext(ckb, seed=1, max_batch=8, bootstrap="ckks")
    ms1, w1, b1 = run(ctxb, ds, a.iters)
    out["real_bootstrap"] = {"ms_per_iteration": round(ms1, 3), "iterations_per_s": round(1000.0 / ms1, 3),
                             "L": ckb.L, "K": ckb.K, "dnum": ckb.dnum, "work_levels": a.work_levels,
                             "bootstrapped_ciphertexts": b1,
                             "bootstrap_share": round(1.0 - ms0 / ms1, 3)}
    out["max_weight_difference"] = [float(np.max(np.abs(x - y))) for x, y in zip(w0, w1)]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
