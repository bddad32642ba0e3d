#!/usr/bin/env python
"""Run exactly the bench workload and bracket ONE training step (after the
bench's warm-up) with cudaProfilerStart/Stop, so that

    ncu --profile-from-start off --metrics gpu__time_duration.sum,... \
        python tools/profile_step.py [--workload paper_mini] [--graph]

lists exactly the launches of one step.  Eager launches by default (the same
kernels the captured graph replays, without graph-node indirection).

    python tools/profile_step.py --steps 2    # profile two consecutive steps
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="paper_mini", choices=list(bench.WORKLOADS))
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--steps", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_2406_13221_b200.ckks import GpuContext
    from paper_2406_13221_b200.driver import FusedTrainer
    from paper_2406_13221_b200.params import CkksParams

    wl = bench.WORKLOADS[a.workload]
    ck = CkksParams.generate(log_n=wl["log_n"], n_q=wl["L"], dnum=wl["dnum"])
    ctx = GpuContext(ck, seed=1, max_batch=max(8, wl["blocks"]))
    ds = bench.make_dataset(wl["data"])
    tr = FusedTrainer(ctx, ds, rows_per_block=wl["rows"], blocks_per_batch=wl["blocks"], mode=wl["mode"],
                      use_graph=a.graph)
    for _ in range(max(1, a.warmup)):
        tr.iterate()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(a.steps):
        tr.iterate()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    tr.close()
    print(f"profiled {a.steps} step(s) of {a.workload}", flush=True)


if __name__ == "__main__":
    main()
