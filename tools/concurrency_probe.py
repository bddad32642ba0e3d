#!/usr/bin/env python
"""How much does the step gain if two independent iterations share the GPU?
Two trainers (two contexts, paper shape, 16 batches each) iterate on their own
streams, alone and interleaved; aggregate iterations/s is compared.  Upper
bound for splitting one iteration's row blocks over two graph branches."""
import json
import sys
import threading
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2406_13221_b200 import data  # noqa: E402
from paper_2406_13221_b200.ckks import GpuContext  # noqa: E402
from paper_2406_13221_b200.driver import FusedTrainer  # noqa: E402
from paper_2406_13221_b200.params import CkksParams  # noqa: E402

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ds = data.paper_dataset(n=128 * blocks * 16)
ck = CkksParams.generate(log_n=16, n_q=8, dnum=2)
trs = []
for seed in (1, 2):
    ctx = GpuContext(ck, seed=seed, max_batch=8)
    trs.append(FusedTrainer(ctx, ds, rows_per_block=128, blocks_per_batch=blocks, mode="mini_batch", use_graph=True))
for tr in trs:
    for _ in range(3):
        tr.iterate()
torch.cuda.synchronize()
N = 60


def timed(which):
    evs = []
    for tr in which:
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(tr.stream)
        evs.append(e0)
    if len(which) == 1:
        for _ in range(N):
            which[0].iterate()
    else:
        th = [threading.Thread(target=lambda t=tr: [t.iterate() for _ in range(N)]) for tr in which]
        for t in th:
            t.start()
        for t in th:
            t.join()
    ends = []
    for tr in which:
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(tr.stream)
        ends.append(e1)
    torch.cuda.synchronize()
    ms = max(a.elapsed_time(b) for a, b in zip(evs, ends))
    return len(which) * N / (ms / 1000.0)


out = {"blocks_per_batch": blocks, "alone": round(timed(trs[:1]), 2), "two_interleaved_aggregate": round(timed(trs), 2),
       "alone_again": round(timed(trs[1:]), 2)}
print(json.dumps(out))
