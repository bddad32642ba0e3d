#!/usr/bin/env python
"""Real CKKS bootstrapping at a given ring (default the paper ring N = 2^16):
precision against the encrypted slots and device time of one batched bootstrap
of `count` ciphertexts (W and V: count = 2), plus the key / plaintext memory.

    python tools/bootstrap_bench.py [--log-n 16] [--count 2] [--reps 3] [--scale-bits 40]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2406_13221_b200.bootstrap import BootstrapConfig, bootstrap_ring  # noqa: E402
from paper_2406_13221_b200.ckks import GpuContext  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log-n", type=int, default=16)
    ap.add_argument("--count", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--scale-bits", type=int, default=40)
    ap.add_argument("--in-bits", type=int, default=48, help="scale of the exhausted input on q_0 (the trainer's W', V')")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--dnum", type=int, default=None)
    ap.add_argument("--p-bits", type=int, default=60)
    ap.add_argument("--c2s", type=int, default=3)
    ap.add_argument("--s2c", type=int, default=3)
    a = ap.parse_args()
    cfg = BootstrapConfig(c2s_groups=a.c2s, s2c_groups=a.s2c)
    P = bootstrap_ring(a.log_n, work_levels=7, scale_bits=a.scale_bits, cfg=cfg, dnum=a.dnum, p_bits=a.p_bits)
    t0 = time.time()
    ctx = GpuContext(P, seed=3, max_batch=max(4, 2 * a.count), bootstrap="ckks")
    bs = ctx.bootstrapper()
    rng = np.random.default_rng(0)
    z = rng.uniform(-1, 1, size=(a.count, P.slots))
    s_in = float(2 ** a.in_bits)
    buf = ctx._empty((a.count, 2, P.L, P.n))
    ctx.encrypt_to(ctx.encoder.encode(z, s_in), buf, 0)      # level-0 ciphertexts at the trainer's bottom scale
    torch.cuda.synchronize()
    boot = lambda: ctx.bootstrap_batch(buf, 0, s_in, use_graph=not a.no_graph)
    out, lvl, sc = boot()                                     # first call: keys, plaintext diagonals, graph capture
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    ms = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out, lvl, sc = boot()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    errs = []
    for b in range(a.count):
        ct = ctx._wrap(out[b], lvl, sc)
        errs.append(float(np.max(np.abs(ctx.dec(ct).real - z[b]))))
    keys = len(ctx._gks) + 1
    key_gb = keys * ctx.rlk.numel() * 8 / 1e9
    pt_gb = sum(t.numel() * 8 for pts, _ in bs._pt_cache.values() for t in pts.values()) / 1e9
    print(json.dumps({"log_n": a.log_n, "L": P.L, "K": P.K, "dnum": P.dnum, "count": a.count, "depth": cfg.depth,
                      "out_level": lvl, "ms_per_bootstrap": round(min(ms), 2), "ms_all": [round(x, 2) for x in ms],
                      "max_err": max(errs), "cuda_graph": not a.no_graph, "switch_keys": keys, "key_gb": round(key_gb, 2),
                      "plaintext_gb": round(pt_gb, 2), "setup_s": round(setup_s, 1),
                      "counters": {k: v for k, v in ctx.counters.items() if v}}))


if __name__ == "__main__":
    main()
