#!/usr/bin/env python
"""NTT microbenchmark at the paper ring (N = 2^16, 40-bit scaling primes, so
every limb but q_0 takes the fp64 path): forward / inverse over B polynomials
x limbs 1..L-1 (fp64 limbs only) and over limb 0 (q_0, integer path).
Reports us per limb-transform and GB/s of algorithmic bytes (16 N per limb).

    python tools/ntt_micro.py [--batch 16] [--reps 20] [--once]
(--once: one forward + one inverse call, for an ncu capture)
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2406_13221_b200 import _lib  # noqa: E402
from paper_2406_13221_b200.ckks import GpuContext  # noqa: E402
from paper_2406_13221_b200.params import CkksParams  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--log-n", type=int, default=16)
    ap.add_argument("--once", action="store_true")
    a = ap.parse_args()
    ck = CkksParams.generate(log_n=a.log_n, n_q=8, dnum=2)
    ctx = GpuContext(ck, seed=3, max_batch=2)
    n, L, B = ck.n, ck.L, a.batch
    g = torch.Generator(device="cuda").manual_seed(3)
    data = torch.empty((B, L, n), dtype=torch.int64, device="cuda")
    for p in range(L):
        data[:, p].copy_(torch.randint(0, int(ck.q[p]), (B, n), device="cuda", generator=g, dtype=torch.int64))
    st = torch.cuda.current_stream().cuda_stream
    if a.once:  # profiled region only (ncu --profile-from-start off)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        _lib.call("helr_ntt_fwd", ctx.handle, data.data_ptr() + 8 * n, 1, L - 1, B, L * n, st)
        _lib.call("helr_ntt_inv", ctx.handle, data.data_ptr() + 8 * n, 1, L - 1, B, L * n, st)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    ref = data.clone()
    out = {}
    big = torch.empty((8 * B, 1, n), dtype=torch.int64, device="cuda")  # q_0 only, 8x the items
    big.copy_(torch.randint(0, int(ck.q[0]), (8 * B, 1, n), device="cuda", generator=g, dtype=torch.int64))
    for name, first, cnt in (("fp64", 1, L - 1), ("int_q0", 0, 1), ("mixed", 0, L), ("int_q0_big", 0, 1)):
        buf, items, stride = (big, 8 * B, n) if name == "int_q0_big" else (data, B, L * n)
        for d in ("fwd", "inv"):
            fn = lambda: _lib.call(f"helr_ntt_{d}", ctx.handle, buf.data_ptr() + 8 * n * first, first, cnt, items, stride,
                                   st)
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            limbs = items * cnt
            out[f"{name}_{d}"] = {"us_per_call": round(ms * 1e3, 2), "limbs": limbs,
                                  "us_per_limb": round(ms * 1e3 / limbs, 4),
                                  "gbs": round(16.0 * n * limbs / (ms * 1e-3) / 1e9, 1)}
    # round trip sanity: (reps+1) forward then (reps+1) inverse per group is identity
    out["roundtrip_identity"] = bool(torch.equal(data, ref))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
