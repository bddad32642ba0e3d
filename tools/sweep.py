#!/usr/bin/env python
"""Primitive sweep (BASELINE.json config 2): batched forward/inverse NTT,
ct x ct multiply + relinearise, rescale and rotate-by-2^k key switch over
N in {2^14, 2^15, 2^16}, L in {8, 16, 24} primes (q0 ~ 2^60, 50-bit scaling
primes here), dnum in {1, 3}, batches of 1..64 ciphertexts with uniformly
random residues.  Device time by CUDA events; algorithmic bytes per
SURVEY.md §8(d):
  NTT        2 * limbs * N * 8          per polynomial (read + write)
  rotate     (2l + 2 beta (l+K) + 2l) N 8
  mul+relin  (4l + 2 beta (l+K) + 2l) N 8   (rescale excluded)
  rescale    (2l + 2(l-1)) N 8

    python tools/sweep.py [--quick] [--json out.json]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2406_13221_b200 import _lib  # noqa: E402
from paper_2406_13221_b200.ckks import GpuContext  # noqa: E402
from paper_2406_13221_b200.params import CkksParams  # noqa: E402


def peak():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6650.0


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


SCALE_BITS = 50


def run(log_n, L, dnum, batch, ops):
    ck = CkksParams.generate(log_n=log_n, n_q=L, dnum=dnum, scale_bits=SCALE_BITS)
    ctx = GpuContext(ck, seed=3, max_batch=batch)
    n, K = ck.n, ck.K
    beta = -(-L // ck.alpha)
    g = torch.Generator(device="cuda").manual_seed(3)
    cts = ctx._empty((batch, 2, L, n))
    for p in range(L):  # uniform residues per limb
        cts[:, :, p].copy_(torch.randint(0, int(ck.q[p]), (batch, 2, n), device="cuda", generator=g,
                                         dtype=torch.int64))
    cts2 = cts.roll(1, dims=0).contiguous()
    out = torch.empty_like(cts)
    st = torch.cuda.current_stream().cuda_stream
    lvl = L - 1
    res = []
    if "ntt" in ops:
        data = cts.clone()
        ms = timed(lambda: _lib.call("helr_ntt_fwd", ctx.handle, data.data_ptr(), 0, L, 2 * batch, L * n, st))
        ms_i = timed(lambda: _lib.call("helr_ntt_inv", ctx.handle, data.data_ptr(), 0, L, 2 * batch, L * n, st))
        by = 2 * L * n * 8 * 2 * batch
        res.append(("ntt_fwd", ms, by))
        res.append(("ntt_inv", ms_i, by))
    if "mul" in ops:
        ms = timed(lambda: _lib.call("helr_mul_relin", ctx.handle, cts.data_ptr(), cts2.data_ptr(), ctx.rlk.data_ptr(),
                                     out.data_ptr(), batch, lvl, st))
        res.append(("mul_relin", ms, (4 * L + 2 * beta * (L + K) + 2 * L) * n * 8 * batch))
    if "rescale" in ops:
        ms = timed(lambda: _lib.call("helr_rescale", ctx.handle, cts.data_ptr(), out.data_ptr(), batch, lvl, st))
        res.append(("rescale", ms, (2 * L + 2 * (L - 1)) * n * 8 * batch))
    if "rotate" in ops:
        gal = ctx.galois_for_rotation(1 << 3)
        gk = ctx.galois_key(gal)
        ms = timed(lambda: _lib.call("helr_rotate", ctx.handle, cts.data_ptr(), gal, gk.data_ptr(), out.data_ptr(), batch,
                                     lvl, 0, st))
        res.append(("rotate", ms, (2 * L + 2 * beta * (L + K) + 2 * L) * n * 8 * batch))
    if "rotsum" in ops:
        import ctypes
        steps = list(range(1, 16))
        gals = [ctx.galois_for_rotation(k) for k in steps]
        keys = [ctx.galois_key(x) for x in gals]
        garr = (ctypes.c_int64 * len(gals))(*gals)
        karr = (ctypes.c_void_p * len(keys))(*[k.data_ptr() for k in keys])
        lv = min(lvl, 6)
        ms = timed(lambda: _lib.call("helr_rotsum", ctx.handle, cts.data_ptr(), len(gals), garr, karr, out.data_ptr(),
                                     batch, lv, 1, st))
        nl = lv + 1
        nd = -(-nl // ck.alpha)
        by = (4 * nl + len(steps) * 2 * nd * (nl + K) / batch + 2 * nd * (nl + K) + 2 * nl) * n * 8 * batch
        res.append(("rotsum15", ms, by))
    del ctx
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--json", default=None)
    ap.add_argument("--ops", default="ntt,mul,rescale,rotate,rotsum")
    ap.add_argument("--scale-bits", type=int, default=50, help="scaling-prime size (< 41 bits: fp64 NTT path)")
    a = ap.parse_args()
    global SCALE_BITS
    SCALE_BITS = a.scale_bits
    ops = a.ops.split(",")
    P = peak()
    grid = [(16, 8, 3, 8), (16, 8, 3, 64)] if a.quick else [
        (ln, L, d, b) for ln in (14, 15, 16) for L in (8, 16, 24) for d in (1, 3) for b in (1, 8, 64)]
    rows = []
    for (ln, L, d, b) in grid:
        mem = 2 * L * (1 << ln) * 8 * b
        if mem * 6 > 60e9:  # keep the sweep bounded in memory
            continue
        try:
            for name, ms, by in run(ln, L, d, b, ops):
                gbs = by / (ms / 1e3) / 1e9
                row = dict(op=name, log_n=ln, L=L, dnum=d, batch=b, scale_bits=SCALE_BITS, ms=ms, gbs=gbs, frac=gbs / P)
                rows.append(row)
                print(json.dumps(row), flush=True)
        except Exception as exc:  # report and continue the sweep
            print(json.dumps(dict(log_n=ln, L=L, dnum=d, batch=b, error=str(exc)[:200])), flush=True)
    if a.json:
        Path(a.json).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
