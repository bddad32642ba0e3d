#!/usr/bin/env python
"""One fused GPU iteration started from the reference's exact state (W, V,
alpha, t) after `t0` iterations, compared with the reference's next state.
Isolates the per-iteration error from the trajectory's amplification."""
import json
import math
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import slotsim  # noqa: E402
from paper_2406_13221_b200 import data  # noqa: E402
from paper_2406_13221_b200.ckks import GpuContext  # noqa: E402
from paper_2406_13221_b200.driver import FusedTrainer  # noqa: E402
from paper_2406_13221_b200.encoding import replicate_rows  # noqa: E402
from paper_2406_13221_b200.optimizer import BASELINE_CUBIC, next_alpha  # noqa: E402
from paper_2406_13221_b200.params import CkksParams  # noqa: E402

QP = BASELINE_CUBIC.complement().padded(3)
CFG = {"medium": (data.medium_dataset, 15, 1024, 1, "mini_batch"),
       "paper_mini": (data.paper_dataset, 16, 128, 8, "mini_batch"),
       "toy": (data.toy_dataset, 13, 128, 1, "mini_batch")}


def slot_states(ds, log_n, m, blocks, iters, mode):
    """(W, V) after each iteration of the slot-level reference circuit."""
    states = []
    orig_boot = slotsim.SlotSim.bootstrap

    def boot(self, a):
        return orig_boot(self, a)
    trace, _ = slotsim.train(ds.X, ds.y, log_n, m, blocks, QP, lambda t: 1 + 10 * math.exp(-t), iters, mode=mode)
    return trace


def main(name, t0):
    make, log_n, m, blocks, mode = CFG[name]
    ds = make()
    # reference states: W after t0 and t0+1 iterations; V via a second sim pass
    sim_trace = slotsim_train_wv(ds, log_n, m, blocks, t0 + 1, mode)
    ck = CkksParams.generate(log_n=log_n, n_q=8, dnum=3)
    ctx = GpuContext(ck, seed=2, max_batch=8)
    tr = FusedTrainer(ctx, ds, rows_per_block=m, blocks_per_batch=blocks, mode=mode)
    (w0, v0), (w1, v1) = sim_trace[t0], sim_trace[t0 + 1]
    lay = tr.layout
    top = ck.top_level
    s = ck.level_scales[top]
    vals = np.stack([np.stack(replicate_rows(w0, lay)), np.stack(replicate_rows(v0, lay))]).reshape(-1, ck.slots)
    ctx.encrypt_to(ctx.encoder.encode(vals, s), tr.wv, top)
    tr.level, tr.s_w, tr.s_v, tr.t = top, s, s, t0
    a0 = 0.01
    a1 = next_alpha(a0)
    for _ in range(t0):
        a0, a1 = a1, next_alpha(a1)
    tr.alpha0, tr.alpha1 = a0, a1
    tr.iterate()
    w = tr.weights()
    # V readout
    C = tr.cols
    out = torch.empty((C, ck.n), dtype=torch.int64, device="cuda")
    ctx._call("helr_decrypt", ctx.sk.data_ptr(), tr.wv[C:].data_ptr(), C, tr.level, out.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    v = np.concatenate([np.real(ctx.encoder.decode(c, tr.s_v).reshape(lay.m, lay.g)[0]) for c in out.cpu().numpy()])
    v = v[: lay.cols]
    print(json.dumps(dict(workload=name, t0=t0, dw=float(np.abs(w - w1).max()), dv=float(np.abs(v - v1).max()),
                          w_absmax=float(np.abs(w1).max()), dw_rel=float(np.abs(w - w1).max() / np.abs(w1 - w0).max()))))


def slotsim_train_wv(ds, log_n, m, blocks, iters, mode):
    """Re-run the slot circuit keeping (W, V) row 0 after each iteration."""
    S = 1 << (log_n - 1)
    g = S // m
    out = []
    orig_train = slotsim.train

    class Cap(slotsim.SlotSim):
        pass
    # minimal re-implementation of slotsim.train's loop capturing V too
    sim = slotsim.SlotSim(log_n, 10 ** 7, 40, 40)
    n, cols = ds.X.shape
    Z = ds.X * ds.y[:, None]
    zb = slotsim._blocks(Z, m, g)
    rb, cb = zb.shape[0], zb.shape[1]
    cz = [[sim.enc(zb[i, j]) for j in range(cb)] for i in range(rb)]
    rpb = m * blocks
    nb = -(-rb // blocks)
    scal = [slotsim.bbar_of(ds.X[k * rpb:min((k + 1) * rpb, n)]) for k in range(nb)]
    cbar = [[sim.enc(v) for v in slotsim._replicate(s_, m, g, cb)] for s_ in scal]
    w = [sim.enc(np.zeros(S)) for _ in range(cb)]
    v = [sim.enc(np.zeros(S)) for _ in range(cb)]
    a0 = 0.01
    a1 = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * a0 * a0))
    row0 = lambda cts: np.concatenate([np.real(c.slots.reshape(m, g)[0]) for c in cts])[:cols]
    out.append((row0(w), row0(v)))
    for t in range(iters):
        b = t % nb
        blk = list(range(b * blocks, min((b + 1) * blocks, rb)))
        rows = min(rpb, n - b * rpb)
        lr = 1 + 10 * math.exp(-t)
        eta = (1.0 - a0) / a1
        gsum = None
        for k in blk:
            gk = slotsim.gradient_block(sim, cz[k], w, QP, m, g)
            gsum = gk if gsum is None else [sim.add(x, y) for x, y in zip(gsum, gk)]
        G = [sim.mul(gj, bj) for gj, bj in zip(gsum, cbar[b])]
        mult = 1.0 + lr / rows
        nw, nv = [], []
        for j in range(cb):
            vt = sim.add(w[j], sim.cmul(G[j], mult))
            nw.append(sim.add(sim.cmul(vt, 1.0 - eta), sim.cmul(v[j], eta)))
            nv.append(vt)
        w = [sim.bootstrap(c) for c in nw]
        v = [sim.bootstrap(c) for c in nv]
        a0, a1 = a1, 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * a1 * a1))
        out.append((row0(w), row0(v)))
    return out


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        name, t0 = spec.split(":")
        main(name, int(t0))
