"""Generate tests/golden/*.npz by running the REFERENCE implementation
(/root/reference/pkg/src/helr, imported read-only) on the BASELINE
synthetic workloads.  Run in the build container only:

    python tools/make_goldens.py [toy medium paper_mini paper_full ops]

The reference is composed exactly as SURVEY.md §8(c) prescribes: its own
SimContext / plan_layout / pack_matrix / replicate_rows / scaler_for /
merge_bbar / enc_gradient / enc_quad_gradient / enc_nag_update, with the
BASELINE cubic (0.5, 0.15012, 0, -0.001593), lr = 1 + 10 e^-t (t = the
0-based NAG step), eps = 1e-8, alpha0 = 0.01, B̄ per 1,024-row batch (or
per batch of the Toy/Medium layouts), gamma = lr / real rows of the batch
(mini) or lr / n (full), and a deep log_q so no refresh is needed (the
simulator's refresh preserves values anyway).  The datasets come from
paper_2406_13221_b200.data (seeded numpy) so the GPU box regenerates the
identical inputs without the reference.
"""

from __future__ import annotations

import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from helr import enctrain as R_enc  # noqa: E402  (reference)
from helr.encoding import pack_matrix, plan_layout, replicate_rows  # noqa: E402
from helr.hesim import HeParams, SimContext  # noqa: E402
from helr.optim import auroc  # noqa: E402
from helr.quadgrad import merge_bbar, scaler_for  # noqa: E402
from helr.sigmoid import PolyApprox  # noqa: E402

from paper_2406_13221_b200.data import medium_dataset, paper_dataset, toy_dataset  # noqa: E402

OUT = ROOT / "tests" / "golden"
CUBIC = PolyApprox((0.5, 0.15012, 0.0, -0.001593), (-8.0, 8.0))


def lr_fn(t):
    return 1.0 + 10.0 * math.exp(-t)


def run(ds, log_n, m, blocks_per_batch, iterations, mode, keep):
    params = HeParams(log_n=log_n, log_q=10 ** 6, log_delta=40, log_delta_c=40)
    ctx = SimContext(params)
    lay = plan_layout(ds.n_samples, ds.n_features, params, m)
    Z = ds.y[:, None] * ds.X
    blocks = pack_matrix(Z, lay)
    ct_z = [[ctx.enc(v) for v in row] for row in blocks]
    rows_per_batch = m * blocks_per_batch
    nb = -(-lay.row_blocks // blocks_per_batch)
    scalers = [scaler_for(ds.X[k * rows_per_batch:min((k + 1) * rows_per_batch, ds.n_samples)]) for k in range(nb)]
    if mode == "full_batch":
        ct_b = [[ctx.enc(v) for v in replicate_rows(merge_bbar(scalers).b, lay)]]
    else:
        ct_b = [[ctx.enc(v) for v in replicate_rows(s.b, lay)] for s in scalers]
    zeros = np.zeros(lay.slots)
    st = R_enc.EncModelState(
        ct_w=tuple(ctx.enc(zeros) for _ in range(lay.col_blocks)),
        ct_v=tuple(ctx.enc(zeros) for _ in range(lay.col_blocks)),
        alpha0=R_enc.ALPHA0_INIT, alpha1=R_enc._next_alpha(R_enc.ALPHA0_INIT))
    trace, aucs, its = [], [], []
    t0 = time.time()
    for t in range(iterations):
        if mode == "mini_batch":
            b = t % nb
            blk = range(b * blocks_per_batch, min((b + 1) * blocks_per_batch, lay.row_blocks))
            rows = min(rows_per_batch, ds.n_samples - b * rows_per_batch)
            bsel = ct_b[b]
        else:
            blk = range(lay.row_blocks)
            rows = ds.n_samples
            bsel = ct_b[0]
        lr = lr_fn(st.t)
        eta = (1.0 - st.alpha0) / st.alpha1
        acc = None
        for k in blk:
            gk = R_enc.enc_gradient(ctx, tuple(ct_z[k]), st.ct_w, CUBIC, lay)
            acc = gk if acc is None else [ctx.add(a, c) for a, c in zip(acc, gk)]
        G = R_enc.enc_quad_gradient(ctx, acc, tuple(bsel))
        st = R_enc.enc_nag_update(ctx, st, G, eta=eta, gamma=lr / rows)
        st = R_enc._refresh(ctx, st)
        if keep(t, iterations):
            w = R_enc.decode_weights(ctx, st.ct_w, lay)
            trace.append(w)
            its.append(t + 1)
            aucs.append(auroc(ds.y, ds.X @ w))
    return dict(weights=np.array(trace), iterations=np.array(its), auc=np.array(aucs),
                seconds=time.time() - t0, final=R_enc.decode_weights(ctx, st.ct_w, lay))


def keep_all(t, n):
    return True


def keep_sparse(t, n):
    return t < 32 or (t + 1) % 16 == 0 or t == n - 1


def ops_vectors():
    """Reference simulator op outputs on small seeded inputs (semantics pins)."""
    rng = np.random.default_rng(77)
    params = HeParams(log_n=6, log_q=500, log_delta=40, log_delta_c=40)
    ctx = SimContext(params)
    lay = plan_layout(8, 3, params, batch_rows=8)  # 8 x 4
    x = rng.normal(size=32)
    y = rng.normal(size=32)
    a, b = ctx.enc(x), ctx.enc(y)
    out = dict(x=x, y=y)
    out["rot1"] = ctx.dec(ctx.rotate(a, 1))
    out["rot_m3"] = ctx.dec(ctx.rotate(a, -3))
    out["mul"] = ctx.dec(ctx.mul(a, b))
    out["cmul"] = ctx.dec(ctx.cmul(a, y))
    out["cadd"] = ctx.dec(ctx.cadd(a, 0.25))
    out["imul"] = ctx.dec(ctx.imul(a))
    out["sum_col_vec"] = ctx.dec(ctx.sum_col_vec(a, lay))
    out["sum_rows"] = ctx.dec(ctx.sum_rows(a, lay))
    out["levels"] = np.array([ctx.mul(a, b).level_bits, ctx.cmul(a, 2.0).level_bits,
                              ctx.sum_col_vec(a, lay).level_bits, ctx.sum_rows(a, lay).level_bits])
    return out


def main(which):
    OUT.mkdir(parents=True, exist_ok=True)
    if "ops" in which:
        np.savez_compressed(OUT / "sim_ops.npz", **ops_vectors())
        print("ops done")
    if "toy" in which:
        ds = toy_dataset()
        r = run(ds, 13, 128, 1, 24, "mini_batch", keep_all)
        np.savez_compressed(OUT / "toy.npz", **r)
        print("toy", r["seconds"], r["auc"][-1])
    if "medium" in which:
        ds = medium_dataset()
        r = run(ds, 15, 1024, 1, 320, "mini_batch", keep_sparse)
        np.savez_compressed(OUT / "medium.npz", **r)
        print("medium", r["seconds"], r["auc"][-1])
    if "paper_mini" in which:
        ds = paper_dataset()
        r = run(ds, 16, 128, 8, 3 * 413, "mini_batch", keep_sparse)
        np.savez_compressed(OUT / "paper_mini.npz", **r)
        print("paper_mini", r["seconds"], r["auc"][-1])
    if "paper_full" in which:
        ds = paper_dataset()
        r = run(ds, 16, 128, 8, 10, "full_batch", keep_all)
        np.savez_compressed(OUT / "paper_full.npz", **r)
        print("paper_full", r["seconds"], r["auc"][-1])


if __name__ == "__main__":
    main(sys.argv[1:] or ["ops", "toy", "medium", "paper_mini", "paper_full"])
