"""Residue-exact parity of whole training runs and of the benchmark ring.

1. ``FusedTrainer`` (CUDA graphs, graphs re-pointed per batch, refresh
   stand-in every iteration) on the Toy config for all 24 iterations: after
   every iteration each RNS residue of W and V equals the CPU oracle's
   restatement of the same schedule (oracle/schedule.py), which keeps its
   OWN W, V state (refreshed with ``oc_refresh``) and is fed only the
   trainer's inputs: the encrypted dataset and B̄ (encrypted on the device,
   encryption itself is pinned in test_gpu_parity.py), the keys, the mask
   plaintext and the per-iteration constants the host planner produced.
   Reference loop body: enctrain.py:344-398.
2. One fused iteration at the benchmark ring: N = 2^16, L = 8, dnum = 2,
   K = 5 40-bit special primes, R = 8 row blocks, C = 1, log g = 8,
   log m = 7, 4-bit hoisted groups (the paper_mini bench configuration).
"""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import schedule as osched
from oracle.oracle import Oracle
from paper_2406_13221_b200 import _lib, data
from paper_2406_13221_b200.ckks import GpuContext
from paper_2406_13221_b200.driver import ITER_DEPTH, FusedTrainer, NagArgs, _bind, grouped_steps, plan_iteration, row_mask
from paper_2406_13221_b200.optimizer import BASELINE_CUBIC
from paper_2406_13221_b200.params import CkksParams

pytestmark = pytest.mark.gpu


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("dnum", [2, 3])
def test_toy_trainer_all_iterations_residue_exact(dnum):
    ck = CkksParams.generate(log_n=13, n_q=8, dnum=dnum)
    ctx = GpuContext(ck, seed=2, max_batch=8)
    tr = FusedTrainer(ctx, data.toy_dataset(), rows_per_block=128, blocks_per_batch=1, mode="mini_batch",
                      use_graph=True)
    plans = []
    upload = tr._upload_consts

    def record(plan):
        plans.append(plan)
        upload(plan)
    tr._upload_consts = record

    orc = Oracle(ck)
    sk = orc.keygen_secret(ctx.key_seed, ck.hw)
    np.testing.assert_array_equal(u64(ctx.sk), sk)
    torch.cuda.synchronize()
    z, bbar = u64(tr.z), u64(tr.bbar)
    C = tr.cols
    wv = u64(tr.wv).copy()          # the oracle's own W, V from here on
    rlk = u64(ctx.rlk)
    gkeys = {g: u64(ctx.galois_key(g)) for g in set(tr.gal_left + tr.gal_right + tr.gal_rows)}
    level, s_w = tr.level, tr.s_w
    top = ck.top_level
    for it in range(24):
        first = ctx._next_ct_id
        b = tr.t % tr.n_batches
        info = tr.iterate()
        if level < ITER_DEPTH:     # the trainer refreshed W, V before the iteration
            assert info["refreshed"]
            ratio = float(2 ** tr.refresh_bits) / s_w
            wv = orc.refresh(sk, wv, level, ratio, top, ctx.enc_seed, first)
            level = top
        plan = plans[-1]
        assert plan.lw == level
        mask = u64(tr._mask(plan.lw, plan.mask_scale))
        w2, v2 = osched.nag_iteration(orc, z[b], wv[:C], wv[C:], bbar[b], level, rlk, gkeys, mask, plan.consts,
                                      tr.log_g, tr.log_m, log_baby=tr.log_baby, log_baby_rows=tr.log_baby_rows)
        level -= ITER_DEPTH
        s_w = plan.s_out
        wv = np.concatenate([w2, v2])
        got = u64(tr.wv)
        np.testing.assert_array_equal(got[:, :, :level + 1], wv[:, :, :level + 1], err_msg=f"iteration {it + 1}")
    tr.close()


def test_bench_ring_fused_iteration_residue_exact():
    """The paper_mini bench ring and schedule, one iteration, every residue."""
    log_n, L, dnum, R, C, log_g = 16, 8, 2, 8, 1, 8
    P = CkksParams.generate(log_n=log_n, n_q=L, dnum=dnum)
    assert P.K == 5 and max(p.bit_length() for p in P.primes[P.L:]) <= 41  # 40-bit specials, as benched
    ctx = GpuContext(P, seed=13, max_batch=R)
    rng = np.random.default_rng(13)
    S, n = P.slots, P.n
    log_m = log_n - 1 - log_g
    top = P.top_level
    s_top = P.level_scales[top]
    # dataset ciphertexts through the DEVICE encoder (the bench default)
    zvals = rng.uniform(-1, 1, size=(R * C, S))
    z = ctx._empty((R, C, 2, L, n))
    ctx.encrypt_to(ctx.encode_slots(zvals, s_top), z.view(R * C, 2, L, n), top)
    wv = ctx._empty((2 * C, 2, L, n))
    ctx.encrypt_to(ctx.encode_slots(rng.normal(scale=0.3, size=(2 * C, S)), 2.0 ** 47), wv, top)
    bbar = ctx._empty((C, 2, L, n))
    ctx.encrypt_to(ctx.encode_slots(rng.uniform(1e-4, 1e-3, size=(C, S)), s_top * 1e3), bbar, top)
    plan = plan_iteration(P, top, 2.0 ** 47, 2.0 ** 47, s_top, s_top * 1e3, BASELINE_CUBIC.complement().padded(3),
                          1.004, 0.37)
    lb, lbr = (log_g + 1) // 2, (log_m + 1) // 2
    steps = [k for grp in grouped_steps(log_g, lb) for k in grp]
    rsteps = [k for grp in grouped_steps(log_m, lbr, 1 << log_g) for k in grp]
    gl = [pow(5, k, 2 * n) for k in steps]
    gr = [pow(5, S - k, 2 * n) for k in steps]
    gw = [pow(5, k % S, 2 * n) for k in rsteps]
    arr = lambda gs: (ctypes.c_void_p * len(gs))(*[ctx.galois_key(g).data_ptr() for g in gs])
    mask = ctx._plain(ctx.encoder.encode(row_mask(S, 1 << log_g), plan.mask_scale), top - 1)
    consts = torch.from_numpy(plan.consts.view(np.int64)).to(ctx.device)
    grad = ctx._empty((C, 2, L, n))
    cs = wv[0].numel() * 8
    lib = _lib.load()
    _bind(lib)
    z_np, w_np, v_np, b_np = u64(z), u64(wv[:C]), u64(wv[C:]), u64(bbar)
    args = NagArgs(z=z.data_ptr(), rows=R, cols=C, log_g=log_g, log_m=log_m, w=wv.data_ptr(),
                   v=wv.data_ptr() + C * cs, bbar=bbar.data_ptr(), lw=top, rlk=ctx.rlk.data_ptr(),
                   rot_left=arr(gl), rot_right=arr(gr), rot_rows=arr(gw), mask_pt=mask.data_ptr(),
                   consts=consts.data_ptr(), grad=grad.data_ptr(), phase=0, log_baby=lb, log_baby_rows=lbr)
    _lib.check(lib.helr_nag_iteration(ctx.handle, ctypes.byref(args), torch.cuda.current_stream().cuda_stream),
               "nag")
    out = u64(wv)
    orc = Oracle(P)
    gkeys = {g: u64(ctx.galois_key(g)) for g in set(gl + gr + gw)}
    w2, v2 = osched.nag_iteration(orc, z_np, w_np, v_np, b_np, top, u64(ctx.rlk), gkeys, u64(mask), plan.consts,
                                  log_g, log_m, log_baby=lb, log_baby_rows=lbr)
    lo = top - ITER_DEPTH + 1
    np.testing.assert_array_equal(out[:C, :, :lo], w2[:, :, :lo])
    np.testing.assert_array_equal(out[C:, :, :lo], v2[:, :, :lo])
