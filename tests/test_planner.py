"""CPU check of the host planner (driver.plan_iteration): the exact-scale
integer constants it emits, executed by the ring oracle's restatement of the
fused schedule (oracle/schedule.py), must reproduce the plaintext NAG update
(enctrain.py:162-239 semantics) within CKKS noise.  No GPU needed."""

import math

import numpy as np
import pytest

from oracle import schedule as osched
from oracle.oracle import Oracle
from paper_2406_13221_b200.driver import plan_iteration, row_mask
from paper_2406_13221_b200.encoder import Encoder
from paper_2406_13221_b200.optimizer import BASELINE_CUBIC
from paper_2406_13221_b200.params import CkksParams


def _gal(k, n):
    return pow(5, k % (n // 2), 2 * n)


@pytest.mark.parametrize("bsgs", [0, 2, 3])
@pytest.mark.parametrize("R,C", [(1, 1), (2, 2)])
def test_planned_iteration_matches_plaintext(R, C, bsgs):
    log_n, L = 10, 8
    P = CkksParams.generate(log_n=log_n, n_q=L, dnum=3)
    orc = Oracle(P)
    enc = Encoder(log_n)
    sk = orc.keygen_secret(3)
    rng = np.random.default_rng(R * 10 + C + bsgs)
    S, N, top = P.slots, P.n, P.top_level
    log_g = 4
    g, log_m = 1 << log_g, log_n - 1 - log_g
    m = S // g
    s_top = P.level_scales[top]
    zv = rng.uniform(-1, 1, size=(R * C, S))
    wvv = rng.normal(scale=0.3, size=(2 * C, S))
    bv = rng.uniform(1e-4, 2e-3, size=(C, S))
    s_b = s_top / float(np.abs(bv).max())
    ids = iter(range(1, 10_000))
    encr = lambda x, s: orc.encrypt(sk, enc.encode(np.atleast_2d(x), s), top, 5, next(ids))[0]
    z = np.stack([encr(v, s_top) for v in zv]).reshape(R, C, 2, L, N)
    w = np.stack([encr(v, s_top) for v in wvv[:C]])
    v = np.stack([encr(v, s_top) for v in wvv[C:]])
    bb = np.stack([encr(x, s_b) for x in bv])
    qp = BASELINE_CUBIC.complement().padded(3)
    mult, eta = 1.02, -0.6
    plan = plan_iteration(P, top, s_top, s_top, s_top, s_b, qp, mult, eta)
    if bsgs:
        steps = [k for grp in osched.grouped_steps(log_g, bsgs) for k in grp]
        rsteps = [k for grp in osched.grouped_steps(log_m, bsgs, g) for k in grp]
    else:
        steps = [1 << i for i in range(log_g)]
        rsteps = [g << i for i in range(log_m)]
    gals = [_gal(k, N) for k in steps] + [_gal(-k, N) for k in steps] + [_gal(k, N) for k in rsteps]
    gk = {x: orc.keygen_switch(sk, x, 3, x) for x in set(gals)}
    rlk = orc.keygen_switch(sk, 0, 3, 0)
    mask = orc.encode_plain(enc.encode(row_mask(S, g), plan.mask_scale), top - 1)[0]
    w2, v2 = osched.nag_iteration(orc, z, w, v, bb, top, rlk, gk, mask, plan.consts, log_g, log_m, log_baby=bsgs,
                                  log_baby_rows=bsgs)
    got_w = enc.decode(orc.decrypt(sk, w2, 0), plan.s_out).real
    got_v = enc.decode(orc.decrypt(sk, v2, 0), plan.s_out).real
    # plaintext model
    W, V = wvv[:C], wvv[C:]
    Zb = zv.reshape(R, C, S)
    G = np.zeros((C, S))
    for r in range(R):
        p = sum(Zb[r, j] * W[j] for j in range(C))
        acc = sum(np.roll(p, -k) for k in range(g)) * row_mask(S, g)
        u = sum(np.roll(acc, k) for k in range(g))
        qu = qp[0] + qp[1] * u + qp[2] * u * u + qp[3] * u ** 3
        for j in range(C):
            G[j] += qu * Zb[r, j]
    for j in range(C):
        G[j] = sum(np.roll(G[j], -k * g) for k in range(m))
    D = G * bv
    vn = W + mult * D
    wn = (1 - eta) * vn + eta * V
    assert np.abs(got_w - wn).max() < 1e-7
    assert np.abs(got_v - vn).max() < 1e-7
