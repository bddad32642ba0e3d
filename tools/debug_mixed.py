#!/usr/bin/env python
"""Per-limb parity of rotate / mul_relin on a ring with 60-bit special primes
above 40-bit scaling primes (GPU vs CPU ring oracle), every level."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle.oracle import Oracle  # noqa: E402
from paper_2406_13221_b200 import _lib  # noqa: E402
from paper_2406_13221_b200.ckks import GpuContext  # noqa: E402
from paper_2406_13221_b200.params import CkksParams  # noqa: E402

for name, P in (("mixed_p60_d2", CkksParams.generate(log_n=12, n_q=6, dnum=2, p_bits=60)),
                ("mixed_p60_d3", CkksParams.generate(log_n=12, n_q=6, dnum=3, p_bits=60)),
                ("mixed_p60_d6", CkksParams.generate(log_n=12, n_q=6, dnum=6, p_bits=60))):
    ctx = GpuContext(P, seed=5, max_batch=4)
    orc = Oracle(P)
    sk = orc.keygen_secret(ctx.key_seed, P.hw)
    rng = np.random.default_rng(0)
    ct = np.zeros((2, 2, P.L, P.n), dtype=np.uint64)
    for p in range(P.L):
        ct[:, :, p] = rng.integers(0, P.q[p], size=(2, 2, P.n), dtype=np.uint64)
    g = 5
    gk_o = orc.keygen_switch(sk, g, ctx.key_seed, g)
    rlk_o = orc.keygen_switch(sk, 0, ctx.key_seed, 0)
    st = torch.cuda.current_stream().cuda_stream
    d = torch.from_numpy(ct.view(np.int64)).cuda()
    print(name, "K", P.K, "alpha", P.alpha, "keys equal", np.array_equal(ctx.galois_key(g).cpu().numpy().view(np.uint64), gk_o))
    for lvl in range(P.L - 1, 0, -1):
        out = torch.empty_like(d)
        _lib.call("helr_rotate", ctx.handle, d.data_ptr(), g, ctx.galois_key(g).data_ptr(), out.data_ptr(), 2, lvl, 0, st)
        exp = orc.rotate(ct.copy(), g, gk_o, lvl)
        got = out.cpu().numpy().view(np.uint64)
        bad_r = [(pl, l) for pl in range(2) for l in range(lvl + 1) if not np.array_equal(got[:, pl, l], exp[:, pl, l])]
        out2 = torch.empty_like(d)
        _lib.call("helr_mul_relin", ctx.handle, d.data_ptr(), d.data_ptr(), ctx.rlk.data_ptr(), out2.data_ptr(), 2, lvl, st)
        exp2 = orc.mul_relin(ct.copy(), ct.copy(), rlk_o, lvl)
        got2 = out2.cpu().numpy().view(np.uint64)
        bad_m = [(pl, l) for pl in range(2) for l in range(lvl + 1) if not np.array_equal(got2[:, pl, l], exp2[:, pl, l])]
        out3 = torch.empty_like(d)
        _lib.call("helr_mul_relin_rescale", ctx.handle, d.data_ptr(), d.data_ptr(), ctx.rlk.data_ptr(), out3.data_ptr(), 2, lvl, st)
        exp3 = orc.mul_relin_rescale(ct.copy(), ct.copy(), rlk_o, lvl)
        got3 = out3.cpu().numpy().view(np.uint64)
        bad_s = [(pl, l) for pl in range(2) for l in range(lvl) if not np.array_equal(got3[:, pl, l], exp3[:, pl, l])]
        print(f"  level {lvl}: rotate bad (poly, limb) {bad_r}  mul_relin bad {bad_m}  mul_relin_rescale bad {bad_s}")
