"""Real CKKS bootstrapping on the GPU evaluator.

The circuit of ``bootstrap.Bootstrapper`` is deterministic given the keys, so
the GPU run (``GpuRing``: helr_* kernels) must equal, residue for residue, the
same circuit driven by the CPU ring oracle (``OracleRing``).  On a larger ring
the reference's contract for ``bootstrap`` (hesim.py:228-236: level restored,
slots preserved, counter bumped) is checked through ``GpuContext``.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from bootstrap_util import LockstepRing, OracleRing
from paper_2406_13221_b200.bootstrap import BootstrapConfig, Bootstrapper, GpuRing, bootstrap_ring

pytestmark = pytest.mark.gpu


def _u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


def test_bootstrap_residue_exact_vs_oracle():
    from paper_2406_13221_b200.ckks import GpuContext

    cfg = BootstrapConfig()
    P = bootstrap_ring(10, work_levels=2, cfg=cfg, secret_hw=32)
    ctx = GpuContext(P, seed=11, max_batch=2)
    oring = OracleRing(P, key_seed=ctx.key_seed)
    assert np.array_equal(_u64(ctx.sk), oring.sk)
    rng = np.random.default_rng(3)
    z = rng.uniform(-1, 1, P.slots) + 1j * rng.uniform(-1, 1, P.slots)
    top = P.top_level
    s = P.level_scales[top]
    coef = ctx.encoder.encode(z, s)
    ct_o = oring.orc.encrypt(oring.sk, coef, top, ctx.enc_seed, 1)
    ct_g = torch.from_numpy(ct_o.view(np.int64)).cuda()
    # every primitive of the circuit runs on both evaluators and is compared
    # on the spot (LockstepRing raises at the first differing residue)
    lock = LockstepRing(GpuRing(ctx), oring)
    (out_g, out_o), lvl_g, sc_g = Bootstrapper(lock, cfg).bootstrap((ct_g, ct_o), top, s)
    assert lock.ops > 300
    got = _u64(out_g)
    assert np.array_equal(got[:, :, : lvl_g + 1], out_o[:, :, : lvl_g + 1])
    dec = ctx.encoder.decode(oring.orc.decrypt(oring.sk, got, lvl_g)[0], sc_g)
    assert np.abs(dec - z).max() < 1e-4


def test_mod_raise_residue_exact():
    from paper_2406_13221_b200.ckks import GpuContext

    P = bootstrap_ring(11, work_levels=2, secret_hw=32)
    ctx = GpuContext(P, seed=2, max_batch=2)
    oring = OracleRing(P, key_seed=ctx.key_seed)
    rng = np.random.default_rng(0)
    ct = np.zeros((2, 2, P.L, P.n), dtype=np.uint64)
    for p in range(P.L):
        ct[:, :, p] = rng.integers(0, P.q[p], size=(2, 2, P.n), dtype=np.uint64)
    want = oring.mod_raise(ct, P.L - 1)
    got = GpuRing(ctx).mod_raise(torch.from_numpy(ct.view(np.int64)).cuda(), P.L - 1)
    assert np.array_equal(_u64(got), want)


def test_context_bootstrap_contract():
    """GpuContext(bootstrap='ckks').bootstrap: the reference's contract on a
    ciphertext whose working levels are spent (hesim.py:228-236)."""
    from paper_2406_13221_b200.ckks import GpuContext

    P = bootstrap_ring(13, work_levels=3, scale_bits=46)
    ctx = GpuContext(P, seed=5, max_batch=2, bootstrap="ckks")
    rng = np.random.default_rng(4)
    z = rng.uniform(-1, 1, P.slots)
    ct = ctx.enc(z)
    full = ct.level_bits
    x = ctx.cmul(ctx.cmul(ctx.cmul(ct, 0.5), 2.0), 1.0)   # three constant products: levels spent
    assert x.level == 0
    y = ctx.bootstrap(x)
    assert ctx.counters["bootstrap"] == 1
    assert y.level_bits == full and y.boot_count == 1
    assert np.abs(ctx.dec(y).real - z).max() < 2e-6       # measured 4e-7 (scale 2^46, EvalMod at 2^59)
    w = ctx.mul(y, y)                                      # usable afterwards
    assert np.abs(ctx.dec(w).real - z * z).max() < 1e-5
    with pytest.raises(ValueError):
        GpuContext(P.__class__.generate(log_n=10, n_q=4, dnum=2), seed=1, bootstrap="ckks")


def test_trainer_with_real_bootstrapping():
    """Toy (BASELINE config 1) through the fused trainer on a bootstrappable
    chain: every iteration after the first starts with a REAL bootstrap of W
    and V (one batched circuit, evaluation keys only) instead of the refresh
    stand-in.  Compared with the reference goldens; the tolerance is the
    bootstrap's own precision (~1e-7 per refresh at N = 2^13) times the
    amplification of the NAG dynamics, not the 1e-6 bar of the stand-in runs."""
    from pathlib import Path

    from paper_2406_13221_b200 import data
    from paper_2406_13221_b200.ckks import GpuContext
    from paper_2406_13221_b200.driver import FusedTrainer

    gold = np.load(Path(__file__).resolve().parent / "golden" / "toy.npz")
    P = bootstrap_ring(13, work_levels=7)
    ctx = GpuContext(P, seed=2, max_batch=8, bootstrap="ckks")
    ds = data.toy_dataset()
    tr = FusedTrainer(ctx, ds, rows_per_block=128, blocks_per_batch=1, mode="mini_batch", use_graph=False)
    assert tr.real_bootstrap
    its = [int(t) for t in gold["iterations"]]
    worst = 0.0
    n_iters = 8
    for t in range(1, n_iters + 1):
        tr.iterate()
        if t in its:
            worst = max(worst, float(np.max(np.abs(tr.weights() - gold["weights"][its.index(t)]))))
    print(f"toy with real bootstrapping, {n_iters} iterations: max |dw| = {worst:.3e}")
    assert ctx.counters["bootstrap"] == 2 * (n_iters - 1)
    assert worst < 1e-4
    tr.close()
