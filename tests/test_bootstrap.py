"""Real CKKS bootstrapping (bootstrap.py), CPU side: the circuit is driven by
the CPU ring oracle through the same evaluator protocol the GPU implements
(tests/bootstrap_util.OracleRing), on a small ring.

The reference only models a bootstrap (hesim.py:228-236: level restored,
slots preserved); these tests check exactly that contract on real
ciphertexts, plus the building blocks (special-FFT factors, the scaled-sine
interpolant).
"""

import numpy as np
import pytest

from bootstrap_util import OracleRing
from paper_2406_13221_b200.bootstrap import (BootstrapConfig, Bootstrapper, _Transform, apply_diagonals,
                                             bootstrap_ring, chebyshev_coefficients, grouped_dft_factors)
from paper_2406_13221_b200.encoder import Encoder


@pytest.mark.parametrize("log_n,groups", [(5, 1), (6, 2), (8, 3)])
def test_grouped_factors_compose_to_the_encoding_map(log_n, groups):
    """Forward factors applied to the bit-reversed coefficient pairs give the
    slot values (the encoder's own map); the un-normalised inverse factors
    undo it up to n."""
    enc = Encoder(log_n)
    n = 1 << (log_n - 1)
    rng = np.random.default_rng(log_n)
    z = rng.normal(size=n) + 1j * rng.normal(size=n)
    w = z.copy()
    for m in grouped_dft_factors(log_n, groups, True):
        w = apply_diagonals(m, w)
    back = w.copy()
    for m in grouped_dft_factors(log_n, groups, False):
        back = apply_diagonals(m, back)
    assert np.abs(back / n - z).max() < 1e-9
    # w / n holds t_i + i t_{i + n} in bit-reversed order, t = the encoder's real coefficients of z
    coef = enc.coefficients(z)
    bits = log_n - 1
    brv = np.array([int(format(i, f"0{bits}b")[::-1], 2) if bits else 0 for i in range(n)])
    assert np.abs(w / n - (coef[:n] + 1j * coef[n:])[brv]).max() < 1e-9


def test_transform_plan_covers_every_diagonal():
    for m in grouped_dft_factors(9, 3, True) + grouped_dft_factors(9, 3, False):
        t = _Transform.plan(m, 256)
        seen = sorted(t.signed[t.baby * i + j] for i, js in t.terms.items() for j in js)
        assert seen == sorted(m)
        # baby-step/giant-step needs about 2 sqrt(#diagonals) rotations, not #diagonals
        assert len(t.rotations(256)) <= 2 * int(np.ceil(np.sqrt(len(m)))) + 2


def test_scaled_sine_interpolant():
    cfg = BootstrapConfig()
    c = chebyshev_coefficients(cfg.k_range, cfg.double_angles, cfg.degree)
    from numpy.polynomial import chebyshev as C

    u = np.linspace(-1, 1, 4001)
    v = C.chebval(u, c)
    for _ in range(cfg.double_angles):
        v = 2 * v * v - 1
    assert np.abs(v - np.sin(2 * np.pi * cfg.k_range * u)).max() < 1e-9


def test_chain_layout():
    cfg = BootstrapConfig()
    P = bootstrap_ring(10, work_levels=3, cfg=cfg)
    assert P.work_levels == 3 and P.top_level == 3
    assert P.L == 1 + 3 + cfg.depth
    assert len(set(P.q) | set(P.p)) == P.L + P.K
    with pytest.raises(ValueError):
        Bootstrapper(OracleRing(bootstrap_ring(6, work_levels=2, cfg=cfg), 1),
                     BootstrapConfig(c2s_groups=5, s2c_groups=5, degree=127))  # deeper than the chain


@pytest.fixture(scope="module")
def small_boot():
    cfg = BootstrapConfig()
    P = bootstrap_ring(9, work_levels=2, cfg=cfg, secret_hw=32)
    ring = OracleRing(P, key_seed=5)
    return P, ring, Bootstrapper(ring, cfg)


def test_bootstrap_restores_level_and_slots(small_boot):
    P, ring, bs = small_boot
    enc = Encoder(P.log_n)
    rng = np.random.default_rng(1)
    z = rng.uniform(-1, 1, P.slots) + 1j * rng.uniform(-1, 1, P.slots)
    top = P.top_level
    s = P.level_scales[top]
    ct = ring.orc.encrypt(ring.sk, enc.encode(z, s), top, 9, 1)
    # exhaust the working levels first: two constant products
    lvl, sc = top, s
    for _ in range(top):
        c = int(round(float(P.q[lvl]) * P.level_scales[lvl - 1] / sc))
        ct = ring.rescale(ring.mul_const(ct, c, lvl), lvl)
        sc = sc * c / float(P.q[lvl])
        lvl -= 1
    assert lvl == 0
    out, out_level, out_scale = bs.bootstrap(ct, lvl, sc)
    assert out_level == P.top_level == bs.out_level
    assert out_scale == pytest.approx(P.level_scales[P.top_level])
    got = enc.decode(ring.orc.decrypt(ring.sk, out, out_level)[0], out_scale)
    assert np.abs(got - z).max() < 1e-4
    # the refreshed ciphertext is usable: one more product at the working top
    sq = ring.mul(out, out, out_level)
    got2 = enc.decode(ring.orc.decrypt(ring.sk, sq, out_level - 1)[0], P.level_scales[out_level - 1])
    assert np.abs(got2 - z * z).max() < 5e-4


def test_bootstrap_refuses_scales_too_close_to_q0(small_boot):
    P, ring, bs = small_boot
    ct = ring.orc.ct_zeros(1)
    with pytest.raises(ValueError):
        bs.bootstrap(ct, 0, float(P.q[0]) / 8.0)
