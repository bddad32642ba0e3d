"""The slot-level oracle (oracle/slotsim.py) reproduces the REFERENCE's own
outputs: simulator op vectors and BASELINE training traces recorded by
running /root/reference (tools/make_goldens.py) -- the pin for every value
check of the GPU trainer."""

import math
from pathlib import Path

import numpy as np
import pytest

from oracle import slotsim
from paper_2406_13221_b200 import data
from paper_2406_13221_b200.optimizer import BASELINE_CUBIC

GOLD = Path(__file__).resolve().parent / "golden"
QPOLY = BASELINE_CUBIC.complement().padded(3)


def lr_fn(t):
    return 1.0 + 10.0 * math.exp(-t)


def test_sim_ops_match_reference():
    g = np.load(GOLD / "sim_ops.npz")
    sim = slotsim.SlotSim(6, 500, 40, 40)
    a, b = sim.enc(g["x"]), sim.enc(g["y"])
    np.testing.assert_array_equal(sim.dec(sim.rotate(a, 1)), g["rot1"])
    np.testing.assert_array_equal(sim.dec(sim.rotate(a, -3)), g["rot_m3"])
    np.testing.assert_array_equal(sim.dec(sim.mul(a, b)), g["mul"])
    np.testing.assert_array_equal(sim.dec(sim.cmul(a, g["y"])), g["cmul"])
    np.testing.assert_array_equal(sim.dec(sim.cadd(a, 0.25)), g["cadd"])
    np.testing.assert_array_equal(sim.dec(sim.imul(a)), g["imul"])
    np.testing.assert_array_equal(sim.dec(sim.sum_col_vec(a, 8, 4)), g["sum_col_vec"])
    np.testing.assert_array_equal(sim.dec(sim.sum_rows(a, 8, 4)), g["sum_rows"])
    lv = [sim.mul(a, b).level_bits, sim.cmul(a, 2.0).level_bits, sim.sum_col_vec(a, 8, 4).level_bits,
          sim.sum_rows(a, 8, 4).level_bits]
    np.testing.assert_array_equal(lv, g["levels"])


def test_sim_level_budget_raises():
    sim = slotsim.SlotSim(4, 100, 40, 40)
    a = sim.enc(np.ones(8))
    b = sim.mul(a, a)
    with pytest.raises(slotsim.SlotNeedsBootstrap):
        sim.mul(b, b)


@pytest.mark.parametrize("name,ds_fn,log_n,m,blocks,iters", [
    ("toy", data.toy_dataset, 13, 128, 1, 24),
    ("medium", data.medium_dataset, 15, 1024, 1, 40),
])
def test_training_trace_matches_reference(name, ds_fn, log_n, m, blocks, iters):
    g = np.load(GOLD / f"{name}.npz")
    ds = ds_fn()
    trace, _ = slotsim.train(ds.X, ds.y, log_n, m, blocks, QPOLY, lr_fn, iters)
    its = list(g["iterations"])
    for t in range(iters):
        if t + 1 in its:
            k = its.index(t + 1)
            np.testing.assert_allclose(trace[t], g["weights"][k], rtol=0, atol=1e-12)
            assert abs(slotsim.auroc(ds.y, ds.X @ trace[t]) - g["auc"][k]) < 1e-12


@pytest.mark.slow
def test_paper_mini_first_iterations_match_reference():
    g = np.load(GOLD / "paper_mini.npz")
    ds = data.paper_dataset()
    trace, _ = slotsim.train(ds.X, ds.y, 16, 128, 8, QPOLY, lr_fn, 6)
    for t in range(6):
        np.testing.assert_allclose(trace[t], g["weights"][t], rtol=0, atol=1e-12)
