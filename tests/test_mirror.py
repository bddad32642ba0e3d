"""Host-side mirror of the reference API (encoding, optimizer scalars,
enctrain driver logic).  Runs on CPU: the encrypted-training driver is
exercised over the slot-level oracle through a SimContext-shaped adapter,
and — where /root/reference is importable (the build container) — compared
value-for-value with the reference's own functions."""

import math
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import slotsim
from paper_2406_13221_b200 import encoding as E
from paper_2406_13221_b200 import enctrain as T
from paper_2406_13221_b200 import optimizer as O
from paper_2406_13221_b200.data import build_z, make_dataset
from paper_2406_13221_b200.errors import NeedsBootstrap
from paper_2406_13221_b200.params import HeParams

REF = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def helr():
    if not REF.exists():
        pytest.skip("reference not mounted (GPU box)")
    sys.path.insert(0, str(REF))
    import helr  # noqa: F401
    return sys.modules["helr"]


class SlotCtx:
    """SimContext-protocol adapter over oracle.slotsim (test harness only)."""

    COUNTER_KEYS = ("enc", "dec", "add", "cadd", "mul", "cmul", "imul", "rotate", "bootstrap")

    def __init__(self, params):
        self.params = params
        self._s = slotsim.SlotSim(params.log_n, params.log_q, params.log_delta, params.log_delta_c)
        self.counters = self._s.counters

    @property
    def counters(self):
        return self._s.counters

    @counters.setter
    def counters(self, v):
        self._s.counters = v

    def reset_counters(self):
        snap = dict(self._s.counters)
        self._s.counters = dict.fromkeys(self.COUNTER_KEYS, 0)
        return snap

    def __getattr__(self, name):
        attr = getattr(self._s, name)
        if not callable(attr):
            return attr

        def call(*args, **kw):
            # the product driver catches only the product's NeedsBootstrap
            try:
                return attr(*args, **kw)
            except slotsim.SlotNeedsBootstrap as e:
                raise NeedsBootstrap(str(e)) from e
        return call

    def sum_col_vec(self, a, layout):
        return self.__getattr__("sum_col_vec")(a, layout.m, layout.g)

    def sum_rows(self, a, layout):
        return self.__getattr__("sum_rows")(a, layout.m, layout.g)


TOY = HeParams(log_n=5, log_q=2000)
TABLE = O.LrSchedule(2.0, 1.0, 36, 2.5)


def toy(rng, n=4, f=3):
    X = rng.uniform(0.0, 1.0, size=(n, f))
    y = rng.choice([-1.0, 1.0], size=n)
    if len(set(y)) == 1:
        y[0] = -y[0]
    return make_dataset(X, y)


def test_scalar_goldens():
    # reference test_optim.py:32-60 golden values
    assert O.f2(O.LrSchedule(2.0, 1.0, 81, 2.5), 41) == pytest.approx(1.8177166108973121, abs=1e-12)
    a1 = O.next_alpha(0.01)
    assert a1 == pytest.approx(1.0000999900019995, abs=1e-15)
    assert (1 - 0.01) / a1 == pytest.approx(0.9899010197950514, abs=1e-15)
    assert O.ExpDecay()(0) == 11.0


def test_layout_and_packing(rng):
    lay = E.plan_layout(6, 3, TOY, batch_rows=4)
    assert (lay.m, lay.g, lay.row_blocks, lay.col_blocks, lay.pad_rows) == (4, 4, 2, 1, 2)
    Z = rng.normal(size=(6, 4))
    blocks = E.pack_matrix(Z, lay)
    np.testing.assert_array_equal(E.unpack_matrix(blocks, lay), Z)
    np.testing.assert_array_equal(E.pack_matrix_array(Z, lay), np.array(blocks))
    with pytest.raises(ValueError, match="power of two"):
        E.plan_layout(6, 3, TOY, batch_rows=3)


def test_mirror_equals_reference(helr, rng):
    from helr import encoding as RE, quadgrad as RQ, optim as RO
    RS = sys.modules["helr.sigmoid"]
    lay = E.plan_layout(300, 20, HeParams(log_n=10), 64)
    rlay = RE.plan_layout(300, 20, helr.HeParams(log_n=10), 64)
    assert lay.__dict__ == rlay.__dict__
    Z = rng.normal(size=(300, 21))
    for a, b in zip(E.pack_matrix(Z, lay), RE.pack_matrix(Z, rlay)):
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
    v = rng.normal(size=21)
    for x, y in zip(E.replicate_rows(v, lay), RE.replicate_rows(v, rlay)):
        np.testing.assert_array_equal(x, y)
    X = rng.uniform(-1, 1, size=(50, 7))
    np.testing.assert_array_equal(O.scaler_for(X).b, RQ.scaler_for(X).b)
    sc = [O.scaler_for(X[i::3]) for i in range(3)]
    rsc = [RQ.scaler_for(X[i::3]) for i in range(3)]
    np.testing.assert_allclose(O.merge_bbar(sc).b, RQ.merge_bbar(rsc).b, rtol=1e-15)
    y = np.where(rng.random(200) < 0.3, 1.0, -1.0)
    s = np.round(rng.normal(size=200), 1)  # ties exercise the midrank path
    assert O.auroc(y, s) == pytest.approx(RO.auroc(y, s), abs=1e-15)
    assert O.G8.complement().coefficients == RS.G8.complement().coefficients
    xs = np.linspace(-8, 8, 101)
    np.testing.assert_array_equal(O.G16(xs), RS.G16(xs))


def test_enctrain_gradient_matches_plaintext(rng):
    ds = toy(rng)
    ctx = SlotCtx(TOY)
    lay = E.plan_layout(4, 3, TOY, batch_rows=4)
    prep = T.client_prepare(ds, ctx, lay)
    w = rng.normal(size=4) * 0.5
    ct_w = [ctx.enc(v) for v in E.replicate_rows(w, lay)]
    g = T.decode_weights(ctx, T.enc_gradient(ctx, prep.ct_z[0], ct_w, O.G8, lay), lay)
    np.testing.assert_allclose(g, O.gradient(build_z(ds).Z, w, O.G8), atol=1e-12)


def test_bootstrap_cadence_and_ledger(rng):
    # reference test_enctrain.py:293-336 expectations, on the mirrored driver
    ds = toy(rng, n=8, f=3)
    cfg = O.TrainConfig(mode="mini_batch", batch_size=8, max_iterations=6, schedule=TABLE, sigmoid="g8")
    params = HeParams(log_n=5)
    res = T.train_encrypted(ds, cfg, params, ctx=SlotCtx(params))
    assert [r["bootstraps"] for r in res.ledger] == [0, 1, 1, 1, 1, 1]
    for row in res.ledger:
        assert row["level_after"] == row["level_start"] - row["consumed_bits"]
        if row["bootstraps"]:
            assert row["level_start"] == params.log_q and row["boot_ops"] == 2 * res.layout.col_blocks
        assert row["level_after"] >= params.log_delta
    with pytest.raises(NeedsBootstrap, match="bits"):
        cfg1 = O.TrainConfig(mode="mini_batch", batch_size=4, max_iterations=1, schedule=TABLE, sigmoid="g8")
        p = HeParams(log_n=5, log_q=100)
        T.train_encrypted(toy(rng), cfg1, p, ctx=SlotCtx(p))


def test_enctrain_equals_reference_train(helr, rng):
    from helr import enctrain as RT, optim as RO
    ds_r = helr.make_dataset(*_feats(rng))
    ds = make_dataset(ds_r.X[:, 1:], ds_r.y)
    for mode in ("mini_batch", "full_batch"):
        rcfg = RO.TrainConfig(mode=mode, batch_size=4, max_iterations=7, schedule=RO.LrSchedule(2.0, 1.0, 36, 2.5),
                              sigmoid="g8")
        cfg = O.TrainConfig(mode=mode, batch_size=4, max_iterations=7, schedule=TABLE, sigmoid="g8")
        p = HeParams(log_n=5, log_q=400)
        ref = RT.train_encrypted(ds_r, rcfg, helr.HeParams(log_n=5, log_q=400), trace_weights=True)
        got = T.train_encrypted(ds, cfg, p, ctx=SlotCtx(p), trace_weights=True)
        for a, b in zip(got.weight_trace, ref.weight_trace):
            np.testing.assert_allclose(a, b, atol=1e-12)
        assert [r["bootstraps"] for r in got.ledger] == [r["bootstraps"] for r in ref.ledger]
        assert [r["consumed_bits"] for r in got.ledger] == [r["consumed_bits"] for r in ref.ledger]


def _feats(rng):
    X = rng.uniform(0, 1, size=(10, 3))
    y = np.where(rng.random(10) < 0.5, 1.0, 0.0)
    y[0], y[1] = 1.0, 0.0
    return X, y
