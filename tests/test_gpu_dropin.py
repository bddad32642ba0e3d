"""The reference's own evaluator and driver tests, run against ``GpuContext``
(real RNS-CKKS on the B200) instead of the slot simulator.

Restates the value and level tests of the reference suite
(pkg/tests/test_hesim.py:93-274 and pkg/tests/test_enctrain.py:68-336,
SURVEY.md §4 reuse plan) with two documented changes:
- values are compared within a tolerance (real CKKS noise, ~1e-9 here)
  instead of bit-exactly;
- level costs stay exact, in the GPU context's units: every rescale drops
  one limb = ``log_delta`` bits, and ``log_delta_c == log_delta``
  (params.CkksParams.he_params), so the reference's "-30 per product,
  -20 per constant product" reads "-log_delta" for both.
The drop-in driver runs (``train_encrypted(..., ctx=GpuContext)``) are
compared with weight traces the unchanged reference ``train_encrypted``
produced (tests/golden/dropin.npz, tools/make_dropin_goldens.py).
"""

from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2406_13221_b200 import enctrain as T
from paper_2406_13221_b200 import optimizer as O
from paper_2406_13221_b200.ckks import GpuCiphertext, GpuContext
from paper_2406_13221_b200.data import build_z, make_dataset
from paper_2406_13221_b200.encoding import plan_layout, replicate_rows
from paper_2406_13221_b200.errors import NeedsBootstrap
from paper_2406_13221_b200.params import CkksParams, HeParams

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "dropin.npz"
TOL = 1e-6


def mk(n_q=10, log_n=5, dnum=2, seed=3):
    return GpuContext(CkksParams.generate(log_n=log_n, n_q=n_q, dnum=dnum), seed=seed, max_batch=4)


@pytest.fixture(scope="module")
def ctx():
    return mk()


def close(a, b, tol=TOL):
    a, b = np.asarray(a), np.asarray(b)
    err = float(np.max(np.abs(a - b))) if a.size else 0.0
    assert err < tol * max(1.0, float(np.max(np.abs(b))) if b.size else 1.0), err


def toy_dataset(rng, n=4, f=3):
    feats = rng.uniform(0.0, 1.0, size=(n, f))
    y = rng.choice([-1.0, 1.0], size=n)
    if len(set(y)) == 1:
        y[0] = -y[0]
    return make_dataset(feats, y)


# --------------------------------------------------------------- evaluator
class TestEncDec:
    def test_roundtrip(self, ctx, rng):
        S = ctx.params.slots
        m = rng.normal(size=S) + 1j * rng.normal(size=S)
        close(ctx.dec(ctx.enc(m)), m)

    def test_fresh_level_is_log_q(self, ctx):
        assert ctx.enc([1.0]).level_bits == ctx.params.log_q

    def test_zero_padding(self, ctx):
        out = ctx.dec(ctx.enc([1.0, 2.0]))
        close(out[:2], [1.0, 2.0])
        close(out[2:], np.zeros(ctx.params.slots - 2))

    def test_oversize_rejected(self, ctx):
        with pytest.raises(ValueError, match="slots"):
            ctx.enc(np.ones(ctx.params.slots + 1))


class TestArithmetic:
    def test_add(self, ctx):
        close(ctx.dec(ctx.add(ctx.enc([1.0, 2.0]), ctx.enc([3.0, 4.0])))[:2], [4.0, 6.0])

    def test_add_takes_min_level(self, ctx):
        a = ctx.enc([1.0])
        b = ctx.mul(ctx.enc([1.0]), ctx.enc([1.0]))
        out = ctx.add(a, b)
        assert out.level_bits == b.level_bits == ctx.params.log_q - ctx.params.log_delta
        close(ctx.dec(out)[:1], [2.0])

    def test_add_scale_mismatch_rejected(self, ctx):
        a = ctx.enc([1.0])
        weird = GpuCiphertext(ctx, a.data, a.level, a.scale, 99)
        with pytest.raises(ValueError, match="scale"):
            ctx.add(a, weird)

    def test_cadd_scalar(self, ctx):
        out = ctx.cadd(ctx.enc([1.0, 2.0]), 5.0)
        close(ctx.dec(out)[:2], [6.0, 7.0])
        assert out.level_bits == ctx.params.log_q

    def test_cadd_vector(self, ctx, rng):
        S = ctx.params.slots
        m, c = rng.normal(size=S), rng.normal(size=S)
        out = ctx.cadd(ctx.enc(m), c)
        close(ctx.dec(out), m + c)
        assert out.level_bits == ctx.params.log_q

    def test_cadd_bad_shape(self, ctx):
        with pytest.raises(ValueError, match="shape"):
            ctx.cadd(ctx.enc([1.0]), np.ones(3))

    def test_mul(self, ctx):
        out = ctx.mul(ctx.enc([1.0, 2.0]), ctx.enc([3.0, 4.0]))
        close(ctx.dec(out)[:2], [3.0, 8.0])
        assert out.level_bits == ctx.params.log_q - ctx.params.log_delta
        assert out.scale_bits == ctx.params.log_delta

    def test_mul_chain_budget(self):
        c = mk(n_q=6)
        d = c.params.log_delta
        ct = c.enc(np.ones(c.params.slots))
        fits = c.params.log_q // d - 1   # every product drops one limb; one must remain
        for _ in range(fits):
            ct = c.mul(ct, c.enc(np.ones(c.params.slots)))
        assert ct.level_bits == c.params.log_q - fits * d
        close(c.dec(ct), np.ones(c.params.slots))
        with pytest.raises(NeedsBootstrap):
            c.mul(ct, c.enc(np.ones(c.params.slots)))

    def test_cmul_scalar_and_vector(self, ctx, rng):
        out = ctx.cmul(ctx.enc([2.0]), 3.0)
        close(ctx.dec(out)[:1], [6.0])
        assert out.level_bits == ctx.params.log_q - ctx.params.log_delta_c
        m = rng.normal(size=ctx.params.slots)
        close(ctx.dec(ctx.cmul(ctx.enc(m), np.ones(ctx.params.slots))), m)

    def test_imul_twice_negates(self, ctx, rng):
        m = rng.normal(size=ctx.params.slots)
        out = ctx.imul(ctx.imul(ctx.enc(m)))
        close(ctx.dec(out), -m)
        assert out.level_bits == ctx.params.log_q


class TestRotate:
    def test_basic_left_rotation(self, ctx):
        out = ctx.dec(ctx.rotate(ctx.enc([1.0, 2.0, 3.0]), 1))
        close(out[:3], [2.0, 3.0, 0.0])
        close(out[-1:], [1.0])

    def test_full_rotation_is_identity(self, ctx, rng):
        m = rng.normal(size=ctx.params.slots)
        close(ctx.dec(ctx.rotate(ctx.enc(m), ctx.params.slots)), m)

    def test_composition(self, ctx, rng):
        m = rng.normal(size=ctx.params.slots)
        a = ctx.rotate(ctx.rotate(ctx.enc(m), 3), 7)
        close(ctx.dec(a), np.roll(m, -10))

    def test_negative_rotates_right(self, ctx):
        out = ctx.dec(ctx.rotate(ctx.enc([1.0, 2.0]), -1))
        close(out[1:3], [1.0, 2.0])


class TestStructuredSums:
    def test_sum_col_vec_matches_row_sums(self, ctx, rng):
        lay = plan_layout(4, 3, ctx.params, batch_rows=4)   # 4 x 4 block
        block = rng.normal(size=(lay.m, lay.g))
        out = ctx.sum_col_vec(ctx.enc(block.reshape(-1)), lay)
        close(np.real(ctx.dec(out)), np.repeat(block.sum(axis=1), lay.g))
        assert out.level_bits == ctx.params.log_q - ctx.params.log_delta_c   # one mask product

    def test_sum_rows_matches_column_sums(self, ctx, rng):
        lay = plan_layout(4, 3, ctx.params, batch_rows=4)
        block = rng.normal(size=(lay.m, lay.g))
        out = ctx.sum_rows(ctx.enc(block.reshape(-1)), lay)
        close(np.real(ctx.dec(out)), np.tile(block.sum(axis=0), lay.m))
        assert out.level_bits == ctx.params.log_q

    def test_layout_mismatch_rejected(self, ctx):
        bad = plan_layout(4, 3, HeParams(log_n=7), batch_rows=4)   # 64 slots, not 16
        with pytest.raises(ValueError, match="slots"):
            ctx.sum_rows(ctx.enc([1.0]), bad)
        with pytest.raises(ValueError, match="slots"):
            ctx.sum_col_vec(ctx.enc([1.0]), bad)


class TestBootstrapStandIn:
    def test_restores_budget_and_slots(self, ctx, rng):
        m = rng.normal(size=ctx.params.slots)
        low = ctx.cmul(ctx.mul(ctx.enc(m), ctx.enc(np.ones(ctx.params.slots))), 1.0)
        out = ctx.bootstrap(low)
        assert out.level_bits == ctx.params.log_q
        assert out.boot_count == 1
        close(ctx.dec(out), m)
        assert ctx.bootstrap(out).boot_count == 2


def test_random_chains_track_plaintext_and_levels(rng):
    """test_hesim.py:221-274 on the GPU: values within tolerance, level =
    log_q - (products since the last refresh) * log_delta exactly."""
    c = mk(n_q=6, seed=9)
    d = c.params.log_delta
    S = c.params.slots
    for _ in range(25):
        vec = rng.uniform(-1, 1, size=S)
        ct, mirror = c.enc(vec), vec.astype(np.complex128)
        spent = boots = 0
        for _ in range(int(rng.integers(1, 10))):
            op = rng.choice(["add", "cadd", "mul", "cmul", "imul", "rotate", "bootstrap"])
            if op == "add":
                o = rng.uniform(-1, 1, size=S)
                ct, mirror = c.add(ct, c.enc(o)), mirror + o
            elif op == "cadd":
                k = float(rng.uniform(-1, 1))
                ct, mirror = c.cadd(ct, k), mirror + k
            elif op in ("mul", "cmul"):
                o = rng.uniform(-1, 1, size=S)
                try:
                    ct = c.mul(ct, c.enc(o)) if op == "mul" else c.cmul(ct, o)
                except NeedsBootstrap:
                    continue
                mirror, spent = mirror * o, spent + d
            elif op == "imul":
                ct, mirror = c.imul(ct), mirror * 1j
            elif op == "rotate":
                k = int(rng.integers(0, S))
                ct, mirror = c.rotate(ct, k), np.roll(mirror, -k)
            else:
                ct, boots, spent = c.bootstrap(ct), boots + 1, 0
            close(c.dec(ct), mirror, tol=1e-6)
            assert ct.level_bits == c.params.log_q - spent >= d
        assert ct.boot_count == boots


def test_counters(ctx):
    a, b = ctx.enc([1.0]), ctx.enc([2.0])
    ctx.reset_counters()
    ctx.mul(a, b)
    ctx.add(a, b)
    ctx.rotate(a, 1)
    ctx.rotate(a, 2)
    counts = ctx.reset_counters()
    assert counts["mul"] == 1 and counts["add"] == 1 and counts["rotate"] == 2
    assert ctx.counters["mul"] == 0


# ------------------------------------------------------------------ driver
class TestEncCircuit:
    def test_initial_weights_zero(self, ctx, rng):
        ds = toy_dataset(rng)
        lay = plan_layout(4, 3, ctx.params, batch_rows=4)
        prep = T.client_prepare(ds, ctx, lay)
        close(T.decode_weights(ctx, prep.state.ct_w, lay, check=False), np.zeros(4))

    def test_zero_weights_give_half_column_sums(self, ctx, rng):
        ds = toy_dataset(rng)
        lay = plan_layout(4, 3, ctx.params, batch_rows=4)
        prep = T.client_prepare(ds, ctx, lay)
        g = T.enc_gradient(ctx, prep.ct_z[0], prep.state.ct_w, O.G8, lay)
        close(T.decode_weights(ctx, g, lay, check=False), 0.5 * build_z(ds).Z.sum(axis=0))

    def test_matches_plaintext_gradient_and_padding(self, ctx, rng):
        ds = toy_dataset(rng, n=6)
        Z = build_z(ds).Z
        lay = plan_layout(6, 3, ctx.params, batch_rows=4)
        prep = T.client_prepare(ds, ctx, lay)
        w = rng.normal(size=4) * 0.5
        ct_w = [ctx.enc(v) for v in replicate_rows(w, lay)]
        g0 = T.decode_weights(ctx, T.enc_gradient(ctx, prep.ct_z[0], ct_w, O.G8, lay), lay, check=False)
        close(g0, O.gradient(Z[:4], w, O.G8))
        g1 = T.decode_weights(ctx, T.enc_gradient(ctx, prep.ct_z[1], ct_w, O.G8, lay), lay, check=False)
        close(g1, O.gradient(Z[4:], w, O.G8))   # padded rows contribute nothing

    def test_quad_gradient_identity_level_and_mismatch(self, ctx, rng):
        ds = toy_dataset(rng)
        lay = plan_layout(4, 3, ctx.params, batch_rows=4)
        prep = T.client_prepare(ds, ctx, lay)
        g = T.enc_gradient(ctx, prep.ct_z[0], prep.state.ct_w, O.G8, lay)
        ones = tuple(ctx.enc(v) for v in replicate_rows(np.ones(4), lay))
        G = T.enc_quad_gradient(ctx, g, ones)
        close(T.decode_weights(ctx, G, lay, check=False), T.decode_weights(ctx, g, lay, check=False))
        assert G[0].level_bits == g[0].level_bits - ctx.params.log_delta
        with pytest.raises(ValueError, match="mismatch"):
            T.enc_quad_gradient(ctx, [ctx.enc([1.0])], tuple())

    def test_nag_update_values_and_levels(self, ctx, rng):
        ds = toy_dataset(rng)
        lay = plan_layout(4, 3, ctx.params, batch_rows=4)
        prep = T.client_prepare(ds, ctx, lay)
        wv, vv = rng.normal(size=4), rng.normal(size=4)
        st = T.EncModelState(ct_w=tuple(ctx.enc(v) for v in replicate_rows(wv, lay)),
                             ct_v=tuple(ctx.enc(v) for v in replicate_rows(vv, lay)),
                             alpha0=prep.state.alpha0, alpha1=prep.state.alpha1)
        zero = [ctx.enc(np.zeros(lay.slots)) for _ in range(lay.col_blocks)]
        out = T.enc_nag_update(ctx, st, zero, eta=0.3, gamma=0.1)
        close(T.decode_weights(ctx, out.ct_w, lay, check=False), 0.7 * wv + 0.3 * vv)
        close(T.decode_weights(ctx, out.ct_v, lay, check=False), wv)
        assert out.t == 1 and out.alpha0 == st.alpha1
        # level costs on the weight path (test_enctrain.py:186-206)
        dc = ctx.params.log_delta_c
        direction = [ctx.mul(c, c) for c in prep.state.ct_w]
        out = T.enc_nag_update(ctx, prep.state, direction, eta=0.3, gamma=0.1)
        vt = min(prep.state.ct_w[0].level_bits, direction[0].level_bits - dc)
        assert out.ct_v[0].level_bits == vt
        assert out.ct_w[0].level_bits == min(vt - dc, prep.state.ct_v[0].level_bits - dc)


# ------------------------------------------- train_encrypted(ctx=GpuContext)
def _golden_case(name):
    g = np.load(GOLD)
    return make_dataset(g[f"{name}_X"], g[f"{name}_y"]), g


@pytest.mark.parametrize("name,mode,sig,enh,sched,iters", [
    ("mini_g8", "mini_batch", "g8", True, (2.0, 1.0, 36, 2.5), 7),
    ("full_g16", "full_batch", "g16", True, (2.0, 1.0, 36, 2.5), 7),
    ("baseline_g8", "mini_batch", "g8", False, (1.0, 1.0, 36, 2.5), 7),
    ("mini_2col", "mini_batch", "g8", True, (2.0, 1.0, 36, 2.5), 6),
])
def test_train_encrypted_matches_reference_trace(name, mode, sig, enh, sched, iters):
    """The reference's driver, unchanged in behaviour, over the GPU context:
    literal depth-9 circuit, on-demand refresh stand-in, weight trace within
    1e-6 of the reference simulator's (same op counts per iteration)."""
    ds, g = _golden_case(name)
    c = mk(n_q=10, seed=5)
    cfg = O.TrainConfig(mode=mode, batch_size=4, max_iterations=iters, schedule=O.LrSchedule(*sched), sigmoid=sig)
    res = T.train_encrypted(ds, cfg, c.params, ctx=c, enhanced=enh, trace_weights=True, metrics=False)
    assert len(res.weight_trace) == len(g[f"{name}_trace"])
    for a, b in zip(res.weight_trace, g[f"{name}_trace"]):
        close(a, b)
    close(res.weights, g[f"{name}_final"])
    assert [r["muls"] for r in res.ledger] == list(g[f"{name}_muls"])
    assert [r["cmuls"] for r in res.ledger] == list(g[f"{name}_cmuls"])
    assert [r["rotations"] for r in res.ledger] == list(g[f"{name}_rotations"])


class FaultyContext(GpuContext):
    """Fault injection: the n-th ``mul`` raises NeedsBootstrap once, so the
    driver's rollback-refresh-retry path (enctrain.py:386-393) runs."""

    fail_at = None

    def mul(self, a, b):
        if self.fail_at is not None:
            self.fail_at -= 1
            if self.fail_at == 0:
                self.fail_at = None
                raise NeedsBootstrap("injected: mul needs a refresh")
        return super().mul(a, b)


def test_forced_needs_bootstrap_retry():
    ds, g = _golden_case("mini_g8")
    c = FaultyContext(CkksParams.generate(log_n=5, n_q=19, dnum=2), seed=6, max_batch=4)
    c.fail_at = 5 + 3    # inside iteration 2 (5 muls per iteration)
    cfg = O.TrainConfig(mode="mini_batch", batch_size=4, max_iterations=7, schedule=O.LrSchedule(2.0, 1.0, 36, 2.5),
                        sigmoid="g8")
    res = T.train_encrypted(ds, cfg, c.params, ctx=c, trace_weights=True, metrics=False)
    for a, b in zip(res.weight_trace, g["mini_g8_trace"]):
        close(a, b)
    row = res.ledger[1]
    assert row["bootstraps"] == 1 and row["boot_ops"] == 2 * res.layout.col_blocks
    assert row["level_start"] == c.params.log_q
    assert row["muls"] == 5   # counters rolled back before the retry


def test_bootstrap_cadence_and_ledger(rng):
    ds = toy_dataset(rng, n=8, f=3)
    cfg = O.TrainConfig(mode="mini_batch", batch_size=8, max_iterations=6, schedule=O.LrSchedule(2.0, 1.0, 36, 2.5),
                        sigmoid="g8")
    c = mk(n_q=10, seed=7)   # room for exactly one literal (depth-9) iteration
    res = T.train_encrypted(ds, cfg, c.params, ctx=c, metrics=False)
    assert [r["bootstraps"] for r in res.ledger] == [0, 1, 1, 1, 1, 1]
    for row in res.ledger:
        assert row["level_after"] == row["level_start"] - row["consumed_bits"]
        if row["bootstraps"]:
            assert row["level_start"] == c.params.log_q and row["boot_ops"] == 2 * res.layout.col_blocks
        else:
            assert row["level_start"] == row["level_before"]
        assert row["level_after"] >= c.params.log_delta
    c2 = mk(n_q=19, seed=7)  # doubled budget halves the refresh rate
    cfg9 = O.TrainConfig(mode="mini_batch", batch_size=8, max_iterations=9, schedule=O.LrSchedule(2.0, 1.0, 36, 2.5),
                         sigmoid="g8")
    boots = [r["bootstraps"] for r in T.train_encrypted(ds, cfg9, c2.params, ctx=c2, metrics=False).ledger]
    assert np.mean(boots[1:]) <= 0.5


def test_impossible_budget_raises(rng):
    c = mk(n_q=5, seed=8)
    cfg = O.TrainConfig(mode="mini_batch", batch_size=4, max_iterations=1, schedule=O.LrSchedule(2.0, 1.0, 36, 2.5),
                        sigmoid="g8")
    with pytest.raises(NeedsBootstrap, match="bits"):
        T.train_encrypted(toy_dataset(rng), cfg, c.params, ctx=c, metrics=False)


def test_exact_sigmoid_rejected(ctx, rng):
    cfg = O.TrainConfig(mode="mini_batch", batch_size=4, max_iterations=1, sigmoid="exact")
    with pytest.raises(ValueError, match="polynomial"):
        T.train_encrypted(toy_dataset(rng), cfg, ctx.params, ctx=ctx)


def test_train_encrypted_with_real_bootstrapping():
    """The reference driver over a GpuContext whose ``bootstrap`` is REAL CKKS
    bootstrapping (bootstrap='ckks', evaluation keys only; SURVEY.md §8(f) row
    1): same cadence and op ledger as with the stand-in, weight trace within
    the bootstrap's precision of the reference simulator's trace."""
    from paper_2406_13221_b200.bootstrap import bootstrap_ring

    ds, g = _golden_case("mini_g8")
    ring = bootstrap_ring(5, work_levels=9)   # ten working limbs = mk(n_q=10): one literal iteration per refresh
    c = GpuContext(ring, seed=5, max_batch=4, bootstrap="ckks")
    cfg = O.TrainConfig(mode="mini_batch", batch_size=4, max_iterations=7, schedule=O.LrSchedule(2.0, 1.0, 36, 2.5),
                        sigmoid="g8")
    res = T.train_encrypted(ds, cfg, c.params, ctx=c, trace_weights=True, metrics=False)
    assert len(res.weight_trace) == len(g["mini_g8_trace"])
    worst = max(float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) for a, b in zip(res.weight_trace, g["mini_g8_trace"]))
    print(f"train_encrypted with real bootstrapping: max |dw| = {worst:.3e}")
    assert worst < 1e-4
    assert [r["bootstraps"] for r in res.ledger] == [0] + [1] * (len(res.ledger) - 1)
    assert [r["muls"] for r in res.ledger] == list(g["mini_g8_muls"])
    assert c.counters["bootstrap"] >= 2 * (len(res.ledger) - 1) or sum(r["boot_ops"] for r in res.ledger) >= 2
