"""Device metrics (helr_metrics) against optimizer.py's restatement of the
reference's log_likelihood / predict / accuracy / auroc (optim.py:123-229)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2406_13221_b200 import data
from paper_2406_13221_b200.ckks import GpuContext
from paper_2406_13221_b200.metrics import DeviceMetrics
from paper_2406_13221_b200.optimizer import accuracy, auroc, log_likelihood, predict
from paper_2406_13221_b200.params import CkksParams

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return GpuContext(CkksParams.generate(log_n=10, n_q=8, dnum=2), seed=1, max_batch=1)


@pytest.mark.parametrize("n,d,ties", [(1, 3, False), (777, 16, False), (5000, 33, True), (70000, 64, False)])
def test_metrics_match_host(ctx, n, d, ties):
    rng = np.random.default_rng(n)
    X = rng.uniform(-1, 1, size=(n, d))
    X[:, 0] = 1.0
    if ties:
        X = np.round(X * 2) / 2  # many tied scores
    y = np.where(rng.uniform(size=n) < 0.3, 1.0, -1.0)
    if n == 1:
        y[:] = 1.0
    w = rng.normal(size=d) * 0.5
    dm = DeviceMetrics(ctx, X, y)
    got = dm.evaluate(w)
    Z = X * y[:, None]
    assert got["log_likelihood"] == pytest.approx(log_likelihood(Z, w), rel=1e-12, abs=1e-12)
    assert got["accuracy"] == accuracy(y, predict(w, X))
    assert got["n_pos"] == int((y > 0).sum())
    if 0 < got["n_pos"] < n:
        assert got["auroc"] == pytest.approx(auroc(y, X @ w), abs=1e-12)
    else:
        assert got["auroc"] is None
        with pytest.raises(ValueError):
            dm.auroc(w)


def test_paper_shape_metrics(ctx):
    ds = data.paper_dataset()
    rng = np.random.default_rng(9)
    w = rng.normal(size=ds.X.shape[1]) * 0.1
    dm = DeviceMetrics(ctx, ds.X, ds.y)
    got = dm.evaluate(w)
    assert got["auroc"] == pytest.approx(auroc(ds.y, ds.X @ w), abs=1e-12)
    assert got["log_likelihood"] == pytest.approx(log_likelihood(ds.X * ds.y[:, None], w), rel=1e-12)


def test_train_encrypted_per_op_path_with_device_metrics():
    """The drop-in surface: train_encrypted (enctrain.py:303-449 mirror) on the
    per-op GpuContext evaluator; its per-iteration metrics come from the
    device and equal the host functions on the decrypted weights."""
    from paper_2406_13221_b200 import enctrain as T
    from paper_2406_13221_b200.optimizer import TrainConfig, ExpDecay
    ds = data.toy_dataset()
    ck = CkksParams.generate(log_n=13, n_q=12, dnum=2)
    g = GpuContext(ck, seed=1)
    cfg = TrainConfig(mode="mini_batch", batch_size=128, max_iterations=2, schedule=ExpDecay(), sigmoid="g8")
    res = T.train_encrypted(ds, cfg, g.params, val=ds, ctx=g, trace_weights=True)
    assert len(res.metrics) == 2
    for m, w in zip(res.metrics, res.weight_trace):
        assert m["train_acc"] == accuracy(ds.y, predict(w, ds.X))
        assert m["auroc"] == pytest.approx(auroc(ds.y, ds.X @ w), abs=1e-12)
        assert m["log_likelihood"] == pytest.approx(log_likelihood(ds.X * ds.y[:, None], w), rel=1e-12)
