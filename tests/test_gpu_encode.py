"""Device-side CKKS encoding / decoding (helr_encode / helr_decode, csrc/encode.cu)
against the host encoder (encoder.py, the canonical embedding behind
SimContext.enc / dec, hesim.py:146-162).  Floating-point parity: a coefficient
may differ by one unit where scale * m lies within rounding error of a
half-integer; decoded slots agree to 1e-9 relative."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2406_13221_b200 import _lib, data
from paper_2406_13221_b200.ckks import GpuContext
from paper_2406_13221_b200.driver import FusedTrainer
from paper_2406_13221_b200.params import CkksParams

pytestmark = pytest.mark.gpu
COEF_TOL = 1          # units of the integer coefficient
DIFF_FRACTION = 0.01  # at most 1% of coefficients may round the other way
SLOT_TOL = 1e-9       # decoded slots, relative to the slot magnitude


@pytest.fixture(scope="module", params=[13, 16])
def ctx(request):
    return GpuContext(CkksParams.generate(log_n=request.param, n_q=8, dnum=2), seed=4, max_batch=2)


@pytest.mark.parametrize("kind", ["real", "complex", "short"])
def test_encode_matches_host(ctx, kind):
    S = ctx.ckks.slots
    rng = np.random.default_rng(11)
    if kind == "real":
        z = rng.uniform(-1, 1, size=(5, S))
    elif kind == "complex":
        z = rng.uniform(-1, 1, size=(3, S)) + 1j * rng.uniform(-1, 1, size=(3, S))
    else:  # fewer than N/2 values: zero padded, like SimContext.enc
        z = rng.uniform(-4, 4, size=(2, S // 3))
    scale = 2.0 ** 40
    want = ctx.encoder.encode(z, scale)
    got = ctx.encode_slots(z, scale).cpu().numpy()
    diff = np.abs(got - want)
    assert diff.max() <= COEF_TOL
    assert (diff > 0).mean() <= DIFF_FRACTION


def test_decode_matches_host(ctx):
    rng = np.random.default_rng(12)
    n = ctx.ckks.n
    coef = rng.integers(-(1 << 45), 1 << 45, size=(4, n), dtype=np.int64)
    scale = 2.0 ** 40
    want = ctx.encoder.decode(coef, scale)
    got = ctx.decode_coefficients(torch.from_numpy(coef).cuda(), scale)
    assert np.max(np.abs(got - want)) <= SLOT_TOL * max(1.0, np.max(np.abs(want)))


def test_roundtrip_and_encrypt_decrypt(ctx):
    ck = ctx.ckks
    rng = np.random.default_rng(13)
    z = rng.uniform(-1, 1, size=(2, ck.slots))
    scale = 2.0 ** 40
    coef = ctx.encode_slots(z, scale)
    back = ctx.decode_coefficients(coef, scale)
    assert np.max(np.abs(back - z)) < 2.0 ** -30
    ct = ctx._empty((2, 2, ck.L, ck.n))
    ctx.encrypt_to(coef, ct, ck.top_level)
    dec = ctx._empty((2, ck.n))
    ctx._call("helr_decrypt", ctx.sk.data_ptr(), ct.data_ptr(), 2, ck.top_level, dec.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    slots = ctx.decode_coefficients(dec, scale)
    assert np.max(np.abs(slots - z)) < 1e-6


def test_encode_overflow_raises(ctx):
    with pytest.raises(_lib.HelrError, match="2\\*\\*62"):
        ctx.encode_slots(np.full((1, 4), 1e9), 2.0 ** 50)
    with pytest.raises(ValueError):
        ctx.encode_slots(np.zeros((1, ctx.ckks.slots + 1)), 1.0)


def test_trainer_device_encoding_matches_host_encoding():
    """client_prepare on the device leaves the training trajectory unchanged
    (weights after 4 toy iterations within 1e-9 of the host-encoded run)."""
    ds = data.toy_dataset()
    ck = CkksParams.generate(log_n=13, n_q=8, dnum=2)
    ws = []
    for dev in (False, True):
        tr = FusedTrainer(GpuContext(ck, seed=2, max_batch=8), ds, rows_per_block=128, mode="mini_batch",
                          device_encode=dev)
        for _ in range(4):
            tr.iterate()
        ws.append(tr.weights())
        tr.close()
    assert np.max(np.abs(ws[0] - ws[1])) < 1e-9
