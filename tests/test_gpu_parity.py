"""Residue-exact parity: every device primitive vs the CPU oracle.

The device library (through its C ABI) and the oracle (oracle/ckks_oracle.c)
get the same ring, the same seeds and the same inputs; every RNS residue of
every output must match bit for bit.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2406_13221_b200.params import CkksParams
from paper_2406_13221_b200.ckks import GpuContext
from paper_2406_13221_b200 import _lib
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


def dev(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def stream():
    return torch.cuda.current_stream().cuda_stream


RINGS = {
    "n32": CkksParams.generate(log_n=5, n_q=4, dnum=2),
    "toy": CkksParams.generate(log_n=13, n_q=8, dnum=3),
    "n2e12": CkksParams.generate(log_n=12, n_q=5, dnum=2),
    "n2e15": CkksParams.generate(log_n=15, n_q=6, dnum=3),
    "n2e16": CkksParams.generate(log_n=16, n_q=8, dnum=3),
    # BASELINE primitive-sweep rings: 50-60-bit primes, so every limb takes the
    # integer (Shoup / 128-bit accumulator) path; dnum 1 and 3, L 16 and 24
    "sweep_i50": CkksParams.generate(log_n=14, n_q=16, dnum=1, scale_bits=50, p_bits=60),
    "sweep_l24": CkksParams.generate(log_n=14, n_q=24, dnum=3, scale_bits=55, p_bits=60),
    # 60-bit special primes above 40-bit scaling primes: the ModDown conversions
    # take the integer path but feed fp64 limbs (the bootstrapping chains' mix)
    "mixed_p60": CkksParams.generate(log_n=12, n_q=6, dnum=2, p_bits=60),
}


@pytest.fixture(scope="module", params=list(RINGS))
def pair(request):
    P = RINGS[request.param]
    ctx = GpuContext(P, seed=5, max_batch=4)
    orc = Oracle(P)
    sk = orc.keygen_secret(ctx.key_seed, P.hw)
    return P, ctx, orc, sk


def test_ntt_roundtrip_and_oracle(pair, rng):
    P, ctx, orc, _ = pair
    n, LK = P.n, P.L + P.K
    data = np.stack([rng.integers(0, q, size=n, dtype=np.uint64) for q in P.primes])[None]
    t = dev(data)
    _lib.call("helr_ntt_fwd", ctx.handle, t.data_ptr(), 0, LK, 1, LK * n, stream())
    fwd = u64(t)
    exp = orc.ntt_batch(data, 0, LK)
    np.testing.assert_array_equal(fwd, exp)
    _lib.call("helr_ntt_inv", ctx.handle, t.data_ptr(), 0, LK, 1, LK * n, stream())
    np.testing.assert_array_equal(u64(t), data)


def test_secret_key(pair):
    P, ctx, orc, sk = pair
    np.testing.assert_array_equal(u64(ctx.sk), sk)


def test_switch_keys(pair):
    P, ctx, orc, sk = pair
    np.testing.assert_array_equal(u64(ctx.rlk), orc.keygen_switch(sk, 0, ctx.key_seed, 0))
    g = ctx.galois_for_rotation(1)
    np.testing.assert_array_equal(u64(ctx.galois_key(g)), orc.keygen_switch(sk, g, ctx.key_seed, g))


def _fresh(ctx, orc, sk, rng, count=2):
    P = ctx.ckks
    z = rng.uniform(-1, 1, size=(count, P.slots))
    scale = P.level_scales[P.top_level]
    coef = ctx.encoder.encode(z, scale)
    first = ctx._next_ct_id
    cts = ctx.encrypt_coefficients(coef, scale)
    ref = orc.encrypt(sk, coef, P.top_level, ctx.enc_seed, first)
    return z, cts, ref


def test_encrypt_decrypt(pair, rng):
    P, ctx, orc, sk = pair
    z, cts, ref = _fresh(ctx, orc, sk, rng)
    got = np.stack([u64(c.data) for c in cts])
    np.testing.assert_array_equal(got, ref)
    dec = np.stack([ctx.decrypt_coefficients(c) for c in cts])
    np.testing.assert_array_equal(dec, orc.decrypt(sk, ref, P.top_level))
    back = ctx.encoder.decode(dec, cts[0].scale)
    assert np.max(np.abs(back - z)) < 1e-6


def test_elementwise(pair, rng):
    P, ctx, orc, sk = pair
    _, cts, ref = _fresh(ctx, orc, sk, rng)
    lvl = P.top_level
    a, b = cts
    for name, sub in (("helr_add", False), ("helr_sub", True)):
        out = ctx._ct_buffer()
        _lib.call(name, ctx.handle, a.data.data_ptr(), b.data.data_ptr(), out.data_ptr(), 1, lvl, stream())
        np.testing.assert_array_equal(u64(out), orc.add(ref[0:1], ref[1:2], lvl, sub=sub)[0])
    k = int(rng.integers(-2**50, 2**50))
    res = ctx._residues(k, lvl)
    cres = np.array([k % q for q in P.q[: lvl + 1]], dtype=np.uint64)
    out = ctx._ct_buffer()
    _lib.call("helr_mul_const", ctx.handle, a.data.data_ptr(), res.data_ptr(), out.data_ptr(), 1, lvl, stream())
    np.testing.assert_array_equal(u64(out), orc.mul_const(ref[0:1], cres, lvl)[0])
    out = ctx._ct_buffer()
    _lib.call("helr_add_const", ctx.handle, a.data.data_ptr(), res.data_ptr(), out.data_ptr(), 1, lvl, stream())
    np.testing.assert_array_equal(u64(out), orc.add_const(ref[0:1], cres, lvl)[0])
    coef = ctx.encoder.encode(rng.normal(size=P.slots), 2.0 ** 30)
    pt = ctx._plain(coef, lvl)
    opt = orc.encode_plain(coef, lvl)[0]
    np.testing.assert_array_equal(u64(pt)[: lvl + 1], opt[: lvl + 1])
    out = ctx._ct_buffer()
    _lib.call("helr_mul_plain", ctx.handle, a.data.data_ptr(), pt.data_ptr(), out.data_ptr(), 1, lvl, stream())
    np.testing.assert_array_equal(u64(out)[:, : lvl + 1], orc.mul_plain(ref[0:1], opt, lvl)[0][:, : lvl + 1])
    # vector cadd (hesim.py:177-184): the plaintext is added to c0 only, residue for residue
    out = ctx._ct_buffer()
    _lib.call("helr_add_plain", ctx.handle, a.data.data_ptr(), pt.data_ptr(), out.data_ptr(), 1, lvl, stream())
    exp = ref[0].copy()
    for p in range(lvl + 1):
        exp[0, p] = (exp[0, p] + opt[p]) % np.uint64(P.q[p])
    np.testing.assert_array_equal(u64(out)[:, : lvl + 1], exp[:, : lvl + 1])
    out = ctx._ct_buffer()
    _lib.call("helr_imul", ctx.handle, a.data.data_ptr(), out.data_ptr(), 1, lvl, stream())
    np.testing.assert_array_equal(u64(out), orc.imul(ref[0:1], lvl)[0])


def test_rescale(pair, rng):
    P, ctx, orc, sk = pair
    _, cts, ref = _fresh(ctx, orc, sk, rng)
    for lvl in (P.top_level, 1):
        out = ctx._empty((2, 2, P.L, P.n))
        both = torch.stack([c.data for c in cts])
        _lib.call("helr_rescale", ctx.handle, both.data_ptr(), out.data_ptr(), 2, lvl, stream())
        exp = orc.rescale(ref, lvl)
        np.testing.assert_array_equal(u64(out)[:, :, :lvl], exp[:, :, :lvl])


def test_mul_relin(pair, rng):
    P, ctx, orc, sk = pair
    _, cts, ref = _fresh(ctx, orc, sk, rng, count=4)
    rlk = orc.keygen_switch(sk, 0, ctx.key_seed, 0)
    for lvl in (P.top_level, 1):
        a = torch.stack([cts[0].data, cts[1].data])
        b = torch.stack([cts[2].data, cts[3].data])
        out = ctx._empty((2, 2, P.L, P.n))
        _lib.call("helr_mul_relin", ctx.handle, a.data_ptr(), b.data_ptr(), ctx.rlk.data_ptr(), out.data_ptr(), 2, lvl,
                  stream())
        exp = orc.mul_relin(ref[0:2].copy(), ref[2:4].copy(), rlk, lvl)
        np.testing.assert_array_equal(u64(out)[:, :, : lvl + 1], exp[:, :, : lvl + 1])


@pytest.mark.parametrize("k", [1, 3, -1])
@pytest.mark.parametrize("acc", [0, 1])
def test_rotate(pair, rng, k, acc):
    P, ctx, orc, sk = pair
    z, cts, ref = _fresh(ctx, orc, sk, rng, count=2)
    g = ctx.galois_for_rotation(k)
    gk = orc.keygen_switch(sk, g, ctx.key_seed, g)
    lvl = P.top_level - 1
    a = torch.stack([c.data for c in cts])
    out = ctx._empty((2, 2, P.L, P.n))
    _lib.call("helr_rotate", ctx.handle, a.data_ptr(), g, ctx.galois_key(g).data_ptr(), out.data_ptr(), 2, lvl, acc,
              stream())
    exp = orc.rotate(ref, g, gk, lvl, accumulate=bool(acc))
    np.testing.assert_array_equal(u64(out)[:, :, : lvl + 1], exp[:, :, : lvl + 1])


def test_refresh(pair, rng):
    P, ctx, orc, sk = pair
    _, cts, ref = _fresh(ctx, orc, sk, rng, count=2)
    a = torch.stack([c.data for c in cts])
    for ratio in (1.0, 0.75):
        out = ctx._empty((2, 2, P.L, P.n))
        _lib.call("helr_refresh", ctx.handle, ctx.sk.data_ptr(), a.data_ptr(), 1, ratio, out.data_ptr(), P.top_level,
                  2, ctx.enc_seed, 777, stream())
        exp = orc.refresh(sk, ref, 1, ratio, P.top_level, ctx.enc_seed, 777)
        np.testing.assert_array_equal(u64(out), exp)


@pytest.mark.parametrize("steps,ident", [((1, 2, 3), 1), ((4, 8, 12), 0), ((-1, -5), 1)])
def test_rotsum_hoisted(pair, rng, steps, ident):
    import ctypes
    P, ctx, orc, sk = pair
    z, cts, ref = _fresh(ctx, orc, sk, rng, count=2)
    gals = [ctx.galois_for_rotation(k) for k in steps]
    keys = [ctx.galois_key(g) for g in gals]
    lvl = P.top_level - 1
    a = torch.stack([c.data for c in cts])
    out = ctx._empty((2, 2, P.L, P.n))
    garr = (ctypes.c_int64 * len(gals))(*gals)
    karr = (ctypes.c_void_p * len(keys))(*[k.data_ptr() for k in keys])
    _lib.call("helr_rotsum", ctx.handle, a.data_ptr(), len(gals), garr, karr, out.data_ptr(), 2, lvl, ident, stream())
    exp = orc.rotsum(ref, gals, [u64(k) for k in keys], lvl, include_identity=bool(ident))
    np.testing.assert_array_equal(u64(out)[:, :, : lvl + 1], exp[:, :, : lvl + 1])
    # values: decrypt == sum of np.roll (hesim.py:222 semantics)
    want = sum(np.roll(z[0], -k) for k in steps) + (z[0] if ident else 0)
    dec = ctx.encoder.decode(orc.decrypt(sk, exp[:1], lvl)[0], cts[0].scale)
    assert np.abs(dec - want).max() < 1e-6


def test_mul_relin_rescale_merged(pair, rng):
    P, ctx, orc, sk = pair
    _, cts, ref = _fresh(ctx, orc, sk, rng, count=4)
    rlk = orc.keygen_switch(sk, 0, ctx.key_seed, 0)
    for lvl in (P.top_level, 1):
        a = torch.stack([cts[0].data, cts[1].data])
        b = torch.stack([cts[2].data, cts[3].data])
        out = ctx._empty((2, 2, P.L, P.n))
        _lib.call("helr_mul_relin_rescale", ctx.handle, a.data_ptr(), b.data_ptr(), ctx.rlk.data_ptr(),
                  out.data_ptr(), 2, lvl, stream())
        exp = orc.mul_relin_rescale(ref[0:2].copy(), ref[2:4].copy(), rlk, lvl)
        np.testing.assert_array_equal(u64(out)[:, :, :lvl], exp[:, :, :lvl])
