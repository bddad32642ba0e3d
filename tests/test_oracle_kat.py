"""Known-answer tests that pin the CPU RNS-CKKS oracle (no GPU needed).

The reference has no ring arithmetic, so the oracle is
pinned by independent big-integer restatements: schoolbook negacyclic
products, exact CRT rescale / basis conversion formulas, and the
reference's own slot semantics (rotation == np.roll, hesim.py:222).
"""

import numpy as np
import pytest

from paper_2406_13221_b200.encoder import Encoder
from paper_2406_13221_b200.params import CkksParams, is_prime
from oracle.oracle import Oracle, prng

SMALL = CkksParams.generate(log_n=5, n_q=4, dnum=2)
MID = CkksParams.generate(log_n=10, n_q=6, dnum=3)


def brv(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2)


def centred(v, q):
    v = int(v) % q
    return v - q if v > q // 2 else v


def crt(residues, primes):
    Q = 1
    for p in primes:
        Q *= p
    x = 0
    for r, p in zip(residues, primes):
        Mi = Q // p
        x += int(r) * Mi * pow(Mi, -1, p)
    return x % Q, Q


@pytest.fixture(scope="module")
def small():
    return Oracle(SMALL)


def test_prng_pinned():
    # counter-based generator spec (modarith.cuh / ckks_oracle.c): fixed outputs
    vals = [prng(0, 0, 0), prng(1, 2, 3), prng(2 ** 63, 5, 10 ** 9)]
    assert vals == [0x568A9B0B1A2C05EC, 0xDAC0B083A7C5FEA9, 0x0CC4863CC59AD0B4]


def test_params_chain():
    for P in (SMALL, MID):
        for q in P.primes:
            assert is_prime(q) and q < 2 ** 61 and (q - 1) % (2 * P.n) == 0
            psi = P.psi[P.primes.index(q)]
            assert pow(psi, P.n, q) == q - 1
        # P exceeds the largest digit modulus (the one holding q_0)
        digit = 1
        for q in P.q[:P.alpha]:
            digit *= q
        prod_p = 1
        for p in P.p:
            prod_p *= p
        assert prod_p > digit
        s = P.level_scales
        for lvl in range(1, P.L):
            assert s[lvl - 1] == pytest.approx(s[lvl] ** 2 / P.q[lvl], rel=1e-15)


@pytest.mark.parametrize("p", range(SMALL.L + SMALL.K))
def test_ntt_is_evaluation_at_odd_powers(small, p, rng):
    q, psi, N = SMALL.primes[p], SMALL.psi[p], SMALL.n
    a = rng.integers(0, q, N, dtype=np.uint64)
    A = small.ntt(a, p)
    for i in range(N):
        e = 2 * brv(i, SMALL.log_n) + 1
        assert int(A[i]) == sum(int(a[k]) * pow(psi, e * k, q) for k in range(N)) % q
    np.testing.assert_array_equal(small.ntt(A, p, inverse=True), a)


@pytest.mark.parametrize("p", [0, 2, 5])
def test_ntt_product_is_negacyclic_schoolbook(small, p, rng):
    q, N = SMALL.primes[p], SMALL.n
    a = rng.integers(0, q, N, dtype=np.uint64)
    b = rng.integers(0, q, N, dtype=np.uint64)
    A, B = small.ntt(a, p), small.ntt(b, p)
    c = small.ntt(np.array([int(x) * int(y) % q for x, y in zip(A, B)], dtype=np.uint64), p, inverse=True)
    ref = [0] * N
    for i in range(N):
        for j in range(N):
            v = int(a[i]) * int(b[j])
            if i + j < N:
                ref[i + j] += v
            else:
                ref[i + j - N] -= v
    assert [x % q for x in ref] == [int(x) for x in c]


def test_rescale_is_rounded_division(rng):
    orc = Oracle(MID)
    sk = orc.keygen_secret(3)
    lvl = MID.top_level
    ct = orc.ct_zeros(1)
    for k in range(2):
        for p in range(lvl + 1):
            ct[0, k, p] = rng.integers(0, MID.q[p], MID.n, dtype=np.uint64)
    out = orc.rescale(ct, lvl)
    ql = MID.q[lvl]
    primes = MID.q[:lvl + 1]
    for k in range(2):
        coef = np.stack([orc.ntt(ct[0, k, p], p, inverse=True) for p in range(lvl + 1)])
        got = np.stack([orc.ntt(out[0, k, p], p, inverse=True) for p in range(lvl)])
        for i in range(0, MID.n, 97):
            x, Q = crt(coef[:, i], primes)
            r = centred(x % ql, ql)
            y = (x - r) // ql
            for p in range(lvl):
                assert int(got[p, i]) == y % MID.q[p]


def test_fast_basis_conversion_formula(rng):
    orc = Oracle(MID)
    src, dst = [0, 1, 2], [3, 4, MID.L, MID.L + 1]
    coef = np.stack([rng.integers(0, MID.primes[s], MID.n, dtype=np.uint64) for s in src])
    out = orc.basis_convert(coef, src, dst)
    D = 1
    for s in src:
        D *= MID.primes[s]
    for i in range(0, MID.n, 61):
        total = 0
        for k, s in enumerate(src):
            pk = MID.primes[s]
            Dk = D // pk
            total += (int(coef[k, i]) * pow(Dk, -1, pk) % pk) * Dk
        for d, t in enumerate(dst):
            assert int(out[d, i]) == total % MID.primes[t]


def test_keyswitch_decrypt_equivalence(rng):
    """k0 + k1 s == d s' up to a small, zero-mean error (centred ModDown)."""
    orc = Oracle(MID)
    sk = orc.keygen_secret(9)
    lvl = MID.top_level
    d = np.stack([rng.integers(0, q, MID.n, dtype=np.uint64) for q in MID.q[:lvl + 1]])
    rlk = orc.keygen_switch(sk, 0, 9, 0)
    k0, k1 = orc.keyswitch(d, rlk, lvl)
    q = MID.q[0]
    s = [int(x) for x in sk[0]]
    err = np.array([(int(k0[0][i]) + int(k1[0][i]) * s[i] - int(d[0][i]) * s[i] * s[i]) % q
                    for i in range(MID.n)], dtype=np.uint64)
    e = orc.ntt(err, 0, inverse=True)
    ec = np.array([centred(x, q) for x in e], dtype=float)
    assert np.abs(ec).max() < 200
    assert abs(ec.mean()) < 5


@pytest.mark.parametrize("k", [1, 5, -1, -7])
def test_rotation_matches_np_roll(k, rng):
    """decrypt(rotate(ct, k)) == np.roll(slots, -k) (hesim.py:218-226)."""
    P = CkksParams.generate(log_n=11, n_q=5, dnum=2)
    orc = Oracle(P)
    enc = Encoder(P.log_n)
    sk = orc.keygen_secret(4)
    z = rng.uniform(-1, 1, P.slots) + 1j * rng.uniform(-1, 1, P.slots)
    s = P.level_scales[P.top_level]
    ct = orc.encrypt(sk, enc.encode(z, s), P.top_level, 6, 1)
    g = pow(5, k % P.slots, 2 * P.n)
    gk = orc.keygen_switch(sk, g, 4, g)
    r = orc.rotate(ct, g, gk, P.top_level)
    got = enc.decode(orc.decrypt(sk, r, P.top_level)[0], s)
    assert np.abs(got - np.roll(z, -k)).max() < 1e-8


def test_mul_relin_rescale_values(rng):
    P = CkksParams.generate(log_n=11, n_q=5, dnum=2)
    orc = Oracle(P)
    enc = Encoder(P.log_n)
    sk = orc.keygen_secret(4)
    a, b = rng.uniform(-2, 2, P.slots), rng.uniform(-2, 2, P.slots)
    top = P.top_level
    s = P.level_scales[top]
    ca = orc.encrypt(sk, enc.encode(a, s), top, 6, 1)
    cb = orc.encrypt(sk, enc.encode(b, s), top, 6, 2)
    rlk = orc.keygen_switch(sk, 0, 4, 0)
    out = orc.rescale(orc.mul_relin(ca, cb, rlk, top), top)
    got = enc.decode(orc.decrypt(sk, out, top - 1)[0], s * s / P.q[top])
    assert np.abs(got - a * b).max() < 1e-8


def test_refresh_keeps_message(rng):
    orc = Oracle(SMALL)
    sk = orc.keygen_secret(2)
    msg = rng.integers(-2 ** 40, 2 ** 40, SMALL.n, dtype=np.int64)
    ct = orc.encrypt(sk, msg, 0, 3, 1)
    m0 = orc.decrypt(sk, ct, 0)[0]
    out = orc.refresh(sk, ct, 0, 1.0, SMALL.top_level, 3, 9)
    m1 = orc.decrypt(sk, out, SMALL.top_level)[0]
    assert np.abs(m1 - m0).max() <= 2 * 21  # fresh error bound (centred binomial, eta = 21)
