"""Oracle restatement of the fused depth-7 NAG iteration (csrc/nag.cu),
composed from the CPU oracle's primitives.  TEST INFRASTRUCTURE ONLY.

Given the same input ciphertexts, keys and per-limb constants as
``helr_nag_iteration``, every residue of the updated W and V must match.
Each step cites the reference circuit piece it computes:
enc_gradient (enctrain.py:162-197), sum_col_vec (hesim.py:240-265),
sum_rows (hesim.py:267-281), enc_quad_gradient (enctrain.py:200-208),
enc_nag_update (enctrain.py:211-239).
"""

from __future__ import annotations

import numpy as np


def _modadd(a, b, level, primes):
    out = a.copy()
    for p in range(level + 1):
        q = np.uint64(primes[p])
        s = a[..., p, :] + b[..., p, :]
        out[..., p, :] = np.where(s >= q, s - q, s)
    return out


def _tensor_sum_relin(orc, pairs, rlk, level):
    """relin(sum_t a_t (x) b_t) for one output ciphertext (no rescale)."""
    primes = orc.params.q
    d = None
    for a, b in pairs:
        t = orc.tensor(a, b, level)
        d = t if d is None else _modadd(d, t, level, primes)
    k0, k1 = orc.keyswitch(np.ascontiguousarray(d[2][: level + 1]), rlk, level)
    out = np.zeros((1, 2, orc.L, orc.N), dtype=np.uint64)
    for p in range(level + 1):
        q = np.uint64(primes[p])
        s0 = d[0, p] + k0[p]
        s1 = d[1, p] + k1[p]
        out[0, 0, p] = np.where(s0 >= q, s0 - q, s0)
        out[0, 1, p] = np.where(s1 >= q, s1 - q, s1)
    return out


def _tensor_sum_relin_rescale(orc, pairs, rlk, level):
    """rescale(relin(sum_t a_t (x) b_t)) with the merged ModDown (device
    op_mul_relin_rescale_sum), output at level-1."""
    primes = orc.params.q
    d = None
    for a, b in pairs:
        t = orc.tensor(a, b, level)
        d = t if d is None else _modadd(d, t, level, primes)
    return orc.relin_rescale_tensor(d, rlk, level)


def _galois(k: int, n: int) -> int:
    return pow(5, k % (n // 2), 2 * n)


def _lincomb(orc, terms, level):
    """sum_t C_t * X_t (per-limb constants), no rescale."""
    acc = None
    for x, cst in terms:
        y = orc.mul_const(x, cst, level)
        acc = y if acc is None else orc.add(acc, y, level)
    return acc


def rotsum_groups(log_total: int, max_bits: int) -> list:
    """Group bit-widths of a grouped rotate-and-sum (helr_rotsum_groups in
    csrc/nag.cu): ceil(log_total / max_bits) groups, bits spread evenly,
    larger groups first."""
    if log_total <= 0 or max_bits <= 0:
        return []
    ng = -(-log_total // max_bits)
    base, rem = divmod(log_total, ng)
    return [base + 1 if j < rem else base for j in range(ng)]


def grouped_steps(log_total: int, max_bits: int, stride: int = 1) -> list:
    """Rotation steps of every group, in key order."""
    out, off = [], 0
    for bits in rotsum_groups(log_total, max_bits):
        out.append([(stride * k) << off for k in range(1, 1 << bits)])
        off += bits
    return out


def _bsgs(orc, x, gkeys, log_g, bs, sign, level, stride=1):
    """sum_{k < 2^log_g} rot(x, sign stride k) as grouped hoisted rotate-and-sums
    (helr_rotsum, one ModUp / ModDown per group)."""
    N = orc.N
    x = np.ascontiguousarray(x)
    for steps in grouped_steps(log_g, bs, stride):
        gal = [_galois(sign * k, N) for k in steps]
        x = orc.rotsum(x, gal, [gkeys[g] for g in gal], level, include_identity=True)
    return x


def nag_iteration(orc, z, w, v, bbar, lw, rlk, gkeys, mask_pt, consts, log_g, log_m, phase=0, grad=None,
                  log_baby=0, log_baby_rows=0):
    """z: u64[R][C][2][L][N]; w, v, bbar, grad: u64[C][2][L][N];
    gkeys: galois element -> key; consts: u64[10][L].
    Returns (w', v') for phase 0, the gradient for phases 1/2, (w', v') for 3."""
    N = orc.N
    R, C = z.shape[0], z.shape[1]
    S = N // 2
    g = 1 << log_g
    K = [np.ascontiguousarray(consts[k]) for k in range(consts.shape[0])]
    if phase != 3:
        rows = []
        for r in range(R):
            # P = Z . W summed over column blocks (enctrain.py:181-183), rescaled
            x = _tensor_sum_relin_rescale(orc, [(z[r, j][None], w[j][None]) for j in range(C)], rlk, lw)
            # sum_col_vec left half (hesim.py:255-257)
            if log_baby > 0:
                x = _bsgs(orc, x, gkeys, log_g, log_baby, +1, lw - 1)
            else:
                for i in range(log_g):
                    ge = _galois(1 << i, N)
                    x = orc.rotate(x, ge, gkeys[ge], lw - 1, accumulate=True)
            # row-start mask (hesim.py:258-260)
            x = orc.rescale(orc.mul_plain(x, mask_pt, lw - 1), lw - 1)
            # right half (hesim.py:262-264)
            if log_baby > 0:
                x = _bsgs(orc, x, gkeys, log_g, log_baby, -1, lw - 2)
            else:
                for i in range(log_g):
                    ge = _galois(S - (1 << i), N)
                    x = orc.rotate(x, ge, gkeys[ge], lw - 2, accumulate=True)
            u = x
            # complement polynomial q0 + q1 u + q2 u^2 + q3 u^3 (enctrain.py:186-191)
            u2 = orc.mul_relin_rescale(u, u, rlk, lw - 2)
            tq = orc.rescale(orc.mul_const(u, K[0], lw - 2), lw - 2)
            qu = orc.mul_relin_rescale(u2, tq, rlk, lw - 3)
            lin = orc.rescale(_lincomb(orc, [(u, K[1]), (u2, K[2])], lw - 3), lw - 3)
            qu = orc.add(qu, lin, lw - 4)
            qu = orc.add_const(qu, K[3], lw - 4)
            rows.append(qu)
        # per column block: sum_r qu_r . Z_rj (enctrain.py:193-196 + block sum 374-379)
        gsum = np.zeros((C, 2, orc.L, N), dtype=np.uint64)
        for j in range(C):
            gsum[j] = _tensor_sum_relin_rescale(orc, [(rows[r], z[r, j][None]) for r in range(R)], rlk, lw - 4)[0]
        if phase == 1:
            return gsum
        if phase == 2:
            return orc.add(grad, gsum, lw - 5)
        G = gsum
    else:
        G = grad
    # sum_rows on the batch total (hesim.py:278-280)
    if log_baby_rows > 0:
        G = _bsgs(orc, G, gkeys, log_m, log_baby_rows, +1, lw - 5, stride=g)
    else:
        for i in range(log_m):
            ge = _galois(g << i, N)
            G = orc.rotate(np.ascontiguousarray(G), ge, gkeys[ge], lw - 5, accumulate=True)
    # quadratic gradient (enctrain.py:200-208)
    D = np.zeros_like(G)
    for j in range(C):
        D[j] = orc.mul_relin_rescale(G[j][None], bbar[j][None], rlk, lw - 5)[0]
    # NAG update (enctrain.py:211-239)
    nv = _lincomb(orc, [(w, K[4]), (D, K[5])], lw - 6)
    nw = _lincomb(orc, [(w, K[6]), (v, K[7]), (D, K[8])], lw - 6)
    return orc.rescale(nw, lw - 6), orc.rescale(nv, lw - 6)
