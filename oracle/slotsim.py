"""Slot-level oracle: a numpy restatement of the reference simulator and its
training circuit.  TEST INFRASTRUCTURE ONLY (and the timed CPU "reference"
arm of bench.py, which runs the reference's own algorithm on host cores).

Restated from the reference (pkg/src/helr):
- ``SlotSim``: hesim.py:110-281 with the noise model off — slots are
  complex128[N/2], level bits drop by log_delta per ct x ct product and
  log_delta_c per constant product (hesim.py:136-142, 186-206), rotations
  are np.roll by -k (hesim.py:218-226), sum_col_vec / sum_rows are the
  rotate-and-add reductions of hesim.py:240-281.
- ``gradient_block``: enc_gradient, enctrain.py:162-197 (literal circuit:
  Z.W, sum_col_vec, u^2, q3 u^2 + q1, u * inner, + q0, * Z, sum_rows).
- ``train``: the BASELINE composition of the reference primitives
  (SURVEY.md §8(c) recipe): per batch of row blocks, sum of block
  gradients, one B̄ product (enctrain.py:200-208) and the NAG update
  (enctrain.py:211-239), gamma = lr / real rows (enhanced), eta =
  (1 - alpha0) / alpha1, alpha recurrence enctrain.py:110-111.

This module does not import the product package; its results are pinned to
the real reference by tests/golden/ (tools/make_goldens.py ran the
reference itself from /root/reference).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np


class SlotNeedsBootstrap(Exception):
    pass


@dataclass
class SlotCt:
    slots: np.ndarray
    level_bits: int
    scale_bits: int
    boot_count: int = 0


class SlotSim:
    def __init__(self, log_n: int, log_q: int, log_delta: int, log_delta_c: int):
        self.S = 1 << (log_n - 1)
        self.log_q, self.log_delta, self.log_delta_c = log_q, log_delta, log_delta_c
        self.counters = {k: 0 for k in ("enc", "dec", "add", "cadd", "mul", "cmul", "imul", "rotate", "bootstrap")}

    def _left(self, level, cost, op):
        rest = level - cost
        if rest < self.log_delta:
            raise SlotNeedsBootstrap(f"{op} needs {cost + self.log_delta} bits but only {level} remain")
        return rest

    def enc(self, m) -> SlotCt:
        m = np.asarray(m, dtype=np.complex128).ravel()
        if m.size > self.S:
            raise ValueError("message too long")
        s = np.zeros(self.S, dtype=np.complex128)
        s[: m.size] = m
        self.counters["enc"] += 1
        return SlotCt(s, self.log_q, self.log_delta)

    def dec(self, a: SlotCt) -> np.ndarray:
        self.counters["dec"] += 1
        return a.slots.copy()

    def add(self, a, b):
        if a.scale_bits != b.scale_bits:
            raise ValueError("scale mismatch")
        self.counters["add"] += 1
        return SlotCt(a.slots + b.slots, min(a.level_bits, b.level_bits), a.scale_bits,
                      max(a.boot_count, b.boot_count))

    def cadd(self, a, c):
        self.counters["cadd"] += 1
        return SlotCt(a.slots + np.asarray(c, dtype=np.complex128), a.level_bits, a.scale_bits, a.boot_count)

    def mul(self, a, b):
        lvl = self._left(min(a.level_bits, b.level_bits), self.log_delta, "mul")
        self.counters["mul"] += 1
        return SlotCt(a.slots * b.slots, lvl, a.scale_bits + b.scale_bits - self.log_delta,
                      max(a.boot_count, b.boot_count))

    def cmul(self, a, c):
        lvl = self._left(a.level_bits, self.log_delta_c, "cmul")
        self.counters["cmul"] += 1
        return SlotCt(a.slots * np.asarray(c, dtype=np.complex128), lvl, a.scale_bits, a.boot_count)

    def imul(self, a):
        self.counters["imul"] += 1
        return SlotCt(a.slots * 1j, a.level_bits, a.scale_bits, a.boot_count)

    def rotate(self, a, k):
        self.counters["rotate"] += 1
        return SlotCt(np.roll(a.slots, -k), a.level_bits, a.scale_bits, a.boot_count)

    def bootstrap(self, a):
        self.counters["bootstrap"] += 1
        return SlotCt(a.slots.copy(), self.log_q, a.scale_bits, a.boot_count + 1)

    def sum_col_vec(self, a, m, g):
        if g == 1:
            return a
        acc, step = a, 1
        while step < g:
            acc = self.add(acc, self.rotate(acc, step))
            step *= 2
        mask = np.zeros(self.S)
        mask[::g] = 1.0
        acc = self.cmul(acc, mask)
        step = 1
        while step < g:
            acc = self.add(acc, self.rotate(acc, -step))
            step *= 2
        return acc

    def sum_rows(self, a, m, g):
        acc, step = a, g
        while step < m * g:
            acc = self.add(acc, self.rotate(acc, step))
            step *= 2
        return acc


def gradient_block(sim: SlotSim, z_row, w, qpoly, m, g):
    """enc_gradient (enctrain.py:162-197) for one row block (list over col blocks)."""
    q0, q1, q2, q3 = qpoly
    acc = None
    for zc, wc in zip(z_row, w):
        p = sim.mul(zc, wc)
        acc = p if acc is None else sim.add(acc, p)
    u = sim.sum_col_vec(acc, m, g)
    u2 = sim.mul(u, u)
    inner = sim.cadd(sim.cmul(u2, q3), q1)
    qu = sim.mul(u, inner)
    if q2 != 0.0:
        qu = sim.add(qu, sim.cmul(u2, q2))
    qu = sim.cadd(qu, q0)
    return [sim.sum_rows(sim.mul(qu, zc), m, g) for zc in z_row]


def _blocks(Z, m, g):
    n, cols = Z.shape
    rb, cb = -(-n // m), -(-cols // g)
    pad = np.zeros((rb * m, cb * g))
    pad[:n, :cols] = Z
    return pad.reshape(rb, m, cb, g).transpose(0, 2, 1, 3).reshape(rb, cb, m * g)


def _replicate(v, m, g, cb):
    seg = np.zeros(cb * g)
    seg[: v.size] = v
    return [np.tile(seg[j * g:(j + 1) * g], m) for j in range(cb)]


def bbar_of(X, eps=1e-8):
    """1 / (eps + sum_k |X'X/4|_jk) (quadgrad.py:53-73)."""
    H = np.abs(0.25 * (X.T @ X))
    return 1.0 / (eps + H.sum(axis=1))


def train(X, y, log_n, m, blocks_per_batch, qpoly, lr_fn, iterations, mode="mini_batch", eps=1e-8,
          log_delta=40, trace=True, stamps=None):
    """BASELINE recipe over the slot simulator; returns (weights trace, final w).

    ``stamps``: optional list that receives time.perf_counter() at the start
    of every iteration and once after the last (bench.py's CPU arm times the
    iterations only, not the encryption of the dataset)."""
    S = 1 << (log_n - 1)
    g = S // m
    sim = SlotSim(log_n, log_q=10 ** 7, log_delta=log_delta, log_delta_c=log_delta)
    n, cols = X.shape
    Z = X * y[:, None]
    zb = _blocks(Z, m, g)
    rb, cb = zb.shape[0], zb.shape[1]
    cz = [[sim.enc(zb[i, j]) for j in range(cb)] for i in range(rb)]
    rows_per_batch = m * blocks_per_batch
    nb = -(-rb // blocks_per_batch)
    scal = [bbar_of(X[k * rows_per_batch:min((k + 1) * rows_per_batch, n)], eps) for k in range(nb)]
    if mode == "full_batch":
        merged = 1.0 / np.sum([1.0 / s for s in scal], axis=0)
        cbar = [[sim.enc(v) for v in _replicate(merged, m, g, cb)]]
    else:
        cbar = [[sim.enc(v) for v in _replicate(s, m, g, cb)] for s in scal]
    w = [sim.enc(np.zeros(S)) for _ in range(cb)]
    v = [sim.enc(np.zeros(S)) for _ in range(cb)]
    a0 = 0.01
    a1 = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * a0 * a0))
    out = []
    for t in range(iterations):
        if stamps is not None:
            stamps.append(time.perf_counter())
        if mode == "mini_batch":
            b = t % nb
            blk = list(range(b * blocks_per_batch, min((b + 1) * blocks_per_batch, rb)))
            rows = min(rows_per_batch, n - b * rows_per_batch)
            bsel = cbar[b]
        else:
            blk = list(range(rb))
            rows = n
            bsel = cbar[0]
        lr = lr_fn(t)
        eta = (1.0 - a0) / a1
        gamma = lr / rows
        gsum = None
        for k in blk:
            gk = gradient_block(sim, cz[k], w, qpoly, m, g)
            gsum = gk if gsum is None else [sim.add(x, y2) for x, y2 in zip(gsum, gk)]
        G = [sim.mul(gj, bj) for gj, bj in zip(gsum, bsel)]
        mult = 1.0 + gamma
        nw, nv = [], []
        for j in range(cb):
            vt = sim.add(w[j], sim.cmul(G[j], mult))
            nw.append(sim.add(sim.cmul(vt, 1.0 - eta), sim.cmul(v[j], eta)))
            nv.append(vt)
        w = [sim.bootstrap(c) for c in nw]
        v = [sim.bootstrap(c) for c in nv]
        a0, a1 = a1, 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * a1 * a1))
        if trace:
            out.append(np.concatenate([np.real(c.slots.reshape(m, g)[0]) for c in w])[:cols])
    if stamps is not None:
        stamps.append(time.perf_counter())
    final = np.concatenate([np.real(c.slots.reshape(m, g)[0]) for c in w])[:cols]
    return out, final


def auroc(y, scores):
    """Midrank AUROC (optim.py:209-229)."""
    y = np.asarray(y)
    s = np.asarray(scores, dtype=np.float64)
    order = np.argsort(s, kind="mergesort")
    ss = s[order]
    ranks = np.empty(s.size)
    i = 0
    while i < s.size:
        j = i
        while j + 1 < s.size and ss[j + 1] == ss[i]:
            j += 1
        ranks[order[i:j + 1]] = 0.5 * (i + j) + 1.0
        i = j + 1
    pos = y > 0
    npos, nneg = int(pos.sum()), int((~pos).sum())
    return (ranks[pos].sum() - npos * (npos + 1) / 2.0) / (npos * nneg)
