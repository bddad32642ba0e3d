#!/usr/bin/env python
"""Where does the fused trainer's weight error come from?  A slot-level
model of the depth-7 fused iteration (csrc/nag.cu) over the paper_mini
workload with individually switchable, *deterministic* CKKS encoding errors
and random per-iteration noise, compared with the reference golden trace
(tests/golden/paper_mini.npz).  CPU only; ~30 s per configuration.

    python tools/precision_probe.py [config ...]

configs: exact | mask:<bits> | z:<bits> | bbar:<bits> | wnoise:<rel> | unoise:<abs> | znoise:<abs> | bnoise:<rel>
(several may be combined with '+', e.g. mask:33+z:40)
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2406_13221_b200.data import paper_dataset  # noqa: E402
from paper_2406_13221_b200.encoder import Encoder  # noqa: E402
from paper_2406_13221_b200.optimizer import BASELINE_CUBIC  # noqa: E402

LOG_N, M, G, R = 16, 128, 256, 8
S = 1 << (LOG_N - 1)


def roundtrip(enc, v, bits):
    """decode(encode(v at scale 2^bits)): the deterministic encoding error."""
    sc = 2.0 ** bits
    return np.real(enc.decode(enc.encode(v, sc), sc))


def run(cfg: dict, ds, gold, iters=None):
    enc = Encoder(LOG_N)
    rng = np.random.default_rng(7)
    X, y = ds.X, ds.y
    n = X.shape[0]
    Z = X * y[:, None]
    cols = Z.shape[1]
    rb = -(-n // M)
    pad = np.zeros((rb * M, G))
    pad[:n, :cols] = Z
    zb = pad.reshape(rb, M * G)
    if "z" in cfg:
        zb = np.stack([roundtrip(enc, zb[i], cfg["z"]) for i in range(rb)])
    if "znoise" in cfg:  # fixed encryption noise of every Z ciphertext (absolute, per slot)
        zb = zb + rng.normal(scale=cfg["znoise"], size=zb.shape)
    nb = -(-rb // R)
    rows_per = M * R
    bb = []
    for k in range(nb):
        Xk = X[k * rows_per:min((k + 1) * rows_per, n)]
        b = 1.0 / (1e-8 + np.abs(0.25 * (Xk.T @ Xk)).sum(axis=1))
        seg = np.zeros(G)
        seg[:cols] = b
        v = np.tile(seg, M)
        if "bbar" in cfg:
            v = roundtrip(enc, v, cfg["bbar"] + round(-math.log2(np.max(np.abs(v)))))
        if "bnoise" in cfg:  # fixed encryption noise relative to max |B̄| (encrypted at s_top / max|B̄|)
            v = v + rng.normal(scale=cfg["bnoise"] * np.max(np.abs(v)), size=S)
        bb.append(v)
    mask = np.zeros(S)
    mask[::G] = 1.0
    if "mask" in cfg:
        mask = roundtrip(enc, mask, cfg["mask"])
    q0, q1, q2, q3 = BASELINE_CUBIC.complement().padded(3)
    W = np.zeros(S)
    V = np.zeros(S)
    a0 = 0.01
    a1 = 0.5 * (1 + math.sqrt(1 + 4 * a0 * a0))
    its = [int(t) for t in gold["iterations"]]
    total = its[-1] if iters is None else iters
    worst = 0.0
    for t in range(total):
        b = t % nb
        blk = range(b * R, min((b + 1) * R, rb))
        rows = min(rows_per, n - b * rows_per)
        lr = 1.0 + 10.0 * math.exp(-t)
        eta = (1 - a0) / a1
        gamma = lr / rows
        T = np.zeros(S)
        for k in blk:
            P = zb[k] * W
            # left rotate-and-sum over g, row-start mask, right rotate-and-sum
            c = np.concatenate([P, P[:G]]).cumsum()
            A = c[G - 1:G - 1 + S] - np.concatenate([[0.0], c[:S - 1]])
            Mk = A * mask
            c2 = np.concatenate([Mk[S - G + 1:], Mk]).cumsum()
            U = c2[G - 1:] - np.concatenate([[0.0], c2[:S - 1]])
            if "unoise" in cfg:
                U = U + rng.normal(scale=cfg["unoise"], size=S)
            qu = q0 + q1 * U + q2 * U * U + q3 * U ** 3
            T += qu * zb[k]
        Gs = np.tile(T.reshape(M, G).sum(axis=0), M)
        D = Gs * bb[b]
        Vn = W + (1 + gamma) * D
        Wn = (1 - eta) * Vn + eta * V
        if "wnoise" in cfg:
            Wn = Wn * (1 + rng.normal(scale=cfg["wnoise"], size=S))
            Vn = Vn * (1 + rng.normal(scale=cfg["wnoise"], size=S))
        W, V = Wn, Vn
        a0, a1 = a1, 0.5 * (1 + math.sqrt(1 + 4 * a1 * a1))
        if t + 1 in its:
            k = its.index(t + 1)
            worst = max(worst, float(np.max(np.abs(W[:cols] - gold["weights"][k]))))
    return worst


def parse(spec: str) -> dict:
    cfg = {}
    for part in spec.split("+"):
        if part == "exact":
            continue
        k, v = part.split(":")
        cfg[k] = float(v)
    return cfg


def main():
    ds = paper_dataset()
    gold = np.load(ROOT / "tests" / "golden" / "paper_mini.npz")
    for spec in sys.argv[1:] or ["exact"]:
        print(spec, f"{run(parse(spec), ds, gold):.3e}", flush=True)


if __name__ == "__main__":
    main()
