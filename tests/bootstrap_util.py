"""Shared helpers for the bootstrapping tests: the CPU ring oracle wrapped in
the evaluator protocol ``bootstrap.Bootstrapper`` drives (test
infrastructure: the product's implementation of the protocol is
``bootstrap.GpuRing``)."""

from __future__ import annotations

import numpy as np

from oracle.oracle import Oracle


class OracleRing:
    def __init__(self, params, key_seed: int):
        self.params = params
        self.orc = Oracle(params)
        self.key_seed = key_seed
        self.sk = self.orc.keygen_secret(key_seed, params.hw)
        self.rlk = self.orc.keygen_switch(self.sk, 0, key_seed, 0)
        self._gk = {}

    def _res(self, value: int, level: int):
        return np.array([int(value) % q for q in self.params.q[: level + 1]], dtype=np.uint64)

    def galois_key(self, g: int):
        g = int(g) % (2 * self.params.n)
        if g not in self._gk:
            self._gk[g] = self.orc.keygen_switch(self.sk, g, self.key_seed, g)
        return self._gk[g]

    def add(self, a, b, level):
        return self.orc.add(np.ascontiguousarray(a), np.ascontiguousarray(b), level)

    def sub(self, a, b, level):
        return self.orc.add(np.ascontiguousarray(a), np.ascontiguousarray(b), level, sub=True)

    def add_const(self, a, value, level):
        return self.orc.add_const(np.ascontiguousarray(a), self._res(value, level), level)

    def mul_const(self, a, value, level):
        return self.orc.mul_const(np.ascontiguousarray(a), self._res(value, level), level)

    def mul_plain(self, a, pt, level):
        return self.orc.mul_plain(np.ascontiguousarray(a), pt, level)

    def encode_plain(self, coef, level):
        return self.orc.encode_plain(coef, level)[0]

    def rescale(self, a, level):
        return self.orc.rescale(np.ascontiguousarray(a), level)

    def mul(self, a, b, level):
        return self.orc.mul_relin_rescale(np.ascontiguousarray(a), np.ascontiguousarray(b), self.rlk, level)

    def rotate(self, a, galois, level):
        return self.orc.rotate(np.ascontiguousarray(a), int(galois), self.galois_key(galois), level)

    def imul(self, a, level):
        return self.orc.imul(np.ascontiguousarray(a), level)

    def mod_raise(self, a, level_out):
        return self.orc.mod_raise(np.ascontiguousarray(a), level_out)

    def cat(self, bufs):
        return np.ascontiguousarray(np.concatenate(list(bufs), axis=0))

    def split(self, buf, parts):
        return [np.ascontiguousarray(c) for c in np.split(buf, parts, axis=0)]


class LockstepRing:
    """Runs every primitive on the GPU evaluator and on the CPU oracle and
    compares all active residues, so a parity failure names the primitive
    (and the level) where the two first differ.  Buffers are (gpu, oracle)
    pairs."""

    def __init__(self, gpu_ring, oracle_ring):
        self.g, self.o = gpu_ring, oracle_ring
        self.params = gpu_ring.params
        self.ops = 0

    def _check(self, name, pair, level):
        g = pair[0].detach().cpu().numpy().view(np.uint64)
        o = pair[1]
        self.ops += 1
        if not np.array_equal(g[:, :, : level + 1], o[:, :, : level + 1]):
            bad = [(int(b), int(p), int(l)) for b, p, l in zip(*np.nonzero((g[:, :, : level + 1] != o[:, :, : level + 1]).any(axis=3)))]
            raise AssertionError(f"op #{self.ops} {name} at level {level}: residues differ in (item, poly, limb) {bad[:8]}")
        return pair

    def _both(self, name, out_level, *args_g, args_o=None):
        args_o = args_g if args_o is None else args_o
        return self._check(name, (getattr(self.g, name)(*args_g), getattr(self.o, name)(*args_o)), out_level)

    def _un(self, name, a, level, out_level=None, *extra):
        out = (getattr(self.g, name)(a[0], *extra, level), getattr(self.o, name)(a[1], *extra, level))
        return self._check(name, out, level if out_level is None else out_level)

    def add(self, a, b, level):
        return self._check("add", (self.g.add(a[0], b[0], level), self.o.add(a[1], b[1], level)), level)

    def sub(self, a, b, level):
        return self._check("sub", (self.g.sub(a[0], b[0], level), self.o.sub(a[1], b[1], level)), level)

    def add_const(self, a, value, level):
        return self._un("add_const", a, level, None, value)

    def mul_const(self, a, value, level):
        return self._un("mul_const", a, level, None, value)

    def mul_plain(self, a, pt, level):
        return self._check("mul_plain", (self.g.mul_plain(a[0], pt[0], level), self.o.mul_plain(a[1], pt[1], level)), level)

    def encode_plain(self, coef, level):
        g, o = self.g.encode_plain(coef, level), self.o.encode_plain(coef, level)
        gn = g.detach().cpu().numpy().view(np.uint64).reshape(-1, self.params.n)
        on = np.asarray(o).reshape(-1, self.params.n)
        if not np.array_equal(gn[: level + 1], on[: level + 1]):
            raise AssertionError(f"encode_plain at level {level}: plaintext residues differ")
        return (g, o)

    def rescale(self, a, level):
        return self._un("rescale", a, level, level - 1)

    def mul(self, a, b, level):
        return self._check("mul", (self.g.mul(a[0], b[0], level), self.o.mul(a[1], b[1], level)), level - 1)

    def rotate(self, a, galois, level):
        return self._check(f"rotate(g={galois})", (self.g.rotate(a[0], galois, level), self.o.rotate(a[1], galois, level)), level)

    def imul(self, a, level):
        return self._un("imul", a, level)

    def mod_raise(self, a, level_out):
        return self._check("mod_raise", (self.g.mod_raise(a[0], level_out), self.o.mod_raise(a[1], level_out)), level_out)

    def cat(self, bufs):
        bufs = list(bufs)
        return (self.g.cat([b[0] for b in bufs]), self.o.cat([b[1] for b in bufs]))

    def split(self, buf, parts):
        return list(zip(self.g.split(buf[0], parts), self.o.split(buf[1], parts)))
