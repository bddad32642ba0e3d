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
