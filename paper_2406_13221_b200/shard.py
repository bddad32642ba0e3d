"""Sharding of the full-batch gradient across ranks.

The reference's full-batch iteration sums every block's gradient with
``SimContext.add`` before one quadratic-gradient / NAG update
(enctrain.py:356-359, 374-381).  The block gradients are independent, so with
one process per GPU each rank computes the sum over its own batches and the
partial sums are combined once per iteration:

* ``partition`` deals batches to ranks round-robin (rank r takes r, r + W, ...);
* the combine is an all-reduce SUM of the raw RNS residue words (int64) over
  NCCL, then ``helr_reduce`` folds each word back to [0, q_i).  Residues are
  < q_i < 2^61, so the sum of W partial gradients is exact in 63 bits while
  W * max(q) < 2^63 (``max_world``: 8 ranks for the 60-bit q_0).

Addition mod q is associative and commutative, so the combined gradient is
residue-for-residue the single-GPU accumulation and every rank then applies
the identical update (replicated W, V; no broadcast needed).
"""

from __future__ import annotations

from typing import Callable, List, Optional

import torch

__all__ = ["partition", "max_world", "ResidueAllReduce"]


def partition(n_batches: int, rank: int, world: int) -> List[int]:
    """Batches of ``rank`` out of ``world``: r, r + world, r + 2 world, ..."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad shard (rank {rank}, world {world})")
    if n_batches < 0:
        raise ValueError("n_batches must be >= 0")
    return list(range(rank, n_batches, world))


def max_world(primes) -> int:
    """Largest world size whose residue sum cannot overflow a signed 64-bit word."""
    return ((1 << 63) - 1) // max(int(q) for q in primes)


class ResidueAllReduce:
    """In-place all-reduce SUM of an int64 residue tensor over a process group
    (NCCL for CUDA tensors), issued on the current stream."""

    def __init__(self, primes, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        if self.world > max_world(primes):
            raise ValueError(f"{self.world} ranks overflow the 63-bit residue sum (max {max_world(primes)})")

    def __call__(self, t: torch.Tensor) -> None:
        if not t.is_contiguous():
            raise ValueError("residue all-reduce needs a contiguous tensor")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)


Reducer = Optional[Callable[[torch.Tensor], None]]
