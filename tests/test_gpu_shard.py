"""Sharded full-batch gradient (shard.py) on one GPU: two
ranks' trainers (shard 0/2 and 1/2) each sum the gradients of their own
batches; the partial sums are added as raw residue words (what the NCCL
all-reduce computes), folded by helr_reduce, and the update that follows must
leave W, V residue-for-residue equal to the unsharded full-batch trainer."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2406_13221_b200 import data
from paper_2406_13221_b200.ckks import GpuContext
from paper_2406_13221_b200.driver import FusedTrainer
from paper_2406_13221_b200.params import CkksParams

pytestmark = pytest.mark.gpu


def _trainer(ck, ds, shard=(0, 1), reducer=None):
    ctx = GpuContext(ck, seed=2, max_batch=8)
    return FusedTrainer(ctx, ds, rows_per_block=16, blocks_per_batch=2, mode="full_batch", use_graph=True,
                        shard=shard, reducer=reducer)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_full_batch_equals_single_rank(world):
    ds = data.toy_dataset()
    ck = CkksParams.generate(log_n=13, n_q=8, dnum=3)
    ref = _trainer(ck, ds)
    assert ref.n_batches >= world
    mailbox = []
    # ranks 1..world-1 only post their partial gradients; rank 0 adds them
    # (raw int64 words, the all-reduce SUM) before helr_reduce
    posts = [(lambda g: mailbox.append(g.clone())) for _ in range(world - 1)]
    others = [_trainer(ck, ds, (r, world), posts[r - 1]) for r in range(1, world)]

    def gather(g):
        for m in mailbox:
            g.add_(m)
        mailbox.clear()

    r0 = _trainer(ck, ds, (0, world), gather)
    for it in range(3):
        for tr in others:  # same W, V and schedule state as rank 0
            tr.wv.copy_(r0.wv)
            tr.iterate()
        torch.cuda.synchronize()  # the mailbox clones live on the other trainers' streams
        r0.iterate()
        ref.iterate()
        torch.cuda.synchronize()  # trainers run on their own streams
        lv = ref.level + 1
        a, b = ref.wv[:, :, :lv].cpu().numpy(), r0.wv[:, :, :lv].cpu().numpy()
        np.testing.assert_array_equal(a, b, err_msg=f"iteration {it + 1}")
        assert ref.level == r0.level
    # every residue word of the combined gradient is canonical
    q = np.array(ck.q, dtype=np.uint64)
    g = r0.grad.cpu().numpy().view(np.uint64)
    glv = r0.level + 7 - 5
    assert np.all(g[:, :, :glv + 1] < q[None, None, :glv + 1, None])
    for tr in [ref, r0] + others:
        tr.close()


def test_reduce_folds_sums_of_eight():
    ck = CkksParams.generate(log_n=13, n_q=8, dnum=3)
    ctx = GpuContext(ck, seed=2, max_batch=2)
    rng = np.random.default_rng(5)
    L, n = ck.L, ck.n
    q = np.array(ck.q, dtype=np.uint64)
    parts = [rng.integers(0, q[None, None, :, None], size=(2, 2, L, n), dtype=np.uint64) for _ in range(8)]
    tot = np.zeros_like(parts[0])
    for p in parts:
        tot += p  # < 8 q < 2^63: no wrap
    dev = torch.from_numpy(tot.view(np.int64)).cuda()
    out = torch.empty_like(dev)
    ctx._call("helr_reduce", dev.data_ptr(), out.data_ptr(), 2, L - 1, torch.cuda.current_stream().cuda_stream)
    got = out.cpu().numpy().view(np.uint64)
    want = tot % q[None, None, :, None]
    np.testing.assert_array_equal(got, want)


def test_concurrent_trainers_do_not_share_scratch():
    """Two trainers (own contexts, own streams) iterating back to back without
    a host synchronisation in between stay bit-identical: the fused driver's
    workspace belongs to the context, not the process."""
    ds = data.toy_dataset()
    ck = CkksParams.generate(log_n=13, n_q=8, dnum=3)
    a, b = _trainer(ck, ds), _trainer(ck, ds)
    for _ in range(3):
        a.iterate()
        b.iterate()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(a.wv.cpu().numpy(), b.wv.cpu().numpy())
    a.close()
    b.close()
