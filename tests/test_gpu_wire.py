"""Wire format on the device path: a trainer's encrypted dataset, W, V and
schedule state saved and loaded into another trainer resume training
residue-for-residue; evaluation keys load into a context with another seed."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2406_13221_b200 import data, wire
from paper_2406_13221_b200.ckks import GpuContext
from paper_2406_13221_b200.driver import FusedTrainer
from paper_2406_13221_b200.params import CkksParams

pytestmark = pytest.mark.gpu


def test_trainer_state_roundtrip(tmp_path):
    ds = data.toy_dataset()
    ck = CkksParams.generate(log_n=13, n_q=8, dnum=2)
    mk = lambda: FusedTrainer(GpuContext(ck, seed=2, max_batch=8), ds, rows_per_block=128, mode="mini_batch",
                              use_graph=True)
    a, b = mk(), mk()
    for _ in range(3):
        a.iterate()
    b.iterate()  # b diverges from a before the load
    torch.cuda.synchronize()
    wire.save_trainer_data(tmp_path, a)
    wire.load_trainer_data(tmp_path, b)
    torch.cuda.synchronize()
    assert (b.t, b.level, b.s_w) == (a.t, a.level, a.s_w)
    np.testing.assert_array_equal(b.z.cpu().numpy(), a.z.cpu().numpy())
    for _ in range(3):
        a.iterate()
        b.iterate()
    torch.cuda.synchronize()
    lv = a.level + 1
    np.testing.assert_array_equal(a.wv[:, :, :lv].cpu().numpy(), b.wv[:, :, :lv].cpu().numpy())
    assert np.max(np.abs(a.weights() - b.weights())) == 0.0
    a.close()
    b.close()


def test_keys_roundtrip(tmp_path):
    ck = CkksParams.generate(log_n=13, n_q=8, dnum=2)
    c1 = GpuContext(ck, seed=2, max_batch=2)
    g = c1.galois_for_rotation(3)
    c1.galois_key(g)
    wire.save_keys(tmp_path, c1)
    c2 = GpuContext(ck, seed=5, max_batch=2)
    assert not torch.equal(c2.rlk, c1.rlk)
    got = wire.load_keys(tmp_path, c2)
    assert set(got) == {g % (2 * ck.n)}
    assert torch.equal(c2.rlk, c1.rlk) and torch.equal(c2.galois_key(g), c1.galois_key(g))
