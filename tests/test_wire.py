"""Wire formats (wire.py): the reference's packed-matrix
files (encoding.py:160-206) and the limb-major ciphertext / key store.
CPU-only: tensors on the host, no device calls."""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2406_13221_b200 import wire
from paper_2406_13221_b200.encoding import pack_matrix, plan_layout
from paper_2406_13221_b200.params import CkksParams, HeParams


def test_packed_roundtrip_matches_reference_layout(tmp_path):
    rng = np.random.default_rng(1)
    Z = rng.uniform(-1, 1, size=(300, 16))
    lay = plan_layout(300, 15, HeParams(log_n=11), 64)
    blocks = pack_matrix(Z, lay)
    wire.save_packed(tmp_path, blocks, lay)
    mf = json.loads((tmp_path / "manifest.json").read_text())
    assert set(mf) == {"n", "f", "m", "g", "row_blocks", "col_blocks", "blocks"}
    assert mf["blocks"][0] == {"row": 0, "col": 0, "key": "block_0_0"}
    back, lay2 = wire.load_packed(tmp_path)
    assert lay2 == lay
    for i in range(lay.row_blocks):
        for j in range(lay.col_blocks):
            np.testing.assert_array_equal(back[i][j], blocks[i][j])


def _ck():
    return CkksParams.generate(log_n=10, n_q=8, dnum=2)


def _random_cts(ck, count, rng):
    q = np.array(ck.q, dtype=np.uint64)
    a = rng.integers(0, q[None, None, :, None], size=(count, 2, ck.L, ck.n), dtype=np.uint64)
    return torch.from_numpy(a.view(np.int64))


def test_cipher_store_roundtrip_active_limbs(tmp_path):
    ck = _ck()
    rng = np.random.default_rng(2)
    cts = _random_cts(ck, 3, rng)
    with wire.CipherStore.create(tmp_path, ck) as st:
        st.put("a", cts, level=4, scale=2.0 ** 40)
        st.put("b", cts[:1], scale=2.0 ** 47)
    st = wire.CipherStore.open(tmp_path)
    st.check_ring(ck)
    a = st.get("a")
    assert st.info("a")["nbytes"] == 3 * 2 * 5 * ck.n * 8  # only limbs 0..4 are stored
    np.testing.assert_array_equal(a[:, :, :5].numpy(), cts[:, :, :5].numpy())
    assert not a[:, :, 5:].any()
    np.testing.assert_array_equal(st.get("b").numpy(), cts[:1].numpy())
    assert st.info("b")["scale"] == 2.0 ** 47 and st.info("b")["level"] == ck.L - 1
    st.close()


def test_cipher_store_rejects_bad_input(tmp_path):
    ck = _ck()
    rng = np.random.default_rng(3)
    cts = _random_cts(ck, 1, rng)
    with wire.CipherStore.create(tmp_path, ck) as st:
        st.put("x", cts, level=2)
        with pytest.raises(ValueError):
            st.put("x", cts)
        with pytest.raises(ValueError):
            st.put("y", cts, level=ck.L)
        with pytest.raises(ValueError):
            st.put("z", cts[0, 0])  # not (..., 2, L, N)
    st = wire.CipherStore.open(tmp_path)
    with pytest.raises(ValueError):
        st.check_ring(CkksParams.generate(log_n=10, n_q=7, dnum=2))
    with pytest.raises(ValueError):
        st.get("x", out=torch.empty((2, 2, ck.L, ck.n), dtype=torch.int64))
    st.close()
    with open(tmp_path / "data.bin", "r+b") as fh:  # truncate
        fh.truncate(100)
    with pytest.raises(ValueError):
        wire.CipherStore.open(tmp_path).get("x")
    (tmp_path / "manifest.json").write_text(json.dumps({"format": "other"}))
    with pytest.raises(ValueError):
        wire.CipherStore.open(tmp_path)


def test_key_groups_are_stored_whole(tmp_path):
    ck = _ck()
    rng = np.random.default_rng(4)
    beta = -(-ck.L // ck.alpha)
    key = torch.from_numpy(rng.integers(0, 1 << 40, size=(beta, 2, ck.L + ck.K, ck.n), dtype=np.int64))
    with wire.CipherStore.create(tmp_path, ck) as st:
        st.put("gk_5", key, kind="key", meta={"galois": 5})
    st = wire.CipherStore.open(tmp_path)
    np.testing.assert_array_equal(st.get("gk_5").numpy(), key.numpy())
    assert st.info("gk_5")["meta"] == {"galois": 5}
    st.close()
