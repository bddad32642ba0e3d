"""CPU-side checks: the C-ABI library loads and exports every symbol that
include/helr_ckks.h declares (no compute calls without a GPU), the product
refuses to run without CUDA, and host-side parameter/encoding logic."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2406_13221_b200 import _lib
from paper_2406_13221_b200.encoder import Encoder
from paper_2406_13221_b200.params import CkksParams, HeParams, ciphertext_size_mb

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "helr_ckks.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(helr_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    names = declared_symbols()
    assert len(names) >= 25
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_covers_header():
    names = set(declared_symbols())
    bound = set(_lib.SIGNATURES)
    extra = {"helr_nag_graph_capture", "helr_nag_graph_update", "helr_nag_graph_launch", "helr_nag_graph_destroy", "helr_prof_enable",
             "helr_prof_collect", "helr_launch_count"}
    assert names - bound <= extra


def test_version_call_is_safe_without_gpu():
    assert _lib.load().helr_version() >= 100


def test_no_cpu_fallback():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2406_13221_b200.ckks import GpuContext
    with pytest.raises(_lib.NativeLibraryError):
        GpuContext(CkksParams.generate(log_n=5, n_q=3, dnum=1))


def test_heparams_surface():
    p = HeParams(log_n=16)
    assert p.slots == 32768
    assert ciphertext_size_mb(HeParams(log_n=16, log_q=275)) == pytest.approx(4.5056)
    with pytest.raises(ValueError, match="exceed"):
        HeParams(log_q=20, log_delta=30)
    with pytest.raises(ValueError, match="noise_sigma"):
        HeParams(noise_sigma=-1.0)


def test_ckks_params_views():
    ck = CkksParams.generate(log_n=16, n_q=8, dnum=3)
    # 40-bit special primes: alpha + 1 of them cover the q_0 digit (2^140) with margin
    assert (ck.L, ck.K, ck.alpha) == (8, 4, 3)
    assert all(p < 2 ** 41 for p in ck.p) and np.prod([float(p) for p in ck.p]) > 2.0 ** 159
    ck61 = CkksParams.generate(log_n=16, n_q=8, dnum=3, p_bits=61)
    assert (ck61.K, ck61.alpha) == (3, 3) and all(p < 2 ** 61 for p in ck61.p)
    assert CkksParams.generate(log_n=16, n_q=8, dnum=2).K == 5
    hp = ck.he_params()
    assert hp.log_q == 40 * 8 and hp.log_delta == 40 == hp.log_delta_c
    assert ck.level_bits(ck.top_level) == hp.log_q
    assert abs(np.log2(ck.q[0]) - 60) < 0.01 and all(abs(np.log2(q) - 40) < 0.01 for q in ck.q[1:])
    assert all(abs(np.log2(s) - 40) < 0.01 for s in ck.level_scales)


@pytest.mark.parametrize("log_n", [3, 6, 13])
def test_encoder_roundtrip(log_n, rng):
    enc = Encoder(log_n)
    z = rng.normal(size=enc.slots) + 1j * rng.normal(size=enc.slots)
    c = enc.encode(z, 2.0 ** 40)
    assert c.dtype == np.int64
    assert np.abs(enc.decode(c, 2.0 ** 40) - z).max() < 1e-9
    with pytest.raises(ValueError, match="slots"):
        enc.encode(np.ones(enc.slots + 1), 1.0)


def test_encoder_constant_is_constant_polynomial():
    enc = Encoder(8)
    c = enc.encode(np.full(enc.slots, 0.75), 2.0 ** 30)
    assert c[0] == round(0.75 * 2 ** 30) and np.all(np.abs(c[1:]) <= 1)


def test_rotsum_groups_host_rule_matches_library():
    """helr_rotsum_groups (csrc/nag.cu) and the driver's / oracle's grouping
    rule agree; it is a host-only entry point, callable without a GPU."""
    import ctypes
    from oracle import schedule as osched
    from paper_2406_13221_b200 import _lib
    from paper_2406_13221_b200.driver import rotsum_groups
    lib = _lib.load()
    bits = (ctypes.c_int * 64)()
    for total in range(0, 17):
        for mx in range(0, 9):
            ng = lib.helr_rotsum_groups(total, mx, bits)
            want = rotsum_groups(total, mx)
            assert list(bits[:ng]) == want == osched.rotsum_groups(total, mx)
            if want:
                assert sum(want) == total and max(want) <= mx
