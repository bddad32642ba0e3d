"""The TMA-fed persistent NTT passes (csrc/ntt_tma.cuh: cp.async.bulk.tensor
tile prefetch on mbarriers) are an opt-in alternative to the plain passes
(measured slower).  They share ntt_body's arithmetic, so every
N = 2^16 parity case must still equal the CPU ring oracle residue for residue
with the path forced on for every launch.  The knobs are read once per
process, hence the subprocess."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_parity_suite_with_tma_passes_forced_on():
    env = dict(os.environ, HELR_NTT_TMA="1", HELR_NTT_TMA_MIN_TILES="1")
    res = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-q", "-m", "gpu", "-k", "n2e16",
                          "-p", "no:cacheprovider"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    tail = res.stdout.strip().splitlines()[-1] if res.stdout.strip() else res.stderr[-400:]
    assert res.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail, tail
