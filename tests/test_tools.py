"""Host-side measurement plumbing: the ncu launch-list summary that feeds
bench.py's roofline.traffic (an NTT "launch" is one two-pass transform) and
bench.py's reader of it.  CPU only."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

HEADER = '"ID","Process ID","Process Name","Host Name","Kernel Name","Context","Stream","Block Size","Grid Size","Device","CC","Section Name","Metric Name","Metric Unit","Metric Value"'


def _rows(lid, name, us, rd_mb, wr_mb):
    base = f'"{lid}","1","python","box","{name}","1","7","(256, 1, 1)","(16, 1, 1)","0","10.0","Command line profiler metrics"'
    return [f'{base},"dram__bytes_read.sum","Mbyte","{rd_mb}"', f'{base},"dram__bytes_write.sum","Mbyte","{wr_mb}"',
            f'{base},"gpu__time_duration.sum","us","{us}"']


def _csv(path, scale):
    lines = ["==PROF== noise line", HEADER]
    k = 0
    for _ in range(3):  # three transforms = six ntt_pass kernels
        for _ in range(2):
            lines += _rows(k, "void ntt_pass<8, 4, 16, 1, 0, 8, LdBuf, StBuf>(T1)", 30.0, 20.0 * scale, 5.0 * scale)
            k += 1
    lines += _rows(k, "void k_modup<4>(ModUpArgs, Tables)", 40.0, 60.0 * scale, 40.0 * scale)
    path.write_text("\n".join(lines) + "\n")


def test_ncu_summary_counts_transforms(tmp_path):
    cold, warm, out = tmp_path / "cold.csv", tmp_path / "warm.csv", tmp_path / "traffic.json"
    _csv(cold, 1.0)
    _csv(warm, 0.5)
    subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(cold), "--traffic", str(out), "--warm",
                    str(warm)], check=True, capture_output=True)
    d = json.loads(out.read_text())
    assert d["ntt_transforms"] == 3.0
    assert d["per_kernel_launch"]["ntt"] == 25e6           # per CUDA kernel
    assert d["per_launch"]["ntt"] == 50e6                  # per two-pass transform
    assert d["per_launch"]["modup"] == 100e6
    assert d["per_launch_warm"]["ntt"] == 25e6
    assert d["per_launch_warm"]["modup"] == 50e6


def test_bench_reads_traffic_file():
    sys.path.insert(0, str(ROOT))
    import bench

    cold, warm = bench.ncu_traffic()
    assert isinstance(cold, dict) and isinstance(warm, dict)
    if cold:  # the committed profile: NTT traffic is per transform, i.e. above one pass's ~40 MB
        assert cold["ntt"] > 5e7
