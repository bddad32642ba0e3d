"""N > 1 host logic on CPU (gloo, world_size 2).  The encrypted mini-batch
path does not shard: each rank
trains an independent replica, the job time is the max over ranks and the
job throughput is steps * world_size / that time; the reference arm runs on
rank 0 only and every other rank exits 0 without work."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, q):
    sys.path.insert(0, str(ROOT))
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        ms = [12.5, 17.25][rank]  # per-rank device times: rank 1 is the slow replica
        m = bench.max_over_ranks(ms, ws)
        q.put((rank, m, bench.job_throughput(10, ws, m)))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, m, thr in out:
        assert m == 17.25
        assert thr == pytest.approx(10 * 2 / 0.01725)


def test_single_rank_is_identity():
    sys.path.insert(0, str(ROOT))
    import bench
    assert bench.max_over_ranks(3.5, 1) == 3.5
    assert bench.job_throughput(4, 1, 2000.0) == 2.0


def test_reference_arm_under_torchrun_two_ranks():
    """`torchrun --nproc-per-node 2 bench.py --impl reference`: exactly one
    JSON line (rank 0), both ranks exit 0."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
           "--impl", "reference", "--workload", "toy", "--steps", "2", "--warmup", "1", "--gpus", "2"]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=str(ROOT), env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] in ("port", "reference")


# ---- sharded full-batch gradient: host logic over gloo -------------------
def test_partition_covers_every_batch_once():
    sys.path.insert(0, str(ROOT))
    from paper_2406_13221_b200.shard import partition
    for nb in (0, 1, 5, 413):
        for ws in (1, 2, 3, 8):
            parts = [partition(nb, r, ws) for r in range(ws)]
            flat = sorted(b for p in parts for b in p)
            assert flat == list(range(nb))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        partition(4, 2, 2)


def test_max_world_bound():
    sys.path.insert(0, str(ROOT))
    from paper_2406_13221_b200.params import CkksParams
    from paper_2406_13221_b200.shard import max_world
    ck = CkksParams.generate(log_n=13, n_q=8, dnum=2)
    assert max_world(ck.q + ck.p) >= 8  # q_0 < 2^60: eight 60-bit residues fit in 63 bits
    assert max_world([(1 << 62) - 57]) == 2 and max_world([(1 << 62) + 135]) == 1


def _residue_worker(rank, ws, port, q, out):
    sys.path.insert(0, str(ROOT))
    import numpy as np
    from paper_2406_13221_b200.shard import ResidueAllReduce
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        rng = np.random.default_rng(100 + rank)
        mine = rng.integers(0, np.array(q, dtype=np.uint64)[:, None], size=(len(q), 64), dtype=np.uint64)
        t = torch.from_numpy(mine.view(np.int64).copy())
        ResidueAllReduce(q)(t)
        out.put((rank, mine, t.numpy().view(np.uint64).copy()))
    finally:
        dist.destroy_process_group()


def test_residue_allreduce_gloo_is_exact():
    """Two ranks' residue words summed by the all-reduce reduce mod q to the
    sum of the residues mod q (what helr_reduce then computes on the GPU)."""
    import numpy as np
    qs = [(1 << 60) - 93, (1 << 40) + 1281, (1 << 40) - 87]
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_residue_worker, args=(r, 2, port, qs, out)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((out.get(timeout=120) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    qv = np.array(qs, dtype=np.uint64)[:, None]
    want = (res[0][1] % qv + res[1][1] % qv) % qv
    for _, _, summed in res:
        assert np.all(summed < (1 << 63))
        np.testing.assert_array_equal(summed % qv, want)
