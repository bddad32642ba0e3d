#!/usr/bin/env python
"""bench.py — encrypted enhanced-NAG logistic-regression training on B200.

Metric (BASELINE.json): encrypted NAG iterations/s at the paper shape
(422,108 x 200 padded to 256, N = 2^16, 1,024-row mini-batches packed as 8
ciphertexts of 128 x 256), plus epoch time and HBM GB/s.  One "step" is one
full NAG iteration over one batch: Z.W products, sum_col_vec, degree-3
sigmoid complement, gradient, sum_rows, quadratic-gradient product, NAG
update, and the refresh stand-in of W/V (every iteration at L = 8 primes).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload paper_mini]
    python bench.py --impl reference ...   # the reference algorithm on host cores

Timing: CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks; every step reads a different batch (64 MiB of
ciphertexts) and streams ~80 Galois keys (~2 GB), far beyond the 126 MB L2,
so no flush is needed between steps.  Multi-GPU: independent replicas
(the mini-batch path does not shard), scaling "weak".
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "encrypted NAG iterations/sec and epoch time at 422,108x200, N=2^16; HBM GB/s"
UNIT = "iterations/s"
CATS = ["ntt", "modup", "ks_inner", "moddown", "tensor", "rescale", "elementwise", "other"]

WORKLOADS = {
    # name: (dataset factory kwargs, log_n, L primes, dnum, rows per block, blocks per batch, mode)
    "paper_mini": dict(data="paper", log_n=16, L=8, dnum=2, rows=128, blocks=8, mode="mini_batch"),
    "paper_full": dict(data="paper", log_n=16, L=8, dnum=2, rows=128, blocks=8, mode="full_batch"),
    "medium": dict(data="medium", log_n=15, L=8, dnum=2, rows=1024, blocks=1, mode="mini_batch"),
    "toy": dict(data="toy", log_n=13, L=8, dnum=2, rows=128, blocks=1, mode="mini_batch"),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None, help="timed iterations (default: one epoch)")
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=list(WORKLOADS), default="paper_mini")
    p.add_argument("--no-graph", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-iters", type=int, default=1000, help="bounded CPU-baseline sample (iterations)")
    p.add_argument("--cpu-rns-iters", type=int, default=1,
                   help="C3 baseline: iterations of the CPU RNS-CKKS oracle on all host cores (0 = skip)")
    p.add_argument("--profile-steps", type=int, default=4)
    p.add_argument("--dnum", type=int, default=None, help="override the key-switching digit count")
    p.add_argument("--bsgs-bits", type=int, default=None, help="max bits per hoisted group (sum_col_vec)")
    p.add_argument("--rows-bits", type=int, default=None, help="max bits per hoisted group (sum_rows)")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_dataset(name):
    from paper_2406_13221_b200 import data
    return {"paper": data.paper_dataset, "medium": data.medium_dataset, "toy": data.toy_dataset}[name]()


def lr_fn(t):
    return 1.0 + 10.0 * math.exp(-t)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)), "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    path = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(path.read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """DRAM bytes per launch of each category from the committed ncu launch
    list (tools/ncu_summary.py --traffic): an NTT "launch" is one whole
    transform (both passes), matching the algorithmic bytes per launch."""
    path = ROOT / "profiles" / "ncu_traffic.json"
    try:
        d = json.loads(path.read_text())
        return d.get("per_launch", d), (d.get("per_launch_warm") or {})
    except Exception:
        return {}, {}


def max_over_ranks(x: float, ws: int) -> float:
    """Max of a per-rank device time over all ranks (the slowest replica sets
    the whole-job time).  Works on nccl (CUDA tensor) and gloo (CPU tensor)."""
    if ws <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(steps: int, ws: int, ms_max: float) -> float:
    """Whole-job iterations/s: every replica runs ``steps`` iterations."""
    return steps * ws / (ms_max / 1000.0)


# ----------------------------------------------------------------- reference arm
def cpu_reference_sample(wl, iters, warm=0):
    """The reference's own algorithm (slot-level simulator circuit, restated
    in oracle/slotsim.py) on host cores: ``warm`` untimed iterations, then
    ``iters`` timed ones (dataset encryption excluded).  Returns
    (iterations/s, timed seconds, timed iterations)."""
    from oracle import slotsim
    from paper_2406_13221_b200.optimizer import BASELINE_CUBIC
    ds = make_dataset(wl["data"])
    qpoly = BASELINE_CUBIC.complement().padded(3)
    mode = wl["mode"]
    if mode == "full_batch":
        iters, warm = max(1, min(iters, 2)), min(warm, 1)
    stamps = []
    slotsim.train(ds.X, ds.y, wl["log_n"], wl["rows"], wl["blocks"], qpoly, lr_fn, warm + iters, mode=mode,
                  trace=False, stamps=stamps)
    dt = stamps[-1] - stamps[warm]
    return iters / dt, dt, iters


def cpu_rns_sample(wl, iters, cores):
    """C3: the build's CPU RNS-CKKS oracle (oracle/, plain C +
    OpenMP on ``cores`` threads) running exactly the arithmetic of one fused
    iteration of this workload's ring and schedule (oracle/schedule.py) on
    uniformly random residues and keys (the cost does not depend on values).
    Returns (iterations/s, timed seconds)."""
    os.environ["OMP_NUM_THREADS"] = str(cores)
    from oracle import schedule as osched
    from oracle.oracle import Oracle
    from paper_2406_13221_b200.driver import grouped_steps
    from paper_2406_13221_b200.params import CkksParams
    ck = CkksParams.generate(log_n=wl["log_n"], n_q=wl["L"], dnum=wl["dnum"])
    orc = Oracle(ck, threads=cores)
    rng = np.random.default_rng(3)
    n, L, S = ck.n, ck.L, ck.slots
    R, C = wl["blocks"], 1
    log_g = int(math.log2(S // wl["rows"]))
    log_m = ck.log_n - 1 - log_g
    lb, lbr = (log_g + 1) // 2, (log_m + 1) // 2
    q = np.array(ck.q, dtype=np.uint64)[:, None]
    ct = lambda *lead: (rng.integers(0, 2 ** 62, size=lead + (2, L, n), dtype=np.uint64) % q)
    beta = -(-L // ck.alpha)
    pq = np.array(list(ck.q) + list(ck.p), dtype=np.uint64)[:, None]
    key = lambda: rng.integers(0, 2 ** 62, size=(beta, 2, L + ck.K, n), dtype=np.uint64) % pq
    steps = [k for grp in grouped_steps(log_g, lb) for k in grp]
    rsteps = [k for grp in grouped_steps(log_m, lbr, 1 << log_g) for k in grp]
    gals = set([pow(5, k, 2 * n) for k in steps] + [pow(5, S - k, 2 * n) for k in steps] +
               [pow(5, k % S, 2 * n) for k in rsteps])
    gk = {g: key() for g in gals}
    z, w, v, b = ct(R, C), ct(C), ct(C), ct(C)
    rlk, mask = key(), ct()[0, 0]
    consts = rng.integers(0, 2 ** 39, size=(10, L), dtype=np.uint64)
    t0 = time.perf_counter()
    for _ in range(iters):
        osched.nag_iteration(orc, z, w, v, b, L - 1, rlk, gk, mask, consts, log_g, log_m, log_baby=lb,
                             log_baby_rows=lbr)
    dt = time.perf_counter() - t0
    return iters / dt, dt


def reference_driver_sample(reps=3):
    """C2: the reference's own driver semantics end to end
    on Toy — the literal depth-9 ``train_encrypted`` loop (per-iteration
    decrypt + log-likelihood metrics included) over the reference slot
    simulator (oracle/slotsim.py behind the SimContext protocol).
    Returns (iterations/s, seconds, iterations)."""
    from oracle import slotsim
    from paper_2406_13221_b200 import enctrain as T
    from paper_2406_13221_b200.data import toy_dataset
    from paper_2406_13221_b200.errors import NeedsBootstrap
    from paper_2406_13221_b200.optimizer import BASELINE_CUBIC, ExpDecay, TrainConfig
    from paper_2406_13221_b200.params import HeParams

    class Ctx:
        COUNTER_KEYS = ("enc", "dec", "add", "cadd", "mul", "cmul", "imul", "rotate", "bootstrap")

        def __init__(self, params):
            self.params = params
            self._s = slotsim.SlotSim(params.log_n, params.log_q, params.log_delta, params.log_delta_c)

        counters = property(lambda self: self._s.counters, lambda self, v: setattr(self._s, "counters", v))

        def reset_counters(self):
            snap = dict(self._s.counters)
            self._s.counters = dict.fromkeys(self.COUNTER_KEYS, 0)
            return snap

        def __getattr__(self, name):
            f = getattr(self._s, name)

            def call(*a, **k):
                try:
                    return f(*a, **k)
                except slotsim.SlotNeedsBootstrap as e:
                    raise NeedsBootstrap(str(e)) from e
            return call

        def sum_col_vec(self, a, lay):
            return self.__getattr__("sum_col_vec")(a, lay.m, lay.g)

        def sum_rows(self, a, lay):
            return self.__getattr__("sum_rows")(a, lay.m, lay.g)

    ds = toy_dataset()
    params = HeParams(log_n=13, log_q=10 ** 6, log_delta=40, log_delta_c=40)
    cfg = TrainConfig(mode="mini_batch", batch_size=128, epochs=3, max_iterations=10 ** 6, schedule=ExpDecay(),
                      sigmoid="g8")
    t0 = time.perf_counter()
    iters = runs = 0
    while runs < reps or time.perf_counter() - t0 < 2.0:   # whole 24-iteration runs, >= 2 s of work
        res = T.train_encrypted(ds, cfg, params, ctx=Ctx(params), poly=BASELINE_CUBIC)
        iters += len(res.ledger)
        runs += 1
    dt = time.perf_counter() - t0
    return iters / dt, dt, iters


def run_reference(args, wl, ws, rank):
    if rank != 0:
        return
    steps = args.steps if args.steps is not None else 100
    warm = max(0, args.warmup)
    from oracle import slotsim  # noqa: F401
    cores = 1  # numpy slot arithmetic is single-threaded
    # warm-up + timed sample, each step one iteration of the reference circuit
    rate, dt, iters = cpu_reference_sample(wl, steps, warm)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": ws, "steps": steps,
        "warmup": warm, "ms_per_step": 1000.0 / rate, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "n": 422108 if "paper" in args.workload else None,
                   "batch_rows": wl["rows"] * wl["blocks"], "log_n": wl["log_n"], "parallelism": "replicas"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{iters} timed iterations (after {warm} warm-up) of the reference simulator circuit "
                                   f"(oracle/slotsim.py), {dt:.2f} s"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "epoch_s": 413.0 / rate if "paper" in args.workload else None,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm
def main():
    args = parse()
    ws, rank, local = dist_env()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl, ws, rank)
        return
    import torch
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2406_13221_b200 import _lib
    from paper_2406_13221_b200.ckks import GpuContext
    from paper_2406_13221_b200.driver import FusedTrainer
    from paper_2406_13221_b200.params import CkksParams

    lib = _lib.load()
    lib.helr_prof_collect.argtypes = [ctypes.POINTER(ctypes.c_double)] * 2 + [ctypes.POINTER(ctypes.c_int)]
    lib.helr_prof_enable.argtypes = [ctypes.c_int]
    lib.helr_launch_count.restype = ctypes.c_ulonglong

    t_setup = time.perf_counter()
    ck = CkksParams.generate(log_n=wl["log_n"], n_q=wl["L"], dnum=args.dnum or wl["dnum"])
    ctx = GpuContext(ck, seed=1, max_batch=max(8, wl["blocks"]))
    ds = make_dataset(wl["data"])
    # full batch on N > 1 GPUs: the ranks share each iteration's batches and
    # all-reduce the gradient residues (shard.py; strong scaling); the
    # mini-batch path does not shard, so N GPUs run N replicas (weak scaling)
    sharded = ws > 1 and wl["mode"] == "full_batch"
    shard_kw = {}
    if sharded:
        from paper_2406_13221_b200.shard import ResidueAllReduce
        shard_kw = dict(shard=(rank, ws), reducer=ResidueAllReduce(tuple(ck.q) + tuple(ck.p)))
    tr = FusedTrainer(ctx, ds, rows_per_block=wl["rows"], blocks_per_batch=wl["blocks"], mode=wl["mode"],
                      use_graph=not args.no_graph, bsgs_bits=args.bsgs_bits, rows_bits=args.rows_bits, **shard_kw)
    job = (lambda n, w, m: n / (m / 1000.0)) if sharded else job_throughput
    setup_s = time.perf_counter() - t_setup
    steps = args.steps if args.steps is not None else tr.n_batches
    warm = max(3, args.warmup)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    stream = tr.stream  # all trainer work (and these events) live on its stream
    for _ in range(warm):
        tr.iterate()
    barrier()

    # ---------------- timed region: device-resident dataset
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        tr.iterate()
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1), ws)
    value = job(steps, ws, ms)

    # ---------------- live per-kernel attribution: CUDA events recorded inside a
    # captured graph (no host launch gaps), one category pair per launch
    c0 = lib.helr_launch_count()
    msa = (ctypes.c_double * 8)()
    bya = (ctypes.c_double * 8)()
    cna = (ctypes.c_int * 8)()
    tot_ms, tot_by, tot_cn = [0.0] * 8, [0.0] * 8, [0] * 8
    prof_ms = 0.0
    for _ in range(args.profile_steps):
        pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pe0.record(stream)
        tr.profile_iteration()
        pe1.record(stream)
        lib.helr_prof_collect(msa, bya, cna)
        prof_ms += pe0.elapsed_time(pe1)
        for i in range(8):
            tot_ms[i] += msa[i]
            tot_by[i] += bya[i]
            tot_cn[i] += cna[i]
    launches_per_step = (lib.helr_launch_count() - c0) / args.profile_steps
    msa, bya, cna = tot_ms, tot_by, tot_cn
    cats = {CATS[i]: {"ms": msa[i] / args.profile_steps, "launches": cna[i] / args.profile_steps,
                      "gb": bya[i] / args.profile_steps / 1e9} for i in range(8)}
    dom = max(range(8), key=lambda i: msa[i])
    peak, peak_kind = peaks()
    achieved = (bya[dom] / cna[dom]) / ((msa[dom] / cna[dom]) / 1000.0) / 1e9
    traffic_cold, traffic_warm = ncu_traffic()
    traffic = traffic_cold.get(CATS[dom])
    # the event-bracketed replay serialises the graph (no programmatic
    # dependent-launch overlap), so per-category times add up to more than a
    # step: shares are reported against the attributed sum
    attributed = sum(msa) / args.profile_steps
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_unit": "DRAM bytes per launch (ncu, profiles/ncu_traffic.json)",
                "traffic_warm_l2": traffic_warm.get(CATS[dom]),
                "kernel": CATS[dom], "peak_kind": peak_kind,
                "share_of_step": (msa[dom] / args.profile_steps) / attributed,
                "attributed_ms_per_step": attributed,
                "algorithmic_bytes_per_launch": bya[dom] / cna[dom],
                "avg_launch_ms": msa[dom] / cna[dom]}
    step_gb = sum(bya) / args.profile_steps / 1e9

    # ---------------- e2e: host-resident encrypted dataset through the public API
    e2e = None
    if not args.no_e2e:
        tr.enable_host_stream()
        for _ in range(2):
            tr.iterate()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(steps):
            tr.iterate()
        tr.finish_host_stream()  # the last step's weight read-back is inside the timed region
        f1.record(stream)
        barrier()
        ems = max_over_ranks(f0.elapsed_time(f1), ws)
        h2d, d2h = tr.bytes_per_step()
        e2e = {"value": job(steps, ws, ems), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ems / steps}
        tr.disable_host_stream()

    # ---------------- CPU baselines (rank 0, N=1 only)
    cpu = None
    if rank == 0 and ws == 1 and args.cpu_iters > 0:
        nproc = os.cpu_count() or 1
        rate, dt, iters = cpu_reference_sample(wl, args.cpu_iters, warm=5)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"C1: {iters} iterations of the reference simulator circuit (oracle/slotsim.py, numpy "
                         f"elementwise: one core of {nproc}), {dt:.1f} s"}
        r2, dt2, it2 = reference_driver_sample()
        cpu["reference_driver"] = {"value": r2, "unit": UNIT, "cores": 1, "kind": "port", "workload": "toy",
                                   "sample": f"C2: {it2} iterations of the literal train_encrypted loop with its "
                                             f"per-iteration metrics over the reference simulator, Toy, {dt2:.1f} s"}
        if args.cpu_rns_iters > 0:
            r3, dt3 = cpu_rns_sample(wl, args.cpu_rns_iters, nproc)
            cpu["rns_oracle"] = {"value": r3, "unit": UNIT, "cores": nproc, "kind": "port",
                                 "sample": f"C3: {args.cpu_rns_iters} fused iteration(s) of the CPU RNS-CKKS oracle "
                                           f"(real HE, same ring and schedule as the GPU), {dt3:.1f} s on {nproc} "
                                           f"OpenMP threads", "gpu_speedup": value / r3}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": steps, "warmup": warm,
            "ms_per_step": ms / steps, "higher_is_better": True, "scaling": "strong" if sharded else "weak",
            "vs_baseline": None,
            "dtype": "u64", "data": "synthetic",
            "config": {"workload": args.workload, "n": ds.n_samples, "features": ds.n_features,
                       "padded_cols": tr.layout.col_blocks * tr.layout.g, "log_n": ck.log_n, "L": ck.L,
                       "K": ck.K, "dnum": ck.dnum, "batch_rows": tr.batch_rows, "cts_per_batch": tr.rows,
                       "batches": tr.n_batches, "mode": wl["mode"],
                       "parallelism": f"shard{ws}" if sharded else "replicas",
                       "cuda_graph": tr.use_graph, "rotsum_group_bits": tr.log_baby, "rows_group_bits": tr.log_baby_rows,
                       "l2": "no flush needed: each step streams a new 64 MiB batch and ~2 GB of keys"},
            "epoch_s": (1.0 / value) if wl["mode"] == "full_batch" else tr.n_batches / (value / ws),
            "hbm_gbs_step": step_gb / (ms / steps / 1000.0),
            "algorithmic_gb_per_step": step_gb,
            "roofline": roofline,
            "kernels": cats,
            "gpu_launches": int(round(launches_per_step * steps)),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "setup_s": setup_s,
            "prepare_s": tr.timings.get("prepare_s"),
        }
        print(json.dumps(line), flush=True)
    tr.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
