#!/usr/bin/env python
"""Brief of an ncu --set full report: per launch the headline SOL, issue,
occupancy and pipe numbers, plus the top stall reasons.

    python tools/ncu_brief.py report.ncu-rep [kernel-regex]
"""
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for row in rows[2:]:
        d = dict(zip(h, row))
        name = d.get("Kernel Name", "")
        if pat and not pat.search(name):
            continue
        print(f"== {d.get('ID')} {name[:100]}")
        for k in KEYS:
            if k in d:
                print(f"   {k:70s} {d[k]}")
        stalls = []
        for k, v in d.items():
            m = re.match(r"smsp__average_warp_latency_issue_stalled_(\w+)\.ratio$", k) or \
                re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+)$", k)
            if m:
                try:
                    stalls.append((float(v), m.group(1)))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("   stalls:", ", ".join(f"{n}={v:g}" for v, n in stalls[:8]))


if __name__ == "__main__":
    main()
