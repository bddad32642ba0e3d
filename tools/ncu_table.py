#!/usr/bin/env python
"""Per-kernel table from an ncu --set full report of one training step:
launches, summed time, and time-weighted averages of the pipe / issue /
memory metrics that show what binds each kernel.

    python tools/ncu_table.py report.ncu-rep [--md out.md]
"""
import argparse
import csv
import io
import re
import subprocess
from collections import defaultdict

M = [("issue %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
     ("fma-heavy %", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
     ("fp64 %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
     ("alu %", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
     ("lsu wavefronts %", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
     ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
     ("DRAM GB/s", None)]


def short(name):
    m = re.match(r"(?:void )?([A-Za-z_0-9]+)(<[^(]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    agg = defaultdict(lambda: defaultdict(float))
    for row in rows[2:]:
        d = dict(zip(h, row))
        try:
            t = float(d["gpu__time_duration.sum"])  # ns or us, same unit for all rows
        except (KeyError, ValueError):
            continue
        k = agg[short(d["Kernel Name"])]
        k["n"] += 1
        k["t"] += t
        for lab, key in M:
            if key is None:
                try:
                    by = float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])
                    k[lab] += by * t  # weighted later
                except (KeyError, ValueError):
                    pass
                continue
            try:
                k[lab] += float(d[key]) * t
            except (KeyError, ValueError):
                pass
    unit = rows[1][h.index("gpu__time_duration.sum")]
    tot = sum(k["t"] for k in agg.values())
    lines = [f"time unit: {unit}; metrics are time-weighted averages over the launches", "",
             "| kernel | launches | time | share | " + " | ".join(l for l, _ in M[:-1]) + " |",
             "|---|---:|---:|---:|" + "---:|" * (len(M) - 1)]
    for name, k in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        vals = " | ".join(f"{k[l] / k['t']:.1f}" for l, _ in M[:-1])
        lines.append(f"| `{name}` | {int(k['n'])} | {k['t']:.1f} | {k['t'] / tot:.3f} | {vals} |")
    text = "\n".join(lines) + "\n"
    print(text)
    if a.md:
        open(a.md, "w").write(text)


if __name__ == "__main__":
    main()
