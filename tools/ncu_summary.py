#!/usr/bin/env python
"""Summarise an ncu launch list (CSV from --csv --log-file, one row per
metric) by kernel category: launches, summed duration, share, and DRAM
bytes per launch when dram__bytes_{read,write}.sum were collected.

    python tools/ncu_summary.py gpurun_out/launches.csv \
        --md profiles/r01_launches.md --traffic profiles/ncu_traffic.json

The category map is the one the in-library profiler uses (csrc/prof.cuh),
so the shares here can be compared with bench.py's "kernels" block.
ncu serialises launches and runs them cold-cache: compare SHARES, not
absolute times.
"""

from __future__ import annotations

import argparse
import csv
import json
import re
from collections import defaultdict

CATS = ["ntt", "modup", "ks_inner", "moddown", "tensor", "rescale", "elementwise", "other"]
RULES = [
    (r"ntt_pass", "ntt"),
    (r"k_modup", "modup"),
    (r"k_ks_inner", "ks_inner"),
    (r"k_moddown|k_mdr_", "moddown"),
    (r"k_tensor", "tensor"),
    (r"k_rescale", "rescale"),
    (r"k_elementwise|k_lincomb|k_plain_fill", "elementwise"),
]


def category(name: str) -> str:
    for pat, cat in RULES:
        if re.search(pat, name):
            return cat
    return "other"


def short(name: str) -> str:
    m = re.match(r"(?:void )?([A-Za-z_0-9]+)(<[^(]*>)?", name)
    if not m:
        return name[:60]
    return (m.group(1) + (m.group(2) or ""))[:90]


def load(path):
    launches = defaultdict(dict)
    with open(path, newline="") as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for row in csv.DictReader(lines):
        lid = int(row["ID"])
        d = launches[lid]
        d["name"] = row["Kernel Name"]
        d["grid"] = row.get("Grid Size", "")
        d["block"] = row.get("Block Size", "")
        try:
            v = float(row["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        unit = row.get("Metric Unit", "")
        key = row["Metric Name"]
        if key == "gpu__time_duration.sum":
            v = v / 1e3 if unit == "ns" else (v if unit == "us" else v * 1e3 if unit == "ms" else v)
            key = "us"
        elif key.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
            v = v * scale.get(unit, 1)
        d[key] = v
    return [launches[k] for k in sorted(launches)]


def summarise(launches):
    cats = {c: dict(launches=0, us=0.0, dram=0.0, has_dram=False) for c in CATS}
    kern = defaultdict(lambda: dict(launches=0, us=0.0, dram=0.0))
    for d in launches:
        c = category(d["name"])
        s = cats[c]
        s["launches"] += 1
        s["us"] += d.get("us", 0.0)
        if "dram__bytes_read.sum" in d:
            s["has_dram"] = True
            b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
            s["dram"] += b
            kern[short(d["name"])]["dram"] += b
        k = kern[short(d["name"])]
        k["launches"] += 1
        k["us"] += d.get("us", 0.0)
    return cats, kern


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--md", default=None)
    ap.add_argument("--traffic", default=None)
    ap.add_argument("--warm", default=None,
                    help="second launch list of the same step captured with --cache-control none (L2 kept warm)")
    ap.add_argument("--title", default="ncu launch list")
    a = ap.parse_args()
    launches = load(a.csv)
    cats, kern = summarise(launches)
    total = sum(s["us"] for s in cats.values()) or 1.0
    out = [f"# {a.title}", "", f"source: `{a.csv}`, {len(launches)} launches, "
           f"sum of serialised kernel time {total / 1e3:.3f} ms", "",
           "| category | launches | ms | share | DRAM MB / launch |", "|---|---:|---:|---:|---:|"]
    for c in CATS:
        s = cats[c]
        if not s["launches"]:
            continue
        per = f"{s['dram'] / s['launches'] / 1e6:.2f}" if s["has_dram"] else "-"
        out.append(f"| {c} | {s['launches']} | {s['us'] / 1e3:.3f} | {s['us'] / total:.3f} | {per} |")
    out += ["", "| kernel | launches | ms | share | DRAM MB / launch |", "|---|---:|---:|---:|---:|"]
    for name, k in sorted(kern.items(), key=lambda kv: -kv[1]["us"]):
        per = f"{k['dram'] / k['launches'] / 1e6:.2f}" if k["dram"] else "-"
        out.append(f"| `{name}` | {k['launches']} | {k['us'] / 1e3:.3f} | {k['us'] / total:.3f} | {per} |")
    text = "\n".join(out) + "\n"
    print(text)
    if a.md:
        with open(a.md, "w") as fh:
            fh.write(text)
    if a.traffic:
        per_kernel = {c: s["dram"] / s["launches"] for c, s in cats.items() if s["launches"] and s["has_dram"]}
        # an NTT "launch" in the library's byte model (ProfScope in ntt_launch)
        # is one whole transform: two ntt_pass kernels (N >= 2^12) or one
        # ntt_cluster kernel, so DRAM bytes are summed over both passes
        n_pass = sum(1 for d in launches if "ntt_pass" in d["name"])
        n_cl = sum(1 for d in launches if "ntt_cluster" in d["name"])
        per_launch = dict(per_kernel)
        if cats["ntt"]["has_dram"] and (n_pass or n_cl):
            per_launch["ntt"] = cats["ntt"]["dram"] / (n_pass / 2.0 + n_cl)
        warm = None
        if a.warm:
            wl = load(a.warm)
            wc, _ = summarise(wl)
            warm = {c: s["dram"] / s["launches"] for c, s in wc.items() if s["launches"] and s["has_dram"]}
            wp = sum(1 for d in wl if "ntt_pass" in d["name"])
            wcl = sum(1 for d in wl if "ntt_cluster" in d["name"])
            if wc["ntt"]["has_dram"] and (wp or wcl):
                warm["ntt"] = wc["ntt"]["dram"] / (wp / 2.0 + wcl)
        tr = {"per_launch": per_launch, "per_launch_warm": warm, "per_kernel_launch": per_kernel,
              "ntt_transforms": n_pass / 2.0 + n_cl, "_source": a.csv,
              "_unit": "DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum, ncu serialised, cold cache); "
                       "per_launch: per library launch (NTT: per two-pass transform), per_kernel_launch: per CUDA kernel; "
                       "per_launch_warm: the same from a capture with --cache-control none (L2 not flushed between "
                       "kernels, as in the real step)"}
        with open(a.traffic, "w") as fh:
            json.dump(tr, fh, indent=1)


if __name__ == "__main__":
    main()
