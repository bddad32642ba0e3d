#!/usr/bin/env python
"""Per-opcode executed-instruction and stall-sample totals from an
`ncu --page source --csv --print-source sass` export (optionally .gz).

    python tools/ncu_src_ops.py file.csv[.gz] [top]
"""
import csv
import gzip
import io
import sys
from collections import Counter


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    raw = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    rows = [r for r in csv.reader(raw)]
    hdr = next(r for r in rows if r and r[0] == "Address")
    data = [r for r in rows if r and r[0].startswith("0x")]
    iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    st, ex = Counter(), Counter()
    for r in data:
        t = r[1].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        op = op.split(".")[0]
        st[op] += int(r[iS] or 0)
        ex[op] += int(r[iE] or 0)
    ts, te = sum(st.values()), sum(ex.values())
    print(f"{rows[0][1][:100]}\n  samples {ts}  warp-instructions {te}")
    for op, v in ex.most_common(top):
        print(f"  {op:10s} exec {v:9d} ({100 * v / te:5.1f}%)  stall {100 * st[op] / max(ts, 1):5.1f}%")


if __name__ == "__main__":
    main()
