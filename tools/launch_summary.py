#!/usr/bin/env python
"""Per-kernel summary of an ncu --metrics gpu__time_duration.sum launch list (CSV).

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/rX_launches.txt
"""
import csv
import sys
from collections import defaultdict


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        d[r[ki][:90]].append(float(r[vi].replace(",", "")))
    print(f"{'launches':>8} {'avg_ns':>12} {'total_ns':>12}  kernel")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):>8} {sum(v) / len(v):>12.0f} {sum(v):>12.0f}  {k}")


if __name__ == "__main__":
    main()
