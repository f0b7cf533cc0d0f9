#!/usr/bin/env python
"""Join ncu per-SASS-instruction counts with nvdisasm line info: where do the
executed instructions of a kernel come from (source file:line)?

    python tools/sass_lines.py <ncu-rep> <cubin> <mangled kernel name> [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def main():
    rep, cubin, fun = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    dis = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
    start = dis.find(f".text.{fun}:")
    end = dis.find("//--------------------- .text.", start + 1)
    dis = dis[start:end if end > 0 else len(dis)]
    line_of = {}
    cur = "?"
    for ln in dis.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            line_of[int(m.group(1), 16)] = cur
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head = rows[1]
    ia, iad, iss = head.index("Instructions Executed"), head.index("Address"), head.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) > ia and r[ia]]
    base = int(data[0][iad], 16)
    cnt, smp = collections.Counter(), collections.Counter()
    tot = tots = 0.0
    for r in data:
        off = int(r[iad], 16) - base
        n = float(r[ia])
        s = float(r[iss] or 0)
        key = line_of.get(off, "?")
        cnt[key] += n
        smp[key] += s
        tot += n
        tots += s
    print(f"total warp instructions {tot:.0f}, stall samples {tots:.0f}")
    for k, n in cnt.most_common(top):
        print(f"{100 * n / tot:5.1f}% inst  {100 * smp[k] / max(tots, 1):5.1f}% samples  {k}")


if __name__ == "__main__":
    main()
