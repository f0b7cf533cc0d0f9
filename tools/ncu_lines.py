#!/usr/bin/env python
"""Per-source-line view of an ncu --set full capture (cuda,sass source page):
executed warp instructions, stall samples and the top stall reasons of every
CUDA source line of the profiled kernel, plus the SASS opcode mix.

    python tools/ncu_lines.py gpurun_out/x.ncu-rep [top] [--sass]
"""
import collections
import csv
import io
import re
import subprocess
import sys

STALLS = ("stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_drain", "stall_lg", "stall_long_sb",
          "stall_math", "stall_membar", "stall_mio", "stall_misc", "stall_no_inst", "stall_not_selected",
          "stall_selected", "stall_short_sb", "stall_sleep", "stall_tex", "stall_wait")


def f(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return 0.0


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    inst, samp = collections.Counter(), collections.Counter()
    reasons = collections.defaultdict(collections.Counter)
    ops = collections.Counter()
    opsamp = collections.Counter()
    fname, line = "?", "?"
    head = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            head = row
            continue
        if head is None or len(row) < len(head):
            continue
        if row[0]:
            line = row[0]
            continue
        d = dict(zip(head[4:], row[4:]))
        key = f"{fname}:{line}"
        n = f(d.get("Instructions Executed"))
        s = f(d.get("Warp Stall Sampling (All Samples)"))
        inst[key] += n
        samp[key] += s
        for r in STALLS:
            reasons[key][r] += f(d.get(r))
        op = row[3].strip().split()
        if op:
            o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
            o = re.sub(r"\..*", "", o)
            ops[o] += n
            opsamp[o] += s
    ti, ts = sum(inst.values()), sum(samp.values())
    print(f"total warp instructions {ti:.0f}, stall samples {ts:.0f}")
    print(f"{'inst%':>6} {'samp%':>6}  line  top stalls")
    for key, s in samp.most_common(top):
        rs = ", ".join(f"{r[6:]} {100 * v / max(s, 1):.0f}%" for r, v in reasons[key].most_common(3) if v)
        print(f"{100 * inst[key] / ti:6.1f} {100 * s / ts:6.1f}  {key}  {rs}")
    print("\nopcode mix (inst% / samp%):")
    for o, n in ops.most_common(25):
        print(f"  {o:12s} {100 * n / ti:6.1f} {100 * opsamp[o] / ts:6.1f}")


if __name__ == "__main__":
    main()
