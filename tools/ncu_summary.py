#!/usr/bin/env python
"""Summarise an ncu --set full capture of the fused kernel into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_cfg3.ncu-rep profiles/ncu_cfg3.json --frames 592

Extracts per-launch duration, DRAM bytes, pipe utilisation, shared-memory
wavefronts, issue/stall breakdown and registers, and the FP32 FLOP rate
implied by the algorithmic FLOP count when --frames/--flops
are given.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

KEEP = (
    "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__warps_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__cluster_dim_x",
    "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
)


SCALE = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep: str) -> list[dict]:
    """Rows of the raw page with values normalised to ns (times) and bytes."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k, u, v in zip(head, units, r):
            x = num(v)
            if isinstance(x, float) and u in SCALE:
                x *= SCALE[u]
            d[k] = x
        res.append(d)
    return res


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except (ValueError, AttributeError):
        return v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--frames", type=int, default=0)
    ap.add_argument("--flops-per-frame", type=float, default=0.0)
    args = ap.parse_args()
    launches = raw(args.rep)
    summary = []
    for r in launches:
        d = {"kernel": r.get("Kernel Name", "")}
        for k in KEEP:
            if k in r:
                d[k] = num(r[k])
        stalls = {k: num(v) for k, v in r.items()
                  if k.startswith("smsp__average_warp_latency_issue_stalled") or
                  (k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"))}
        top = sorted(((v, k) for k, v in stalls.items() if isinstance(v, float)), reverse=True)[:8]
        d["top_stalls"] = {k: v for v, k in top}
        summary.append(d)
    res = {"rep": Path(args.rep).name, "launches": summary}
    if summary:
        first = summary[0]
        t_ns = first.get("gpu__time_duration.sum")
        dram = (first.get("dram__bytes_read.sum") or 0) + (first.get("dram__bytes_write.sum") or 0)
        res["dram_bytes_per_launch"] = dram
        if args.frames and isinstance(t_ns, float):
            res["frames_per_launch"] = args.frames
            res["dram_bytes_per_frame"] = dram / args.frames
            res["duration_ns_per_frame"] = t_ns / args.frames
            if args.flops_per_frame:
                res["achieved_tflops_under_ncu"] = args.frames * args.flops_per_frame / (t_ns * 1e-9) / 1e12
            shared = first.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
            if isinstance(shared, float):
                res["smem_wavefronts_per_frame"] = shared / args.frames
            inst = first.get("smsp__inst_executed.sum")
            if isinstance(inst, float):
                res["warp_instructions_per_frame"] = inst / args.frames
    Path(args.out).write_text(json.dumps(res, indent=1))
    print(json.dumps(res, indent=1)[:4000])


if __name__ == "__main__":
    main()
