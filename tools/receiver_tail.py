#!/usr/bin/env python
"""Tail of the batch-1 receiver latency: per-stage event times over many runs
(which stage the p99.9 outliers come from).

    python tools/receiver_tail.py [--M 16384 --N 32 --runs 2000]
"""
import argparse
import gc
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2604_02266_b200 as pkg  # noqa: E402
from paper_2604_02266_b200.synth import synthesize_packets  # noqa: E402
from paper_2604_02266_b200.zak import dzt_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=16384)
    ap.add_argument("--N", type=int, default=32)
    ap.add_argument("--runs", type=int, default=2000)
    args = ap.parse_args()
    M, N = args.M, args.N
    s = pkg.SsCgaSolver(M, N, 10, precision="fp32", modulation="qam16")
    pk = synthesize_packets(s, 1, snr_db=25.0, nu_max_hz=100.0, modulation="qam16", seed=3, cdtype=s.cdtype)
    for _ in range(10):
        s.receive(pk.pilot_rx, pk.data_rx, pk.lam, 0.08, tx_labels=pk.tx_labels, trace=False)
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()
    import time
    rows = []
    for _ in range(args.runs):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        h0 = time.perf_counter()
        ev[0].record()
        pending = []
        paths = s.detect(pk.pilot_rx, 0.08, _deferred=pending)
        ev[1].record()
        y = dzt_device(pk.data_rx, M, N, colmajor=True)
        ev[2].record()
        s.solve(y, paths, pk.lam, tx_labels=pk.tx_labels, trace=False)
        ev[3].record()
        pending[0][0].tolist()
        ev[4].record()
        ev[4].synchronize()
        h1 = time.perf_counter()
        rows.append([ev[i].elapsed_time(ev[i + 1]) for i in range(4)] + [ev[0].elapsed_time(ev[4]),
                                                                         (h1 - h0) * 1e3])
    gc.enable()
    names = ["detect", "data_dzt", "solve", "check", "total_dev", "total_host"]
    out = {}
    for j, nme in enumerate(names):
        v = sorted(r[j] for r in rows)
        out[nme] = {"p50": v[len(v) // 2], "p99": v[int(len(v) * 0.99)], "p999": v[int(len(v) * 0.999)],
                    "max": v[-1]}
    worst = sorted(rows, key=lambda r: -r[4])[:5]
    out["worst_rows"] = [[round(x, 3) for x in r] for r in worst]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
