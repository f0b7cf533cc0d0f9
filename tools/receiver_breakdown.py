#!/usr/bin/env python
"""Stage times of a batch-1 SsCgaSolver.receive (device events around each stage).

    python tools/receiver_breakdown.py [--M 16384 --N 32]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2604_02266_b200 as pkg  # noqa: E402
from paper_2604_02266_b200 import _native as nat  # noqa: E402
from paper_2604_02266_b200.synth import synthesize_packets  # noqa: E402
from paper_2604_02266_b200.zak import dzt_device  # noqa: E402


def timed(fn, reps=50):
    out = None
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2], out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=16384)
    ap.add_argument("--N", type=int, default=32)
    ap.add_argument("--batch", type=int, default=1)
    args = ap.parse_args()
    M, N, B = args.M, args.N, args.batch
    s = pkg.SsCgaSolver(M, N, 10, precision="fp32", modulation="qam16")
    pk = synthesize_packets(s, B, snr_db=25.0, nu_max_hz=100.0, modulation="qam16", seed=3, cdtype=s.cdtype)
    MN = M * N
    amp = float(MN ** 0.5)
    res = {}
    res["pilot_dzt_ms"], heff = timed(lambda: dzt_device(pk.pilot_rx, M, N, colmajor=False, pilot_amplitude=amp,
                                                         fp64=True))
    cnt = torch.empty(B, dtype=torch.int32, device="cuda")
    kk = torch.empty(B, 64, dtype=torch.int32, device="cuda")
    ll = torch.empty_like(kk)
    gg = torch.empty(B, 64, dtype=torch.complex128, device="cuda")
    lib = nat.load()
    import ctypes as C
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    res["detect_kernel_ms"], _ = timed(lambda: lib.ddb_detect_paths(B, M, N, p(heff), 0.08, 64, p(cnt), p(kk), p(ll),
                                                                     p(gg), st))
    res["detect_total_ms"], paths = timed(lambda: s.detect(pk.pilot_rx, 0.08))
    res["data_dzt_ms"], y = timed(lambda: dzt_device(pk.data_rx, M, N, colmajor=True))
    out = s.alloc(B, trace=False, bit_errors=True)
    res["solve_ms"], _ = timed(lambda: s.solve(y, paths, pk.lam, tx_labels=pk.tx_labels, out=out, trace=False))
    res["receive_ms"], _ = timed(lambda: s.receive(pk.pilot_rx, pk.data_rx, pk.lam, 0.08, tx_labels=pk.tx_labels,
                                                   trace=False))
    res["taps"] = int(cnt[0].item())
    res["plan"] = s.plan()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
