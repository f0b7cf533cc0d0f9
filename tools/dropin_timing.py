#!/usr/bin/env python
"""Per-call host time of the drop-ins on run_packet's pilot path at (32, 32)
(harness.py:153-168), sparse and dense branches: what criterion 10's
dense/sparse pilot-time ratio (tests/test_acceptance.py:301-332) measures
when the reference runs through the patcher."""

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2604_02266_b200 as pkg  # noqa: E402
from paper_2604_02266_b200 import dense, pilot, sparse, zak  # noqa: E402


def timed(fn, reps=200):
    for _ in range(10):
        fn()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    t.sort()
    return 1e6 * t[len(t) // 2]


def main():
    M, N = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (32, 32)))
    cfg = pkg.GridConfig(M, N)
    rng = np.random.default_rng(0)
    kern = zak.build_zak_kernel(N)
    twist = pilot.build_twist_kernel(cfg)
    y = rng.normal(size=M * N) + 1j * rng.normal(size=M * N)
    Y = zak.dzt_gemm(y, kern, cfg)
    h = pilot.estimate_heff(Y, twist, cfg)
    h = np.zeros_like(h)
    h[M // 2, N // 2] = 1.0
    h[M // 2 + 3, N // 2] = 0.3
    h[M // 2 + 7, N // 2 + 1] = 0.2
    taps = sparse.detect_paths(h, 0.08, cfg)
    res = {
        "dzt_gemm_us": timed(lambda: zak.dzt_gemm(y, kern, cfg)),
        "estimate_heff_us": timed(lambda: pilot.estimate_heff(Y, twist, cfg)),
        "detect_paths_us": timed(lambda: sparse.detect_paths(h, 0.08, cfg)),
        "build_ss_channel_us": timed(lambda: sparse.build_ss_channel(taps, cfg)),
        "threshold_frame_us": timed(lambda: dense.threshold_frame(h, 0.08, cfg), 50),
        "build_dense_hdd_us": timed(lambda: dense.build_dense_hdd(h, cfg), 50),
    }
    sp = res["dzt_gemm_us"] + res["estimate_heff_us"] + res["detect_paths_us"] + res["build_ss_channel_us"]
    dn = res["dzt_gemm_us"] + res["estimate_heff_us"] + res["detect_paths_us"] + res["threshold_frame_us"] + \
        res["build_dense_hdd_us"]
    res["sparse_pilot_us"], res["dense_pilot_us"], res["ratio"] = sp, dn, dn / sp
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
