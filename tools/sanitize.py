#!/usr/bin/env python
"""Small fused solves for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize.py --kernel tmem --grid cfg3 --batch 4

--kernel tmem | row | global (DDB_KERNEL, csrc/capi.cu) selects sscga_tm_kernel,
sscga_kernel or the workspace path (g_persist for batch <= 8, else the
multi-kernel sequence; --no-persist forces the latter).  Every solve is
checked against the numpy oracle, so a sanitizer run is also a parity run.
"""

from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

GRIDS = {"cfg1": (64, 16, 4), "cfg2": (256, 16, 4), "cfg3": (512, 32, 6), "cfg4": (1024, 64, 8),
         "paper128": (128, 32, 6), "odd": (48, 32, 5)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", choices=("tmem", "row", "global"), default="tmem")
    ap.add_argument("--grid", choices=sorted(GRIDS), default="cfg1")
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--precision", choices=("fp32", "fp64"), default="fp32")
    ap.add_argument("--doppler", action="store_true", help="taps with Doppler shifts (DSMEM route)")
    ap.add_argument("--no-persist", action="store_true")
    a = ap.parse_args()
    os.environ["DDB_KERNEL"] = {"tmem": "tmem", "row": "row", "global": "global"}[a.kernel]
    if a.no_persist:
        os.environ["DDB_NO_PERSIST"] = "1"
    import torch
    import ddlink_oracle as orc
    import paper_2604_02266_b200 as pkg

    M, N, P = GRIDS[a.grid]
    rng = np.random.default_rng(7)
    B = a.batch
    off = np.arange(B + 1, dtype=np.int32) * P
    k = (M // 2 + rng.integers(0, min(M // 2, 40), size=B * P)).astype(np.int32)
    l = np.full(B * P, N // 2, np.int32)
    if a.doppler:
        l += rng.integers(-1, 2, size=B * P).astype(np.int32)
    g = (rng.normal(size=B * P) + 1j * rng.normal(size=B * P)) * 0.3
    g[::P] = 1.0
    y = rng.normal(size=(B, M * N)) + 1j * rng.normal(size=(B, M * N))
    lam = np.full(B, 0.01)
    s = pkg.SsCgaSolver(M, N, 10, precision=a.precision, modulation="qam16")
    cd = np.complex64 if a.precision == "fp32" else np.complex128
    paths = pkg.PathBatch.from_arrays(off, k, l, g, cdtype=s.cdtype)
    res = s.solve(torch.as_tensor(y.astype(cd), device="cuda"), paths, lam, llr=True,
                  tx_labels=torch.zeros(B, M * N, dtype=torch.uint8, device="cuda"))
    torch.cuda.synchronize()
    x = res.x.cpu().numpy()
    worst = 0.0
    for f in range(B):
        taps = [orc.Tap(int(k[i]), int(l[i]), complex(g[i])) for i in range(off[f], off[f + 1])]
        xr, _ = orc.cga(orc.build_tables(taps, M, N), y[f].astype(cd).astype(np.complex128), 10, lam[f])
        worst = max(worst, float(np.linalg.norm(x[f] - xr) / np.linalg.norm(xr)))
    tol = 1e-4 if a.precision == "fp32" else 1e-10
    print(f"sanitize {a.kernel} {a.grid} B={B} {a.precision} doppler={a.doppler} plan={s.plan()['kernel']}: "
          f"worst rel L2 {worst:.2e} ({'ok' if worst < tol else 'FAIL'})")
    sys.exit(0 if worst < tol else 1)


if __name__ == "__main__":
    main()
