#!/usr/bin/env python
"""Per-phase cycle breakdown of the fused solve (clock64 on thread 0 per CTA).

    python tools/phase_profile.py [--M 512 --N 32 --batch 4096 --paths 6]
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
from paper_2604_02266_b200.synth import make_frames  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=512)
    ap.add_argument("--N", type=int, default=32)
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--paths", type=int, default=6)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--nu", type=float, default=100.0)
    args = ap.parse_args()
    s = pkg.SsCgaSolver(args.M, args.N, args.iters, precision="fp32", modulation="qam16")
    fb = make_frames(s, args.batch, snr_db=25.0, nu_max_hz=args.nu, seed=7, n_paths=args.paths)
    out = s.alloc(args.batch, llr=True, bit_errors=True)
    for _ in range(3):
        s.solve(fb.y, fb.paths, fb.lam, tx_labels=fb.tx_labels, out=out)
    prof = torch.zeros(4736, nat.kProfPhases if hasattr(nat, "kProfPhases") else 12, dtype=torch.int64,
                       device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = s.solve(fb.y, fb.paths, fb.lam, tx_labels=fb.tx_labels, out=out, phase_cycles=prof)
    e1.record()
    torch.cuda.synchronize()
    it_done = res.iterations_done.float().mean().item() if res.iterations_done is not None else None
    flat = prof.cpu().reshape(-1)
    p = flat[:4096 - 4096 % 12].reshape(-1, 12)
    rows = p[p.sum(dim=1) > 0]
    # per-warp timers [cta][warp][fwd MVM, herm MVM, arrive, wait, arrive parts] (kProfWarpBase)
    wt = flat[4096:4096 + rows.shape[0] * 16 * 8].reshape(rows.shape[0], 16, 8).double()
    tot = rows.sum(dim=0).double()
    frames_per_cta = args.batch / (rows.shape[0] / s.plan()["cluster"])
    res = {"plan": s.plan(), "ms": e0.elapsed_time(e1), "ctas": int(rows.shape[0]), "mean_iterations": it_done,
           "cycles_per_frame": float(tot.sum() / rows.shape[0] / frames_per_cta),
           "phases_pct": {name: round(100 * float(tot[i] / tot.sum()), 2) for i, name in enumerate(nat.PHASES)},
           "phase_cycles_per_frame": {name: round(float(tot[i] / rows.shape[0] / frames_per_cta))
                                      for i, name in enumerate(nat.PHASES)},
           "per_warp_cycles_per_frame": {
               k: [round(float(v)) for v in (wt[:, :, i].mean(dim=0) / frames_per_cta)]
               for i, k in enumerate(("mvm_fwd", "mvm_herm", "arrive", "wait", "a_tmem_st", "a_cta_bar", "a_fold", "a_arrive"))}}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
