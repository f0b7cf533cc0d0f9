#!/usr/bin/env python
"""Time the receiver front end's pieces on a cfg3 batch: fp64 pilot DZT with the
fused estimate, detect_paths, CSR construction, fp32 data DZT."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes as C  # noqa: E402

import paper_2604_02266_b200 as pkg  # noqa: E402
from paper_2604_02266_b200 import _native as nat  # noqa: E402
from paper_2604_02266_b200.synth import make_frames, time_domain_frames  # noqa: E402
from paper_2604_02266_b200.zak import dzt_device  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


s = pkg.SsCgaSolver(512, 32, 10, precision="fp32", modulation="qam16")
B, M, N, MN = 4096, 512, 32, 512 * 32
fb = make_frames(s, B, seed=3)
pil, dat = time_domain_frames(s, fb)
pil64 = pil.to(torch.complex128)
heff = dzt_device(pil64, M, N, colmajor=False, pilot_amplitude=MN ** 0.5)
cnt = torch.empty(B, dtype=torch.int32, device="cuda")
kk = torch.empty(B, 64, dtype=torch.int32, device="cuda")
ll = torch.empty_like(kk)
gg = torch.empty(B, 64, dtype=torch.complex128, device="cuda")
lib = nat.load()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
res = {
    "pilot_cast_fp64_ms": timed(lambda: pil.to(torch.complex128)),
    "pilot_dzt_fp64_ms": timed(lambda: dzt_device(pil64, M, N, colmajor=False, pilot_amplitude=MN ** 0.5, out=heff)),
    "detect_kernel_ms": timed(lambda: lib.ddb_detect_paths(B, M, N, C.c_void_p(heff.data_ptr()), 0.08, 64,
                                                          C.c_void_p(cnt.data_ptr()), C.c_void_p(kk.data_ptr()),
                                                          C.c_void_p(ll.data_ptr()), C.c_void_p(gg.data_ptr()), st)),
    "detect_api_ms": timed(lambda: s.detect(pil, 0.08)),
    "data_dzt_fp32_ms": timed(lambda: dzt_device(dat, M, N, colmajor=True)),
    "solve_ms": timed(lambda: s.solve(fb.y, fb.paths, fb.lam, tx_labels=fb.tx_labels, trace=False)),
    "receive_ms": timed(lambda: s.receive(pil, dat, fb.lam, 0.08, tx_labels=fb.tx_labels, trace=False)),
}
print({k: round(v, 3) for k, v in res.items()})
