import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2604_02266_b200 as pkg
from paper_2604_02266_b200.synth import make_frames
s = pkg.SsCgaSolver(512, 32, 10, precision="fp32", modulation="qam16")
fb = make_frames(s, 4096, snr_db=25.0, nu_max_hz=100.0, seed=7)
for trace in (True, False):
    for llr in (True, False):
        out = s.alloc(4096, llr=llr, trace=trace, bit_errors=True)
        for _ in range(3):
            s.solve(fb.y, fb.paths, fb.lam, tx_labels=fb.tx_labels, out=out, trace=trace)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            s.solve(fb.y, fb.paths, fb.lam, tx_labels=fb.tx_labels, out=out, trace=trace)
        b.record(); b.synchronize()
        ms = a.elapsed_time(b) / 10
        print(f"trace={trace} llr={llr}: {ms:.3f} ms  {4096*16384/ms/1e6:.2f} Gsym/s")
