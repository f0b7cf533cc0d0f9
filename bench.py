#!/usr/bin/env python
"""Benchmark of the SS-CGA equalizer hot path (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], the metric's configuration): OTFS M=512,
N=32, P=6 Veh-A taps, 16-QAM, Xi=10 fixed CG iterations, 25 dB, a batch of
4096 frames per GPU (weak scaling: every rank solves its own 4096 frames, no
collective on the data path).  A step = one fused solve of the whole batch
(coefficients on the fly + CG + hard decisions + max-log LLRs + bit errors).

One JSON line on rank 0: symbols/s (value, device-resident inputs), the same
metric end to end from pinned host buffers (e2e), p50/p99 single-frame
latency (CUDA graph replays), the FP32 roofline of the fused kernel against
the FP32 peak measured on this box by an FFMA probe, the HBM fraction, the
oracle port timed on the host cores (cpu_baseline) and the clocks seen.
`--impl reference` times the reference algorithm's CPU implementation (the
numpy oracle port of ddlink, oracle/ddlink_oracle.py) on all host cores.
"""

from __future__ import annotations

import os

# The CPU reference legs run one single-threaded numpy process per core, as
# run_packets does with OPENBLAS_NUM_THREADS=1 (harness.py:217-232; SURVEY.md
# 8c: multithreaded OpenBLAS makes cga_equalize ~10x slower).  BLAS pools are
# sized when numpy first loads, so this has to precede every import.
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse  # noqa: E402
import json  # noqa: E402
import math  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import tempfile  # noqa: E402
import time  # noqa: E402
from pathlib import Path  # noqa: E402

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

METRIC = "DD-equalized symbols/sec (M=512,N=32,P=6, 16-QAM); p50 per-frame latency"
CONFIGS = {
    "cfg1": dict(M=64, N=16, P=4, mod="qpsk", batch=4096, nu=0.0),
    "cfg2": dict(M=256, N=16, P=4, mod="qam16", batch=1024, nu=300.0),
    "cfg3": dict(M=512, N=32, P=6, mod="qam16", batch=4096, nu=100.0),
    # BASELINE config 4: high mobility (nu_max 1000 Hz: Doppler taps), 8 paths, 64-QAM (build extension)
    "cfg4": dict(M=1024, N=64, P=8, mod="qam64", batch=1024, nu=1000.0),
    # cfg3 grid with the taps the reference's detect_paths finds on fractional-Doppler
    # Veh-A channels (tests/golden/frames_sweep.npz: 8-10 taps per frame, 2-4 of them
    # Doppler-leakage taps at l = L0 +- 1), cycled over the batch
    "cfg3det": dict(M=512, N=32, P=0, mod="qam16", batch=4096, nu=100.0, taps="frames_sweep"),
    # the paper's real-time grid: beyond a cluster's on-chip
    # memory, so the workspace-backed kernels run it
    "paper": dict(M=16384, N=32, P=6, mod="qam16", batch=128, nu=100.0),
    # the grid the paper times its SS-CGA equalization on (PAPER.md:1529, 1627-1629:
    # (128, 32), QPSK; 0.54-0.78 ms per frame on H200)
    "paper128": dict(M=128, N=32, P=6, mod="qpsk", batch=4096, nu=100.0),
    # SURVEY.md 8(d)(3)'s fixed-P kernel benchmark: a dominant unit tap plus 5
    # taps of magnitude 0.05-0.2 at distinct random bins anywhere on the grid
    # (tests/test_acceptance.py:40-50, random_tap_frame), so most taps shift
    # Doppler (DSMEM / per-element route); y = Hx + AWGN as for the others (the
    # survey's y ~ CN(0, 1) changes nothing: the solve's cost is data-independent)
    "cfg3rand": dict(M=512, N=32, P=6, mod="qam16", batch=4096, nu=0.0, taps="random"),
}
BPS = {"qpsk": 2, "qam16": 4, "qam64": 6}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg3")
    ap.add_argument("--batch", type=int, default=0, help="frames per GPU (default: config's)")
    ap.add_argument("--snr", type=float, default=25.0)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--paths", type=int, default=0, help="override taps per frame (analysis only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-frontend", action="store_true")
    ap.add_argument("--e2e-chunk", type=int, default=444, help="frames per HostPipeline chunk (6 waves of 74 clusters)")
    ap.add_argument("--e2e-depth", type=int, default=2)
    ap.add_argument("--lat-runs", type=int, default=2000)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="weak: every rank solves the config's batch; strong: the batch is split over the ranks "
                         "(dist.shard)")
    ap.add_argument("--precision", choices=("fp32", "fp64"), default="fp32",
                    help="fp64 = the drop-in cga_equalize default (complex128, bit-identical decisions)")
    ap.add_argument("--no-dropin", action="store_true", help="skip the drop-in cga_equalize per-call latency")
    ap.add_argument("--delay-scale", type=float, default=1.0, help="scale the Veh-A delays (kernel analysis only)")
    ap.add_argument("--no-geometry", action="store_true",
                    help="skip the cfg3det / cfg3rand tap-geometry lines reported beside the headline")
    return ap.parse_args()


def median_ms(fn, stream, reps: int = 5) -> float:
    """Median device time of fn() over reps calls (CUDA events on `stream`,
    synchronised on both sides): robust to one-off host stalls in calls that
    include host round trips (the receiver's tap CSR)."""
    import torch
    times = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        times.append(a.elapsed_time(b))
    return sorted(times)[len(times) // 2]


def flops_per_frame(P, MN, iters):
    return 8 * P * MN * (2 * iters + 1) + 24 * MN * iters + 4 * MN


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows
                                                        if r[3].replace(".", "").isdigit())}


# ------------------------------------------------------------------ CPU side (oracle port)
def _cpu_frames(cfg, S, snr_db, iters, seed):
    """Synthetic frames of the workload, built with the oracle on the host."""
    import numpy as np
    import ddlink_oracle as orc
    rng = np.random.default_rng(seed)
    M, N = cfg["M"], cfg["N"]
    const = orc.qam(cfg["mod"])
    B = M * 30e3
    P = cfg["P"] or 6
    delays = np.round(np.array([0.0, 0.31, 0.71, 1.09, 1.73, 2.51])[:P] * 1e-6 * B).astype(int)
    pw = 10 ** (np.array([0.0, -1.0, -9.0, -10.0, -15.0, -20.0])[:P] / 10)
    mags = np.sqrt(pw / pw.sum())
    frames = []
    for _ in range(S):
        dop = np.round(cfg["nu"] * np.cos(2 * np.pi * rng.random(P)) / (30e3 / N)).astype(int)
        taps = [orc.Tap(int((M // 2 + d) % M), int((N // 2 + o) % N), complex(m * np.exp(2j * np.pi * rng.random())))
                for d, o, m in zip(delays, dop, mags)]
        lab = rng.integers(0, len(const.points), M * N)
        t = orc.build_tables(taps, M, N)
        hx = orc.forward(t, const.points[lab])
        snr = 10 ** (snr_db / 10)
        sigma = math.sqrt(np.mean(np.abs(hx) ** 2) / snr / 2)
        y = hx + sigma * (rng.normal(size=M * N) + 1j * rng.normal(size=M * N))
        frames.append((taps, y, 1.0 / snr))
    return frames, const


_WORK = None


def _single_thread_blas():
    """Pin every BLAS / OpenMP pool of this process to one thread (the parent may
    already have loaded numpy with the default pool, e.g. under torch)."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except ImportError:
        pass


def _init_worker(frames, cfg, iters):
    global _WORK
    _single_thread_blas()
    _WORK = (frames, cfg, iters)


def _solve_chunk(idx):
    import ddlink_oracle as orc
    frames, cfg, iters = _WORK
    const = orc.qam(cfg["mod"])
    times = []
    for i in idx:
        taps, y, lam = frames[i % len(frames)]
        t0 = time.perf_counter()
        orc.receive(taps, y, cfg["M"], cfg["N"], iters, lam, const)
        times.append(time.perf_counter() - t0)
    return times


def _solve_chunk_ref(idx):
    """The unmodified reference (baseline/_ref ddlink): build_ss_channel ->
    cga_equalize -> hard_demod per frame (harness.py:163, 189-194)."""
    import numpy as np
    from ddlink import grid as G, sparse as SP
    from ddlink.equalize import CgaConfig, cga_equalize
    frames, cfg, iters = _WORK
    g = G.GridConfig(cfg["M"], cfg["N"], 30e3)
    const = G.make_constellation(cfg["mod"])
    times = []
    for i in idx:
        taps, y, lam = frames[i % len(frames)]
        paths = [SP.DominantPath(t.k, t.l, t.gain) for t in taps]
        t0 = time.perf_counter()
        ch = SP.build_ss_channel(paths, g)
        x, _ = cga_equalize(ch, np.asarray(y), CgaConfig(iterations=iters, lam=lam))
        G.hard_demod(G.unflatten(x, g), const, g)
        times.append(time.perf_counter() - t0)
    return times


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def have_reference() -> bool:
    return (ROOT / "baseline" / "_ref" / "ddlink" / "__init__.py").exists()


class CpuArm:
    """The reference hot path (build_ss_channel -> cga_equalize -> hard_demod)
    on the host cores, one process per core like run_packets (harness.py:217-232):
    the unmodified reference from baseline/_ref when it is installed
    (kind "reference"), else its numpy restatement (kind "port")."""

    def __init__(self, cfg, snr_db, iters, seed=123, prefer_reference=True, frames=None):
        import multiprocessing as mp
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        os.environ["OMP_NUM_THREADS"] = "1"
        self.cores = len(os.sched_getaffinity(0))
        self.cfg, self.iters = cfg, iters
        self.kind = "port"
        self.fn = _solve_chunk
        # the reference demodulates QPSK / 16-QAM only (grid.py:126-154); 64-QAM runs the port
        if prefer_reference and have_reference() and cfg["mod"] in ("qpsk", "qam16"):
            ref = str(ROOT / "baseline" / "_ref")
            if ref not in sys.path:
                sys.path.insert(0, ref)
            try:
                import ddlink  # noqa: F401
                self.kind, self.fn = "reference", _solve_chunk_ref
            except ImportError:
                pass
        if frames is None:
            frames, _ = _cpu_frames(cfg, 8, snr_db, iters, seed)
        self.pool = mp.get_context("fork").Pool(self.cores, initializer=_init_worker,
                                                initargs=(frames, cfg, iters))
        self.pool.map(self.fn, [[0]] * self.cores)  # warm every worker
        _init_worker(frames, cfg, iters)
        t = self.fn([0, 1])
        self.frame_s = sum(t) / len(t)
        self.frame_times = []

    def run(self, frames_total):
        per = max(1, frames_total // self.cores)
        chunks = [list(range(i * per, (i + 1) * per)) for i in range(self.cores)]
        t0 = time.perf_counter()
        parts = self.pool.map(self.fn, chunks)
        dt = time.perf_counter() - t0
        times = [x for p in parts for x in p]
        self.frame_times.extend(times)
        return len(times), dt

    def frame_stats(self) -> dict:
        t = sorted(self.frame_times)
        if not t:
            return {}
        return {"p50_frame_ms": 1e3 * t[len(t) // 2], "p99_frame_ms": 1e3 * t[min(len(t) - 1, int(len(t) * 0.99))],
                "frames_timed": len(t)}

    def close(self):
        self.pool.terminate()


def sample_frames(arm, seconds):
    """Frames per step so one step is ~`seconds` of CPU work in total."""
    return max(arm.cores, int(seconds / max(arm.frame_s, 1e-4)))


# ------------------------------------------------------------------ reference arm
def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    arm = CpuArm(cfg, args.snr, args.iters)
    MN = cfg["M"] * cfg["N"]
    per_step = max(arm.cores, int(min(args.cpu_seconds, 8.0) / arm.frame_s))
    for _ in range(args.warmup):
        arm.run(arm.cores)
    arm.frame_times = []
    total_frames, total_t = 0, 0.0
    for _ in range(args.steps):
        n, dt = arm.run(per_step)
        total_frames += n
        total_t += dt
    stats = arm.frame_stats()
    arm.close()
    arm.frame_stats = lambda: stats  # noqa: E731 (pool closed; keep the sample's statistics)
    value = total_frames * MN / total_t
    what = ("ddlink (baseline/_ref, unmodified) build_ss_channel -> cga_equalize -> hard_demod"
            if arm.kind == "reference" else "numpy port of build_ss_channel -> cga_equalize -> hard_demod")
    sample = (f"{per_step} frames per step (~{per_step * arm.frame_s:.1f} s CPU work) of {what}, "
              f"{arm.cores} processes, OPENBLAS_NUM_THREADS=1")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "symbols/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "fp64 (complex128)", "data": "synthetic (host numpy, Veh-A taps)",
        "config": _config_json(args, cfg),
        "cpu_baseline": {"value": value, "unit": "symbols/s", "cores": arm.cores, "kind": arm.kind,
                         "sample": sample, "cpu_model": cpu_model(), **arm.frame_stats()},
        "e2e": {"value": value, "unit": "symbols/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "latency": {"p50_ms": arm.frame_stats().get("p50_frame_ms"), "p99_ms": arm.frame_stats().get("p99_frame_ms"),
                    "what": "single-core per-frame time of the reference path"},
    }
    print(json.dumps(line), flush=True)


def _config_json(args, cfg):
    B = args.batch or cfg["batch"]
    ptxt = f"P={cfg['P']}" if cfg["P"] else f"P=detect_paths taps of {cfg['taps']}"
    per = "frames/GPU" if args.scaling == "weak" else f"frames in all over {args.gpus} GPU(s)"
    return {"workload": f"{args.config}: OTFS M={cfg['M']} N={cfg['N']} {ptxt} {cfg['mod']} "
                        f"batch {B} {per}, Xi={args.iters}, {args.snr:g} dB, {args.precision}",
            "M": cfg["M"], "N": cfg["N"], "P": cfg["P"], "modulation": cfg["mod"],
            "batch_per_gpu": B if args.scaling == "weak" else -(-B // max(1, args.gpus)), "scaling": args.scaling,
            "iterations": args.iters, "snr_db": args.snr, "nu_max_hz": cfg["nu"],
            "parallelism": f"frame-sharded x{args.gpus}, no collective on the solve path",
            "l2": "inputs exceed L2 (y alone is batch*MN*8 B per GPU)"}


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2604_02266_b200 import dist as ddist
    rank, local, world = ddist.world()
    # one process per GPU (local rank = device); the modulo and DDB_DIST_BACKEND=gloo
    # only serve to exercise the multi-rank path with several ranks on one device
    torch.cuda.set_device(local % torch.cuda.device_count())
    ddist.init(os.environ.get("DDB_DIST_BACKEND", "nccl"))

    import ctypes as C
    import paper_2604_02266_b200 as pkg
    from paper_2604_02266_b200 import _native as nat
    from paper_2604_02266_b200.synth import make_frames

    M, N, P = cfg["M"], cfg["N"], (args.paths or cfg["P"])
    MN = M * N
    B_job = args.batch or cfg["batch"]
    if args.scaling == "strong":  # the job's batch split over the ranks, no collective
        lo, hi = ddist.shard(B_job, rank, world)
        B = hi - lo
    else:
        B = B_job
    bps = BPS[cfg["mod"]]
    s = pkg.SsCgaSolver(M, N, args.iters, precision=args.precision, modulation=cfg["mod"])
    given = None
    if cfg.get("taps") == "random":
        from paper_2604_02266_b200.synth import random_paths
        given = random_paths(B, M, N, P, ddist.rank_seed(3000, rank), s.cdtype)
    elif cfg.get("taps"):
        import numpy as np
        from paper_2604_02266_b200.synth import cycle_paths
        with np.load(ROOT / "tests" / "golden" / f"{cfg['taps']}.npz") as z:
            given = cycle_paths(B, z["path_off"], z["path_k"], z["path_l"], z["path_g"], "cuda", s.cdtype)
    fb = make_frames(s, B, snr_db=args.snr, nu_max_hz=cfg["nu"], modulation=cfg["mod"],
                     seed=ddist.rank_seed(1000, rank), n_paths=P or 6, paths=given, delay_scale=args.delay_scale)
    out = s.alloc(B, llr=True, trace=True, bit_errors=True)
    stream = torch.cuda.current_stream()

    def step():
        s.solve(fb.y, fb.paths, fb.lam, tx_labels=fb.tx_labels, out=out)

    barrier = ddist.barrier

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    ms = ddist.max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms / args.steps
    frames_job = world * B if args.scaling == "weak" else B_job
    value = frames_job * MN * args.steps / (ms * 1e-3)
    bit_errors = ddist.sum_over_ranks(int(out.bit_errors.sum().item()))
    ber = bit_errors / (frames_job * MN * bps)

    # ---- the same grid with other tap geometries (reported beside the headline):
    #      the taps detect_paths finds on fractional-Doppler Veh-A channels
    #      (Doppler-leakage taps) and SURVEY 8(d)(3)'s random P = 6 taps
    geometry = None
    if args.config == "cfg3" and not args.no_geometry:
        from paper_2604_02266_b200.synth import cycle_paths, random_paths
        with np.load(ROOT / "tests" / "golden" / "frames_sweep.npz") as z:
            det = cycle_paths(B, z["path_off"], z["path_k"], z["path_l"], z["path_g"], "cuda", s.cdtype)
        geometry = {}
        for name, pb in (("cfg3det", det), ("cfg3rand", random_paths(B, M, N, 6, 4321, s.cdtype))):
            for _ in range(3):
                s.solve(fb.y, pb, fb.lam, tx_labels=fb.tx_labels, out=out)
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(5):
                s.solve(fb.y, pb, fb.lam, tx_labels=fb.tx_labels, out=out)
            g1.record(stream)
            g1.synchronize()
            gms = g0.elapsed_time(g1) / 5
            p_avg = float((pb.offsets[-1] - pb.offsets[0]).item()) / B
            geometry[name] = {"value": B * MN / (gms * 1e-3), "unit": "symbols/s", "ms_per_step": gms,
                              "taps_per_frame": p_avg, "flops_per_frame": flops_per_frame(p_avg, MN, args.iters)}
        s.solve(fb.y, fb.paths, fb.lam, tx_labels=fb.tx_labels, out=out)  # restore the headline's outputs

    # ---- FP32 peak of this box (FFMA / FFMA2 probe), HBM peak from MEASURED_PEAKS
    scratch = torch.empty(148 * 8, dtype=torch.float32, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    lib = nat.load()
    peak_tflops = 0.0
    probe = {}
    for mode in ((0, 1) if args.precision == "fp32" else (2,)):
        blocks, iters = sms * 8, 2000 if mode < 2 else 200
        for _ in range(2):
            nat.check(lib.ddb_probe_fp32(mode, blocks, iters, C.c_void_p(scratch.data_ptr()),
                                         C.c_void_p(stream.cuda_stream)), "probe")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        nat.check(lib.ddb_probe_fp32(mode, blocks, iters, C.c_void_p(scratch.data_ptr()),
                                     C.c_void_p(stream.cuda_stream)), "probe")
        b.record(stream)
        b.synchronize()
        tf = blocks * 256 * iters * 256 * 2 / (a.elapsed_time(b) * 1e-3) / 1e12
        probe[("ffma", "ffma2", "dfma")[mode]] = tf
        peak_tflops = max(peak_tflops, tf)
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    hbm_peak = json.loads(peaks_path.read_text())["hbm_gbs"] if peaks_path.exists() else 6650.0
    P_avg = float((fb.paths.offsets[-1] - fb.paths.offsets[0]).item()) / B
    fl = flops_per_frame(P_avg, MN, args.iters)
    achieved = B * fl / (ms_step * 1e-3) / 1e12
    eb = 8 if args.precision == "fp32" else 16  # complex element bytes
    io_bytes = B * (eb * MN + eb * MN + 4 * bps * MN + MN + MN + 16 * P_avg)  # y, x, llr, labels, tx, taps
    workspace = s.plan()["kernel"] == "workspace"
    # workspace path: c, u, p stream through HBM every phase -- per iteration
    # g_fwd reads c (gather), u, p and writes u, p; g_herm reads u (gather), p,
    # x, c and writes x, c (11 vector passes); g_init reads y, writes c and x
    ws_bytes = B * (11 * args.iters + 3) * eb * MN if workspace else 0
    hbm_gbs = (io_bytes + ws_bytes) / (ms_step * 1e-3) / 1e9
    traffic = None
    ncu_sum = ROOT / "profiles" / f"ncu_{args.config}.json"
    if ncu_sum.exists():  # per-frame DRAM bytes of the committed ncu --set full capture, scaled to this launch
        per_frame = json.loads(ncu_sum.read_text()).get("dram_bytes_per_frame")
        traffic = per_frame * B if per_frame else None

    # ---- receiver front end (row f1): batched DZT of time-domain data frames
    #      (HBM-bound: 8 B read + 8 B written per symbol at fp32) and the pilot
    #      path (fp64 DZT + estimate fused, detect_paths) on the same batch
    frontend = None
    if not args.no_frontend:
        from paper_2604_02266_b200.zak import dzt_device
        y_time = torch.randn(B, MN, dtype=torch.complex64, device="cuda")
        y_dd = torch.empty_like(y_time)
        for _ in range(3):
            dzt_device(y_time, M, N, out=y_dd)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        a.record(stream)
        for _ in range(reps):
            dzt_device(y_time, M, N, out=y_dd)
        b.record(stream)
        b.synchronize()
        dzt_ms = a.elapsed_time(b) / reps
        dzt_gbs = B * MN * 16 / (dzt_ms * 1e-3) / 1e9
        pil = torch.zeros(B, MN, dtype=torch.complex128, device="cuda")
        pil[:, (N // 2) * M + M // 2] = math.sqrt(MN)  # an identity channel's pilot frame, time domain
        s.detect(pil, 0.08)
        torch.cuda.synchronize()
        a.record(stream)
        s.detect(pil, 0.08)
        b.record(stream)
        b.synchronize()
        det_ms = a.elapsed_time(b)
        # the whole receiver from time-domain pilot and data frames (SsCgaSolver.receive)
        from paper_2604_02266_b200.synth import time_domain_frames
        pil_rx, dat_rx = time_domain_frames(s, fb)
        for _ in range(2):
            rres = s.receive(pil_rx, dat_rx, fb.lam, 0.08, tx_labels=fb.tx_labels, trace=False)
        rx_ms = median_ms(lambda: s.receive(pil_rx, dat_rx, fb.lam, 0.08, tx_labels=fb.tx_labels, trace=False),
                          stream)
        rres = s.receive(pil_rx, dat_rx, fb.lam, 0.08, tx_labels=fb.tx_labels, trace=False)
        rx_ber = int(rres.bit_errors.sum().item()) / (B * MN * bps)
        del pil_rx, dat_rx, rres
        # frame synthesis on the device (row f2) and the receiver on those
        # continuous-Doppler packets (fractional Doppler leaks into extra taps)
        from paper_2604_02266_b200.channel import apply_channel_device
        from paper_2604_02266_b200.synth import synthesize_packets
        pb = synthesize_packets(s, B, snr_db=args.snr, nu_max_hz=cfg["nu"], modulation=cfg["mod"],
                                seed=ddist.rank_seed(2000, rank), cdtype=s.cdtype)
        torch.cuda.synchronize()
        a.record(stream)
        pb = synthesize_packets(s, B, snr_db=args.snr, nu_max_hz=cfg["nu"], modulation=cfg["mod"],
                                seed=ddist.rank_seed(2000, rank), cdtype=s.cdtype)
        b.record(stream)
        b.synchronize()
        synth_ms = a.elapsed_time(b)
        ych = torch.empty_like(pb.data_rx)
        apply_channel_device(pb.data_rx, pb.channel, pkg.GridConfig(M, N), out=ych)
        a.record(stream)
        for _ in range(reps):
            apply_channel_device(pb.data_rx, pb.channel, pkg.GridConfig(M, N), out=ych)
        b.record(stream)
        b.synchronize()
        ch_ms = a.elapsed_time(b) / reps
        del ych
        rres = s.receive(pb.pilot_rx, pb.data_rx, pb.lam, 0.08, tx_labels=pb.tx_labels, trace=False)
        frx_ms = median_ms(lambda: s.receive(pb.pilot_rx, pb.data_rx, pb.lam, 0.08, tx_labels=pb.tx_labels,
                                             trace=False), stream)
        frx_ber = int(rres.bit_errors.sum().item()) / (B * MN * bps)
        del pb, rres
        frontend = {"dzt_ms": dzt_ms, "dzt_gbs": dzt_gbs, "dzt_hbm_frac": dzt_gbs / hbm_peak,
                    "synth_ms": synth_ms, "apply_channel_ms": ch_ms,
                    "apply_channel_gbs": B * MN * 16 / (ch_ms * 1e-3) / 1e9,
                    "fracdop_receiver_ms": frx_ms, "fracdop_receiver_sym_s": B * MN / (frx_ms * 1e-3),
                    "fracdop_receiver_ber": frx_ber,
                    "receiver_ms": rx_ms, "receiver_sym_s": B * MN / (rx_ms * 1e-3), "receiver_ber": rx_ber,
                    "dzt_bytes_per_frame": MN * 16, "detect_ms_per_batch": det_ms,
                    "what": "ddb_dzt fp32 batch (zak.py:50-55) vs HBM peak; pilot path = fp64 DZT + estimate_heff "
                            "+ detect_paths + CSR for the batch (pilot.py:40-49, sparse.py:69-88); receiver = "
                            "SsCgaSolver.receive (median of 5 calls) on time-domain pilot + data frames (harness.py:156-194): pilot "
                            "path, data DZT, fused solve + demod + bit errors; synth = synthesize_packets "
                            "(modulate, idzt, Veh-A apply_channel with continuous Doppler, AWGN; pilot + data, "
                            "channel.py:62-119, harness.py:141-149) on the device; fracdop_receiver = receive on "
                            "those packets (detected taps include Doppler leakage)"}

    # ---- single-frame latency: CUDA graph of a batch-1 solve, replayed
    latency = None
    if not args.no_latency and rank == 0:
        # the whole receiver for one packet from time-domain pilot and data frames
        # (SsCgaSolver.receive: pilot DZT + detect_paths + CSR, data DZT, solve), as
        # the paper's full-receiver p99.9; not graph-captured (the
        # tap CSR is sized on the host), so host round trips are inside the time
        from paper_2604_02266_b200.synth import synthesize_packets
        pk1 = synthesize_packets(s, 1, snr_db=args.snr, nu_max_hz=cfg["nu"], modulation=cfg["mod"], seed=7,
                                 cdtype=s.cdtype)
        for _ in range(10):
            s.receive(pk1.pilot_rx, pk1.data_rx, pk1.lam, 0.08, tx_labels=pk1.tx_labels, trace=False)
        torch.cuda.synchronize()
        import gc
        gc.collect()
        gc.disable()  # a collector pass inside the loop is host jitter, not receiver time
        rlat = []
        for _ in range(args.lat_runs):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            s.receive(pk1.pilot_rx, pk1.data_rx, pk1.lam, 0.08, tx_labels=pk1.tx_labels, trace=False)
            b.record()
            b.synchronize()
            rlat.append(a.elapsed_time(b))
        gc.enable()
        rlat.sort()
        del pk1
        y1 = fb.y[:1].clone()
        lam1 = fb.lam[:1].clone()
        tx1 = fb.tx_labels[:1].clone()
        paths1 = pkg.PathBatch(fb.paths.offsets[:2].clone(), fb.paths.k, fb.paths.l, fb.paths.gain)
        o1 = s.alloc(1, llr=True, trace=True, bit_errors=True)
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            for _ in range(3):
                s.solve(y1, paths1, lam1, tx_labels=tx1, out=o1, stream=side)
        side.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            s.solve(y1, paths1, lam1, tx_labels=tx1, out=o1, stream=side)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.lat_runs)]
        for a, b in ev:
            a.record()
            g.replay()
            b.record()
        torch.cuda.synchronize()
        lat = sorted(a.elapsed_time(b) for a, b in ev)
        pl = s.plan()  # persistent clusters: ctas_per_sm frames-slices per SM (measured TMEM residency)
        n_clu = max(1, sms * max(1, pl["ctas_per_sm"]) // max(1, pl["cluster"]))
        latency = {"p50_ms": lat[len(lat) // 2], "p99_ms": lat[int(len(lat) * 0.99)],
                   "p999_ms": lat[int(len(lat) * 0.999)],
                   "max_ms": lat[-1], "runs": len(lat), "frame_duration_ms": 1e3 * N / 30e3,
                   "receiver_p50_ms": rlat[len(rlat) // 2], "receiver_p99_ms": rlat[int(len(rlat) * 0.99)],
                   "receiver_p999_ms": rlat[int(len(rlat) * 0.999)], "receiver_runs": len(rlat),
                   # in a full batch every cluster solves B / clusters frames back to back
                   "in_batch_frame_residency_ms": ms_step * n_clu / B if s.plan()["kernel"] != "workspace" else None,
                   "what": ("batch-1 solve (the lean + general fused launches" if s.plan()["kernel"] == "tmem" else
                            "batch-1 solve (one fused launch" if s.plan()["kernel"] != "workspace" else
                            "batch-1 solve (workspace-backed kernels, one graph") + ", CUDA graph replay), device events; "
                           "receiver_*: one packet through SsCgaSolver.receive from time-domain pilot + data "
                           "frames (device-synthesised), events around the call"}

    # ---- end to end from pinned host buffers (HostPipeline)
    e2e = None
    if not args.no_e2e:
        pipe = pkg.HostPipeline(s, chunk=args.e2e_chunk, depth=args.e2e_depth)
        hy = fb.y.cpu().pin_memory()
        hl = fb.lam.cpu().pin_memory()
        # transmitted labels as bits (bps bits per symbol, packed) like the reference's tx_bits
        tx_in = pkg.pack_labels(fb.tx_labels, bps) if bps in (2, 4) else fb.tx_labels
        ht = tx_in.cpu().pin_memory()
        hp = tuple(t.cpu().pin_memory() for t in (fb.paths.offsets, fb.paths.k, fb.paths.l, fb.paths.gain))
        lab_h = torch.empty(B, MN, dtype=torch.uint8).pin_memory()
        err_h = torch.empty(B, dtype=torch.int32).pin_memory()
        k2 = max(1, min(args.steps, 5))

        def timed(tx):
            """Device time of k2 HostPipeline passes (the first H2D to the last D2H)."""
            pipe.run(hy, hp, hl, tx, lab_h, err_h)
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(pipe.h2d)
            for _ in range(k2):
                pipe.run(hy, hp, hl, tx, lab_h, err_h)
            b.record(pipe.d2h)
            b.synchronize()
            return ddist.max_over_ranks(a.elapsed_time(b))

        # the equalizer end to end -- y, taps and lam in, hard decisions out: the
        # work of the reference arm's build_ss_channel -> cga_equalize -> hard_demod
        ems = timed(None)
        assert torch.equal(lab_h.to("cuda"), out.labels)
        # the same with the transmitted labels in and per-frame bit errors out
        ems_ber = timed(ht)
        assert torch.equal(err_h, out.bit_errors.cpu())
        h2d = hy.numel() * hy.element_size() + hl.numel() * hl.element_size() + \
            sum(t.numel() * t.element_size() for t in hp)
        d2h = lab_h.numel()
        # the bound: this box's pinned H2D copy bandwidth (one 512 MB copy, device events)
        probe_h = torch.empty(1 << 29, dtype=torch.uint8).pin_memory()
        probe_d = torch.empty(1 << 29, dtype=torch.uint8, device="cuda")
        probe_d.copy_(probe_h, non_blocking=True)
        a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a2.record()
        probe_d.copy_(probe_h, non_blocking=True)
        b2.record()
        b2.synchronize()
        h2d_peak = (1 << 29) / (a2.elapsed_time(b2) * 1e-3) / 1e9
        del probe_h, probe_d
        h2d_gbs = h2d / (ems / k2 * 1e-3) / 1e9
        e2e = {"value": frames_job * MN * k2 / (ems * 1e-3), "unit": "symbols/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": k2, "ms_per_step": ems / k2,
               "pcie": {"h2d_gbs": h2d_gbs, "h2d_peak_gbs": h2d_peak, "frac": h2d_gbs / h2d_peak,
                        "peak_source": "one 512 MB pinned H2D copy on this box"},
               "what": "HostPipeline (SsCgaSolver through three streams, chunks overlapped): pinned H2D of "
                       "y / taps / lam, fused solve + demod, D2H of the hard decisions -- the reference arm's "
                       "build_ss_channel -> cga_equalize -> hard_demod, end to end",
               "with_bit_errors": {
                   "value": frames_job * MN * k2 / (ems_ber * 1e-3), "ms_per_step": ems_ber / k2,
                   "h2d_bytes_per_step": h2d + ht.numel(), "d2h_bytes_per_step": d2h + err_h.numel() * 4,
                   "what": "the same plus the transmitted labels in (bps bits per symbol) and per-frame bit "
                           "errors out (run_packet's BER, harness.py:198)"}}

    # ---- CPU baseline (oracle port on the host cores), rank 0 at N=1 only
    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        # the GPU arm's own frames (taps, y, lam), copied to the host
        import ddlink_oracle as orc
        offs = fb.paths.offsets.cpu().numpy()
        kk, ll = fb.paths.k.cpu().numpy(), fb.paths.l.cpu().numpy()
        gg = fb.paths.gain.cpu().numpy().astype(np.complex128)
        own = []
        for f in range(min(B, 16)):
            a0, a1 = int(offs[f]), int(offs[f + 1])
            taps = [orc.Tap(int(kk[i]), int(ll[i]), complex(gg[i])) for i in range(a0, a1)]
            own.append((taps, fb.y[f].cpu().numpy().astype(np.complex128), float(fb.lam[f])))
        arm = CpuArm(cfg, args.snr, args.iters, frames=own)
        n = sample_frames(arm, args.cpu_seconds)
        done, dt = arm.run(n)
        stats = arm.frame_stats
        arm.close()
        cpu = {"value": done * MN / dt, "unit": "symbols/s", "cores": arm.cores, "kind": arm.kind,
               "sample": f"{done} frames cycled from the first {len(own)} frames of the GPU arm's batch "
                         f"({'ddlink from baseline/_ref' if arm.kind == 'reference' else 'numpy port'}"
                         f": build_ss_channel->cga_equalize->hard_demod), {arm.cores} processes, {dt:.1f} s wall",
               "cpu_model": cpu_model(), **stats()}

    if geometry:
        for g in geometry.values():
            g["fp32_frac"] = g["value"] / MN * g["flops_per_frame"] / 1e12 / peak_tflops
    roof_fp = {"bound": args.precision, "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
               "frac": achieved / peak_tflops, "traffic": None if workspace else traffic,
               "flops_per_frame": fl, "peak_source": f"FMA probe on this GPU {probe}"}
    roof_hbm = {"bound": "hbm", "achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": hbm_gbs / hbm_peak, "traffic": traffic if workspace else None,
                "bytes_per_frame": (io_bytes + ws_bytes) / B, "workspace_bytes_per_frame": ws_bytes / B,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks_path.exists() else "fallback"}

    # ---- the drop-in a ddlink user calls: cga_equalize(ch, y, cfg) on numpy
    #      arrays, one frame per call (host wall clock around the call)
    dropin = None
    if not args.no_dropin and rank == 0:
        from paper_2604_02266_b200 import equalize as eqz
        o0, o1 = int(fb.paths.offsets[0]), int(fb.paths.offsets[1])
        taps = [pkg.DominantPath(int(k), int(l), complex(g)) for k, l, g in
                zip(fb.paths.k[o0:o1].tolist(), fb.paths.l[o0:o1].tolist(), fb.paths.gain[o0:o1].cpu().numpy())]
        ch = pkg.build_ss_channel(taps, pkg.GridConfig(M, N))
        y0 = fb.y[0].cpu().numpy().astype(np.complex128)
        ccfg = pkg.CgaConfig(iterations=args.iters, lam=float(fb.lam[0]))
        dropin = {"what": "drop-in cga_equalize (numpy complex128 in/out, one frame per call, H2D + solve + "
                          "D2H), host wall clock, median of 50 calls"}
        prev = eqz.get_precision()
        for prec in ("fp64", "fp32"):
            eqz.set_precision(prec)
            for _ in range(5):
                eqz.cga_equalize(ch, y0, ccfg)
            t = []
            for _ in range(50):
                t0 = time.perf_counter()
                eqz.cga_equalize(ch, y0, ccfg)
                t.append(time.perf_counter() - t0)
            t.sort()
            dropin[f"{prec}_p50_ms"] = 1e3 * t[len(t) // 2]
            dropin[f"{prec}_p99_ms"] = 1e3 * t[-1]
        eqz.set_precision(prev)
        dropin["default_precision"] = prev

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "symbols/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": args.precision,
            "data": "synthetic (device-generated Veh-A taps, uniform labels, y = Hx + AWGN)",
            "config": _config_json(args, cfg),
            "latency": latency,
            # the bound of the dominant kernel: the fused kernels keep the CG state on chip
            # (FP32 / FP64 FMA bound); the workspace path streams it through HBM
            "roofline": (roof_hbm if workspace else roof_fp),
            ("roofline_fp" if workspace else "roofline_hbm"): (roof_fp if workspace else roof_hbm),
            "dropin": dropin,
            "tap_geometry": geometry,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "frontend": frontend,
            # our kernels per step: the TMEM kernel's lean + general instantiations
            # (csrc/sscga_tm.cu launch_r), one row-slice launch, one cooperative launch
            # (workspace path, <= 8 frames), else the workspace phase sequence
            "gpu_launches": args.steps * (2 if s.plan()["kernel"] == "tmem" else
                                          1 if s.plan()["kernel"] != "workspace" or B <= 8
                                          else 4 * args.iters + 5),
            "clocks": clocks,
            "plan": s.plan(),
            "ber": ber,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
