"""Config 5 (BASELINE.json configs[4]): the SNR sweep 0-30 dB at M=512, N=32,
16-QAM, Veh-A at nu_max 100 Hz, theta 0.08, Xi 10 -- run by the UNMODIFIED
reference (`ddlink`, imported from baseline/_ref or /root/reference/pkg/src).

`reference_packet(d, snr_db, idx)` is run_packet (harness.py:131-205) with its
intermediates kept: the same draws on default_rng([SEED, idx]), the same
receiver calls.  Besides the reference's own result on the fp64 frame it also
runs cga_equalize + hard_demod on the complex64-rounded y, the input the fp32
device path consumes, so both device precisions are compared with the
reference on bit-identical inputs.

Used twice: make_golden.py stores the compact per-packet results of this
container's run (sweep_cfg5.npz); tests/test_sweep_parity.py regenerates the
packets with the reference on the GPU box (a process pool over the host
cores), checks them against that fixture, then compares the device path.
Test infrastructure only.
"""

from __future__ import annotations

import math

import numpy as np

M, N, MOD, NU, THETA, ITERS, SEED = 512, 32, "qam16", 100.0, 0.08, 10, 505
SNRS = (0.0, 5.0, 10.0, 15.0, 20.0, 25.0, 30.0)
PACKETS = 64  # per SNR


def _labels(bits, b):
    return (np.asarray(bits).reshape(-1, b) @ (1 << np.arange(b - 1, -1, -1))).astype(np.uint8)


def reference_packet(d, snr_db: float, idx: int, keep_frames: bool = True) -> dict:
    from ddlink.harness import Workspace
    cfg = d.SimConfig(m=M, n=N, mod=MOD, snr_db=snr_db, nu_max_hz=NU, theta=THETA, iters=ITERS, seed=SEED)
    ws = _ws_cache.get(snr_db)
    if ws is None:
        ws = _ws_cache[snr_db] = Workspace(cfg)
    grid, const = ws.grid, ws.const
    b = const.bits_per_symbol
    rng = np.random.default_rng([SEED, idx])
    pset = d.draw_veha(cfg.nu_max_hz, grid, rng)
    tx_bits = rng.integers(0, 2, size=b * grid.size)
    data_tx = d.idzt(d.modulate(tx_bits, const, grid), grid)
    pilot_rx = d.add_awgn(d.apply_channel(ws.pilot_tx, pset, grid), cfg.snr_db, rng)
    data_rx = d.add_awgn(d.apply_channel(data_tx, pset, grid), cfg.snr_db, rng)
    heff = d.estimate_heff(d.dzt_gemm(pilot_rx, ws.zak_kernel, grid), ws.twist, grid)
    taps = d.detect_paths(heff, cfg.theta, grid)
    lam = 0.0 if math.isinf(cfg.snr_linear) else 1.0 / cfg.snr_linear
    out = {"P": len(taps), "tx": _labels(tx_bits, b), "lam": lam,
           "tap_k": np.array([t.k_p for t in taps], np.int32), "tap_l": np.array([t.l_p for t in taps], np.int32),
           "tap_g": np.array([t.gain for t in taps], np.complex128)}
    y = d.flatten(d.dzt_gemm(data_rx, ws.zak_kernel, grid), grid)
    if not taps:  # EmptyChannel: run_packet scores bits / 2 (harness.py:170-178)
        out.update(errors=b * grid.size // 2, errors32=b * grid.size // 2, failed=True, c_norm=np.zeros(ITERS + 1),
                   c_norm32=np.zeros(ITERS + 1))
    else:
        ch = d.build_ss_channel(taps, grid)
        x, tr = d.cga_equalize(ch, y, d.CgaConfig(iterations=cfg.iters, lam=lam))
        _, rx_bits = d.hard_demod(d.unflatten(x, grid), const, grid)
        y32 = y.astype(np.complex64).astype(np.complex128)
        x32, tr32 = d.cga_equalize(ch, y32, d.CgaConfig(iterations=cfg.iters, lam=lam))
        _, rx32 = d.hard_demod(d.unflatten(x32, grid), const, grid)
        out.update(errors=int(np.sum(tx_bits != rx_bits)), errors32=int(np.sum(tx_bits != rx32)), failed=False,
                   c_norm=np.array(tr.c_norm), c_norm32=np.array(tr32.c_norm), rx=_labels(rx_bits, b),
                   rx32=_labels(rx32, b))
        if keep_frames:
            out.update(x=x, x32=x32)
    if keep_frames:
        out.update(pilot_rx=pilot_rx, data_rx=data_rx, y=y)
    return out


_ws_cache: dict = {}
_D = None


def _worker_init(paths):
    import sys
    global _D
    for p in paths:
        if p not in sys.path:
            sys.path.insert(0, p)
    import ddlink
    _D = ddlink


def _job(args):
    snr, idx, keep = args
    return snr, idx, reference_packet(_D, snr, idx, keep)


def run_all(sys_paths, keep_frames: bool = True, processes: int | None = None, snrs=SNRS, packets=PACKETS):
    """Every (SNR, packet) of the sweep through the reference, over a process pool."""
    import multiprocessing as mp
    import os
    jobs = [(s, i, keep_frames) for s in snrs for i in range(packets)]
    n = processes or max(1, min(len(os.sched_getaffinity(0)), 32))
    # one single-threaded numpy per worker (run_packets' setting);
    # spawned workers: the caller may hold a CUDA context, which fork must not copy
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    ctx = mp.get_context("spawn")
    with ctx.Pool(n, initializer=_worker_init, initargs=(list(sys_paths),)) as pool:
        res = pool.map(_job, jobs, chunksize=4)
    return {(s, i): r for s, i, r in res}
