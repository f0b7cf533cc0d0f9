"""Packet pipeline on the device: drop-in for ddlink.harness.

Same configuration, result and statistics types as
/root/reference/pkg/src/ddlink/harness.py -- SimConfig (38-87), PacketResult
(90-107), LatencyStats (110-116), latency_stats (235-244), throughput_mbps
(247-253), aggregate (256-274), apply_axis / run_sweep (277-299),
benchmark_latency (302-316) -- with the packets received by the B200 kernels:

* synthesis (run_packet's untimed TX side, harness.py:141-149) keeps the
  reference's draw order on the same per-packet generators
  (default_rng([seed, idx]), harness.py:212): Veh-A fading, TX bits, pilot
  noise, data noise.  The random variates are drawn on the host; modulate,
  idzt and apply_channel run batched on the device (fp64, rounding-level
  agreement with numpy) and the noise is added there at the reference's
  per-frame power;
* the receiver (harness.py:155-198) is one device batch per chunk:
  pilot DZT + estimate + detect_paths (ddb_dzt, ddb_detect_paths,
  ddb_paths_csr), data DZT, and the fused SS-CGA solve with hard decisions and
  the per-packet bit-error count (ddb_sscga_solve); equalizer="lmmse" runs the
  dense branch (dense.receive_lmmse).  A packet without taps is failed and
  scored bits / 2 (harness.py:170-178).

Timing: run_packets receives a chunk of packets at once and fills each
PacketResult's stage times with the chunk's stage times (CUDA events on the
launch stream) divided by the packets in it -- the per-packet cost in
throughput mode.  benchmark_latency receives one packet per launch sequence,
so its stage times are true single-packet latencies (pilot path = DZT +
estimate + detection + CSR, data path = DZT + fused solve and demod).
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, replace
from typing import Optional, Sequence

import numpy as np
import torch

from . import channel as chan
from .batch import PathBatch, SsCgaSolver
from .grid import GridConfig, make_constellation_ext
from .pilot import make_pilot_frame

MODULATIONS = ("qpsk", "qam16", "qam64")  # qam64: the build's 64-QAM extension
EQUALIZERS = ("ss-cga", "lmmse")
SWEEP_AXES = ("snr", "nu_max", "m", "theta")
CSV_COLUMNS = (
    "m", "n", "delta_f_hz", "mod", "snr_db", "nu_max_hz", "theta", "iters",
    "equalizer", "seed", "packets", "ber_mean", "bits_total", "bit_errors",
    "lat_median_us", "lat_p99_us", "lat_p999_us", "deadline_us",
    "deadline_met_rate", "throughput_mbps",
)


@dataclass(frozen=True)
class SimConfig:
    """One experiment configuration (harness.py:38-87), same fields and checks."""

    m: int = 32
    n: int = 32
    delta_f: float = 30e3
    mod: str = "qpsk"
    snr_db: float = 25.0
    nu_max_hz: float = 100.0
    theta: float = 0.08
    iters: int = 10
    equalizer: str = "ss-cga"
    packets: int = 200
    seed: int = 0
    deadline_frames: float = 2.0
    workers: int = 1

    def __post_init__(self):
        if self.mod not in MODULATIONS:
            raise ValueError(f"mod must be one of {MODULATIONS}, got {self.mod!r}")
        if self.equalizer not in EQUALIZERS:
            raise ValueError(f"equalizer must be one of {EQUALIZERS}, got {self.equalizer!r}")
        if self.packets < 1:
            raise ValueError("packets must be >= 1")
        if self.iters < 1:
            raise ValueError("iters must be >= 1")
        if self.theta < 0:
            raise ValueError("theta must be nonnegative")
        if self.nu_max_hz < 0:
            raise ValueError("nu_max must be nonnegative")
        if self.deadline_frames <= 0:
            raise ValueError("deadline_frames must be positive")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        GridConfig(self.m, self.n, self.delta_f)  # validates geometry

    @property
    def grid(self):
        return GridConfig(self.m, self.n, self.delta_f)

    @property
    def deadline_s(self):
        return self.deadline_frames * self.n / self.delta_f

    @property
    def snr_linear(self):
        return 10.0 ** (self.snr_db / 10.0) if not math.isinf(self.snr_db) else math.inf


@dataclass
class PacketResult:
    """harness.py:90-107."""

    ber: float
    bits_total: int
    bit_errors: int
    time_dzt_s: float
    time_est_s: float
    time_build_s: float
    time_eq_s: float
    time_demod_s: float
    pilot_time_s: float
    data_time_s: float
    deadline_met: bool
    failed: bool = False

    @property
    def rx_time_s(self):
        return self.pilot_time_s + self.data_time_s


@dataclass(frozen=True)
class LatencyStats:
    median_s: float
    p99_s: float
    p999_s: float
    max_s: float
    met_rate: float


# ----------------------------------------------------------------- synthesis
@dataclass
class PacketBatchRx:
    """Received packets of a chunk on the device, as run_packet produces them."""

    indices: np.ndarray      # packet indices
    pilot_rx: torch.Tensor   # complex128 [n, MN] time samples of the pilot frame
    data_rx: torch.Tensor    # complex128 [n, MN] time samples of the data frame
    tx_labels: torch.Tensor  # uint8 [n, MN] transmitted labels (bits MSB first)


def synthesize(cfg: SimConfig, indices: Sequence[int], device=None, pset=None) -> PacketBatchRx:
    """run_packet's TX side and channel (harness.py:141-149) for the packets
    `indices`, in the reference's draw order on default_rng([seed, idx])."""
    from .sparse import _dev
    dev = device or _dev()
    g = cfg.grid
    const = make_constellation_ext(cfg.mod)
    b = const.bits_per_symbol
    MN = g.size
    idx = np.asarray(list(indices), dtype=np.int64)
    n = idx.size
    psets, labels = [], np.empty((n, MN), np.uint8)
    noiseless = math.isinf(cfg.snr_db)
    noise = None if noiseless else np.empty((2, n, MN), np.complex128)
    weights = 1 << np.arange(b - 1, -1, -1)
    for i, pi in enumerate(idx):
        rng = np.random.default_rng([cfg.seed, int(pi)])
        ps = pset if pset is not None else chan.draw_veha(cfg.nu_max_hz, g, rng)
        bits = rng.integers(0, 2, size=b * MN)
        labels[i] = bits.reshape(-1, b) @ weights
        if not noiseless:  # add_awgn's draws: pilot frame first, then data (channel.py:106-119)
            for j in range(2):
                re = rng.standard_normal(MN)
                noise[j, i] = re + 1j * rng.standard_normal(MN)
        psets.append(ps)
    lab = torch.as_tensor(labels, device=dev)
    X = chan.modulate_device(lab, b, torch.complex128)          # grid.py:157-169 (flattened q order)
    data_tx = chan.idzt_device(X, g.M, g.N)                    # zak.py:14-21
    pilot_tx = chan.idzt_device(torch.as_tensor(np.ascontiguousarray(make_pilot_frame(g).reshape(-1, order="F")),
                                                device=dev)[None], g.M, g.N).expand(n, MN).contiguous()
    chb = chan.ChannelBatch.from_pathsets(psets, dev)
    pil = chan.apply_channel_device(pilot_tx, chb, g)          # channel.py:86-95
    dat = chan.apply_channel_device(data_tx, chb, g)
    if not noiseless:
        snr_lin = 10.0 ** (cfg.snr_db / 10.0)
        nz = torch.as_tensor(noise, device=dev)
        for j, y in enumerate((pil, dat)):
            sigma = torch.sqrt((y.real ** 2 + y.imag ** 2).mean(dim=1) / snr_lin)
            y.add_((sigma / math.sqrt(2.0))[:, None] * nz[j])
    return PacketBatchRx(idx, pil, dat, lab)


# ----------------------------------------------------------------- receiver
class Receiver:
    """The receive path of run_packet (harness.py:155-198) for packet batches of
    one configuration, on the device, with per-stage CUDA-event timing."""

    def __init__(self, cfg: SimConfig, precision: str = "fp64", max_paths: int = 1024, device=None):
        self.cfg = cfg
        self.solver = SsCgaSolver(cfg.m, cfg.n, cfg.iters, precision=precision, modulation=cfg.mod, device=device)
        self.max_paths = int(max_paths)
        self.bps = self.solver.bps

    def receive(self, pk: PacketBatchRx) -> dict:
        """Returns per-packet bit_errors / failed (host arrays) and the stage
        times of the batch in seconds."""
        from .dense import receive_lmmse
        from .zak import dzt_device
        cfg, s = self.cfg, self.solver
        n = pk.pilot_rx.shape[0]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        lam = 0.0 if math.isinf(cfg.snr_linear) else 1.0 / cfg.snr_linear
        if cfg.equalizer == "lmmse":
            ev[0].record()
            out = receive_lmmse(s, pk.pilot_rx, pk.data_rx, cfg.snr_db, cfg.theta, tx_labels=pk.tx_labels)
            ev[4].record()
            ev[4].synchronize()
            t = ev[0].elapsed_time(ev[4]) / 1e3
            return {"bit_errors": out["bit_errors"].cpu().numpy(), "failed": out["failed"].cpu().numpy(),
                    "times": {"pilot": t, "data": 0.0, "dzt": 0.0, "est": 0.0, "build": t, "eq": 0.0}}
        pending: list = []
        ev[0].record()
        paths = s.detect(pk.pilot_rx, cfg.theta, max_paths=self.max_paths, _deferred=pending)
        ev[1].record()
        y = dzt_device(pk.data_rx.to(s.cdtype), cfg.m, cfg.n, colmajor=True)
        ev[2].record()
        lam_t = torch.full((n,), lam, dtype=s.rdtype, device=s.device)
        res = s.solve(y, paths, lam_t, tx_labels=pk.tx_labels, trace=True)
        ev[3].record()
        ev[3].synchronize()
        stats, mp = pending[0]
        cmin, cmax, _ = (int(v) for v in stats.tolist())
        if cmin < 0:
            raise RuntimeError("ddb_detect_paths: candidate list exceeds the per-frame capacity")
        if cmax > mp:
            raise ValueError(f"a frame has {cmax} taps above threshold > max_paths={mp}")
        pilot = ev[0].elapsed_time(ev[1]) / 1e3
        ddzt = ev[1].elapsed_time(ev[2]) / 1e3
        eq = ev[2].elapsed_time(ev[3]) / 1e3
        return {"bit_errors": res.bit_errors.cpu().numpy(), "failed": (res.status.cpu().numpy() & 1).astype(bool),
                "times": {"pilot": pilot, "data": ddzt + eq, "dzt": ddzt, "est": pilot, "build": 0.0, "eq": eq}}


def _results(cfg: SimConfig, out: dict, n: int, per_packet_share: bool) -> list:
    const = make_constellation_ext(cfg.mod)
    bits_total = const.bits_per_symbol * cfg.grid.size
    t = out["times"]
    k = float(n) if per_packet_share else 1.0
    res = []
    for e, f in zip(out["bit_errors"], out["failed"]):
        e = int(e)
        pilot, data = t["pilot"] / k, (0.0 if f else t["data"] / k)
        res.append(PacketResult(
            ber=e / bits_total, bits_total=bits_total, bit_errors=e,
            time_dzt_s=t["dzt"] / k, time_est_s=t["est"] / k, time_build_s=t["build"] / k,
            time_eq_s=0.0 if f else t["eq"] / k, time_demod_s=0.0,
            pilot_time_s=pilot, data_time_s=data,
            deadline_met=(pilot + data) <= cfg.deadline_s, failed=bool(f)))
    return res


def run_packets(cfg: SimConfig, packets: Optional[int] = None, *, chunk: int = 1024, precision: str = "fp64",
                max_paths: int = 1024, receiver: Optional[Receiver] = None, pset=None) -> list:
    """harness.py:217-232 on the device: deterministic in (seed, config),
    results in packet order.  Packets are synthesised and received in chunks
    of `chunk`; cfg.workers is accepted and ignored (one device)."""
    count = cfg.packets if packets is None else int(packets)
    rx = receiver or Receiver(cfg, precision=precision, max_paths=max_paths)
    out = []
    for c0 in range(0, count, chunk):
        idx = range(c0, min(count, c0 + chunk))
        pk = synthesize(cfg, idx, rx.solver.device, pset=pset)
        out.extend(_results(cfg, rx.receive(pk), len(idx), per_packet_share=True))
    return out


def latency_stats(results, deadline_s):
    """harness.py:235-244."""
    times = np.array([r.rx_time_s for r in results])
    met = float(np.mean([t <= deadline_s for t in times]))
    return LatencyStats(median_s=float(np.median(times)), p99_s=float(np.percentile(times, 99)),
                        p999_s=float(np.percentile(times, 99.9)), max_s=float(times.max()), met_rate=met)


def throughput_mbps(cfg, mean_ber):
    """harness.py:247-253: half the symbol rate times bits/symbol times (1 - BER)."""
    if not 0.0 <= mean_ber <= 1.0:
        raise ValueError("mean_ber must lie in [0, 1]")
    const = make_constellation_ext(cfg.mod)
    return 0.5 * cfg.m * cfg.delta_f * const.bits_per_symbol * (1.0 - mean_ber) / 1e6


def aggregate(cfg, results):
    """harness.py:256-274: one CSV row dict."""
    stats = latency_stats(results, cfg.deadline_s)
    ber_mean = float(np.mean([r.ber for r in results]))
    return {
        "m": cfg.m, "n": cfg.n, "delta_f_hz": cfg.delta_f, "mod": cfg.mod,
        "snr_db": cfg.snr_db, "nu_max_hz": cfg.nu_max_hz, "theta": cfg.theta,
        "iters": cfg.iters, "equalizer": cfg.equalizer, "seed": cfg.seed,
        "packets": len(results), "ber_mean": ber_mean,
        "bits_total": int(sum(r.bits_total for r in results)),
        "bit_errors": int(sum(r.bit_errors for r in results)),
        "lat_median_us": stats.median_s * 1e6, "lat_p99_us": stats.p99_s * 1e6,
        "lat_p999_us": stats.p999_s * 1e6, "deadline_us": cfg.deadline_s * 1e6,
        "deadline_met_rate": stats.met_rate, "throughput_mbps": throughput_mbps(cfg, ber_mean),
    }


def apply_axis(cfg, axis, value):
    """harness.py:277-292."""
    if axis == "snr":
        return replace(cfg, snr_db=float(value))
    if axis == "nu_max":
        return replace(cfg, nu_max_hz=float(value))
    if axis == "m":
        m = int(value)
        if m != value:
            raise ValueError(f"m sweep value {value!r} is not an integer")
        return replace(cfg, m=m)
    if axis == "theta":
        return replace(cfg, theta=float(value))
    raise ValueError(f"unknown sweep axis {axis!r}, expected one of {SWEEP_AXES}")


def run_sweep(cfg, axis, values, **kw):
    """harness.py:295-299: one aggregated row per axis value."""
    return [aggregate(p, run_packets(p, **kw)) for p in (apply_axis(cfg, axis, v) for v in values)]


def benchmark_latency(cfg, packets, *, precision: str = "fp64", max_paths: int = 1024, warmup: int = 3):
    """harness.py:302-316: the latency distribution of the receive path, one
    packet per launch sequence (batch 1), after `warmup` untimed packets."""
    if packets < 100:
        warnings.warn(f"{packets} packets is too few for stable percentiles; use >= 100", stacklevel=2)
    elif packets < 10_000:
        warnings.warn(f"p99.9 needs >= 10000 packets to be meaningful; got {packets}", stacklevel=2)
    rx = Receiver(cfg, precision=precision, max_paths=max_paths)
    pk = synthesize(cfg, range(packets), rx.solver.device)
    for i in range(min(warmup, packets)):
        rx.receive(_one(pk, i))
    results = []
    for i in range(packets):
        results.extend(_results(cfg, rx.receive(_one(pk, i)), 1, per_packet_share=False))
    return latency_stats(results, cfg.deadline_s), results


def _one(pk: PacketBatchRx, i: int) -> PacketBatchRx:
    return PacketBatchRx(pk.indices[i:i + 1], pk.pilot_rx[i:i + 1], pk.data_rx[i:i + 1], pk.tx_labels[i:i + 1])
