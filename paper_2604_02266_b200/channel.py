"""Multipath channel and frame synthesis on the device.

Drop-in for the numeric parts of /root/reference/pkg/src/ddlink/channel.py and
the transmit side of harness.py:141-149, plus a batched device API that
synthesises whole packet batches in HBM (so the receiver can be fed without
PCIe in the way):

  apply_channel   -> ddb_apply_channel  (channel.py:95-103), fp64, same result to rounding
  idzt            -> ddb_dzt with DDB_DZT_INVERSE (zak.py:14-21)
  modulate        -> ddb_modulate       (grid.py:157-169)
  add_awgn_device -> ddb_add_awgn       (channel.py:106-119 with a counter-based RNG)

The host-side path objects (`PathSpec`, `PathSet`, `make_path`, `draw_veha`)
follow channel.py:20-92 so a reference PathSet can be passed in unchanged;
`add_awgn` keeps the caller's numpy generator (the reference's noise stream is
part of its seeded known answers), so it stays a host operation.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .grid import GridConfig, check_frame, check_signal, flatten
from .sparse import _dev, _p, _stream

VEHA_DELAYS_US = (0.00, 0.31, 0.71, 1.09, 1.73, 2.51)
VEHA_POWERS_DB = (0.0, -1.0, -9.0, -10.0, -15.0, -20.0)


@dataclass(frozen=True)
class PathSpec:
    """One propagation path (channel.py:20-28)."""

    gain: complex
    delay_s: float
    doppler_hz: float
    delay_bin: int
    doppler_frac: float


@dataclass(frozen=True)
class PathSet:
    paths: tuple

    @property
    def P(self):
        return len(self.paths)

    def total_power(self):
        return float(sum(abs(p.gain) ** 2 for p in self.paths))


def make_path(gain, delay_s, doppler_hz, cfg):
    """PathSpec on the grid of cfg with the range checks of channel.py:44-59."""
    delay_bin = int(round(delay_s * cfg.B))
    doppler_frac = doppler_hz / cfg.delta_nu
    if not 0 <= delay_bin < cfg.M:
        raise ValueError(f"delay {delay_s * 1e6:.3f} us maps to bin {delay_bin}, "
                         f"outside the delay period of {cfg.M} bins")
    if abs(doppler_frac) > cfg.N / 2:
        raise ValueError(f"Doppler {doppler_hz:.1f} Hz exceeds half the Doppler period "
                         f"({cfg.N / 2 * cfg.delta_nu:.1f} Hz)")
    return PathSpec(complex(gain), float(delay_s), float(doppler_hz), delay_bin, doppler_frac)


def draw_veha(nu_max, cfg, rng):
    """One Vehicular-A realisation from the caller's numpy generator, drawing
    the same variates in the same order as channel.py:62-92 (phases, then
    Doppler angles), so a shared seed gives the reference's channel."""
    if nu_max < 0:
        raise ValueError("nu_max must be nonnegative")
    delays = np.asarray(VEHA_DELAYS_US) * 1e-6
    if delays[-1] >= cfg.M * cfg.delta_tau:
        raise ValueError(f"delay spread {delays[-1] * 1e6:.2f} us exceeds the delay period "
                         f"{cfg.M * cfg.delta_tau * 1e6:.2f} us; increase M or delta_f")
    w = 10.0 ** (np.asarray(VEHA_POWERS_DB) / 10.0)
    mags = np.sqrt(w / w.sum())
    phases = rng.uniform(0.0, 2.0 * np.pi, size=len(mags))
    nus = nu_max * np.cos(2.0 * np.pi * rng.uniform(0.0, 1.0, size=len(mags)))
    return PathSet(tuple(make_path(m * np.exp(1j * ph), d, nu, cfg)
                         for m, ph, d, nu in zip(mags, phases, delays, nus)))


# ---------------------------------------------------------------- batched device API
@dataclass
class ChannelBatch:
    """Per-frame physical paths as CSR on the device (delay bins int32, Doppler
    and delay float64, complex gains)."""

    offsets: torch.Tensor     # int32 [B+1]
    delay_bin: torch.Tensor   # int32 [P]
    doppler_hz: torch.Tensor  # float64 [P]
    delay_s: torch.Tensor     # float64 [P]
    gain: torch.Tensor        # complex [P]

    @property
    def batch(self) -> int:
        return self.offsets.numel() - 1

    @classmethod
    def from_pathsets(cls, psets, device=None, cdtype=torch.complex128) -> "ChannelBatch":
        dev = device or _dev()
        off = np.zeros(len(psets) + 1, np.int32)
        off[1:] = np.cumsum([len(ps.paths) for ps in psets])
        flat = [p for ps in psets for p in ps.paths]
        return cls(torch.as_tensor(off, device=dev),
                   torch.as_tensor(np.array([p.delay_bin for p in flat], np.int32), device=dev),
                   torch.as_tensor(np.array([p.doppler_hz for p in flat], np.float64), device=dev),
                   torch.as_tensor(np.array([p.delay_s for p in flat], np.float64), device=dev),
                   torch.as_tensor(np.array([p.gain for p in flat], np.complex128), device=dev).to(cdtype))


def draw_veha_batch(B: int, cfg: GridConfig, nu_max: float, gen: torch.Generator, device=None,
                    cdtype=torch.complex128) -> ChannelBatch:
    """B Veh-A realisations drawn on the device (torch RNG): the distribution
    of channel.py:62-92, not the reference's numpy stream."""
    if nu_max < 0:
        raise ValueError("nu_max must be nonnegative")
    dev = device or _dev()
    delays = np.asarray(VEHA_DELAYS_US) * 1e-6
    if delays[-1] >= cfg.M * cfg.delta_tau:
        raise ValueError("Veh-A delay spread exceeds the delay period; increase M or delta_f")
    P = len(delays)
    w = 10.0 ** (np.asarray(VEHA_POWERS_DB) / 10.0)
    mags = torch.as_tensor(np.sqrt(w / w.sum()), device=dev)
    phase = torch.rand(B, P, generator=gen, device=dev, dtype=torch.float64) * (2 * math.pi)
    nus = nu_max * torch.cos(2 * math.pi * torch.rand(B, P, generator=gen, device=dev, dtype=torch.float64))
    kb = torch.as_tensor(np.round(delays * cfg.B).astype(np.int32), device=dev).expand(B, P)
    ds = torch.as_tensor(delays, device=dev).expand(B, P)
    gain = torch.polar(mags.expand(B, P), phase).to(cdtype)
    off = torch.arange(0, (B + 1) * P, P, device=dev, dtype=torch.int32)
    return ChannelBatch(off, kb.reshape(-1).contiguous(), nus.reshape(-1).contiguous(),
                        ds.reshape(-1).contiguous(), gain.reshape(-1).contiguous())


def _dtype_of(t: torch.Tensor) -> int:
    if t.dtype == torch.complex64:
        return nat.DDB_F32
    if t.dtype == torch.complex128:
        return nat.DDB_F64
    raise ValueError("complex64 or complex128 expected")


def apply_channel_device(x: torch.Tensor, ch: ChannelBatch, cfg: GridConfig,
                         out: torch.Tensor | None = None) -> torch.Tensor:
    """Noiseless channel output of time-domain frames x [B, MN] (channel.py:95-103)."""
    if x.dim() != 2 or x.shape[1] != cfg.size or x.shape[0] != ch.batch:
        raise ValueError(f"x must be [{ch.batch}, {cfg.size}], got {tuple(x.shape)}")
    x = x.contiguous()
    dt = _dtype_of(x)
    gain = ch.gain.to(x.dtype).contiguous()
    if out is None:
        out = torch.empty_like(x)
    nat.check(nat.load().ddb_apply_channel(x.shape[0], cfg.M, cfg.N, dt, _p(x), _p(ch.offsets), _p(ch.delay_bin),
                                           _p(ch.doppler_hz), _p(ch.delay_s), _p(gain), float(cfg.B), _p(out),
                                           _stream()), "ddb_apply_channel")
    return out


def add_awgn_device(y: torch.Tensor, snr_db: float, seed: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """y [B, L] plus complex AWGN at snr_db relative to each frame's mean power
    (channel.py:106-119); counter-based normals, reproducible for a seed."""
    if y.dim() != 2:
        raise ValueError("y must be [B, L]")
    y = y.contiguous()
    if out is None:
        out = torch.empty_like(y)
    power = torch.empty(y.shape[0], dtype=torch.float64, device=y.device)
    nat.check(nat.load().ddb_add_awgn(y.shape[0], y.shape[1], _dtype_of(y), _p(y), float(snr_db),
                                      C.c_uint64(seed & (2 ** 64 - 1)), _p(power), _p(out), _stream()),
              "ddb_add_awgn")
    return out


def modulate_device(labels: torch.Tensor, bits_per_symbol: int, cdtype=torch.complex128) -> torch.Tensor:
    """Constellation points of uint8 labels (grid.py:157-169 after `groups @ weights`)."""
    labels = labels.to(torch.uint8).contiguous()
    out = torch.empty(labels.shape, dtype=cdtype, device=labels.device)
    nat.check(nat.load().ddb_modulate(labels.numel(), nat.DDB_F64 if cdtype == torch.complex128 else nat.DDB_F32,
                                      _p(labels), int(bits_per_symbol), _p(out), _stream()), "ddb_modulate")
    return out


def idzt_device(X: torch.Tensor, M: int, N: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """Inverse Zak transform of flattened DD vectors X [B, MN] (q = l M + k) to
    time samples (zak.py:14-21)."""
    if X.dim() != 2 or X.shape[1] != M * N:
        raise ValueError(f"X must be [B, {M * N}], got {tuple(X.shape)}")
    X = X.contiguous()
    if out is None:
        out = torch.empty_like(X)
    nat.check(nat.load().ddb_dzt(X.shape[0], M, N, _dtype_of(X), _p(X), None,
                                 nat.DDB_DZT_COLMAJOR | nat.DDB_DZT_INVERSE, 1.0, _p(out), _stream()), "ddb_dzt")
    return out


# ---------------------------------------------------------------- drop-in (numpy in / out)
def apply_channel(x, pset, cfg):
    """channel.py:95-103 on the device, complex128."""
    x = check_signal(x, cfg)
    dev = _dev()
    xt = torch.as_tensor(np.ascontiguousarray(x, dtype=np.complex128), device=dev)[None, :]
    y = apply_channel_device(xt, ChannelBatch.from_pathsets([pset], dev), cfg)
    torch.cuda.current_stream().synchronize()
    return y[0].cpu().numpy()


def idzt(X_dd, cfg):
    """zak.py:14-21 on the device, complex128."""
    X_dd = check_frame(X_dd, cfg)
    dev = _dev()
    xt = torch.as_tensor(np.ascontiguousarray(flatten(X_dd, cfg), dtype=np.complex128), device=dev)[None, :]
    out = idzt_device(xt, cfg.M, cfg.N)
    torch.cuda.current_stream().synchronize()
    return out[0].cpu().numpy()


def add_awgn(y, snr_db, rng):
    """channel.py:106-119 with the caller's numpy generator (host: the
    reference's seeded known answers depend on its noise stream)."""
    y = np.asarray(y)
    if math.isinf(snr_db):
        return y.copy()
    sigma = math.sqrt(float(np.mean(np.abs(y) ** 2)) / 10.0 ** (snr_db / 10.0))
    noise = rng.standard_normal(y.shape) + 1j * rng.standard_normal(y.shape)
    return y + sigma / math.sqrt(2.0) * noise
