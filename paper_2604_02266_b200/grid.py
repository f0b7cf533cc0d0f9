"""Grid geometry, constellations and demod — drop-in for ddlink.grid.

Same names, argument meaning and errors as the reference module
(/root/reference/pkg/src/ddlink/grid.py).  Layout helpers (flatten/unflatten,
checks) are host bookkeeping; the decision arithmetic of `hard_demod` runs in
the ddb CUDA library (ddb_hard_demod), never on the CPU.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat


@dataclass(frozen=True)
class GridConfig:
    """DD grid geometry (grid.py:14-65): M delay bins, N Doppler bins, spacing delta_f."""

    M: int
    N: int
    delta_f: float = 30e3

    def __post_init__(self):
        if self.M < 2 or self.N < 2:
            raise ValueError(f"grid must be at least 2x2, got ({self.M},{self.N})")
        if self.M % 2 or self.N % 2:
            raise ValueError(
                f"M and N must be even so the pilot sits on a bin center, got ({self.M},{self.N})")
        if self.delta_f <= 0:
            raise ValueError("delta_f must be positive")

    @property
    def B(self):
        return self.M * self.delta_f

    @property
    def T(self):
        return self.N / self.delta_f

    @property
    def delta_tau(self):
        return 1.0 / self.B

    @property
    def delta_nu(self):
        return self.delta_f / self.N

    @property
    def K0(self):
        return self.M // 2

    @property
    def L0(self):
        return self.N // 2

    @property
    def size(self):
        return self.M * self.N


def check_frame(frame, cfg):
    """Raise unless frame is (M, N) (grid.py:68-75)."""
    frame = np.asarray(frame)
    if frame.shape != (cfg.M, cfg.N):
        raise ValueError(f"frame shape {frame.shape} does not match grid ({cfg.M},{cfg.N})")
    return frame


def check_signal(x, cfg):
    """Raise unless x has length M*N (grid.py:78-83)."""
    x = np.asarray(x)
    if x.shape != (cfg.size,):
        raise ValueError(f"signal length {x.shape} != M*N = {cfg.size}")
    return x


def flatten(frame, cfg):
    """q = l*M + k, a fresh copy (grid.py:86-89)."""
    return np.ascontiguousarray(check_frame(frame, cfg).T).reshape(cfg.size).copy()


def unflatten(v, cfg):
    """frame[k, l] = v[l*M + k], a fresh copy (grid.py:92-95)."""
    return np.ascontiguousarray(check_signal(v, cfg).reshape(cfg.N, cfg.M).T)


def _axis_levels(bits_per_axis: int) -> np.ndarray:
    if bits_per_axis not in (1, 2, 3):
        raise ValueError("only 1, 2 or 3 bits per axis supported")
    lv = np.empty(1 << bits_per_axis)
    for i in range(lv.size):
        mag = 1
        for m in range(bits_per_axis - 1, 0, -1):
            cm = (i >> (bits_per_axis - 1 - m)) & 1
            mag = (1 << (bits_per_axis - m)) - (1 - 2 * cm) * mag
        lv[i] = (1 - 2 * ((i >> (bits_per_axis - 1)) & 1)) * mag
    return lv


@dataclass(frozen=True)
class Constellation:
    """Gray-mapped unit-energy constellation (grid.py:112-123)."""

    name: str
    points: np.ndarray
    bits_per_symbol: int
    bit_map: np.ndarray = field(repr=False)


def _build(key: str, bits_per_axis: int) -> Constellation:
    b = 2 * bits_per_axis
    lv = _axis_levels(bits_per_axis)
    order = 1 << b
    bit_map = np.array([[(s >> (b - 1 - i)) & 1 for i in range(b)] for s in range(order)], np.int8)
    pts = np.empty(order, complex)
    for s in range(order):
        i_idx = int("".join(str(v) for v in bit_map[s, 0::2]), 2)
        q_idx = int("".join(str(v) for v in bit_map[s, 1::2]), 2)
        pts[s] = lv[i_idx] + 1j * lv[q_idx]
    pts /= np.sqrt(np.mean(np.abs(pts) ** 2))
    pts.setflags(write=False)
    bit_map.setflags(write=False)
    return Constellation(name=key, points=pts, bits_per_symbol=b, bit_map=bit_map)


def make_constellation(name):
    """'qpsk' or 'qam16' (grid.py:126-154); anything else raises like the reference."""
    key = name.lower().replace("-", "").replace("_", "")
    if key == "qpsk":
        return _build(key, 1)
    if key in ("qam16", "16qam"):
        return _build("qam16", 2)
    raise ValueError(f"unknown constellation {name!r}")


def make_constellation_ext(name):
    """make_constellation plus the 64-QAM build extension (TS 38.211 levels / sqrt42)."""
    key = name.lower().replace("-", "").replace("_", "")
    if key in ("qam64", "64qam"):
        return _build("qam64", 3)
    return make_constellation(name)


def modulate(bits, const, cfg):
    """TX-side bit mapping (grid.py:157-169); off the receive path."""
    bits = np.asarray(bits, dtype=np.int64).ravel()
    b = const.bits_per_symbol
    if bits.size != b * cfg.size:
        raise ValueError(f"need {b * cfg.size} bits for a ({cfg.M},{cfg.N}) {const.name} frame, got {bits.size}")
    labels = bits.reshape(-1, b) @ (1 << np.arange(b - 1, -1, -1))
    return unflatten(const.points[labels], cfg)


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("hard_demod runs on the CUDA device only (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def demod_labels(v: np.ndarray, points: np.ndarray) -> np.ndarray:
    """Nearest-point labels of a complex vector on the device (ddb_hard_demod)."""
    dev = _device()
    xv = torch.as_tensor(np.ascontiguousarray(v, dtype=np.complex128), device=dev)
    pts = torch.as_tensor(np.ascontiguousarray(points, dtype=np.complex128), device=dev)
    lab = torch.empty(xv.numel(), dtype=torch.int32, device=dev)
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    nat.check(nat.load().ddb_hard_demod(xv.numel(), nat.DDB_F64, C.c_void_p(xv.data_ptr()),
                                        C.c_void_p(pts.data_ptr()), pts.numel(),
                                        C.c_void_p(lab.data_ptr()), stream), "ddb_hard_demod")
    return lab.cpu().numpy().astype(np.int64)


def hard_demod(x_hat, const, cfg):
    """Nearest-point hard decisions, lowest label on ties (grid.py:172-183).

    Returns (symbol frame, int64 bits in flattened-index order, MSB first).
    """
    x_hat = check_frame(x_hat, cfg)
    labels = demod_labels(flatten(x_hat, cfg), const.points)
    symbols = unflatten(np.asarray(const.points)[labels], cfg)
    bits = np.asarray(const.bit_map)[labels].reshape(-1).astype(np.int64)
    return symbols, bits


def ber(tx_bits, rx_bits):
    """Bit error rate (grid.py:186-194)."""
    tx = np.asarray(tx_bits).ravel()
    rx = np.asarray(rx_bits).ravel()
    if tx.size != rx.size:
        raise ValueError(f"bit sequences differ in length: {tx.size} vs {rx.size}")
    if tx.size == 0:
        raise ValueError("empty bit sequences")
    return float(np.count_nonzero(tx != rx)) / tx.size
