"""Dense LMMSE baseline on the device — small grids.

Drop-ins for the reference's dense branch (run_packet with
equalizer="lmmse", harness.py:160-168, 191-192):

  threshold_frame   -> ddb_threshold_frame   (sparse.py:163-169)
  build_dense_hdd   -> ddb_build_dense_hdd   (sparse.py:172-206), MN <= 4096
  lmmse_equalize    -> Gram + Cholesky solve (equalize.py:80-94) with cuBLAS /
                       cuSOLVER through torch (a library factorisation is what
                       the survey asks for on this cross-check path)

plus `receive_lmmse`, the whole dense receiver for a packet batch, used to
reproduce the reference's acceptance criterion 6 (iterative vs dense BER).
"""

from __future__ import annotations

import ctypes as C
import math
from typing import Optional

import numpy as np
import torch

from . import _native as nat
from .grid import check_frame
from .sparse import DENSE_GUARD, _dev, _p, _stream


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.complex128:
        return nat.DDB_F64
    if t.dtype == torch.complex64:
        return nat.DDB_F32
    raise ValueError("complex64 or complex128 expected")


def threshold_frame_device(heff: torch.Tensor, theta: float) -> torch.Tensor:
    """heff [B, M, N] -> bins with |h| <= theta * peak zeroed (per frame)."""
    if heff.dim() != 3:
        raise ValueError("heff must be [B, M, N]")
    heff = heff.contiguous()
    out = torch.empty_like(heff)
    B, M, N = heff.shape
    nat.check(nat.load().ddb_threshold_frame(B, M, N, _dt(heff), _p(heff), float(theta), _p(out), _stream()),
              "ddb_threshold_frame")
    return out


def build_dense_device(heff: torch.Tensor) -> torch.Tensor:
    """heff [B, M, N] -> H [B, MN, MN] (sparse.py:172-206)."""
    if heff.dim() != 3:
        raise ValueError("heff must be [B, M, N]")
    B, M, N = heff.shape
    if M * N > DENSE_GUARD:
        raise ValueError(f"dense channel matrix limited to MN <= {DENSE_GUARD}, got {M * N}")
    heff = heff.contiguous()
    H = torch.empty(B, M * N, M * N, dtype=heff.dtype, device=heff.device)
    nat.check(nat.load().ddb_build_dense_hdd(B, M, N, _dt(heff), _p(heff), _p(H), _stream()), "ddb_build_dense_hdd")
    return H


def lmmse_device(H: torch.Tensor, y: torch.Tensor, lam: torch.Tensor) -> torch.Tensor:
    """x = (H^H H + lam I)^{-1} H^H y per frame: H [B, MN, MN], y [B, MN], lam [B]."""
    Hh = H.conj().transpose(1, 2)
    gram = Hh @ H
    gram.diagonal(dim1=1, dim2=2).add_(lam.to(gram.real.dtype)[:, None])
    rhs = Hh @ y.unsqueeze(-1)
    L = torch.linalg.cholesky(gram)
    return torch.cholesky_solve(rhs, L).squeeze(-1)


# ---------------------------------------------------------------- drop-ins (numpy in / out)
def threshold_frame(heff, theta, cfg):
    """sparse.py:163-169 on the device."""
    heff = check_frame(heff, cfg)
    t = torch.as_tensor(np.ascontiguousarray(heff, dtype=np.complex128), device=_dev())[None]
    out = threshold_frame_device(t, theta)
    torch.cuda.current_stream().synchronize()
    return out[0].cpu().numpy()


def build_dense_hdd(heff, cfg, row_block=512):
    """sparse.py:172-206 on the device (row_block is accepted for signature parity)."""
    heff = check_frame(heff, cfg)
    if cfg.size > DENSE_GUARD:
        raise ValueError(f"dense channel matrix limited to MN <= {DENSE_GUARD}, got {cfg.size}")
    t = torch.as_tensor(np.ascontiguousarray(heff, dtype=np.complex128), device=_dev())[None]
    H = build_dense_device(t)
    torch.cuda.current_stream().synchronize()
    return H[0].cpu().numpy()


def lmmse_equalize(h_dense, y_dd, snr_linear):
    """equalize.py:80-94: the same errors, the Cholesky solve on the device."""
    h_dense = np.asarray(h_dense)
    y_dd = np.asarray(y_dd)
    mn = y_dd.size
    if h_dense.shape != (mn, mn):
        raise ValueError(f"matrix shape {h_dense.shape} does not match y ({mn})")
    if snr_linear <= 0:
        raise ValueError("snr_linear must be positive")
    lam = 0.0 if np.isinf(snr_linear) else 1.0 / snr_linear
    dev = _dev()
    H = torch.as_tensor(np.ascontiguousarray(h_dense, dtype=np.complex128), device=dev)[None]
    y = torch.as_tensor(np.ascontiguousarray(y_dd, dtype=np.complex128), device=dev)[None]
    x = lmmse_device(H, y, torch.tensor([lam], dtype=torch.float64, device=dev))
    return x[0].cpu().numpy()


# ---------------------------------------------------------------- batched dense receiver
def receive_lmmse(solver, pilot_rx: torch.Tensor, data_rx: torch.Tensor, snr_db: float, theta: float = 0.08,
                  tx_labels: Optional[torch.Tensor] = None, max_frames_per_chunk: Optional[int] = None) -> dict:
    """run_packet's dense branch (harness.py:156-168, 184-198) for a batch, in
    fp64: pilot DZT + estimate, detect_paths (only to flag EmptyChannel, as
    run_packet does), threshold_frame -> build_dense_hdd -> lmmse_equalize,
    data DZT, hard decisions and bit errors.  Frames with no taps score
    bits / 2 errors (harness.py:170-178).  Returns labels [B, MN], bit_errors
    [B] (if tx_labels), failed [B]."""
    from .zak import dzt_device
    M, N, MN = solver.M, solver.N, solver.MN
    if MN > DENSE_GUARD:
        raise ValueError(f"dense channel matrix limited to MN <= {DENSE_GUARD}, got {MN}")
    dev = solver.device
    B = pilot_rx.shape[0]
    bps = solver.bps
    amp = float(np.sqrt(MN))
    heff = dzt_device(pilot_rx.to(device=dev), M, N, colmajor=False, pilot_amplitude=amp, fp64=True)
    heff = heff.view(B, M, N)
    peak_cnt = torch.empty(B, dtype=torch.int32, device=dev)
    nat.check(nat.load().ddb_detect_paths(B, M, N, _p(heff), float(theta), 0, _p(peak_cnt), None, None, None,
                                          _stream()), "ddb_detect_paths")
    failed = peak_cnt == 0
    y = dzt_device(data_rx.to(device=dev, dtype=torch.complex128), M, N, colmajor=True)
    snr_lin = 10.0 ** (snr_db / 10.0)
    lam = torch.full((B,), 0.0 if math.isinf(snr_lin) else 1.0 / snr_lin, dtype=torch.float64, device=dev)
    chunk = max_frames_per_chunk or max(1, int(2 ** 32 // (MN * MN * 16)))
    x = torch.empty(B, MN, dtype=torch.complex128, device=dev)
    for c0 in range(0, B, chunk):
        c1 = min(B, c0 + chunk)
        H = build_dense_device(threshold_frame_device(heff[c0:c1], theta))
        x[c0:c1] = lmmse_device(H, y[c0:c1], lam[c0:c1])
        del H
    labels = torch.empty(B, MN, dtype=torch.uint8, device=dev)
    nat.check(nat.load().ddb_qam_demod(B * MN, nat.DDB_F64, _p(x), bps, 1.0, _p(labels), None, _stream()),
              "ddb_qam_demod")
    out = {"x": x, "labels": labels, "failed": failed}
    if tx_labels is not None:
        diff = (labels ^ tx_labels.to(device=dev, dtype=torch.uint8)).to(torch.int32)
        bits = torch.zeros_like(diff)
        for b in range(bps):
            bits += (diff >> b) & 1
        errs = bits.sum(dim=1).to(torch.int64)
        out["bit_errors"] = torch.where(failed, torch.full_like(errs, bps * MN // 2), errs)
    return out
