"""Discrete Zak transform — drop-in for ddlink.zak's receive-side GEMM.

Same names, signatures, layouts and errors as
/root/reference/pkg/src/ddlink/zak.py.  The transform itself runs in the ddb
CUDA library:

  dzt_gemm           -> ddb_dzt            (zak.py:50-55; honours any N x N kernel)
  build_zak_kernel   -> the constant table of zak.py:33-47 (host setup, as the
                        reference builds it once per Workspace, harness.py:125)

The transmit-side `idzt` / defining-sum `dzt` are channel simulation, outside
the hot path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .grid import check_signal
from .sparse import _dev, _p, _stream


def build_zak_kernel(N, half_shift=False):
    """N x N transform kernel: kernel[i, l] = (1/sqrt(N)) e^{-j2pi i l/N} (zak.py:33-47)."""
    if N < 1:
        raise ValueError("N must be positive")
    n = np.arange(N)
    kernel = np.exp(-2j * np.pi * np.outer(n, n) / N) / np.sqrt(N)
    if half_shift:
        kernel = kernel * np.where(n % 2, -1.0, 1.0)[None, :]
    kernel.setflags(write=False)
    return kernel


def dzt_device(y_time: torch.Tensor, M: int, N: int, *, kernel: torch.Tensor | None = None,
               colmajor: bool = True, pilot_amplitude: float | None = None, out: torch.Tensor | None = None,
               stream: torch.cuda.Stream | None = None, fp64: bool = False) -> torch.Tensor:
    """Batched Zak transform of received frames on the device.

    y_time: complex64/complex128 [B, M*N] (time index k + i*M).  Returns [B, M*N]
    of the same dtype (complex128 with fp64=True): flattened q = l*M + k when
    colmajor (the solver's input layout), else the (M, N) frame row-major
    (dzt_gemm's).  With pilot_amplitude the point-pilot estimate of
    pilot.py:40-49 is fused in.
    """
    if y_time.dim() != 2 or y_time.shape[1] != M * N:
        raise ValueError(f"y_time must be [B, {M * N}], got {tuple(y_time.shape)}")
    if y_time.dtype not in (torch.complex64, torch.complex128):
        raise ValueError("y_time must be complex64 or complex128")
    y_time = y_time.contiguous()
    # fp64 on complex64 samples without a widening pass (default kernel, power-of-two N)
    mixed = fp64 and y_time.dtype == torch.complex64 and kernel is None and N >= 2 and N & (N - 1) == 0
    if fp64 and y_time.dtype == torch.complex64 and not mixed:
        y_time = y_time.to(torch.complex128)
    dtype = nat.DDB_F64 if (mixed or y_time.dtype == torch.complex128) else nat.DDB_F32
    if out is None:
        out = torch.empty(y_time.shape, dtype=torch.complex128 if dtype == nat.DDB_F64 else torch.complex64,
                          device=y_time.device)
    kptr = None
    if kernel is not None:
        kernel = kernel.to(device=y_time.device, dtype=y_time.dtype).contiguous()
        if kernel.shape != (N, N):
            raise ValueError(f"kernel shape {tuple(kernel.shape)} does not match N={N}")
        kptr = _p(kernel)
    flags = ((nat.DDB_DZT_COLMAJOR if colmajor else 0) | (nat.DDB_DZT_PILOT if pilot_amplitude is not None else 0)
             | (nat.DDB_DZT_INPUT_F32 if mixed else 0))
    st = stream.cuda_stream if stream is not None else torch.cuda.current_stream(y_time.device).cuda_stream
    import ctypes as C
    nat.check(nat.load().ddb_dzt(int(y_time.shape[0]), M, N, dtype, _p(y_time), kptr, flags,
                                 float(pilot_amplitude or 1.0), _p(out), C.c_void_p(st)), "ddb_dzt")
    return out


def dzt_gemm(y, kernel, cfg):
    """DZT as one GEMM: reshape y column-major to (M, N), multiply by the kernel (zak.py:50-55)."""
    y = check_signal(y, cfg)
    kernel = np.asarray(kernel)
    if kernel.shape != (cfg.N, cfg.N):
        raise ValueError(f"kernel shape {kernel.shape} does not match N={cfg.N}")
    _dev()
    # one host round trip (ddb_host_dzt: copy in, the GEMM-form kernel, copy out)
    yh = np.ascontiguousarray(y, dtype=np.complex128)
    kh = np.ascontiguousarray(kernel, dtype=np.complex128)
    out = np.empty((cfg.M, cfg.N), dtype=np.complex128)
    nat.check(nat.load().ddb_host_dzt(cfg.M, cfg.N, yh.ctypes.data, kh.ctypes.data, out.ctypes.data),
              "ddb_host_dzt")
    return out
