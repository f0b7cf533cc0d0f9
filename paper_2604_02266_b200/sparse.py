"""Structured-sparse DD channel operator — drop-in for ddlink.sparse.

Same names, signatures, array layouts (complex128 / int32 tables of shape
(P, MN)) and errors as /root/reference/pkg/src/ddlink/sparse.py.  Every
numeric step runs in the ddb CUDA library:

  detect_paths      -> ddb_detect_paths   (sparse.py:69-88)
  build_ss_channel  -> ddb_build_tables   (sparse.py:124-144)
  forward_index / inverse_index / coefficient
                    -> ddb_build_tables for the single tap (sparse.py:91-121)
  ss_mvm / ss_mvm_hermitian
                    -> ddb_ss_mvm_tables  (sparse.py:147-160), honouring
                       arbitrary (e.g. perturbed) tables
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .grid import check_frame

DENSE_GUARD = 4096


class EmptyChannel(Exception):
    """No taps survived thresholding; there is no channel to equalize against."""


@dataclass(frozen=True)
class DominantPath:
    """One detected tap on the absolute grid (sparse.py:27-37)."""

    k_p: int
    l_p: int
    gain: complex

    def offsets(self, cfg):
        return cfg.K0 - self.k_p, cfg.L0 - self.l_p


@dataclass(frozen=True)
class StructuredSparseChannel:
    """Path-major tables for both product directions (sparse.py:40-66)."""

    M: int
    N: int
    paths: tuple
    fwd_coef: np.ndarray
    fwd_col: np.ndarray
    herm_coef: np.ndarray
    herm_row: np.ndarray
    # set by build_ss_channel only: the tables are the closed form of `paths`,
    # so the fused solve may regenerate them on the fly.  dataclasses.replace
    # (e.g. oracle_check's perturbed fwd_coef, harness.py:368-369) resets it.
    canonical: bool = field(default=False, init=False, repr=False, compare=False)

    @property
    def P(self):
        return len(self.paths)

    @property
    def size(self):
        return self.M * self.N

    def entries_per_direction(self):
        return int(self.fwd_coef.size)


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("the structured-sparse operator runs on the CUDA device only (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t):
    return C.c_void_p(t.data_ptr())


def _device_tables(paths, M: int, N: int):
    dev = _dev()
    P = len(paths)
    k = torch.tensor([int(p.k_p) for p in paths], dtype=torch.int32, device=dev)
    l = torch.tensor([int(p.l_p) for p in paths], dtype=torch.int32, device=dev)
    g = torch.tensor(np.array([complex(p.gain) for p in paths], np.complex128), device=dev)
    MN = M * N
    fc = torch.empty(P, MN, dtype=torch.complex128, device=dev)
    fi = torch.empty(P, MN, dtype=torch.int32, device=dev)
    hc = torch.empty(P, MN, dtype=torch.complex128, device=dev)
    hi = torch.empty(P, MN, dtype=torch.int32, device=dev)
    nat.check(nat.load().ddb_build_tables(M, N, P, _p(k), _p(l), _p(g), _p(fc), _p(fi), _p(hc), _p(hi),
                                          _stream()), "ddb_build_tables")
    return fc, fi, hc, hi


def _single_tap_tables(path, cfg):
    fc, fi, hc, hi = _device_tables([path], cfg.M, cfg.N)
    return fc[0].cpu().numpy(), fi[0].cpu().numpy(), hi[0].cpu().numpy()


def _index(table: np.ndarray, q):
    qa = np.asarray(q)
    out = table[qa]
    if qa.ndim == 0:
        return int(out)
    return out.astype(np.int64)


def forward_index(path, q, cfg):
    """Column feeding output q: 2D circular shift of q (sparse.py:91-96)."""
    _, fi, _ = _single_tap_tables(path, cfg)
    return _index(fi, q)


def inverse_index(path, r, cfg):
    """Output fed by column r (sparse.py:99-104)."""
    _, _, hi = _single_tap_tables(path, cfg)
    return _index(hi, r)


def coefficient(path, q, cfg):
    """Phase-corrected gain multiplying v[forward_index(path, q)] in row q (sparse.py:107-121)."""
    fc, _, _ = _single_tap_tables(path, cfg)
    qa = np.asarray(q)
    out = fc[qa]
    return complex(out) if qa.ndim == 0 else out


_TABLES = ("fwd_coef", "fwd_col", "herm_coef", "herm_row")


class _LazyTablesChannel(StructuredSparseChannel):
    """A StructuredSparseChannel whose four (P, MN) tables are generated on
    the device (ddb_build_tables) the first time one is read.  The fused solve
    needs only M, N and the paths (it regenerates the coefficients on the
    fly), so a receiver that never looks at the tables (run_packet,
    harness.py:163-190) pays nothing for them; any reader (ss_mvm, the
    reference's table tests, dataclasses.replace) sees the same arrays
    build_ss_channel used to return eagerly."""

    def __getattribute__(self, name):
        if name in _TABLES and object.__getattribute__(self, name) is None:
            fc, fi, hc, hi = _device_tables(object.__getattribute__(self, "paths"),
                                            object.__getattribute__(self, "M"), object.__getattribute__(self, "N"))
            for key, t in zip(_TABLES, (fc, fi, hc, hi)):
                object.__setattr__(self, key, t.cpu().numpy())
        return object.__getattribute__(self, name)


def build_ss_channel(paths, cfg):
    """Forward and Hermitian tables for the detected taps (sparse.py:124-144);
    the tables are materialised on first access."""
    if len(paths) == 0:
        raise EmptyChannel("no taps above threshold")
    ch = _LazyTablesChannel(M=cfg.M, N=cfg.N, paths=tuple(paths),
                            fwd_coef=None, fwd_col=None, herm_coef=None, herm_row=None)
    object.__setattr__(ch, "canonical", True)
    return ch


def _checked_tables(coef, index, size):
    """The reference's einsum("pq,pq->q", coef, v[index]) semantics on the host
    side of the boundary: matching (P, size) shapes (ValueError otherwise),
    numpy's negative-index wrap and IndexError outside [-size, size)."""
    c = np.asarray(coef)
    i = np.asarray(index)
    if c.ndim != 2 or i.shape != c.shape or c.shape[1] != size:
        raise ValueError(f"table shapes {c.shape} / {i.shape} do not match (P, {size})")
    if not np.issubdtype(i.dtype, np.integer):
        raise IndexError("arrays used as indices must be of integer type")
    if i.size and (i.min() < -size or i.max() >= size):
        bad = int(i.max()) if i.max() >= size else int(i.min())
        raise IndexError(f"index {bad} is out of bounds for axis 0 with size {size}")
    if i.size and i.min() < 0:
        i = np.where(i < 0, i + size, i)
    return c, i


def _mvm_tables(coef, index, v, size):
    dev = _dev()
    v = np.asarray(v)
    if v.shape != (size,):
        raise ValueError(f"vector length {v.shape} != {size}")
    coef, index = _checked_tables(coef, index, size)
    c = torch.as_tensor(np.ascontiguousarray(coef, dtype=np.complex128), device=dev)
    i = torch.as_tensor(np.ascontiguousarray(index, dtype=np.int32), device=dev)
    vv = torch.as_tensor(np.ascontiguousarray(v, dtype=np.complex128), device=dev)
    u = torch.empty(size, dtype=torch.complex128, device=dev)
    P = int(c.shape[0]) if c.dim() == 2 else 0
    nat.check(nat.load().ddb_ss_mvm_tables(size, P, _p(c), _p(i), _p(vv), _p(u), _stream()),
              "ddb_ss_mvm_tables")
    return u.cpu().numpy()


def ss_mvm(ch, v):
    """u[q] = sum_p fwd_coef[p, q] * v[fwd_col[p, q]] (sparse.py:147-152)."""
    return _mvm_tables(ch.fwd_coef, ch.fwd_col, v, ch.M * ch.N)


def ss_mvm_hermitian(ch, v):
    """u[r] = sum_p herm_coef[p, r] * v[herm_row[p, r]] (sparse.py:155-160)."""
    return _mvm_tables(ch.herm_coef, ch.herm_row, v, ch.M * ch.N)


def detect_paths(heff, theta, cfg):
    """Keep |h| > theta*max|h|, sorted by descending magnitude, stable (sparse.py:69-88)."""
    heff = check_frame(heff, cfg)
    if theta < 0:
        raise ValueError("theta must be nonnegative")
    _dev()
    M, N = cfg.M, cfg.N
    # one host round trip (ddb_host_detect_paths): every candidate, ranked
    h = np.ascontiguousarray(heff, dtype=np.complex128)
    cap = M * N
    cnt = np.zeros(1, dtype=np.int32)
    kk = np.empty(cap, dtype=np.int32)
    ll = np.empty(cap, dtype=np.int32)
    gg = np.empty(cap, dtype=np.complex128)
    nat.check(nat.load().ddb_host_detect_paths(M, N, h.ctypes.data, float(theta), cap, cnt.ctypes.data,
                                               kk.ctypes.data, ll.ctypes.data, gg.ctypes.data), "ddb_host_detect_paths")
    n = int(cnt[0])
    return [DominantPath(int(a), int(b), complex(c)) for a, b, c in zip(kk[:n], ll[:n], gg[:n])]
