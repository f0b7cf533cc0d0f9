"""Batched device API of the SS-CGA equalizer.

`SsCgaSolver` runs the fused sm_100a kernel (ddb_sscga_solve) over a batch
of independent frames that share one grid: y [B, M*N] complex on the GPU,
per-frame taps as CSR (`PathBatch`), per-frame ridge lam [B].  It mirrors
cga_equalize (equalize.py:43-77) frame by frame and fuses the hard demod
(grid.py:172-183), the bit-error count (harness.py:198) and max-log LLRs.

PyTorch is used only for device memory and streams; all arithmetic happens in
libddb.so.  `HostPipeline` is the end-to-end entry point for host buffers:
chunked pinned-memory H2D, solve and D2H overlapped on separate streams.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native as nat

_BPS = {"qpsk": 2, "qam16": 4, "16qam": 4, "qam64": 6, "64qam": 6}


def bits_per_symbol(modulation) -> int:
    if modulation is None:
        return 0
    if isinstance(modulation, int):
        if modulation not in (0, 2, 4, 6):
            raise ValueError(f"bits_per_symbol must be 0, 2, 4 or 6, got {modulation}")
        return modulation
    if hasattr(modulation, "bits_per_symbol"):
        return int(modulation.bits_per_symbol)
    key = str(modulation).lower().replace("-", "").replace("_", "")
    if key not in _BPS:
        raise ValueError(f"unknown modulation {modulation!r}")
    return _BPS[key]


def _precision(precision: str):
    if precision in ("fp32", "float32", "single"):
        return nat.DDB_F32, torch.float32, torch.complex64
    if precision in ("fp64", "float64", "double"):
        return nat.DDB_F64, torch.float64, torch.complex128
    raise ValueError(f"precision must be 'fp32' or 'fp64', got {precision!r}")


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream_handle(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the SS-CGA equalizer runs only on a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass
class PathBatch:
    """Per-frame taps as CSR on the device: frame b owns [offsets[b], offsets[b+1])."""

    offsets: torch.Tensor  # int32 [B+1]
    k: torch.Tensor        # int32 [T] absolute delay index k_p
    l: torch.Tensor        # int32 [T] absolute Doppler index l_p
    gain: torch.Tensor     # complex [T]

    @property
    def batch(self) -> int:
        return self.offsets.numel() - 1

    @classmethod
    def from_arrays(cls, offsets, k, l, gain, device=None, cdtype=torch.complex64) -> "PathBatch":
        device = device or default_device()
        off = torch.as_tensor(np.asarray(offsets), dtype=torch.int32).to(device)
        kk = torch.as_tensor(np.asarray(k), dtype=torch.int32).to(device)
        ll = torch.as_tensor(np.asarray(l), dtype=torch.int32).to(device)
        gg = torch.as_tensor(np.asarray(gain, dtype=np.complex128)).to(cdtype).to(device)
        return cls(off, kk, ll, gg)

    @classmethod
    def from_taps(cls, taps_per_frame: Sequence[Sequence], device=None,
                  cdtype=torch.complex64) -> "PathBatch":
        """Each tap needs .k_p, .l_p, .gain (DominantPath, sparse.py:27-37)."""
        off = [0]
        k, l, g = [], [], []
        for taps in taps_per_frame:
            for t in taps:
                k.append(int(t.k_p))
                l.append(int(t.l_p))
                g.append(complex(t.gain))
            off.append(len(k))
        if not k:  # keep valid (non-null) device pointers for all-empty batches
            k, l, g = [0], [0], [0j]
        return cls.from_arrays(off, k, l, g, device, cdtype)

    def to(self, cdtype) -> "PathBatch":
        return PathBatch(self.offsets, self.k, self.l, self.gain.to(cdtype))

    def validate(self, M: int, N: int) -> None:
        """Host-side range checks (one device sync; not for the timed path)."""
        if self.offsets.numel() < 1:
            raise ValueError("offsets must have B+1 entries")
        off = self.offsets.cpu()
        if int(off[0]) != 0 or bool((off[1:] < off[:-1]).any()):
            raise ValueError("path offsets must start at 0 and be non-decreasing")
        n = int(off[-1])
        if n > self.k.numel() or n > self.l.numel() or n > self.gain.numel():
            raise ValueError("path arrays shorter than offsets[-1]")
        if n:
            kk, ll = self.k[:n].cpu(), self.l[:n].cpu()
            if bool(((kk < 0) | (kk >= M)).any()) or bool(((ll < 0) | (ll >= N)).any()):
                raise ValueError("tap indices outside the grid")


@dataclass
class SolveResult:
    x: torch.Tensor                          # [B, MN] complex
    c_norm: Optional[torch.Tensor] = None    # [B, iters+1] real
    iterations_done: Optional[torch.Tensor] = None  # int32 [B]
    status: Optional[torch.Tensor] = None    # uint8 [B] (FRAME_* bits)
    labels: Optional[torch.Tensor] = None    # uint8 [B, MN]
    llr: Optional[torch.Tensor] = None       # float32 [B, MN, bps]
    bit_errors: Optional[torch.Tensor] = None  # int32 [B]
    snapshots: Optional[torch.Tensor] = None   # [B, iters, MN] complex


class SsCgaSolver:
    """Fixed-grid batched SS-CGA equalizer (matrix-free, fused CG + demod)."""

    def __init__(self, M: int, N: int, iterations: int = 10, precision: str = "fp32",
                 modulation=None, device=None):
        if M < 2 or N < 2 or M % 2 or N % 2:
            raise ValueError(f"M and N must be even and >= 2, got ({M},{N})")
        if iterations < 1:
            raise ValueError("need at least one iteration")
        self.M, self.N, self.MN = int(M), int(N), int(M) * int(N)
        self.iterations = int(iterations)
        self.dtype_code, self.rdtype, self.cdtype = _precision(precision)
        self.precision = "fp64" if self.dtype_code == nat.DDB_F64 else "fp32"
        self.bps = bits_per_symbol(modulation)
        self.device = torch.device(device) if device is not None else default_device()
        self.lib = nat.load()
        self._plan = nat.plan(self.M, self.N, self.dtype_code)

    # -- introspection -----------------------------------------------------
    def plan(self) -> dict:
        p = self._plan
        return {"cluster": p.cluster, "cols_per_cta": p.cols_per_cta,
                "cols_per_thread": p.cols_per_thread, "threads": p.threads,
                "smem_bytes": p.smem_bytes, "ctas_per_sm": p.ctas_per_sm, "halo_rows": p.halo_rows,
                "kernel": {0: "rows", 1: "tmem", 2: "workspace"}[p.kernel], "rows_per_thread": p.rows_per_thread}

    # -- buffers -------------------------------------------------------------
    def alloc(self, B: int, *, llr: bool = False, labels: bool = True, trace: bool = True,
              bit_errors: bool = False, profile: bool = False) -> SolveResult:
        dev = self.device
        r = SolveResult(x=torch.empty(B, self.MN, dtype=self.cdtype, device=dev))
        if trace:
            r.c_norm = torch.empty(B, self.iterations + 1, dtype=self.rdtype, device=dev)
            r.iterations_done = torch.empty(B, dtype=torch.int32, device=dev)
            r.status = torch.empty(B, dtype=torch.uint8, device=dev)
        if self.bps and labels:
            r.labels = torch.empty(B, self.MN, dtype=torch.uint8, device=dev)
        if self.bps and llr:
            r.llr = torch.empty(B, self.MN, self.bps, dtype=torch.float32, device=dev)
        if self.bps and bit_errors:
            r.bit_errors = torch.empty(B, dtype=torch.int32, device=dev)
        if profile:
            r.snapshots = torch.empty(B, self.iterations, self.MN, dtype=self.cdtype, device=dev)
        return r

    def _problem(self, y: torch.Tensor, paths: PathBatch, lam: torch.Tensor) -> nat.Problem:
        B = y.shape[0]
        return nat.Problem(B, self.M, self.N, self.iterations, self.dtype_code,
                           _ptr(paths.offsets), _ptr(paths.k), _ptr(paths.l), _ptr(paths.gain),
                           _ptr(y), _ptr(lam))

    def _check_inputs(self, y, paths, lam):
        if not isinstance(y, torch.Tensor) or y.device.type != "cuda":
            raise ValueError("y must be a CUDA tensor")
        if y.dim() != 2 or y.shape[1] != self.MN:
            raise ValueError(f"y must be [B, {self.MN}], got {tuple(y.shape)}")
        if y.dtype != self.cdtype or not y.is_contiguous():
            raise ValueError(f"y must be contiguous {self.cdtype}")
        B = y.shape[0]
        if paths.batch != B:
            raise ValueError(f"paths describe {paths.batch} frames, y has {B}")
        if paths.gain.dtype != self.cdtype:
            raise ValueError(f"path gains must be {self.cdtype}")
        if lam.shape != (B,) or lam.dtype != self.rdtype or lam.device != y.device:
            raise ValueError(f"lam must be a [{B}] {self.rdtype} tensor on {y.device}")

    def lam_tensor(self, lam, B: int) -> torch.Tensor:
        if isinstance(lam, torch.Tensor):
            return lam.to(device=self.device, dtype=self.rdtype).reshape(B)
        arr = np.broadcast_to(np.asarray(lam, dtype=np.float64), (B,))
        if (arr < 0).any():
            raise ValueError("lam must be nonnegative")
        return torch.as_tensor(arr.copy(), dtype=self.rdtype, device=self.device)

    # -- the fused solve -----------------------------------------------------
    def solve(self, y: torch.Tensor, paths: PathBatch, lam, *, tx_labels: Optional[torch.Tensor] = None,
              noise_var: Optional[torch.Tensor] = None, out: Optional[SolveResult] = None,
              llr: bool = False, trace: bool = True, profile: bool = False,
              stream: Optional[torch.cuda.Stream] = None,
              phase_cycles: Optional[torch.Tensor] = None) -> SolveResult:
        """phase_cycles (measurement only): zeroed int64 CUDA tensor [4736, 12] that
        receives per-CTA clock64 phase totals (ddb_sscga_profile_phases)."""
        B = y.shape[0]
        lam = self.lam_tensor(lam, B)
        self._check_inputs(y, paths, lam)
        if out is None:
            out = self.alloc(B, llr=llr, trace=trace, bit_errors=tx_labels is not None, profile=profile)
        packed = 0
        if tx_labels is not None:
            packed = int(self.bps in (2, 4) and tuple(tx_labels.shape) == (B, self.MN * self.bps // 8))
            if (not packed and tuple(tx_labels.shape) != (B, self.MN)) or tx_labels.dtype != torch.uint8:
                raise ValueError(f"tx_labels must be uint8 [{B}, {self.MN}] (or packed by pack_labels)")
            if out.bit_errors is None:
                out.bit_errors = torch.empty(B, dtype=torch.int32, device=self.device)
        if noise_var is not None:
            noise_var = noise_var.to(device=self.device, dtype=self.rdtype).reshape(B)
        prob = self._problem(y, paths, lam)
        outs = nat.Outputs(
            _ptr(out.x), _ptr(out.c_norm), _ptr(out.iterations_done), _ptr(out.status),
            _ptr(out.snapshots), self.bps if (out.labels is not None or out.llr is not None
                                              or tx_labels is not None) else 0,
            _ptr(out.labels), _ptr(out.llr), _ptr(noise_var), _ptr(tx_labels),
            _ptr(out.bit_errors if tx_labels is not None else None), packed)
        if phase_cycles is not None:
            nat.check(self.lib.ddb_sscga_profile_phases(C.byref(prob), C.byref(outs), _ptr(phase_cycles),
                                                        _stream_handle(stream)), "ddb_sscga_profile_phases")
        else:
            ws_bytes = int(self.lib.ddb_sscga_workspace_bytes(C.byref(prob)))
            ws = self._workspace(ws_bytes, stream)
            nat.check(self.lib.ddb_sscga_solve(C.byref(prob), C.byref(outs), _ptr(ws), ws_bytes,
                                               _stream_handle(stream)), "ddb_sscga_solve")
        return out

    def _workspace(self, nbytes: int, stream: Optional[torch.cuda.Stream] = None) -> Optional[torch.Tensor]:
        """Device workspace of the workspace-backed path (grown, never shrunk).

        One buffer per launch stream: two solves on different streams never
        share c / u / p.  The buffer is allocated with that stream current, so
        the caching allocator orders its reuse after the stream's pending
        kernels when it is regrown (the old block is freed on the same stream)."""
        if nbytes == 0:
            return None
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        pool = self.__dict__.setdefault("_ws", {})
        ws = pool.get(s.cuda_stream)
        if ws is None or ws.numel() < nbytes:
            with torch.cuda.stream(s):
                ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            pool[s.cuda_stream] = ws
        return ws

    # -- receiver front end ---------------------------
    def detect(self, pilot_rx: torch.Tensor, theta: float = 0.08, *, max_paths: int = 64,
               amplitude: Optional[float] = None, stream=None, _deferred: Optional[list] = None) -> PathBatch:
        """Taps of every frame from its received pilot frame, on the device.

        pilot_rx: complex [B, M*N] time-domain samples of the point-pilot frame.
        Zak transform fused with the pilot estimate (dzt_gemm + estimate_heff,
        zak.py:50-55, pilot.py:40-49) in fp64, then detect_paths
        (sparse.py:69-88); the result is the solver's CSR tap batch.  A frame
        with more than max_paths taps raises (truncation would change the
        operator); theta < 0 raises as in the reference.
        """
        from .zak import dzt_device
        if theta < 0:
            raise ValueError("theta must be nonnegative")
        B = pilot_rx.shape[0]
        amp = float(np.sqrt(self.MN)) if amplitude is None else float(amplitude)
        heff = dzt_device(pilot_rx.to(device=self.device), self.M, self.N, colmajor=False, pilot_amplitude=amp,
                          stream=stream, fp64=True)
        cnt = torch.empty(B, dtype=torch.int32, device=self.device)
        kk = torch.empty(B, max_paths, dtype=torch.int32, device=self.device)
        ll = torch.empty(B, max_paths, dtype=torch.int32, device=self.device)
        gg = torch.empty(B, max_paths, dtype=torch.complex128, device=self.device)
        nat.check(self.lib.ddb_detect_paths(B, self.M, self.N, _ptr(heff), float(theta), max_paths, _ptr(cnt),
                                            _ptr(kk), _ptr(ll), _ptr(gg), _stream_handle(stream)),
                  "ddb_detect_paths")
        # CSR on the device (ddb_paths_csr); one 12-byte read checks and sizes the batch
        cap = max(1, B * max_paths)
        off = torch.empty(B + 1, dtype=torch.int32, device=self.device)
        k = torch.empty(cap, dtype=torch.int32, device=self.device)
        l = torch.empty(cap, dtype=torch.int32, device=self.device)
        g = torch.empty(cap, dtype=self.cdtype, device=self.device)
        stats = torch.empty(3, dtype=torch.int32, device=self.device)
        nat.check(self.lib.ddb_paths_csr(B, max_paths, _ptr(cnt), _ptr(kk), _ptr(ll), _ptr(gg), self.dtype_code,
                                         _ptr(off), _ptr(k), _ptr(l), _ptr(g), _ptr(stats), _stream_handle(stream)),
                  "ddb_paths_csr")
        if _deferred is not None:  # receive(): checked after the solve is queued (no mid-pipeline sync)
            _deferred.append((stats, max_paths))
            return PathBatch(off, k, l, g)
        if stream is not None:
            stream.synchronize()
        cmin, cmax, total = (int(v) for v in stats.tolist())
        if cmin < 0:
            raise nat.DdbError(nat.DDB_ERR_UNSUPPORTED, "ddb_detect_paths",
                               "candidate list exceeds the per-frame shared-memory capacity")
        if cmax > max_paths:
            raise ValueError(f"a frame has {cmax} taps above threshold > max_paths={max_paths}")
        n = max(total, 1)  # all frames empty: keep valid device pointers
        return PathBatch(off, k[:n], l[:n], g[:n])

    def receive(self, pilot_rx: torch.Tensor, data_rx: torch.Tensor, lam, theta: float = 0.08, *,
                max_paths: int = 64, tx_labels: Optional[torch.Tensor] = None, llr: bool = False,
                trace: bool = True, stream=None) -> SolveResult:
        """The whole receiver of run_packet (harness.py:156-194) on the device for a batch:
        pilot DZT + estimate + detect_paths -> taps; data DZT -> y_dd; fused SS-CGA
        solve with hard decisions (and LLRs / bit errors).  data_rx: complex
        [B, M*N] time-domain samples of the data frame."""
        from .zak import dzt_device
        pending: list = []
        paths = self.detect(pilot_rx, theta, max_paths=max_paths, stream=stream, _deferred=pending)
        y = dzt_device(data_rx.to(device=self.device, dtype=self.cdtype), self.M, self.N, colmajor=True,
                       stream=stream)
        res = self.solve(y, paths, lam, tx_labels=tx_labels, llr=llr, trace=trace, stream=stream)
        # the tap batch's checks, after everything is queued: one small read
        stats, mp = pending[0]
        if stream is not None:
            stream.synchronize()
        cmin, cmax, _ = (int(v) for v in stats.tolist())
        if cmin < 0:
            raise nat.DdbError(nat.DDB_ERR_UNSUPPORTED, "ddb_detect_paths",
                               "candidate list exceeds the per-frame shared-memory capacity")
        if cmax > mp:
            raise ValueError(f"a frame has {cmax} taps above threshold > max_paths={mp}")
        return res

    # -- matrix-free operator -------------------------------------------------
    def apply(self, v: torch.Tensor, paths: PathBatch, hermitian: bool = False,
              out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """H v or H^H v for every frame (ss_mvm / ss_mvm_hermitian, sparse.py:147-160)."""
        B = v.shape[0]
        if v.dim() != 2 or v.shape[1] != self.MN or v.dtype != self.cdtype or not v.is_contiguous():
            raise ValueError(f"v must be contiguous {self.cdtype} [B, {self.MN}]")
        if paths.batch != B:
            raise ValueError("paths/v batch mismatch")
        if out is None:
            out = torch.empty_like(v)
        dummy_lam = torch.empty(0, dtype=self.rdtype, device=self.device)
        prob = nat.Problem(B, self.M, self.N, self.iterations, self.dtype_code,
                           _ptr(paths.offsets), _ptr(paths.k), _ptr(paths.l), _ptr(paths.gain),
                           _ptr(v), _ptr(dummy_lam))
        nat.check(self.lib.ddb_ss_apply(C.byref(prob), _ptr(out), int(bool(hermitian)), _stream_handle(stream)),
                  "ddb_ss_apply")
        return out


def pack_labels(labels: torch.Tensor, bps: int) -> torch.Tensor:
    """[B, MN] uint8 labels -> [B, MN * bps / 8] bytes, bps bits per symbol LSB-first
    (QPSK 4 and 16-QAM 2 symbols per byte): the tx_labels_packed layout of
    include/ddb.h, which halves (16-QAM) the transmitted-label bytes an
    end-to-end run moves over PCIe."""
    if bps not in (2, 4):
        raise ValueError("packing needs 2 or 4 bits per symbol")
    per = 8 // bps
    B, MN = labels.shape
    if MN % per:
        raise ValueError("M*N must be a multiple of the symbols per byte")
    v = labels.reshape(B, MN // per, per).to(torch.int32)
    shifts = torch.arange(per, device=labels.device, dtype=torch.int32) * bps
    return (v << shifts).sum(dim=2).to(torch.uint8)


class HostPipeline:
    """End-to-end solve from host buffers (the call a user with numpy data makes).

    Frames are processed in chunks; chunk i+1's pinned H2D copy overlaps chunk
    i's solve and chunk i-1's D2H copy (three streams, events between them).
    Returns hard-decision labels on the host, and per-frame bit errors when
    the transmitted labels are given (tx_host; None: the equalizer alone, the
    work the reference's build_ss_channel -> cga_equalize -> hard_demod does).
    """

    def __init__(self, solver: SsCgaSolver, chunk: int = 512, depth: int = 2):
        self.s = solver
        self.chunk = int(chunk)
        self.depth = int(depth)
        dev = solver.device
        self.h2d = torch.cuda.Stream(dev)
        self.comp = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        MN = solver.MN
        self.slots = []
        for _ in range(depth):
            self.slots.append(dict(
                y=torch.empty(self.chunk, MN, dtype=solver.cdtype, device=dev),
                lam=torch.empty(self.chunk, dtype=solver.rdtype, device=dev),
                tx=None,  # allocated at the first run with the host labels' width (packed or not)
                res=solver.alloc(self.chunk, trace=False, bit_errors=True),
                loaded=torch.cuda.Event(), solved=torch.cuda.Event(), drained=torch.cuda.Event(),
            ))

    def run(self, y_host: torch.Tensor, paths_host: tuple, lam_host: torch.Tensor,
            tx_host: Optional[torch.Tensor], labels_host: torch.Tensor,
            errors_host: Optional[torch.Tensor] = None) -> None:
        """All host tensors must be pinned.  paths_host = (offsets, k, l, gain) host tensors."""
        s = self.s
        B = y_host.shape[0]
        off, kk, ll, gg = paths_host
        dev = s.device
        for slot in self.slots:  # TX labels one byte per symbol, or packed (pack_labels)
            if tx_host is not None and (slot["tx"] is None or slot["tx"].shape[1] != tx_host.shape[1]):
                torch.cuda.synchronize(dev)
                slot["tx"] = torch.empty(self.chunk, tx_host.shape[1], dtype=torch.uint8, device=dev)
        # taps are tiny: one copy for the whole batch, rebased per chunk on the device
        with torch.cuda.stream(self.h2d):
            d_off = off.to(dev, non_blocking=True)
            d_k = kk.to(dev, non_blocking=True)
            d_l = ll.to(dev, non_blocking=True)
            d_g = gg.to(dev, non_blocking=True)
        for ci, start in enumerate(range(0, B, self.chunk)):
            n = min(self.chunk, B - start)
            slot = self.slots[ci % self.depth]
            with torch.cuda.stream(self.h2d):
                self.h2d.wait_event(slot["drained"])
                slot["y"][:n].copy_(y_host[start:start + n], non_blocking=True)
                slot["lam"][:n].copy_(lam_host[start:start + n], non_blocking=True)
                if tx_host is not None:
                    slot["tx"][:n].copy_(tx_host[start:start + n], non_blocking=True)
                slot["loaded"].record(self.h2d)
            with torch.cuda.stream(self.comp):
                self.comp.wait_event(slot["loaded"])
                # offsets are absolute into the shared tap arrays: a slice is a valid CSR
                paths = PathBatch(d_off[start:start + n + 1], d_k, d_l, d_g)
                res = slot["res"]
                tx = slot["tx"][:n] if tx_host is not None else None
                view = SolveResult(x=res.x[:n], labels=res.labels[:n],
                                   bit_errors=res.bit_errors[:n] if tx is not None else None)
                s.solve(slot["y"][:n], paths, slot["lam"][:n], tx_labels=tx, out=view, trace=False, stream=self.comp)
                slot["solved"].record(self.comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(slot["solved"])
                labels_host[start:start + n].copy_(res.labels[:n], non_blocking=True)
                if tx_host is not None and errors_host is not None:
                    errors_host[start:start + n].copy_(res.bit_errors[:n], non_blocking=True)
                slot["drained"].record(self.d2h)
        self.d2h.synchronize()
