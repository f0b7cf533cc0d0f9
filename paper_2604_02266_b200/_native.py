"""ctypes binding of libddb.so (include/ddb.h).

The library is loaded from this package directory only.  There is no
fallback: if the shared object is missing or CUDA is unavailable every
entry point raises, so a silent CPU path can never stand in for the kernels.
"""

from __future__ import annotations

import ctypes as C
import os
import re
import threading
from pathlib import Path

# DDB_LIB: an alternative build of the same library (A/B measurement builds of build.py --variant)
LIB_PATH = Path(os.environ["DDB_LIB"]).resolve() if os.environ.get("DDB_LIB") else \
    Path(__file__).resolve().parent / "libddb.so"
HEADER_PATH = Path(__file__).resolve().parent.parent / "include" / "ddb.h"

DDB_OK = 0
DDB_ERR_INVALID = 1
DDB_ERR_SHAPE = 2
DDB_ERR_UNSUPPORTED = 3
DDB_ERR_CUDA = 4
DDB_ERR_WORKSPACE = 5
DDB_F32 = 0
DDB_F64 = 1
FRAME_EMPTY_CHANNEL = 0x1
FRAME_EXACT_CONVERGED = 0x2


class DdbError(RuntimeError):
    """A ddb entry point returned a non-zero status."""

    def __init__(self, status: int, where: str, message: str):
        super().__init__(f"{where}: status {status}: {message}")
        self.status = status


class Problem(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("M", C.c_int32), ("N", C.c_int32), ("iterations", C.c_int32),
        ("dtype", C.c_int32),
        ("path_offsets", C.c_void_p), ("path_k", C.c_void_p), ("path_l", C.c_void_p),
        ("path_gain", C.c_void_p), ("y", C.c_void_p), ("lam", C.c_void_p),
    ]


class Outputs(C.Structure):
    _fields_ = [
        ("x", C.c_void_p), ("c_norm", C.c_void_p), ("iterations_done", C.c_void_p),
        ("status", C.c_void_p), ("snapshots", C.c_void_p),
        ("bits_per_symbol", C.c_int32),
        ("labels", C.c_void_p), ("llr", C.c_void_p), ("noise_var", C.c_void_p),
        ("tx_labels", C.c_void_p), ("bit_errors", C.c_void_p), ("tx_labels_packed", C.c_int32),
    ]


ABI_VERSION = 3  # include/ddb.h DDB_ABI_VERSION
DDB_DZT_COLMAJOR = 1
DDB_DZT_PILOT = 2
DDB_DZT_INPUT_F32 = 4
DDB_DZT_INVERSE = 8


class Plan(C.Structure):
    _fields_ = [
        ("cluster", C.c_int32), ("cols_per_cta", C.c_int32), ("cols_per_thread", C.c_int32),
        ("threads", C.c_int32), ("smem_bytes", C.c_int32), ("ctas_per_sm", C.c_int32),
        ("halo_rows", C.c_int32), ("kernel", C.c_int32), ("rows_per_thread", C.c_int32),
    ]


_SIGNATURES = {
    "ddb_abi_version": (C.c_int32, []),
    "ddb_last_error": (C.c_char_p, []),
    "ddb_build_info": (C.c_char_p, []),
    "ddb_sscga_plan": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(Plan)]),
    "ddb_sscga_workspace_bytes": (C.c_size_t, [C.POINTER(Problem)]),
    "ddb_sscga_solve": (C.c_int32, [C.POINTER(Problem), C.POINTER(Outputs), C.c_void_p, C.c_size_t,
                                    C.c_void_p]),
    "ddb_ss_apply": (C.c_int32, [C.POINTER(Problem), C.c_void_p, C.c_int32, C.c_void_p]),
    "ddb_build_tables": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ddb_ss_mvm_tables": (C.c_int32, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p]),
    "ddb_hard_demod": (C.c_int32, [C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                   C.c_void_p]),
    "ddb_qam_demod": (C.c_int32, [C.c_int64, C.c_int32, C.c_void_p, C.c_int32, C.c_double, C.c_void_p,
                                  C.c_void_p, C.c_void_p]),
    "ddb_detect_paths": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_double, C.c_int32,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ddb_dzt": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                            C.c_double, C.c_void_p, C.c_void_p]),
    "ddb_estimate_heff": (C.c_int32, [C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                      C.c_void_p]),
    "ddb_host_dzt": (C.c_int32, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ddb_host_estimate_heff": (C.c_int32, [C.c_int64, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p]),
    "ddb_host_detect_paths": (C.c_int32, [C.c_int32, C.c_int32, C.c_void_p, C.c_double, C.c_int32, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_void_p]),
    "ddb_paths_csr": (C.c_int32, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ddb_modulate": (C.c_int32, [C.c_int64, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "ddb_apply_channel": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                      C.c_void_p]),
    "ddb_add_awgn": (C.c_int32, [C.c_int32, C.c_int64, C.c_int32, C.c_void_p, C.c_double, C.c_uint64,
                                 C.c_void_p, C.c_void_p, C.c_void_p]),
    "ddb_threshold_frame": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_double,
                                        C.c_void_p, C.c_void_p]),
    "ddb_build_dense_hdd": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                        C.c_void_p]),
    "ddb_probe_fp32": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "ddb_sscga_profile_phases": (C.c_int32, [C.POINTER(Problem), C.POINTER(Outputs), C.c_void_p, C.c_void_p]),
}
PHASES = ("setup", "arrive", "mvm_local", "wait", "mvm_remote", "read", "step1", "step3", "epilogue", "tail")

_lock = threading.Lock()
_lib = None


def header_symbols() -> list[str]:
    """Every function name declared in include/ddb.h."""
    text = HEADER_PATH.read_text()
    return sorted(set(re.findall(r"\b(ddb_[a-z0-9_]+)\s*\(", text)))


def load(build_if_missing: bool = False):
    """Load (once) and return the configured ctypes library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            if build_if_missing:
                from .build import build
                build()
            else:
                raise RuntimeError(
                    f"native library {LIB_PATH} is missing; run "
                    "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.ddb_abi_version() != ABI_VERSION:
            raise RuntimeError("libddb ABI version mismatch")
        _lib = lib
        return lib


# per-entry-point call counts (status checks), so a run through the patcher can
# show which kernels the reference's code actually reached (pytest_plugin)
CALLS: dict = {}


def check(status: int, where: str) -> None:
    CALLS[where] = CALLS.get(where, 0) + 1
    if status != DDB_OK:
        msg = load().ddb_last_error().decode(errors="replace")
        raise DdbError(status, where, msg)


def plan(M: int, N: int, dtype: int) -> Plan:
    p = Plan()
    check(load().ddb_sscga_plan(M, N, dtype, C.byref(p)), "ddb_sscga_plan")
    return p
