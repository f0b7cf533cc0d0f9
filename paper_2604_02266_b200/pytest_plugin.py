"""pytest plugin: run a test-suite written against `ddlink` through the B200 kernels.

    pytest -p paper_2604_02266_b200.pytest_plugin <ddlink tests>

The patch is installed at configure time, i.e. before test modules execute
their `from ddlink import ...` lines, so those names resolve to the GPU path.
Environment: DDB_PATCH_PRECISION (fp64 default, or fp32), DDB_PATCH_SYNTHESIS=1
(also rebind the transmit side, patch.install(synthesis=True)), and
DDB_PATCH_REPORT=<file>: at exit a JSON record of the rebound names, the ddb
entry points called (with counts) and whether libddb.so was mapped into the
process, so a caller can prove the kernels ran.
"""

import json
import os

_STATE = {}


def pytest_configure(config):
    from .patch import install
    saved = install(precision=os.environ.get("DDB_PATCH_PRECISION", "fp64"),
                    synthesis=os.environ.get("DDB_PATCH_SYNTHESIS", "0") == "1")
    _STATE["rebound"] = sorted(f"{m}.{n}" for (m, n) in saved)


def pytest_report_header(config):
    return f"ddb patch: {len(_STATE.get('rebound', []))} ddlink names rebound onto libddb.so"


def pytest_unconfigure(config):
    path = os.environ.get("DDB_PATCH_REPORT")
    if not path:
        return
    from . import _native
    try:
        maps = open("/proc/self/maps").read()
    except OSError:
        maps = ""
    rec = {"rebound": _STATE.get("rebound", []), "calls": dict(sorted(_native.CALLS.items())),
           "libddb_mapped": str(_native.LIB_PATH) in maps}
    with open(path, "w") as f:
        json.dump(rec, f, indent=1)
