"""In-tree build of the native library (libddb.so) with nvcc for sm_100a.

The shared object is written next to this file so it travels with the repo
snapshot to the GPU box; nothing is JIT-compiled or cached outside the tree.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
LIB_PATH = PKG_DIR / "libddb.so"
SOURCES = ("sscga.cu", "sscga_tm.cu", "sscga_global.cu", "aux.cu", "frontend.cu", "channel.cu", "dense.cu", "capi.cu")
# sscga_tm.cu is compiled once per part (TM_PART, see the end of that file), in parallel
PARTS = {"sscga_tm.cu": ("0", "1", "2", "3")}
HEADERS = ("common.cuh", "cg.cuh", "demod.cuh", "internal.h")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the ddb native library cannot be built")


def _inputs():
    yield REPO_DIR / "include" / "ddb.h"
    for name in SOURCES + HEADERS:
        yield CSRC / name


def is_stale() -> bool:
    if not LIB_PATH.exists():
        return True
    mtime = LIB_PATH.stat().st_mtime
    return any(p.stat().st_mtime > mtime for p in _inputs())


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> Path:
    """Compile every CUDA source into libddb.so (no-op when up to date).  A
    variant (measurement A/B builds) goes to libddb_<variant>.so with extra
    -D defines; select it at run time with DDB_LIB."""
    lib_path = LIB_PATH if not variant else PKG_DIR / f"libddb_{variant}.so"
    if not variant and not force and not is_stale():
        return LIB_PATH
    nvcc = nvcc_path()
    objdir = PKG_DIR / ("build" if not variant else f"build_{variant}")
    objdir.mkdir(exist_ok=True)
    hdr_mtime = max(p.stat().st_mtime for p in [REPO_DIR / "include" / "ddb.h", *(CSRC / h for h in HEADERS)])
    objs, cmds = [], []
    units = [(src, None) for src in SOURCES if src not in PARTS]
    units += [(src, part) for src in SOURCES if src in PARTS for part in PARTS[src]]
    for src, part in units:
        obj = objdir / (Path(src).stem + (f"_p{part}" if part is not None else "") + ".o")
        objs.append(str(obj))
        if not force and obj.exists() and obj.stat().st_mtime > max(hdr_mtime, (CSRC / src).stat().st_mtime):
            continue  # object up to date
        extra = [f"-DTM_PART={part}"] if part is not None else []
        cmd = [nvcc, *NVCC_FLAGS, *extra, *(f"-D{d}" for d in defines), "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        cmds.append(cmd)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as pool:
        for fut in [pool.submit(_run, c, verbose) for c in cmds]:
            fut.result()
    tmp = lib_path.with_suffix(".so.tmp")
    _run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
          *objs, "-o", str(tmp)], verbose)
    os.replace(tmp, lib_path)
    return lib_path


def _run(cmd, verbose):
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout)
        sys.stderr.write(res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"command failed ({res.returncode}): {' '.join(cmd)}")


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--variant", default="")
    ap.add_argument("-D", action="append", default=[])
    args = ap.parse_args()
    print(build(force=args.force, verbose=args.v, variant=args.variant, defines=args.D))
