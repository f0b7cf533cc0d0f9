"""Recipe: make the unmodified reference (`ddlink`, /root/reference/pkg) importable
on the GPU box, as test infrastructure and as the bench's reference arm.

    python oracle/make_ref.py        # run in the build container (build() calls it)

* baseline/_ref/  -- `pip install --no-index --no-deps --target` of a /tmp copy
                     of /root/reference/pkg (the build writes into its source
                     tree, and /root/reference is read-only): the reference's own
                     package, untouched.  Used by `bench.py --impl reference`
                     and by the -m gpu tests that run the reference itself.
* oracle/_ref/tests/ -- the reference's own test-suite (pkg/tests), run through
                     the patcher on the B200 by tests/test_reference_suite.py.

Both directories are git-ignored (no reference source enters the history) and
not gpurun-ignored, so they travel to the GPU box with the snapshot.  Nothing
in the product package imports either of them.
"""

from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

REF_PKG = Path("/root/reference/pkg")
ROOT = Path(__file__).resolve().parent.parent
BASE = ROOT / "baseline" / "_ref"
TESTS = ROOT / "oracle" / "_ref" / "tests"


def _stamp(p: Path) -> float:
    return max((f.stat().st_mtime for f in p.rglob("*") if f.is_file()), default=0.0)


def make(force: bool = False) -> bool:
    """Install / refresh both trees; False when the reference is absent (GPU box)."""
    if not REF_PKG.is_dir():
        return False
    if force or not (BASE / "ddlink" / "__init__.py").exists() or _stamp(REF_PKG / "src") > _stamp(BASE / "ddlink"):
        with tempfile.TemporaryDirectory() as tmp:
            src = Path(tmp) / "pkg"
            shutil.copytree(REF_PKG, src)
            if BASE.exists():
                shutil.rmtree(BASE)
            subprocess.run([sys.executable, "-m", "pip", "install", "--quiet", "--no-index", "--no-build-isolation",
                            "--no-deps", "--find-links", "/opt/wheelhouse", "--target", str(BASE), str(src)],
                           check=True)
    if force or not TESTS.exists() or _stamp(REF_PKG / "tests") > _stamp(TESTS):
        if TESTS.exists():
            shutil.rmtree(TESTS)
        shutil.copytree(REF_PKG / "tests", TESTS, ignore=shutil.ignore_patterns("__pycache__", ".hypothesis"))
    return True


if __name__ == "__main__":
    print("reference trees ready" if make(force="--force" in sys.argv) else "reference absent: nothing to do")
