"""The reference's own test-suite (pkg/tests, 177 tests) run through the patcher
on the B200 (substitution mechanism 2).

`oracle/make_ref.py` (run by build() in the build container) installs the
unmodified reference into baseline/_ref and copies its tests to
oracle/_ref/tests; both travel to the GPU box.  The suite runs in a
subprocess with `-p paper_2604_02266_b200.pytest_plugin`, which rebinds
ddlink's hot-path names (patch.install: detect_paths, build_ss_channel,
ss_mvm(_hermitian), cga_equalize, hard_demod, dzt_gemm, estimate_heff, the
dense branch) onto libddb.so before the test modules import them.  Expected:
everything passes except criterion 12, which the reference documents as a
designed FAIL (README.md:57-65, test_output.txt:240).
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import xml.etree.ElementTree as ET
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BASE = ROOT / "baseline" / "_ref"
SUITE = ROOT / "oracle" / "_ref" / "tests"
DESIGNED_FAIL = {"test_criterion_12_threshold_tradeoff"}


def _have_reference() -> bool:
    return (BASE / "ddlink" / "__init__.py").exists() and (SUITE / "test_sparse.py").exists()


def _run_suite(tmp_path: Path, extra_env: dict, select: list[str] | None = None):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT), str(BASE), env.get("PYTHONPATH", "")])
    env.update({"OPENBLAS_NUM_THREADS": "1", "OMP_NUM_THREADS": "1", "DDB_PATCH_REPORT": str(tmp_path / "patch.json")})
    env.update(extra_env)
    junit = tmp_path / "junit.xml"
    targets = select or [str(SUITE)]
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "paper_2604_02266_b200.pytest_plugin",
           f"--junitxml={junit}", "-rA", *targets]
    proc = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=2400)
    tree = ET.parse(junit)
    passed, failed, skipped = set(), set(), set()
    for case in tree.iter("testcase"):
        name = case.get("name")
        if case.find("failure") is not None or case.find("error") is not None:
            failed.add(name)
        elif case.find("skipped") is not None:
            skipped.add(name)
        else:
            passed.add(name)
    report = json.loads((tmp_path / "patch.json").read_text())
    return proc, passed, failed, skipped, report


@pytest.mark.gpu
@pytest.mark.skipif(not _have_reference(), reason="reference trees absent (run oracle/make_ref.py in the build container)")
def test_reference_suite_fp64_through_patcher(tmp_path):
    proc, passed, failed, skipped, report = _run_suite(tmp_path, {"DDB_PATCH_PRECISION": "fp64"})
    tail = proc.stdout[-6000:]
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "reference_suite_fp64.log").write_text(proc.stdout + proc.stderr)
    assert report["libddb_mapped"], "libddb.so was not loaded by the patched suite"
    for name in ("ddb_sscga_solve", "ddb_build_tables", "ddb_ss_mvm_tables", "ddb_host_detect_paths", "ddb_host_dzt",
                 "ddb_host_estimate_heff"):
        assert report["calls"].get(name, 0) > 0, f"{name} never called through the patcher: {report['calls']}"
    assert len(passed) + len(failed) >= 170, tail
    assert failed == DESIGNED_FAIL, f"unexpected failures {sorted(failed - DESIGNED_FAIL)}\n{tail}"


@pytest.mark.gpu
@pytest.mark.skipif(not _have_reference(), reason="reference trees absent (run oracle/make_ref.py in the build container)")
def test_reference_unit_suites_with_device_synthesis(tmp_path):
    """The module-level suites with the transmit side on the device too
    (patch.install(synthesis=True): idzt, apply_channel)."""
    sel = [str(SUITE / f) for f in ("test_sparse.py", "test_equalize.py", "test_grid.py", "test_zak.py",
                                    "test_pilot.py", "test_channel.py", "test_harness.py")]
    proc, passed, failed, skipped, report = _run_suite(tmp_path, {"DDB_PATCH_SYNTHESIS": "1"}, sel)
    assert report["libddb_mapped"]
    assert report["calls"].get("ddb_apply_channel", 0) > 0 and report["calls"].get("ddb_dzt", 0) > 0
    assert not failed, f"failures {sorted(failed)}\n{proc.stdout[-6000:]}"
    assert len(passed) >= 120
