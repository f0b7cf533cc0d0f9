"""INTEGRATION.md's reference-side ctypes stub (Option B), executed as written:
the code block is extracted into a throw-away `ddlink`-shaped package (its
`from .equalize import CgaTrace` resolved to this build's CgaTrace), pointed at
the in-tree libddb.so, and run on golden CG cases against the reference's
fp64 results."""

import re
import sys
import types
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import load_golden  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


def _stub_module():
    text = (ROOT / "INTEGRATION.md").read_text()
    m = re.search(r"```python\n# ddlink/_b200\.py\n(.*?)```", text, re.S)
    assert m, "INTEGRATION.md lost its ctypes stub"
    code = m.group(1).replace("/path/to/paper_2604_02266_b200/libddb.so",
                              str(ROOT / "paper_2604_02266_b200" / "libddb.so"))
    import paper_2604_02266_b200 as b200
    pkg = types.ModuleType("ddlink_stub")
    pkg.__path__ = []
    eq = types.ModuleType("ddlink_stub.equalize")
    eq.CgaTrace = b200.CgaTrace
    mod = types.ModuleType("ddlink_stub._b200")
    mod.__package__ = "ddlink_stub"
    sys.modules.update({"ddlink_stub": pkg, "ddlink_stub.equalize": eq, "ddlink_stub._b200": mod})
    exec(compile(code, "INTEGRATION.md:_b200.py", "exec"), mod.__dict__)
    return mod


def test_documented_stub_solves_reference_cases():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_02266_b200 as b200
    stub = _stub_module()
    d = load_golden("cga")
    for c in range(int(d["n_cases"])):
        p = f"c{c}_"
        M, N, iters, prof, ident = (int(v) for v in d[p + "meta"])
        paths = [b200.DominantPath(int(a), int(b), complex(g))
                 for a, b, g in zip(d[p + "tap_k"], d[p + "tap_l"], d[p + "tap_g"])]
        ch = types.SimpleNamespace(M=M, N=N, paths=paths)
        x, tr = stub.cga_equalize(ch, d[p + "y"], b200.CgaConfig(iterations=iters, lam=float(d[p + "lam"])))
        ref = d[p + "x"]
        assert np.linalg.norm(x - ref) <= 1e-10 * max(np.linalg.norm(ref), 1e-300) + 1e-12, c
        np.testing.assert_allclose(tr.c_norm, d[p + "c_norm"], rtol=1e-9, atol=1e-12 * d[p + "c_norm"][0])
        assert tr.exact_converged == bool(d[p + "exact"])
        assert tr.mvm_count == int(d[p + "mvm_count"])


def test_documented_frontend_stub_matches_reference_goldens():
    """INTEGRATION.md's host-pointer front-end stub (Option B'), executed as
    written, against the reference's own pilot DZT and detect_paths outputs
    (tests/golden/frontend.npz, made by running ddlink)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_02266_b200 as b200
    text = (ROOT / "INTEGRATION.md").read_text()
    m = re.search(r"```python\n# ddlink/_b200_frontend\.py\n(.*?)```", text, re.S)
    assert m, "INTEGRATION.md lost its front-end stub"
    code = m.group(1).replace("/path/to/paper_2604_02266_b200/libddb.so",
                              str(ROOT / "paper_2604_02266_b200" / "libddb.so"))
    pkg = types.ModuleType("ddlink_fe")
    pkg.__path__ = []
    sp = types.ModuleType("ddlink_fe.sparse")
    sp.DominantPath = b200.DominantPath
    mod = types.ModuleType("ddlink_fe._b200_frontend")
    mod.__package__ = "ddlink_fe"
    sys.modules.update({"ddlink_fe": pkg, "ddlink_fe.sparse": sp, "ddlink_fe._b200_frontend": mod})
    exec(compile(code, "INTEGRATION.md:_b200_frontend.py", "exec"), mod.__dict__)
    d = load_golden("frontend")
    for tag in ("c1", "c3"):
        M, N = (int(v) for v in d[tag + "_meta"][:2])
        cfg = b200.GridConfig(M, N)
        off = d[tag + "_path_off"]
        for f in range(d[tag + "_pilot_rx"].shape[0]):
            ypil = mod.dzt_gemm(d[tag + "_pilot_rx"][f], b200.build_zak_kernel(N), cfg)
            np.testing.assert_allclose(ypil, d[tag + "_ypil"][f], atol=1e-12 * np.abs(d[tag + "_ypil"][f]).max())
            taps = mod.detect_paths(d[tag + "_heff"][f], float(d[tag + "_theta"]), cfg)
            assert [(t.k_p, t.l_p) for t in taps] == list(zip(d[tag + "_path_k"][off[f]:off[f + 1]].tolist(),
                                                              d[tag + "_path_l"][off[f]:off[f + 1]].tolist()))
