"""C-ABI boundary and host logic, CPU only (no kernel launches)."""

import ctypes as C

import numpy as np
import pytest

from paper_2604_02266_b200 import _native as nat


@pytest.fixture(scope="module")
def lib():
    return nat.load(build_if_missing=True)


def test_exports_every_header_symbol(lib):
    names = nat.header_symbols()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    assert lib.ddb_abi_version() == nat.ABI_VERSION == 3
    assert b"sm_100a" in lib.ddb_build_info()


def test_library_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(nat.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("M,N,dt,cluster", [
    (64, 16, nat.DDB_F32, 1), (256, 16, nat.DDB_F32, 1), (512, 32, nat.DDB_F32, 2),
    (512, 32, nat.DDB_F64, 4), (128, 32, nat.DDB_F64, 1), (8, 2, nat.DDB_F64, 1),
])
def test_plan_without_gpu(lib, M, N, dt, cluster):
    p = nat.plan(M, N, dt)
    assert p.cluster == cluster
    assert p.cols_per_cta * p.cluster == N
    assert p.cols_per_cta % p.cols_per_thread == 0
    assert p.threads % 32 == 0 and p.threads <= 1024
    assert p.smem_bytes <= 227 * 1024
    # the Veh-A delay spread (<= 39 bins at M=512) fits the quasi-periodic halo;
    # the TMEM kernel's small grids stop at M / 2 rows, which covers every
    # delay shift (|d_k| <= M / 2, sparse.py:35-37)
    assert p.halo_rows >= (min(M // 2, 64) if p.kernel == 1 else min(M, 64))


def test_plan_large_grid_uses_bigger_clusters(lib):
    p = nat.plan(1024, 64, nat.DDB_F32)
    assert p.cluster in (8, 16)
    assert p.kernel == 1 and p.rows_per_thread == 16  # TMEM-operand kernel
    p = nat.plan(512, 32, nat.DDB_F32)
    assert (p.kernel, p.cluster, p.rows_per_thread, p.threads) == (1, 2, 16, 512)
    assert nat.plan(512, 32, nat.DDB_F64).kernel == 0  # fp64: row-slice kernel


def test_paper_grid_uses_workspace_path(lib):
    """(16384, 32) exceeds a 16-CTA cluster's on-chip memory: the
    planner picks the workspace-backed kernels and sizes their workspace."""
    for dt, eb in ((nat.DDB_F32, 8), (nat.DDB_F64, 16)):
        p = nat.plan(16384, 32, dt)
        assert p.kernel == 2
        prob = _prob(batch=3, M=16384, N=32, dtype=dt)
        ws = lib.ddb_sscga_workspace_bytes(C.byref(prob))
        assert ws >= 3 * 3 * 16384 * 32 * eb  # c, u, p of every frame
    assert lib.ddb_sscga_workspace_bytes(C.byref(_prob(M=512, N=32))) == 0  # fused: state on chip


def _prob(**kw):
    base = dict(batch=1, M=8, N=4, iterations=10, dtype=nat.DDB_F32)
    base.update(kw)
    return nat.Problem(base["batch"], base["M"], base["N"], base["iterations"], base["dtype"],
                       C.c_void_p(8), C.c_void_p(8), C.c_void_p(8), C.c_void_p(8), C.c_void_p(8), C.c_void_p(8))


@pytest.mark.parametrize("kw,code", [
    (dict(iterations=0), nat.DDB_ERR_INVALID),      # equalize.py:26-27
    (dict(M=7), nat.DDB_ERR_SHAPE),                  # grid.py:25-29
    (dict(N=1), nat.DDB_ERR_SHAPE),
    (dict(batch=-1), nat.DDB_ERR_INVALID),
    (dict(dtype=7), nat.DDB_ERR_INVALID),
])
def test_solve_validates_before_launch(lib, kw, code):
    out = nat.Outputs()
    out.x = C.c_void_p(8)
    r = lib.ddb_sscga_solve(C.byref(_prob(**kw)), C.byref(out), None, 0, None)
    assert r == code
    assert lib.ddb_last_error()


def test_solve_rejects_bad_demod_request(lib):
    out = nat.Outputs()
    out.x = C.c_void_p(8)
    out.bits_per_symbol = 3
    assert lib.ddb_sscga_solve(C.byref(_prob()), C.byref(out), None, 0, None) == nat.DDB_ERR_INVALID
    out.bits_per_symbol = 0
    out.bit_errors = C.c_void_p(8)
    assert lib.ddb_sscga_solve(C.byref(_prob()), C.byref(out), None, 0, None) == nat.DDB_ERR_INVALID


def test_empty_batch_is_ok(lib):
    out = nat.Outputs()
    assert lib.ddb_sscga_solve(C.byref(_prob(batch=0)), C.byref(out), None, 0, None) == nat.DDB_OK


def test_detect_rejects_negative_theta(lib):
    r = lib.ddb_detect_paths(1, 8, 4, C.c_void_p(8), -0.5, 4, C.c_void_p(8), C.c_void_p(8), C.c_void_p(8),
                             C.c_void_p(8), None)
    assert r == nat.DDB_ERR_INVALID


def test_build_tables_empty_channel(lib):
    r = lib.ddb_build_tables(8, 4, 0, None, None, None, None, None, None, None, None)
    assert r == nat.DDB_ERR_INVALID
    assert b"no taps" in lib.ddb_last_error()


class TestHostMirror:
    def test_config_errors_match_reference(self):
        from paper_2604_02266_b200 import CgaConfig, GridConfig, make_constellation
        with pytest.raises(ValueError):
            CgaConfig(iterations=0)
        with pytest.raises(ValueError):
            CgaConfig(iterations=5, lam=-1.0)
        for m, n in [(1, 4), (3, 4), (4, 3), (0, 2), (4, 1)]:
            with pytest.raises(ValueError):
                GridConfig(m, n)
        with pytest.raises(ValueError):
            make_constellation("qam64")

    def test_constellations_match_oracle(self):
        import ddlink_oracle as orc
        from paper_2604_02266_b200 import make_constellation, make_constellation_ext
        for name in ("qpsk", "qam16"):
            a, b = make_constellation(name), orc.qam(name)
            np.testing.assert_allclose(a.points, b.points, atol=1e-15)
            np.testing.assert_array_equal(a.bit_map, b.bit_map)
        a, b = make_constellation_ext("qam64"), orc.qam("qam64")
        np.testing.assert_allclose(a.points, b.points, atol=1e-15)

    def test_flatten_layout(self):
        from paper_2604_02266_b200 import GridConfig, flatten, unflatten
        gc = GridConfig(4, 2)
        frame = np.arange(8, dtype=complex).reshape(4, 2, order="F")
        v = flatten(frame, gc)
        np.testing.assert_array_equal(v, np.arange(8))
        np.testing.assert_array_equal(unflatten(v, gc), frame)
        v[0] = 9
        assert frame[0, 0] == 0

    def test_bits_per_symbol(self):
        from paper_2604_02266_b200 import bits_per_symbol
        assert bits_per_symbol("qpsk") == 2 and bits_per_symbol("16-QAM") == 4 and bits_per_symbol("qam64") == 6
        with pytest.raises(ValueError):
            bits_per_symbol("qam256")

    def test_product_path_never_imports_oracle(self):
        import pathlib
        pkg = pathlib.Path(nat.__file__).parent
        for f in pkg.rglob("*.py"):
            assert "oracle" not in f.read_text().replace("oracle_check", ""), f


def test_pack_labels_layout():
    import torch
    from paper_2604_02266_b200 import pack_labels
    lab = torch.tensor([[1, 2, 3, 0, 15, 14, 13, 12]], dtype=torch.uint8)
    assert pack_labels(lab & 3, 2).tolist() == [[1 | 2 << 2 | 3 << 4, 3 | 2 << 2 | 1 << 4]]
    assert pack_labels(lab, 4).tolist() == [[0x21, 0x03, 0xEF, 0xCD]]
    with pytest.raises(ValueError):
        pack_labels(lab, 6)
