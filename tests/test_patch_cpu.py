"""The opt-in ddlink patcher rebinds the hot-path names (CPU only; skipped
where the reference package is not importable, e.g. on the GPU box)."""

import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture
def ddlink():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    return pytest.importorskip("ddlink")


def test_install_and_uninstall(ddlink):
    import paper_2604_02266_b200 as b200
    from paper_2604_02266_b200 import patch

    orig_cga = ddlink.harness.cga_equalize
    saved = patch.install(ddlink)
    try:
        assert ddlink.harness.cga_equalize is b200.cga_equalize
        assert ddlink.equalize.cga_equalize is b200.cga_equalize
        assert ddlink.sparse.build_ss_channel is b200.build_ss_channel
        assert ddlink.grid.hard_demod is b200.hard_demod
        assert ddlink.detect_paths is b200.detect_paths
        assert ddlink.harness.dzt_gemm is b200.dzt_gemm and ddlink.zak.dzt_gemm is b200.dzt_gemm
        assert ddlink.pilot.estimate_heff is b200.estimate_heff
        assert ddlink.harness.lmmse_equalize is b200.lmmse_equalize
        assert ddlink.sparse.build_dense_hdd is b200.build_dense_hdd
        assert ddlink.sparse.threshold_frame is b200.threshold_frame
        # the reference's EmptyChannel is what the drop-in raises (harness.py:170)
        with pytest.raises(ddlink.EmptyChannel):
            b200.build_ss_channel([], ddlink.GridConfig(8, 4))
    finally:
        patch.uninstall(saved)
        import paper_2604_02266_b200.sparse as sp
        sp.EmptyChannel = b200.EmptyChannel
    assert ddlink.harness.cga_equalize is orig_cga
    assert ddlink.harness.dzt_gemm is not b200.dzt_gemm


def test_install_with_synthesis(ddlink):
    import paper_2604_02266_b200 as b200
    from paper_2604_02266_b200 import channel as pch
    from paper_2604_02266_b200 import patch

    orig_idzt, orig_apply = ddlink.harness.idzt, ddlink.channel.apply_channel
    saved = patch.install(ddlink, synthesis=True)
    try:
        assert ddlink.harness.idzt is pch.idzt and ddlink.zak.idzt is pch.idzt and ddlink.idzt is pch.idzt
        assert ddlink.channel.apply_channel is pch.apply_channel and ddlink.apply_channel is pch.apply_channel
        assert ddlink.channel.add_awgn is not pch.add_awgn  # the reference's noise stream stays
    finally:
        patch.uninstall(saved)
        import paper_2604_02266_b200.sparse as sp
        sp.EmptyChannel = b200.EmptyChannel
    assert ddlink.harness.idzt is orig_idzt and ddlink.channel.apply_channel is orig_apply
