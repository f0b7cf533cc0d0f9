"""Pin the CPU oracle (oracle/ddlink_oracle.py) to the reference's golden vectors.

The fixtures in tests/golden were produced by running the reference package
itself (tests/golden/make_golden.py).  CPU only.
"""

import numpy as np
import pytest

import ddlink_oracle as orc
from conftest import load_golden


def taps_from(d, p):
    return [orc.Tap(int(k), int(l), complex(g)) for k, l, g in zip(d[p + "tap_k"], d[p + "tap_l"], d[p + "tap_g"])]


def frame_taps(d, f):
    a, b = int(d["path_off"][f]), int(d["path_off"][f + 1])
    return [orc.Tap(int(k), int(l), complex(g)) for k, l, g in zip(d["path_k"][a:b], d["path_l"][a:b], d["path_g"][a:b])]


class TestTables:
    def test_worked_example(self):
        d = load_golden("tables")
        r0 = orc.forward_source(orc.Tap(4, 1, 1.0), 7, 8, 2)
        r1 = orc.forward_source(orc.Tap(0, 0, 0.5), 7, 8, 2)
        q1 = orc.inverse_source(orc.Tap(0, 0, 0.5), 11, 8, 2)
        assert [int(r0), int(r1), int(q1)] == [7, 11, 7] == list(d["worked"])

    def test_tables_and_products(self):
        d = load_golden("tables")
        for c in range(int(d["n_cases"])):
            p = f"c{c}_"
            M, N = (int(v) for v in d[p + "grid"])
            t = orc.build_tables(taps_from(d, p), M, N)
            np.testing.assert_array_equal(t.fwd_col, d[p + "fwd_col"])
            np.testing.assert_array_equal(t.herm_row, d[p + "herm_row"])
            np.testing.assert_allclose(t.fwd_coef, d[p + "fwd_coef"], rtol=0, atol=1e-13)
            np.testing.assert_allclose(t.herm_coef, d[p + "herm_coef"], rtol=0, atol=1e-13)
            np.testing.assert_allclose(orc.forward(t, d[p + "v"]), d[p + "Hv"], rtol=0, atol=1e-12)
            np.testing.assert_allclose(orc.adjoint(t, d[p + "v"]), d[p + "HHv"], rtol=0, atol=1e-12)
            if p + "dense_Hv" in d:
                np.testing.assert_allclose(orc.forward(t, d[p + "v"]), d[p + "dense_Hv"], atol=1e-10)

    def test_empty_channel(self):
        with pytest.raises(orc.EmptyChannel):
            orc.build_tables([], 8, 4)

    def test_matrix_free_closed_form(self):
        """The closed forms the CUDA kernels evaluate equal the reference tables."""
        d = load_golden("tables")
        for c in range(int(d["n_cases"])):
            p = f"c{c}_"
            M, N = (int(v) for v in d[p + "grid"])
            MN = M * N
            k = np.arange(M)[:, None]
            l = np.arange(N)[None, :]
            for i, tap in enumerate(taps_from(d, p)):
                dk, dl = M // 2 - tap.k, N // 2 - tap.l
                a = k + dk
                n = np.floor_divide(a, M)
                ks = a - n * M
                e = np.mod(-dl * ks + n * M * l, MN)
                fwd = (tap.gain * np.exp(2j * np.pi * e / MN)).T.reshape(-1)
                np.testing.assert_allclose(fwd, d[p + "fwd_coef"][i], atol=1e-13)
                b = k - dk
                m = np.floor_divide(b, M)
                e2 = np.mod(dl * (k - m * M) + m * M * l, MN)
                herm = (np.conj(tap.gain) * np.exp(2j * np.pi * e2 / MN)).T.reshape(-1)
                np.testing.assert_allclose(herm, d[p + "herm_coef"][i], atol=1e-13)


class TestCga:
    def test_against_reference_runs(self):
        d = load_golden("cga")
        for c in range(int(d["n_cases"])):
            p = f"c{c}_"
            M, N, iters, prof, ident = (int(v) for v in d[p + "meta"])
            t = orc.build_tables(taps_from(d, p), M, N)
            x, tr = orc.cga(t, d[p + "y"], iters, float(d[p + "lam"]), profile=bool(prof))
            ref = d[p + "x"]
            assert np.linalg.norm(x - ref) <= 1e-10 * max(np.linalg.norm(ref), 1e-300) + 1e-12
            np.testing.assert_allclose(tr.c_norm, d[p + "c_norm"], rtol=1e-9, atol=1e-12 * d[p + "c_norm"][0])
            assert tr.mvm_count == int(d[p + "mvm_count"])
            assert tr.exact_converged == bool(d[p + "exact"])
            if prof:
                np.testing.assert_allclose(np.stack(tr.snapshots), d[p + "snapshots"], atol=1e-12)

    def test_config_errors(self):
        t = orc.build_tables([orc.Tap(4, 2, 1.0)], 8, 4)
        with pytest.raises(ValueError):
            orc.cga(t, np.zeros(32), 0)
        with pytest.raises(ValueError):
            orc.cga(t, np.zeros(32), 3, lam=-1.0)


class TestDemod:
    @pytest.mark.parametrize("name", ["qpsk", "qam16"])
    def test_constellation_and_bits(self, name):
        d = load_golden("demod")
        c = orc.qam(name)
        np.testing.assert_allclose(c.points, d[name + "_points"], atol=1e-15)
        np.testing.assert_array_equal(c.bit_map, d[name + "_bitmap"])
        _, bits = orc.hard_demod(d[name + "_x"], c)
        np.testing.assert_array_equal(bits, d[name + "_bits"])

    @pytest.mark.parametrize("name", ["qpsk", "qam16", "qam64"])
    def test_llr_sign_reproduces_hard_decisions(self, name):
        rng = np.random.default_rng(3)
        c = orc.qam(name)
        v = rng.normal(size=4000) * 0.7 + 1j * rng.normal(size=4000) * 0.7
        _, bits = orc.hard_demod(v, c)
        llr = orc.llr_maxlog(v, c, 0.1)
        np.testing.assert_array_equal((llr < 0).astype(np.int64).reshape(-1), bits)

    def test_qam64_extension_shape(self):
        c = orc.qam("qam64")
        assert c.bits_per_symbol == 6 and len(c.points) == 64
        assert np.mean(np.abs(c.points) ** 2) == pytest.approx(1.0)
        pts = c.points * np.sqrt(42)
        for i in range(64):  # Gray: axis neighbours differ in one bit
            for j in range(64):
                dd = pts[i] - pts[j]
                if abs(abs(dd) - 2.0) < 1e-9:
                    assert bin(i ^ j).count("1") == 1


class TestDetect:
    def test_against_reference(self):
        d = load_golden("detect")
        for c in range(int(d["n_cases"])):
            p = f"c{c}_"
            taps = orc.detect_paths(d[p + "heff"], float(d[p + "theta"]))
            np.testing.assert_array_equal([t.k for t in taps], d[p + "k"])
            np.testing.assert_array_equal([t.l for t in taps], d[p + "l"])
            np.testing.assert_array_equal([t.gain for t in taps], d[p + "g"])

    def test_negative_theta(self):
        with pytest.raises(ValueError):
            orc.detect_paths(np.ones((4, 2)), -0.1)

    def test_zero_frame(self):
        assert orc.detect_paths(np.zeros((8, 4), complex), 0.1) == []


@pytest.mark.parametrize("name", ["frames_cfg1", "frames_cfg2", "frames_cfg3"])
def test_frames_reproduce_reference(name):
    d = load_golden(name)
    M, N, iters, b = (int(v) for v in d["meta"])
    const = orc.qam({2: "qpsk", 4: "qam16"}[b])
    for f in range(d["y"].shape[0]):
        x, tr, lab, _ = orc.receive(frame_taps(d, f), d["y"][f].astype(np.complex128), M, N, iters,
                                    float(d["lam"][f]), const)
        ref = d["x_ref"][f]
        assert np.linalg.norm(x - ref) <= 1e-9 * np.linalg.norm(ref)
        np.testing.assert_allclose(tr.c_norm, d["c_norm"][f], rtol=1e-9)
        np.testing.assert_array_equal(lab, d["rx_labels"][f])


class TestFrontEnd:
    """Receiver front end pinned to the reference's own
    dzt_gemm / estimate_heff / detect_paths outputs (tests/golden/frontend.npz)."""

    @pytest.mark.parametrize("tag", ["c1", "c3"])
    def test_dzt_estimate_detect(self, tag):
        d = load_golden("frontend")
        M, N, _, _ = (int(v) for v in d[tag + "_meta"])
        theta = float(d[tag + "_theta"])
        off = d[tag + "_path_off"]
        for i in range(d[tag + "_pilot_rx"].shape[0]):
            yp = orc.dzt_gemm(d[tag + "_pilot_rx"][i], M, N)
            np.testing.assert_allclose(yp, d[tag + "_ypil"][i], rtol=0, atol=1e-12)
            h = orc.estimate_heff(yp, M, N)
            np.testing.assert_allclose(h, d[tag + "_heff"][i], rtol=0, atol=1e-13)
            taps = orc.detect_paths(h, theta)
            a, e = int(off[i]), int(off[i + 1])
            assert [(t.k, t.l) for t in taps] == list(zip(d[tag + "_path_k"][a:e], d[tag + "_path_l"][a:e]))
            y = orc.to_vector(orc.dzt_gemm(d[tag + "_data_rx"][i], M, N))
            np.testing.assert_allclose(y, d[tag + "_y"][i], rtol=0, atol=1e-12)
        half = orc.dzt_gemm(d[tag + "_pilot_rx"][0], M, N, orc.zak_kernel(N, half_shift=True))
        np.testing.assert_allclose(half, d[tag + "_ypil_half"], rtol=0, atol=1e-12)


def test_oracle_receiver_reproduces_criterion6():
    """The oracle's receive chain (dzt_gemm -> estimate_heff -> detect_paths ->
    tables -> CG -> hard_demod) on the stored criterion-6 packets gives the
    reference run_packets' per-packet bit errors (143 in 200 packets)."""
    d = load_golden("harness_c6")
    M, N, iters, b, P = (int(v) for v in d["meta"])
    const = orc.qam("qpsk")
    lam = 1.0 / 10 ** (float(d["snr_db"]) / 10)
    errs = []
    for i in range(P):
        h = orc.estimate_heff(orc.dzt_gemm(d["pilot_rx"][i], M, N), M, N)
        taps = orc.detect_paths(h, float(d["theta"]))
        y = orc.to_vector(orc.dzt_gemm(d["data_rx"][i], M, N))
        _, _, lab, _ = orc.receive(taps, y, M, N, iters, lam, const)
        diff = (lab ^ d["tx_labels"][i]).astype(np.uint8)
        errs.append(int(np.unpackbits(diff[:, None], axis=1).sum()))
    np.testing.assert_array_equal(np.array(errs), d["bit_errors"])


class TestSynthesis:
    """Frame synthesis pinned to the reference's draw_veha,
    modulate, idzt and apply_channel outputs (tests/golden/channel.npz)."""

    @pytest.mark.parametrize("tag", ["c1", "c3"])
    def test_modulate_idzt_apply_channel(self, tag):
        d = load_golden("channel")
        M, N, b, _, count = (int(v) for v in d[tag + "_meta"])
        const = orc.qam({2: "qpsk", 4: "qam16"}[b])
        off = d[tag + "_path_off"]
        for f in range(count):
            X = orc.modulate_labels(d[tag + "_labels"][f], const)
            np.testing.assert_allclose(X, d[tag + "_X"][f], rtol=0, atol=1e-15)
            x = orc.idzt(X, M, N)
            np.testing.assert_allclose(x, d[tag + "_x"][f], rtol=0, atol=1e-12)
            a, e = int(off[f]), int(off[f + 1])
            y = orc.apply_channel(x, d[tag + "_gain"][a:e], d[tag + "_delay_s"][a:e], d[tag + "_doppler_hz"][a:e],
                                  d[tag + "_delay_bin"][a:e], M * 30e3)
            np.testing.assert_allclose(y, d[tag + "_y"][f], rtol=0, atol=1e-12)

    @pytest.mark.parametrize("tag", ["c1", "c3"])
    def test_host_draw_veha_reproduces_reference_draws(self, tag):
        """paper_2604_02266_b200.channel.draw_veha on run_packet's seeded generator
        draws the reference's paths (same variates, same order)."""
        from paper_2604_02266_b200.channel import draw_veha
        from paper_2604_02266_b200.grid import GridConfig
        d = load_golden("channel")
        M, N, _, seed, count = (int(v) for v in d[tag + "_meta"])
        off = d[tag + "_path_off"]
        for f in range(count):
            ps = draw_veha(float(d[tag + "_nu_max"]), GridConfig(M, N), np.random.default_rng([seed, f]))
            a, e = int(off[f]), int(off[f + 1])
            np.testing.assert_array_equal([p.gain for p in ps.paths], d[tag + "_gain"][a:e])
            np.testing.assert_array_equal([p.doppler_hz for p in ps.paths], d[tag + "_doppler_hz"][a:e])
            np.testing.assert_array_equal([p.delay_bin for p in ps.paths], d[tag + "_delay_bin"][a:e])
            np.testing.assert_array_equal([p.delay_s for p in ps.paths], d[tag + "_delay_s"][a:e])

    def test_make_path_range_errors(self):
        from paper_2604_02266_b200.channel import draw_veha, make_path
        from paper_2604_02266_b200.grid import GridConfig
        g = GridConfig(64, 16)
        with pytest.raises(ValueError):
            make_path(1.0, 64 / g.B, 0.0, g)          # delay bin outside the period
        with pytest.raises(ValueError):
            make_path(1.0, 0.0, 9 * g.delta_nu, g)     # beyond half the Doppler period
        with pytest.raises(ValueError):
            draw_veha(-1.0, g, np.random.default_rng(0))
        with pytest.raises(ValueError):
            draw_veha(100.0, GridConfig(8, 16, 1e6), np.random.default_rng(0))  # delay spread > period (1 us)


class TestDense:
    """Dense LMMSE baseline pinned to the reference's
    threshold_frame / build_dense_hdd / lmmse_equalize (tests/golden/dense.npz)."""

    @pytest.mark.parametrize("tag", ["s1", "s2"])
    def test_threshold_dense_lmmse(self, tag):
        d = load_golden("dense")
        M, N = (int(v) for v in d[tag + "_meta"])
        thr = orc.threshold_frame(d[tag + "_heff"], float(d[tag + "_theta"]))
        np.testing.assert_array_equal(thr, d[tag + "_thr"])
        H = orc.dense_channel(thr, M, N)
        np.testing.assert_allclose(H, d[tag + "_H"], rtol=0, atol=1e-14)
        x = orc.lmmse(d[tag + "_H"], d[tag + "_y"], 1.0 / float(d[tag + "_snr_linear"]))
        np.testing.assert_allclose(x, d[tag + "_x"], rtol=0, atol=1e-10 * np.abs(d[tag + "_x"]).max())

    def test_criterion6_dense_arm_known_answer(self):
        d = load_golden("dense")
        assert d["c6_bit_errors"].sum() == 150 and not d["c6_failed"].any()
        assert abs(d["c6_ber"].mean() - 3.662e-4) < 5e-8  # test_output.txt:234
