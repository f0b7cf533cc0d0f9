"""Generate the golden fixtures by running the UNMODIFIED reference package.

Run in the build container (the reference is importable only there):

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

Every array stored here is an output of the reference's own functions
(/root/reference/pkg/src/ddlink).  The oracle (oracle/ddlink_oracle.py) is
pinned to them by tests/test_oracle.py, and the GPU parity tests compare the
CUDA path with the oracle on the fixture inputs.  Nothing on the GPU box reads
/root/reference: only these .npz files travel.

Frame fixtures follow run_packet's draw order exactly (harness.py:141-149:
fading draw, bits, modulate, IDZT, channel + AWGN for pilot then data) and
its receiver path (harness.py:155-194); y is rounded to complex64 first and
the reference is re-run on the rounded input, so the fixtures are
self-consistent for an fp32 device path.
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _ref():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import ddlink  # noqa: F401
    return ddlink


def pack_taps(taps_list):
    off = [0]
    k, l, g = [], [], []
    for taps in taps_list:
        for t in taps:
            k.append(t.k_p)
            l.append(t.l_p)
            g.append(t.gain)
        off.append(len(k))
    return (np.asarray(off, np.int32), np.asarray(k, np.int32), np.asarray(l, np.int32),
            np.asarray(g, np.complex128))


def tables_fixture(d):
    """Index maps / coefficient tables / MVMs on random channels."""
    rng = np.random.default_rng(20261017)
    out = {}
    cases = [(8, 2), (16, 8), (48, 32), (12, 6), (64, 16)]
    for ci, (M, N) in enumerate(cases):
        g = d.GridConfig(M, N)
        frame = np.zeros((M, N), complex)
        frame[rng.integers(M), rng.integers(N)] = 1.0
        for _ in range(4):
            frame[rng.integers(M), rng.integers(N)] += rng.uniform(0.05, 0.3) * np.exp(2j * np.pi * rng.random())
        taps = d.detect_paths(frame, 0.01, g)
        ch = d.build_ss_channel(taps, g)
        v = rng.normal(size=M * N) + 1j * rng.normal(size=M * N)
        p = f"c{ci}_"
        out[p + "grid"] = np.array([M, N], np.int32)
        out[p + "heff"] = frame
        out[p + "tap_k"] = np.array([t.k_p for t in taps], np.int32)
        out[p + "tap_l"] = np.array([t.l_p for t in taps], np.int32)
        out[p + "tap_g"] = np.array([t.gain for t in taps], np.complex128)
        out[p + "fwd_coef"] = ch.fwd_coef
        out[p + "fwd_col"] = ch.fwd_col
        out[p + "herm_coef"] = ch.herm_coef
        out[p + "herm_row"] = ch.herm_row
        out[p + "v"] = v
        out[p + "Hv"] = d.ss_mvm(ch, v)
        out[p + "HHv"] = d.ss_mvm_hermitian(ch, v)
        if M * N <= d.sparse.DENSE_GUARD:
            H = d.build_dense_hdd(frame, g)
            out[p + "dense_Hv"] = H @ v
    out["n_cases"] = np.array(len(cases))
    # worked example (harness.py:349-358; reference tests/test_sparse.py:49-55)
    g = d.GridConfig(8, 2)
    out["worked"] = np.array([
        d.forward_index(d.DominantPath(4, 1, 1.0), 7, g),
        d.forward_index(d.DominantPath(0, 0, 0.5), 7, g),
        d.inverse_index(d.DominantPath(0, 0, 0.5), 11, g),
    ], np.int64)
    np.savez_compressed(OUT / "tables.npz", **out)


def cga_fixture(d):
    """cga_equalize on small problems: lam sweep, full-Krylov, identity, profile."""
    rng = np.random.default_rng(77)
    out = {}
    cases = []
    for (M, N) in [(16, 8), (8, 4), (32, 16)]:
        for lam in (0.0, 1e-3, 0.1):
            for iters in (10, M * N if M * N <= 128 else 25):
                cases.append((M, N, lam, iters, False))
    cases.append((8, 4, 0.0, 4, True))
    cases.append((8, 4, 0.0, 10, "identity"))
    for ci, (M, N, lam, iters, kind) in enumerate(cases):
        g = d.GridConfig(M, N)
        frame = np.zeros((M, N), complex)
        if kind == "identity":
            frame[g.K0, g.L0] = 1.0
        else:
            frame[rng.integers(M), rng.integers(N)] = 1.0
            placed = 0
            while placed < 3:
                k, l = rng.integers(M), rng.integers(N)
                if frame[k, l] == 0:
                    frame[k, l] = rng.uniform(0.05, 0.2) * np.exp(2j * np.pi * rng.random())
                    placed += 1
        taps = d.detect_paths(frame, 0.01, g)
        ch = d.build_ss_channel(taps, g)
        y = rng.normal(size=M * N) + 1j * rng.normal(size=M * N)
        x, tr = d.cga_equalize(ch, y, d.CgaConfig(iterations=iters, lam=lam, profile=kind is True))
        p = f"c{ci}_"
        out[p + "meta"] = np.array([M, N, iters, int(kind is True), int(kind == "identity")], np.int64)
        out[p + "lam"] = np.array(lam)
        out[p + "tap_k"] = np.array([t.k_p for t in taps], np.int32)
        out[p + "tap_l"] = np.array([t.l_p for t in taps], np.int32)
        out[p + "tap_g"] = np.array([t.gain for t in taps], np.complex128)
        out[p + "y"] = y
        out[p + "x"] = x
        out[p + "c_norm"] = np.array(tr.c_norm)
        out[p + "mvm_count"] = np.array(tr.mvm_count)
        out[p + "exact"] = np.array(tr.exact_converged)
        if kind is True:
            out[p + "snapshots"] = np.stack(tr.snapshots)
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(OUT / "cga.npz", **out)


def demod_fixture(d):
    rng = np.random.default_rng(5)
    out = {}
    for name in ("qpsk", "qam16"):
        c = d.make_constellation(name)
        g = d.GridConfig(16, 8)
        pts = c.points
        # noisy points, exact points and exact midpoints (lowest-label ties)
        v = rng.normal(size=g.size) * 0.6 + 1j * rng.normal(size=g.size) * 0.6
        v[:len(pts)] = pts
        mids = (pts[:, None] + pts[None, :]) / 2
        mids = mids[np.triu_indices(len(pts), 1)]
        v[len(pts):len(pts) + min(len(mids), 64)] = mids[:64]
        _, bits = d.hard_demod(d.unflatten(v, g), c, g)
        out[name + "_points"] = pts
        out[name + "_bitmap"] = c.bit_map
        out[name + "_x"] = v
        out[name + "_bits"] = bits
    np.savez_compressed(OUT / "demod.npz", **out)


def run_frames(d, M, N, mod, snr_db, nu, theta, iters, seed, count, pset_fn=None):
    """run_packet (harness.py:131-205) with the receiver's intermediates kept."""
    from ddlink.harness import Workspace
    cfg = d.SimConfig(m=M, n=N, mod=mod, snr_db=snr_db, nu_max_hz=nu, theta=theta, iters=iters,
                      packets=count, seed=seed)
    ws = Workspace(cfg)
    grid, const = ws.grid, ws.const
    rec = {"y": [], "taps": [], "lam": [], "tx": [], "x": [], "c_norm": [], "rx": [], "heff": []}
    for idx in range(count):
        rng = np.random.default_rng([seed, idx])
        pset = pset_fn(grid, rng) if pset_fn else d.draw_veha(cfg.nu_max_hz, grid, rng)
        tx_bits = rng.integers(0, 2, size=const.bits_per_symbol * grid.size)
        data_tx = d.idzt(d.modulate(tx_bits, const, grid), grid)
        pilot_rx = d.add_awgn(d.apply_channel(ws.pilot_tx, pset, grid), cfg.snr_db, rng)
        data_rx = d.add_awgn(d.apply_channel(data_tx, pset, grid), cfg.snr_db, rng)
        heff = d.estimate_heff(d.dzt_gemm(pilot_rx, ws.zak_kernel, grid), ws.twist, grid)
        taps = d.detect_paths(heff, cfg.theta, grid)
        ch = d.build_ss_channel(taps, grid)
        y = d.flatten(d.dzt_gemm(data_rx, ws.zak_kernel, grid), grid)
        y = y.astype(np.complex64).astype(np.complex128)  # fp32-representable input
        lam = 0.0 if math.isinf(cfg.snr_linear) else 1.0 / cfg.snr_linear
        x, tr = d.cga_equalize(ch, y, d.CgaConfig(iterations=cfg.iters, lam=lam))
        _, rx_bits = d.hard_demod(d.unflatten(x, grid), const, grid)
        rec["y"].append(y)
        rec["taps"].append(taps)
        rec["lam"].append(lam)
        rec["tx"].append(tx_bits)
        rec["x"].append(x)
        rec["c_norm"].append(np.array(tr.c_norm))
        rec["rx"].append(rx_bits)
        rec["heff"].append(heff)
    return rec, const


def save_frames(name, d, rec, const, M, N, iters, x_dtype=np.complex128, keep_heff=False):
    b = const.bits_per_symbol
    off, k, l, g = pack_taps(rec["taps"])
    wts = 1 << np.arange(b - 1, -1, -1)
    tx_lab = np.stack([t.reshape(-1, b) @ wts for t in rec["tx"]]).astype(np.uint8)
    rx_lab = np.stack([t.reshape(-1, b) @ wts for t in rec["rx"]]).astype(np.uint8)
    out = dict(
        meta=np.array([M, N, iters, b], np.int64),
        y=np.stack(rec["y"]).astype(np.complex64),
        path_off=off, path_k=k, path_l=l, path_g=g,
        lam=np.array(rec["lam"]),
        tx_labels=tx_lab, rx_labels=rx_lab,
        x_ref=np.stack(rec["x"]).astype(x_dtype),
        c_norm=np.stack(rec["c_norm"]),
    )
    if keep_heff:
        out["heff"] = np.stack(rec["heff"])
    np.savez_compressed(OUT / f"{name}.npz", **out)


def frames_fixtures(d):
    # cfg1: M=64, N=16, 4 integer delay/Doppler paths, QPSK (BASELINE.json configs[0])
    def four_integer_paths(grid, rng):
        dn = grid.delta_nu
        paths = []
        for dly, dop, pw in ((0, 0, 1.0), (3, 1, 0.6), (7, -2, 0.35), (12, 3, 0.2)):
            ph = np.exp(2j * np.pi * rng.random())
            paths.append(d.make_path(pw * ph, dly / grid.B, dop * dn, grid))
        return d.PathSet(tuple(paths))

    rec, c = run_frames(d, 64, 16, "qpsk", 25.0, 0.0, 0.08, 10, 1, 8, four_integer_paths)
    save_frames("frames_cfg1", d, rec, c, 64, 16, 10, keep_heff=True)

    # cfg2: M=256, N=16, 4 paths with fractional Doppler, 16-QAM, 25 dB
    def four_fractional_paths(grid, rng):
        paths = []
        for dly_us, pw in ((0.0, 1.0), (0.31, 0.7), (0.71, 0.35), (1.09, 0.25)):
            nu = 300.0 * np.cos(2 * np.pi * rng.random())
            ph = np.exp(2j * np.pi * rng.random())
            paths.append(d.make_path(pw * ph, dly_us * 1e-6, nu, grid))
        return d.PathSet(tuple(paths))

    rec, c = run_frames(d, 256, 16, "qam16", 25.0, 0.0, 0.08, 10, 2, 4, four_fractional_paths)
    save_frames("frames_cfg2", d, rec, c, 256, 16, 10)

    # cfg3: M=512, N=32, Veh-A (6 paths, fractional Doppler), 16-QAM, 25 dB
    rec, c = run_frames(d, 512, 32, "qam16", 25.0, 100.0, 0.08, 10, 3, 2)
    save_frames("frames_cfg3", d, rec, c, 512, 32, 10)

    # cfg5: SNR sweep 0..30 dB at cfg3 (one frame per SNR)
    recs = {key: [] for key in ("y", "taps", "lam", "tx", "x", "c_norm", "rx", "heff")}
    for snr in (0.0, 5.0, 10.0, 15.0, 20.0, 25.0, 30.0):
        r, c = run_frames(d, 512, 32, "qam16", snr, 100.0, 0.08, 10, 5, 1)
        for key in recs:
            recs[key].extend(r[key])
    save_frames("frames_sweep", d, recs, c, 512, 32, 10, x_dtype=np.complex64)

    # cfg4: M=1024, N=64, high mobility (1000 Hz), equalizer parity with 16-QAM
    rec, c = run_frames(d, 1024, 64, "qam16", 25.0, 1000.0, 0.08, 10, 4, 1)
    save_frames("frames_cfg4", d, rec, c, 1024, 64, 10, x_dtype=np.complex64)


def detect_fixture(d):
    out = {}
    i = 0
    for (M, N, nu, snr, theta) in [(64, 16, 100.0, 25.0, 0.08), (128, 32, 500.0, 10.0, 0.03),
                                   (128, 32, 100.0, 30.0, 0.001), (32, 32, 100.0, 25.0, 0.08)]:
        rec, _ = run_frames(d, M, N, "qpsk", snr, nu, theta, 10, 9, 2)
        for heff in rec["heff"]:
            g = d.GridConfig(M, N)
            taps = d.detect_paths(heff, theta, g)
            p = f"c{i}_"
            out[p + "heff"] = heff
            out[p + "theta"] = np.array(theta)
            out[p + "k"] = np.array([t.k_p for t in taps], np.int32)
            out[p + "l"] = np.array([t.l_p for t in taps], np.int32)
            out[p + "g"] = np.array([t.gain for t in taps], np.complex128)
            i += 1
    out["n_cases"] = np.array(i)
    np.savez_compressed(OUT / "detect.npz", **out)


def frontend_fixture(d):
    """Receiver front end: run_packet's time-domain pilot
    and data frames with the reference's dzt_gemm / estimate_heff /
    detect_paths outputs and the full receive (harness.py:141-194), on the
    unrounded fp64 data path."""
    from ddlink.harness import Workspace
    out = {}
    cases = [("c1", 64, 16, "qpsk", 25.0, 300.0, 0.08, 31, 3), ("c3", 512, 32, "qam16", 25.0, 100.0, 0.08, 33, 1)]
    for tag, M, N, mod, snr, nu, theta, seed, count in cases:
        cfg = d.SimConfig(m=M, n=N, mod=mod, snr_db=snr, nu_max_hz=nu, theta=theta, iters=10, packets=count,
                          seed=seed)
        ws = Workspace(cfg)
        grid, const = ws.grid, ws.const
        rec = {k: [] for k in ("pilot_rx", "data_rx", "ypil", "heff", "y", "tx", "rx", "x", "taps")}
        for idx in range(count):
            rng = np.random.default_rng([seed, idx])
            pset = d.draw_veha(cfg.nu_max_hz, grid, rng)
            tx_bits = rng.integers(0, 2, size=const.bits_per_symbol * grid.size)
            data_tx = d.idzt(d.modulate(tx_bits, const, grid), grid)
            pilot_rx = d.add_awgn(d.apply_channel(ws.pilot_tx, pset, grid), cfg.snr_db, rng)
            data_rx = d.add_awgn(d.apply_channel(data_tx, pset, grid), cfg.snr_db, rng)
            ypil = d.dzt_gemm(pilot_rx, ws.zak_kernel, grid)
            heff = d.estimate_heff(ypil, ws.twist, grid)
            taps = d.detect_paths(heff, cfg.theta, grid)
            y = d.flatten(d.dzt_gemm(data_rx, ws.zak_kernel, grid), grid)
            lam = 1.0 / cfg.snr_linear
            x, _ = d.cga_equalize(d.build_ss_channel(taps, grid), y, d.CgaConfig(iterations=cfg.iters, lam=lam))
            _, rx_bits = d.hard_demod(d.unflatten(x, grid), const, grid)
            for key, v in (("pilot_rx", pilot_rx), ("data_rx", data_rx), ("ypil", ypil), ("heff", heff), ("y", y),
                           ("tx", tx_bits), ("rx", rx_bits), ("x", x), ("taps", taps)):
                rec[key].append(v)
        b = const.bits_per_symbol
        wts = 1 << np.arange(b - 1, -1, -1)
        off, k, l, g = pack_taps(rec["taps"])
        out[tag + "_meta"] = np.array([M, N, 10, b], np.int64)
        out[tag + "_theta"] = np.array(theta)
        out[tag + "_lam"] = np.full(count, 1.0 / cfg.snr_linear)
        for key in ("pilot_rx", "data_rx", "ypil", "heff", "y"):
            out[f"{tag}_{key}"] = np.stack(rec[key])
        out[tag + "_x"] = np.stack(rec["x"]).astype(np.complex64)
        out[tag + "_tx_labels"] = np.stack([t.reshape(-1, b) @ wts for t in rec["tx"]]).astype(np.uint8)
        out[tag + "_rx_labels"] = np.stack([t.reshape(-1, b) @ wts for t in rec["rx"]]).astype(np.uint8)
        out[tag + "_path_off"], out[tag + "_path_k"], out[tag + "_path_l"], out[tag + "_path_g"] = off, k, l, g
        # the reference kernel / twist tables and one half-shift kernel case for dzt_gemm
        out[tag + "_ypil_half"] = d.dzt_gemm(rec["pilot_rx"][0], d.build_zak_kernel(N, half_shift=True), grid)
    np.savez_compressed(OUT / "frontend.npz", **out)


def harness_fixture(d):
    """Acceptance criterion 6 of the reference (tests/test_acceptance.py:179-192):
    run_packets(SimConfig(m=32, n=32, packets=200, seed=11)), i.e. 200 QPSK
    packets at 25 dB, nu_max 100 Hz, theta 0.08, Xi 10.  Stores every packet's
    time-domain pilot and data frames in run_packet's draw order
    (harness.py:141-149), the TX labels, and the reference's own per-packet
    results from run_packets, so the device receiver can be scored against
    the reference's BER known answer (3.491e-4, test_output.txt:234)."""
    from ddlink.harness import Workspace
    cfg = d.SimConfig(m=32, n=32, packets=200, seed=11)
    ws = Workspace(cfg)
    grid, const = ws.grid, ws.const
    pil, dat, tx = [], [], []
    for idx in range(cfg.packets):
        rng = np.random.default_rng([cfg.seed, idx])
        pset = d.draw_veha(cfg.nu_max_hz, grid, rng)
        tx_bits = rng.integers(0, 2, size=const.bits_per_symbol * grid.size)
        data_tx = d.idzt(d.modulate(tx_bits, const, grid), grid)
        pil.append(d.add_awgn(d.apply_channel(ws.pilot_tx, pset, grid), cfg.snr_db, rng))
        dat.append(d.add_awgn(d.apply_channel(data_tx, pset, grid), cfg.snr_db, rng))
        tx.append(tx_bits)
    res = d.run_packets(cfg)
    b = const.bits_per_symbol
    wts = 1 << np.arange(b - 1, -1, -1)
    np.savez_compressed(
        OUT / "harness_c6.npz",
        meta=np.array([cfg.m, cfg.n, cfg.iters, b, cfg.packets], np.int64),
        snr_db=np.array(cfg.snr_db), theta=np.array(cfg.theta),
        pilot_rx=np.stack(pil), data_rx=np.stack(dat),
        tx_labels=np.stack([t.reshape(-1, b) @ wts for t in tx]).astype(np.uint8),
        bit_errors=np.array([r.bit_errors for r in res], np.int64),
        failed=np.array([r.failed for r in res], bool),
        ber=np.array([r.ber for r in res]),
    )


def channel_fixture(d):
    """Frame synthesis: the reference's draw_veha on seeded
    generators (channel.py:62-92), modulate (grid.py:157-169), idzt
    (zak.py:14-21) and the noiseless apply_channel (channel.py:95-103) on
    run_packet's data frames, at two grids with continuous Doppler."""
    out = {}
    for tag, M, N, mod, nu, seed, count in (("c1", 64, 16, "qpsk", 300.0, 41, 3), ("c3", 512, 32, "qam16", 100.0, 43, 2)):
        grid = d.GridConfig(M, N)
        const = d.make_constellation(mod)
        b = const.bits_per_symbol
        wts = 1 << np.arange(b - 1, -1, -1)
        rec = {k: [] for k in ("labels", "X", "x", "y")}
        pg, pd, pn, pk, off = [], [], [], [], [0]
        for idx in range(count):
            rng = np.random.default_rng([seed, idx])
            pset = d.draw_veha(nu, grid, rng)
            bits = rng.integers(0, 2, size=b * grid.size)
            X = d.modulate(bits, const, grid)
            x = d.idzt(X, grid)
            rec["labels"].append((bits.reshape(-1, b) @ wts).astype(np.uint8))
            rec["X"].append(d.flatten(X, grid))
            rec["x"].append(x)
            rec["y"].append(d.apply_channel(x, pset, grid))
            for p in pset.paths:
                pg.append(p.gain)
                pd.append(p.delay_s)
                pn.append(p.doppler_hz)
                pk.append(p.delay_bin)
            off.append(len(pg))
        out[tag + "_meta"] = np.array([M, N, b, seed, count], np.int64)
        out[tag + "_nu_max"] = np.array(nu)
        for key in rec:
            out[f"{tag}_{key}"] = np.stack(rec[key])
        out[tag + "_path_off"] = np.asarray(off, np.int32)
        out[tag + "_gain"] = np.asarray(pg, np.complex128)
        out[tag + "_delay_s"] = np.asarray(pd, np.float64)
        out[tag + "_doppler_hz"] = np.asarray(pn, np.float64)
        out[tag + "_delay_bin"] = np.asarray(pk, np.int32)
    np.savez_compressed(OUT / "channel.npz", **out)


def dense_fixture(d):
    """Dense LMMSE baseline: the reference's
    threshold_frame / build_dense_hdd / lmmse_equalize on estimated
    effective channels of small grids, and acceptance criterion 6's dense
    arm (run_packets with equalizer="lmmse" on the criterion's 200 packets,
    tests/test_acceptance.py:179-192; mean BER 3.662e-4, test_output.txt:234)."""
    from ddlink.harness import Workspace
    out = {}
    for tag, M, N, seed in (("s1", 16, 8, 51), ("s2", 32, 8, 52)):
        cfg = d.SimConfig(m=M, n=N, mod="qpsk", snr_db=20.0, nu_max_hz=300.0, theta=0.08, packets=1, seed=seed)
        ws = Workspace(cfg)
        grid = ws.grid
        rng = np.random.default_rng([seed, 0])
        pset = d.draw_veha(cfg.nu_max_hz, grid, rng)
        tx_bits = rng.integers(0, 2, size=2 * grid.size)
        data_tx = d.idzt(d.modulate(tx_bits, ws.const, grid), grid)
        pilot_rx = d.add_awgn(d.apply_channel(ws.pilot_tx, pset, grid), cfg.snr_db, rng)
        data_rx = d.add_awgn(d.apply_channel(data_tx, pset, grid), cfg.snr_db, rng)
        heff = d.estimate_heff(d.dzt_gemm(pilot_rx, ws.zak_kernel, grid), ws.twist, grid)
        thr = d.threshold_frame(heff, cfg.theta, grid)
        H = d.build_dense_hdd(thr, grid)
        y = d.flatten(d.dzt_gemm(data_rx, ws.zak_kernel, grid), grid)
        out[tag + "_meta"] = np.array([M, N], np.int64)
        out[tag + "_theta"] = np.array(cfg.theta)
        out[tag + "_snr_linear"] = np.array(cfg.snr_linear)
        out[tag + "_heff"] = heff
        out[tag + "_thr"] = thr
        out[tag + "_H"] = H
        out[tag + "_y"] = y
        out[tag + "_x"] = d.lmmse_equalize(H, y, cfg.snr_linear)
    cfg = d.SimConfig(m=32, n=32, packets=200, seed=11, equalizer="lmmse")
    res = d.run_packets(cfg)
    out["c6_bit_errors"] = np.array([r.bit_errors for r in res], np.int64)
    out["c6_failed"] = np.array([r.failed for r in res], bool)
    out["c6_ber"] = np.array([r.ber for r in res])
    np.savez_compressed(OUT / "dense.npz", **out)


def sweep_fixture(d):
    """Config 5 (BASELINE.json configs[4]): SNR 0..30 dB in 5 dB steps, 64
    run_packet packets per SNR at (512, 32), 16-QAM (tests/golden/ref_sweep.py).
    Stores the reference's compact per-packet results -- taps, bit errors on
    the fp64 frame and on its complex64 rounding, residual traces -- so the GPU
    box's own reference run is checked against this container's."""
    sys.path.insert(0, str(OUT))
    import ref_sweep as rs
    res = rs.run_all([str(REF)], keep_frames=False)
    keys = sorted(res)
    taps = [res[k] for k in keys]
    off = np.concatenate([[0], np.cumsum([t["P"] for t in taps])]).astype(np.int32)
    np.savez_compressed(
        OUT / "sweep_cfg5.npz",
        meta=np.array([rs.M, rs.N, rs.ITERS, rs.SEED, rs.PACKETS], np.int64),
        snr=np.array([k[0] for k in keys]), idx=np.array([k[1] for k in keys], np.int32),
        path_off=off,
        path_k=np.concatenate([t["tap_k"] for t in taps]).astype(np.int32),
        path_l=np.concatenate([t["tap_l"] for t in taps]).astype(np.int32),
        path_g=np.concatenate([t["tap_g"] for t in taps]),
        errors=np.array([t["errors"] for t in taps], np.int64),
        errors32=np.array([t["errors32"] for t in taps], np.int64),
        failed=np.array([t["failed"] for t in taps], bool),
        c_norm=np.stack([t["c_norm"] for t in taps]),
        c_norm32=np.stack([t["c_norm32"] for t in taps]),
    )


def main():
    d = _ref()
    if len(sys.argv) > 1:  # regenerate selected fixtures only, e.g. `make_golden.py frontend`
        for name in sys.argv[1:]:
            globals()[f"{name}_fixture"](d)
        return
    tables_fixture(d)
    cga_fixture(d)
    demod_fixture(d)
    detect_fixture(d)
    frames_fixtures(d)
    frontend_fixture(d)
    harness_fixture(d)
    channel_fixture(d)
    dense_fixture(d)
    sweep_fixture(d)
    for p in sorted(OUT.glob("*.npz")):
        print(f"{p.name:24s} {p.stat().st_size / 1024:8.1f} KiB")


if __name__ == "__main__":
    main()
