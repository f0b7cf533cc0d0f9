"""Synthetic frame batches for benchmarks and full-size property tests.

Taps follow the reference's Veh-A geometry (channel.py:17-18, 62-85): six
paths with the ITU delays rounded to delay bins (channel.py:46) and unit total
power, uniform phases, Doppler nu_max cos(2 pi U) rounded to the Doppler grid,
placed on the absolute grid at (K0 + delay, L0 + doppler) like the pilot
estimate (pilot.py:1-6).  Data are uniform random constellation labels; the
received vector is y = H x + n computed with the device operator
(ddb_ss_apply), n ~ CN(0, mean|Hx|^2 / SNR) as in add_awgn (channel.py:99-111).
Everything is generated on the GPU with torch's RNG (this is input
generation, not the measured path).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .batch import PathBatch, SsCgaSolver
from .grid import GridConfig, make_constellation_ext

VEHA_DELAYS_US = (0.00, 0.31, 0.71, 1.09, 1.73, 2.51)
VEHA_POWERS_DB = (0.0, -1.0, -9.0, -10.0, -15.0, -20.0)


@dataclass
class FrameBatch:
    y: torch.Tensor          # [B, MN] complex
    x: torch.Tensor          # [B, MN] complex transmitted symbols
    tx_labels: torch.Tensor  # uint8 [B, MN]
    paths: PathBatch
    lam: torch.Tensor        # [B] real
    snr_db: float


def veha_paths(B: int, grid: GridConfig, nu_max_hz: float, gen: torch.Generator, device,
               cdtype=torch.complex64, n_paths: int = 6, delay_scale: float = 1.0) -> PathBatch:
    # beyond the six Veh-A paths, extra taps model fractional-Doppler leakage:
    # the same delays one Doppler bin away, 25 dB down (analysis / stress only)
    base = np.asarray(VEHA_DELAYS_US)
    idx = np.arange(n_paths) % len(base)
    # delay_scale != 1 compresses the delay profile (kernel analysis only)
    delays = np.round(base[idx] * delay_scale * 1e-6 * grid.B).astype(np.int64)
    if delays.max() >= grid.M:
        raise ValueError("Veh-A delay spread exceeds the delay period; increase M")
    pdb = np.where(np.arange(n_paths) < len(base), np.asarray(VEHA_POWERS_DB)[idx], -25.0)
    powers = 10.0 ** (pdb / 10.0)
    mags = torch.as_tensor(np.sqrt(powers / powers.sum()), device=device, dtype=torch.float64)
    phase = torch.rand(B, n_paths, generator=gen, device=device, dtype=torch.float64) * 2 * np.pi
    u = torch.rand(B, n_paths, generator=gen, device=device, dtype=torch.float64)
    dop = torch.round(nu_max_hz * torch.cos(2 * np.pi * u) / grid.delta_nu).to(torch.int64)
    leak = torch.as_tensor((np.arange(n_paths) >= len(base)).astype(np.int64), device=device)
    dop = (dop + leak[None, :]).clamp(-(grid.N // 2) + 1, grid.N // 2 - 1)
    k = (grid.K0 + torch.as_tensor(delays, device=device)[None, :]).expand(B, n_paths) % grid.M
    l = (grid.L0 + dop) % grid.N
    gain = torch.polar(mags[None, :].expand(B, n_paths), phase)
    off = torch.arange(0, (B + 1) * n_paths, n_paths, device=device, dtype=torch.int32)
    return PathBatch(off, k.reshape(-1).to(torch.int32).contiguous(), l.reshape(-1).to(torch.int32).contiguous(),
                     gain.reshape(-1).to(cdtype).contiguous())


def random_paths(B: int, M: int, N: int, P: int, seed: int, cdtype=torch.complex64, device="cuda") -> PathBatch:
    """SURVEY.md 8(d)(3)'s kernel-benchmark taps: per frame a dominant unit tap
    plus P - 1 taps of magnitude U(0.05, 0.2) and uniform phase, all at
    distinct uniformly random (k, l) bins (tests/test_acceptance.py:40-50,
    random_tap_frame).  Benchmark input generation only (host numpy)."""
    rng = np.random.default_rng(seed)
    k = np.empty((B, P), np.int32)
    l = np.empty((B, P), np.int32)
    g = np.empty((B, P), np.complex128)
    for f in range(B):
        bins = rng.choice(M * N, P, replace=False)
        k[f], l[f] = bins // N, bins % N
        g[f, 0] = 1.0
        g[f, 1:] = rng.uniform(0.05, 0.2, P - 1) * np.exp(2j * np.pi * rng.random(P - 1))
    off = np.arange(0, (B + 1) * P, P, dtype=np.int32)
    return PathBatch.from_arrays(off, k.reshape(-1), l.reshape(-1), g.reshape(-1), device, cdtype)


def cycle_paths(B: int, offsets, k, l, gain, device, cdtype) -> PathBatch:
    """B frames whose tap sets cycle through the given CSR tap sets (e.g. the
    reference's detect_paths output on fractional-Doppler Veh-A channels)."""
    offsets, k, l, gain = (np.asarray(v) for v in (offsets, k, l, gain))
    F = len(offsets) - 1
    sets = [slice(int(offsets[i]), int(offsets[i + 1])) for i in range(F)]
    ks, ls, gs, off = [], [], [], [0]
    for b in range(B):
        sl = sets[b % F]
        ks.append(k[sl])
        ls.append(l[sl])
        gs.append(gain[sl])
        off.append(off[-1] + (sl.stop - sl.start))
    return PathBatch.from_arrays(off, np.concatenate(ks), np.concatenate(ls), np.concatenate(gs), device, cdtype)


def make_frames(solver: SsCgaSolver, B: int, snr_db: float = 25.0, nu_max_hz: float = 100.0,
                modulation: str = "qam16", seed: int = 0, n_paths: int = 6, delta_f: float = 30e3,
                paths: PathBatch | None = None, delay_scale: float = 1.0) -> FrameBatch:
    """paths: use these taps instead of drawing Veh-A ones."""
    dev = solver.device
    grid = GridConfig(solver.M, solver.N, delta_f)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    const = make_constellation_ext(modulation)
    pts = torch.as_tensor(np.array(const.points), device=dev).to(solver.cdtype)
    labels = torch.randint(0, len(const.points), (B, solver.MN), generator=gen, device=dev, dtype=torch.int64)
    x = pts[labels].contiguous()
    if paths is None:
        paths = veha_paths(B, grid, nu_max_hz, gen, dev, solver.cdtype, n_paths, delay_scale)
    hx = solver.apply(x, paths)
    if np.isinf(snr_db):
        y = hx
        lam = torch.zeros(B, dtype=solver.rdtype, device=dev)
    else:
        snr = 10.0 ** (snr_db / 10.0)
        power = (hx.real ** 2 + hx.imag ** 2).mean(dim=1, keepdim=True)
        sigma = torch.sqrt(power / snr / 2)
        noise = torch.complex(torch.randn(B, solver.MN, generator=gen, device=dev, dtype=solver.rdtype),
                              torch.randn(B, solver.MN, generator=gen, device=dev, dtype=solver.rdtype))
        y = (hx + sigma * noise).contiguous()
        lam = torch.full((B,), 1.0 / snr, dtype=solver.rdtype, device=dev)
    return FrameBatch(y=y, x=x, tx_labels=labels.to(torch.uint8).contiguous(), paths=paths, lam=lam,
                      snr_db=snr_db)


def time_domain_frames(solver: SsCgaSolver, fb: FrameBatch, seed: int = 1) -> tuple[torch.Tensor, torch.Tensor]:
    """Received pilot and data frames in the time domain for the batched receiver
    (`SsCgaSolver.receive`), from a DD-domain FrameBatch: the point pilot of
    pilot.py:18-26 through the same channel plus AWGN at the frame's SNR, and
    both frames taken to the time domain by the inverse Zak transform
    x[k + nM] = (1/sqrt N) sum_l X[k, l] e^{+j2pi n l/N} (zak.py:14-21), i.e.
    ddb_dzt with the conjugate kernel.  The transform is unitary, so the AWGN
    statistics are the DD domain's.  Benchmark input generation only."""
    from .zak import build_zak_kernel, dzt_device
    dev, B, M, N, MN = solver.device, fb.y.shape[0], solver.M, solver.N, solver.MN
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    pil = torch.zeros(B, MN, dtype=solver.cdtype, device=dev)
    pil[:, (N // 2) * M + M // 2] = float(np.sqrt(MN))
    hp = solver.apply(pil, fb.paths)
    if not np.isinf(fb.snr_db):
        snr = 10.0 ** (fb.snr_db / 10.0)
        sigma = torch.sqrt((hp.real ** 2 + hp.imag ** 2).mean(dim=1, keepdim=True) / snr / 2)
        hp = hp + sigma * torch.complex(torch.randn(B, MN, generator=gen, device=dev, dtype=solver.rdtype),
                                        torch.randn(B, MN, generator=gen, device=dev, dtype=solver.rdtype))
    kinv = torch.as_tensor(np.conj(build_zak_kernel(N)), device=dev).to(solver.cdtype)
    pilot_rx = dzt_device(hp.contiguous(), M, N, kernel=kinv, colmajor=True)
    data_rx = dzt_device(fb.y, M, N, kernel=kinv, colmajor=True)
    return pilot_rx, data_rx


@dataclass
class PacketBatch:
    """Time-domain received pilot and data frames of a packet batch (the
    channel side of run_packet, harness.py:141-149), all on the device."""

    pilot_rx: torch.Tensor    # [B, MN] complex, time samples k + n M
    data_rx: torch.Tensor     # [B, MN] complex
    tx_labels: torch.Tensor   # uint8 [B, MN] (label of DD symbol q = l M + k)
    channel: "ChannelBatch"   # physical paths (fractional Doppler)
    lam: torch.Tensor         # [B] real, 1/SNR (0 when noiseless)
    snr_db: float


def synthesize_packets(solver: SsCgaSolver, B: int, snr_db: float = 25.0, nu_max_hz: float = 100.0,
                       modulation: str = "qam16", seed: int = 0, delta_f: float = 30e3,
                       cdtype=torch.complex128) -> PacketBatch:
    """B packets through Veh-A channels with continuous Doppler, generated on
    the GPU with the ddb synthesis kernels:
    labels -> modulate (grid.py:157-169) -> idzt (zak.py:14-21) ->
    apply_channel (channel.py:95-103) -> add_awgn (channel.py:106-119), and the
    same channel and noise level for the point pilot (pilot.py:18-26), as
    run_packet does per packet.  Fractional Doppler leaks into neighbouring
    Doppler bins, so detect_paths finds more taps than paths, as it does for
    the reference.  The RNG streams are the device's, not numpy's."""
    from .channel import add_awgn_device, apply_channel_device, draw_veha_batch, idzt_device, modulate_device
    from .grid import make_constellation_ext
    dev = solver.device
    M, N, MN = solver.M, solver.N, solver.MN
    grid = GridConfig(M, N, delta_f)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    bps = make_constellation_ext(modulation).bits_per_symbol
    labels = torch.randint(0, 1 << bps, (B, MN), generator=gen, device=dev, dtype=torch.uint8)
    ch = draw_veha_batch(B, grid, nu_max_hz, gen, dev, cdtype)
    data_tx = idzt_device(modulate_device(labels, bps, cdtype), M, N)
    pil_dd = torch.zeros(1, MN, dtype=cdtype, device=dev)
    pil_dd[0, grid.L0 * M + grid.K0] = float(np.sqrt(MN))
    pilot_tx = idzt_device(pil_dd, M, N).expand(B, MN).contiguous()
    s0 = int(torch.randint(0, 2 ** 62, (1,), generator=gen, device=dev).item())
    pilot_rx = add_awgn_device(apply_channel_device(pilot_tx, ch, grid), snr_db, s0)
    data_rx = add_awgn_device(apply_channel_device(data_tx, ch, grid), snr_db, s0 + 1)
    lam = torch.full((B,), 0.0 if np.isinf(snr_db) else 10.0 ** (-snr_db / 10.0), dtype=solver.rdtype,
                     device=dev)
    return PacketBatch(pilot_rx, data_rx, labels, ch, lam, snr_db)
