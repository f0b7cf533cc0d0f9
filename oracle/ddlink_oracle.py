"""CPU oracle for the SS-CGA hot path — TEST INFRASTRUCTURE ONLY.

A float64 numpy restatement of the reference package's algorithm
(/root/reference/pkg/src/ddlink, "ddlink" 0.1.0).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this module, and only as the checker or the timed CPU baseline —
never as part of the product path (paper_2604_02266_b200 never imports it).

Parity status: PINNED.  tests/test_oracle.py checks every function here
against golden vectors produced by running the reference itself
(tests/golden/make_golden.py, committed with its outputs), plus the
reference's own worked examples (tests/test_sparse.py:49-55 of the reference).

Each function cites the reference file:line it restates.  The hot path
 is:
    detect_paths -> build_tables -> cga -> hard_demod
and the receiver front end before it (section 8f row f1):
    dzt_gemm (pilot, data) -> estimate_heff
and the frame synthesis that feeds it (section 8f row f2):
    modulate_labels -> idzt -> apply_channel
and the dense cross-check (section 8f row f4):
    threshold_frame -> dense_channel -> lmmse
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------
# grid geometry (grid.py:14-95)


def check_grid(M: int, N: int) -> None:
    """GridConfig validation (grid.py:23-31)."""
    if M < 2 or N < 2:
        raise ValueError(f"grid must be at least 2x2, got ({M},{N})")
    if M % 2 or N % 2:
        raise ValueError(f"M and N must be even, got ({M},{N})")


def to_vector(frame: np.ndarray) -> np.ndarray:
    """Column-major vectorisation q = l*M + k (grid.py:86-89)."""
    return np.asarray(frame).T.reshape(-1).copy()


def to_frame(vec: np.ndarray, M: int, N: int) -> np.ndarray:
    """Inverse of to_vector (grid.py:92-95)."""
    return np.asarray(vec).reshape(N, M).T.copy()


# --------------------------------------------------------------------------
# constellations (grid.py:98-154)


def axis_levels(bits_per_axis: int) -> np.ndarray:
    """Gray PAM levels indexed by the axis bits read MSB first.

    grid.py:98-109 for 1 and 2 bits per axis; 3 bits (64-QAM) follows the same
    TS 38.211 recursion and is a build extension (the reference raises).
    """
    if bits_per_axis not in (1, 2, 3):
        raise ValueError("bits_per_axis must be 1, 2 or 3")
    out = np.empty(1 << bits_per_axis)
    for idx in range(out.size):
        bits = [(idx >> (bits_per_axis - 1 - i)) & 1 for i in range(bits_per_axis)]
        mag = 1
        for m in range(bits_per_axis - 1, 0, -1):
            mag = (1 << (bits_per_axis - m)) - (1 - 2 * bits[m]) * mag
        out[idx] = (1 - 2 * bits[0]) * mag
    return out


@dataclass(frozen=True)
class Qam:
    name: str
    points: np.ndarray      # complex128 [2**b], unit mean energy
    bit_map: np.ndarray     # int8 [2**b, b], MSB first
    bits_per_symbol: int


def qam(name: str) -> Qam:
    """make_constellation (grid.py:126-154) + 64-QAM extension."""
    key = name.lower().replace("-", "").replace("_", "")
    per_axis = {"qpsk": 1, "qam16": 2, "16qam": 2, "qam64": 3, "64qam": 3}.get(key)
    if per_axis is None:
        raise ValueError(f"unknown constellation {name!r}")
    b = 2 * per_axis
    lv = axis_levels(per_axis)
    labels = np.arange(1 << b)
    bit_map = ((labels[:, None] >> np.arange(b - 1, -1, -1)[None, :]) & 1).astype(np.int8)
    i_idx = np.zeros(labels.size, dtype=int)
    q_idx = np.zeros(labels.size, dtype=int)
    for pos in range(b):
        if pos % 2 == 0:
            i_idx = (i_idx << 1) | bit_map[:, pos]
        else:
            q_idx = (q_idx << 1) | bit_map[:, pos]
    pts = lv[i_idx] + 1j * lv[q_idx]
    pts = pts / np.sqrt(np.mean(np.abs(pts) ** 2))
    return Qam(key, pts, bit_map, b)


def modulate_labels(labels: np.ndarray, const: Qam) -> np.ndarray:
    """Labels -> symbols in q order (grid.py:157-169 without the bit grouping)."""
    return const.points[np.asarray(labels)]


def labels_from_bits(bits: np.ndarray, b: int) -> np.ndarray:
    """MSB-first bit groups -> integer labels (grid.py:166-168)."""
    g = np.asarray(bits, dtype=np.int64).reshape(-1, b)
    return g @ (1 << np.arange(b - 1, -1, -1))


def hard_demod(x_vec: np.ndarray, const: Qam):
    """Nearest point, lowest label on ties (grid.py:172-183).

    Returns (labels, bits int64 [b * len]).
    """
    v = np.asarray(x_vec).reshape(-1)
    dist = np.abs(v[:, None] - const.points[None, :]) ** 2
    lab = np.argmin(dist, axis=1)
    return lab, const.bit_map[lab].reshape(-1).astype(np.int64)


def decision_margin(x_vec: np.ndarray, const: Qam) -> np.ndarray:
    """Second-smallest minus smallest squared distance per symbol (tie band)."""
    v = np.asarray(x_vec).reshape(-1)
    dist = np.sort(np.abs(v[:, None] - const.points[None, :]) ** 2, axis=1)
    return dist[:, 1] - dist[:, 0]


def llr_maxlog(x_vec: np.ndarray, const: Qam, noise_var: float) -> np.ndarray:
    """Build-defined max-log LLR (absent in the reference).

    llr[s, i] = (min_{c: bit_i=1} |x-c|^2 - min_{c: bit_i=0} |x-c|^2) / noise_var,
    so llr > 0 favours bit 0 and (llr < 0) reproduces hard_demod's bits.
    """
    v = np.asarray(x_vec).reshape(-1)
    dist = np.abs(v[:, None] - const.points[None, :]) ** 2
    out = np.empty((v.size, const.bits_per_symbol))
    for i in range(const.bits_per_symbol):
        one = const.bit_map[:, i] == 1
        out[:, i] = dist[:, one].min(axis=1) - dist[:, ~one].min(axis=1)
    scale = 1.0 / noise_var if noise_var > 0 else 1.0
    return out * scale


# --------------------------------------------------------------------------
# receiver front end (zak.py:33-55, pilot.py:13-49) — SURVEY.md 8f row f1


def zak_kernel(N: int, half_shift: bool = False) -> np.ndarray:
    """kernel[i, l] = e^{-j2pi i l/N} / sqrt(N), optional (-1)^l columns (zak.py:33-47)."""
    n = np.arange(N)
    k = np.exp(-2j * np.pi * np.outer(n, n) / N) / np.sqrt(N)
    if half_shift:
        k = k * np.where(n % 2, -1.0, 1.0)[None, :]
    return k


def dzt_gemm(y: np.ndarray, M: int, N: int, kernel: np.ndarray | None = None) -> np.ndarray:
    """Received samples (index k + i*M) -> (M, N) DD frame, one GEMM (zak.py:50-55)."""
    kernel = zak_kernel(N) if kernel is None else kernel
    return np.asarray(y).reshape(M, N, order="F") @ kernel


def twist_kernel(M: int, N: int) -> np.ndarray:
    """e^{-j2pi K0 (l - L0) / MN}, constant along delay (pilot.py:29-37)."""
    l = np.arange(N)
    return np.broadcast_to(np.exp(-2j * np.pi * (M // 2) * (l - N // 2) / (M * N)), (M, N))


def estimate_heff(Y_dd: np.ndarray, M: int, N: int, amplitude: float | None = None) -> np.ndarray:
    """Y_dd * twist / amplitude, amplitude defaulting to sqrt(MN) (pilot.py:13-15, 40-49)."""
    amp = math.sqrt(M * N) if amplitude is None else amplitude
    return Y_dd * twist_kernel(M, N) / amp


# --------------------------------------------------------------------------
# frame synthesis (zak.py:14-21, channel.py:95-103) — SURVEY.md 8f row f2


def idzt(X_vec: np.ndarray, M: int, N: int) -> np.ndarray:
    """Flattened DD vector (q = l*M + k) -> time samples k + n*M:
    x[k + nM] = (1/sqrt N) sum_l X[k, l] e^{+j2pi n l/N} (zak.py:14-21)."""
    X = np.asarray(X_vec).reshape(M, N, order="F")
    return (X @ np.conj(zak_kernel(N))).reshape(M * N, order="F")


def apply_channel(x: np.ndarray, gains, delay_s, doppler_hz, delay_bin, bandwidth: float) -> np.ndarray:
    """Noiseless channel y[i] = sum_p h_p x[(i - k_p) mod MN] e^{j2pi nu_p (i/B - tau_p)}
    (channel.py:95-103)."""
    x = np.asarray(x, dtype=np.complex128)
    i = np.arange(x.size)
    y = np.zeros(x.size, dtype=np.complex128)
    for h, tau, nu, k in zip(gains, delay_s, doppler_hz, delay_bin):
        y += h * np.roll(x, int(k)) * np.exp(2j * np.pi * nu * (i / bandwidth - tau))
    return y


# --------------------------------------------------------------------------
# dense LMMSE baseline (sparse.py:163-206, equalize.py:80-94) — SURVEY.md 8f row f4


def threshold_frame(heff: np.ndarray, theta: float) -> np.ndarray:
    """Keep bins with |h| > theta * peak, all of them if the peak is 0 (sparse.py:163-169)."""
    mags = np.abs(heff)
    peak = mags.max()
    return np.where(mags > theta * peak, heff, 0.0) if peak > 0 else np.array(heff, copy=True)


def dense_channel(heff: np.ndarray, M: int, N: int) -> np.ndarray:
    """MN x MN DD channel matrix of an effective-channel frame (sparse.py:172-206):
    entry (l'M + k', lM + k) = heff[K0 + dk, L0 + dl] e^{j2pi (dl (k + nM) / MN + n l / N)}
    with the unique wraps n, m that bring (dk, dl) into the signed fundamental range."""
    MN, K0, L0 = M * N, M // 2, N // 2
    q = np.arange(MN)
    kc, lc = q % M, q // M
    kr, lr = kc[:, None], lc[:, None]
    n = (kr - kc[None, :] + K0) // M
    m = (lr - lc[None, :] + L0) // N
    dk = kr - kc[None, :] - n * M
    dl = lr - lc[None, :] - m * N
    ph = np.exp(2j * np.pi * (dl * (kc[None, :] + n * M) / MN + n * lc[None, :] / N))
    return heff[K0 + dk, L0 + dl] * ph


def lmmse(H: np.ndarray, y: np.ndarray, lam: float) -> np.ndarray:
    """(H^H H + lam I)^{-1} H^H y by a Cholesky solve (equalize.py:80-94)."""
    g = H.conj().T @ H + lam * np.eye(H.shape[1])
    L = np.linalg.cholesky(g)
    z = np.linalg.solve(L, H.conj().T @ y)
    return np.linalg.solve(L.conj().T, z)


# --------------------------------------------------------------------------
# structured-sparse operator (sparse.py:27-160)


@dataclass(frozen=True)
class Tap:
    k: int
    l: int
    gain: complex


def detect_paths(heff: np.ndarray, theta: float) -> list[Tap]:
    """Strict relative threshold, stable descending |h| (sparse.py:69-88)."""
    if theta < 0:
        raise ValueError("theta must be nonnegative")
    h = np.asarray(heff)
    mag = np.abs(h)
    peak = mag.max()
    if peak == 0.0:
        return []
    flat = np.flatnonzero(mag.reshape(-1) > theta * peak)   # row-major (k, l) order
    order = np.argsort(-mag.reshape(-1)[flat], kind="stable")
    n = h.shape[1]
    return [Tap(int(i // n), int(i % n), complex(h.reshape(-1)[i])) for i in flat[order]]


def tap_offsets(tap: Tap, M: int, N: int) -> tuple[int, int]:
    """(d_k, d_l) = (K0 - k_p, L0 - l_p) (sparse.py:35-37)."""
    return M // 2 - tap.k, N // 2 - tap.l


def forward_source(tap: Tap, q, M: int, N: int):
    """Input index feeding output q: 2D circular shift (sparse.py:91-96)."""
    dk, dl = tap_offsets(tap, M, N)
    q = np.asarray(q)
    return ((q // M + dl) % N) * M + (q % M + dk) % M


def inverse_source(tap: Tap, r, M: int, N: int):
    """Output fed by input r (sparse.py:99-104)."""
    dk, dl = tap_offsets(tap, M, N)
    r = np.asarray(r)
    return ((r // M - dl) % N) * M + (r % M - dk) % M


def tap_coefficient(tap: Tap, q, M: int, N: int):
    """h_p exp(j phi), phi = 2 pi / MN [(l_p - L0) a + n l_img M] (sparse.py:107-121)."""
    q = np.asarray(q)
    k_q, l_q = q % M, q // M
    a = M // 2 + k_q - tap.k
    wrap = np.floor_divide(a, M)
    l_img = (N // 2 + l_q - tap.l) % N
    phase_idx = (tap.l - N // 2) * a + wrap * l_img * M
    return tap.gain * np.exp(1j * (2.0 * np.pi / (M * N)) * phase_idx)


@dataclass(frozen=True)
class Tables:
    M: int
    N: int
    taps: tuple
    fwd_coef: np.ndarray
    fwd_col: np.ndarray
    herm_coef: np.ndarray
    herm_row: np.ndarray


class EmptyChannel(Exception):
    """No taps survived thresholding (sparse.py:23-24)."""


def build_tables(taps, M: int, N: int) -> Tables:
    """Path-major forward/Hermitian tables (sparse.py:124-144)."""
    taps = tuple(taps)
    if not taps:
        raise EmptyChannel("no taps above threshold")
    q = np.arange(M * N)
    fc = np.stack([tap_coefficient(t, q, M, N) for t in taps]).astype(complex)
    fi = np.stack([forward_source(t, q, M, N) for t in taps]).astype(np.int32)
    hr = np.stack([inverse_source(t, q, M, N) for t in taps]).astype(np.int32)
    hc = np.conj(np.take_along_axis(fc, hr.astype(np.int64), axis=1))
    return Tables(M, N, taps, fc, fi, hc, hr)


def apply_tables(coef: np.ndarray, index: np.ndarray, v: np.ndarray) -> np.ndarray:
    """u[q] = sum_p coef[p, q] v[index[p, q]] (sparse.py:147-160)."""
    v = np.asarray(v)
    if v.shape != (coef.shape[1],):
        raise ValueError(f"vector length {v.shape} != {coef.shape[1]}")
    return (coef * v[index]).sum(axis=0)


def forward(t: Tables, v):
    return apply_tables(t.fwd_coef, t.fwd_col, v)


def adjoint(t: Tables, v):
    return apply_tables(t.herm_coef, t.herm_row, v)


# --------------------------------------------------------------------------
# conjugate gradient (equalize.py:14-77)


@dataclass
class Trace:
    c_norm: list = field(default_factory=list)
    mvm_count: int = 0
    exact_converged: bool = False
    snapshots: list = field(default_factory=list)


def cga(t: Tables, y, iterations: int, lam: float = 0.0, profile: bool = False):
    """Fixed-iteration CG on (H^H H + lam I) x = H^H y (equalize.py:43-77)."""
    if iterations < 1:
        raise ValueError("need at least one iteration")
    if lam < 0:
        raise ValueError("lam must be nonnegative")
    tr = Trace()
    rhs = adjoint(t, np.asarray(y))
    tr.mvm_count = 1
    x = np.zeros_like(rhs)
    r = rhs.copy()
    d = rhs.copy()
    rr = float(np.vdot(r, r).real)
    tr.c_norm.append(rr)
    for _ in range(iterations):
        ad = adjoint(t, forward(t, d))
        tr.mvm_count += 2
        if lam:
            ad = ad + lam * d
        curv = float(np.vdot(d, ad).real)
        if curv == 0.0:
            tr.exact_converged = True
            break
        step = rr / curv
        x = x + step * d
        r = r - step * ad
        rr_new = float(np.vdot(r, r).real)
        d = r + (rr_new / rr) * d
        rr = rr_new
        tr.c_norm.append(rr)
        if profile:
            tr.snapshots.append(x.copy())
    return x, tr


def lam_from_snr(snr_db: float) -> float:
    """harness.py:85-87, 188: lam = 1/SNR_linear, 0 when noiseless."""
    return 0.0 if math.isinf(snr_db) else 1.0 / (10.0 ** (snr_db / 10.0))


# --------------------------------------------------------------------------
# the timed receiver hot path of harness.py:159-194


def receive(taps, y_vec, M: int, N: int, iterations: int, lam: float, const: Qam):
    """build_ss_channel -> cga_equalize -> hard_demod for one data frame."""
    t = build_tables(taps, M, N)
    x, tr = cga(t, y_vec, iterations, lam)
    lab, bits = hard_demod(x, const)
    return x, tr, lab, bits


def flop_count(P: int, MN: int, iterations: int) -> int:
    """Algorithmic FLOPs of one frame: complex MAC = 8 FLOP."""
    return 8 * P * MN * (2 * iterations + 1) + 24 * MN * iterations + 4 * MN
