"""CPU checks of the device harness's host logic (row f3) against the reference:
configuration validation and messages (harness.py:38-87), the statistics
and CSV row (235-274), sweep axes (277-292) -- and the config-5 sweep fixture
against a fresh run of the reference when it is importable here."""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
BASE = ROOT / "baseline" / "_ref"
sys.path.insert(0, str(ROOT))

from paper_2604_02266_b200 import harness as hz  # noqa: E402


def _ref():
    if not (BASE / "ddlink" / "__init__.py").exists():
        pytest.skip("baseline/_ref absent")
    if str(BASE) not in sys.path:
        sys.path.insert(0, str(BASE))
    import ddlink
    return ddlink


BAD = [dict(mod="bpsk"), dict(equalizer="zf"), dict(packets=0), dict(iters=0), dict(theta=-1.0),
       dict(nu_max_hz=-1.0), dict(deadline_frames=0.0), dict(workers=0), dict(m=31)]


@pytest.mark.parametrize("kw", BAD)
def test_simconfig_errors_match_reference(kw):
    d = _ref()
    with pytest.raises(ValueError) as ours:
        hz.SimConfig(**kw)
    with pytest.raises(ValueError) as theirs:
        d.SimConfig(**kw)
    if "mod" not in kw:  # the build adds qam64 to the modulation list
        assert str(ours.value) == str(theirs.value)


def test_properties_stats_and_rows_match_reference():
    d = _ref()
    from ddlink import harness as rh
    cfg, rcfg = hz.SimConfig(m=64, n=16, snr_db=12.0), d.SimConfig(m=64, n=16, snr_db=12.0)
    assert cfg.deadline_s == rcfg.deadline_s and cfg.snr_linear == rcfg.snr_linear
    assert math.isinf(hz.SimConfig(snr_db=math.inf).snr_linear)
    rng = np.random.default_rng(3)
    mk = [dict(ber=float(b), bits_total=128, bit_errors=int(b * 128), time_dzt_s=t, time_est_s=t, time_build_s=t,
               time_eq_s=t, time_demod_s=t, pilot_time_s=t, data_time_s=2 * t, deadline_met=True)
          for b, t in zip(rng.random(50) * 0.1, rng.random(50) * 1e-3)]
    ours = [hz.PacketResult(**k) for k in mk]
    theirs = [rh.PacketResult(**k) for k in mk]
    import dataclasses
    assert (dataclasses.astuple(hz.latency_stats(ours, cfg.deadline_s))
            == dataclasses.astuple(rh.latency_stats(theirs, rcfg.deadline_s)))
    assert hz.aggregate(cfg, ours) == rh.aggregate(rcfg, theirs)
    assert hz.CSV_COLUMNS == rh.CSV_COLUMNS
    for axis, v in (("snr", 3), ("nu_max", 5), ("m", 128), ("theta", 0.1)):
        assert hz.apply_axis(cfg, axis, v).__dict__ == rh.apply_axis(rcfg, axis, v).__dict__
    with pytest.raises(ValueError):
        hz.apply_axis(cfg, "m", 12.5)
    with pytest.raises(ValueError):
        hz.apply_axis(cfg, "bogus", 1)
    assert hz.throughput_mbps(cfg, 0.01) == rh.throughput_mbps(rcfg, 0.01)


def test_sweep_fixture_matches_reference_spot_packets():
    """tests/golden/sweep_cfg5.npz (config 5) against the reference, 3 packets."""
    _ref()
    sys.path.insert(0, str(ROOT / "tests" / "golden"))
    import ref_sweep as rs
    import ddlink
    with np.load(ROOT / "tests" / "golden" / "sweep_cfg5.npz") as z:
        fx = {k: z[k] for k in z.files}
    for snr, idx in ((0.0, 3), (15.0, 17), (30.0, 63)):
        j = int(np.nonzero((fx["snr"] == snr) & (fx["idx"] == idx))[0][0])
        r = rs.reference_packet(ddlink, snr, idx, keep_frames=False)
        assert r["errors"] == fx["errors"][j] and r["errors32"] == fx["errors32"][j]
        assert r["P"] == fx["path_off"][j + 1] - fx["path_off"][j]
        np.testing.assert_allclose(r["c_norm"], fx["c_norm"][j], rtol=1e-12)
