"""Profiler: GPU statistics and report against the frozen outputs of the
reference profiler (tests/golden/profile_reports.json, written by
tests/golden/make_profile_golden.py from the live reference), plus the
host-side logic on hand-built cases (mirroring pkg/tests/test_profiler.py).

Tolerances: the sweep's ratios and the S2R order statistics are exact; r
is compared at 1e-12 (the reference's own bar, pkg/tests/test_profiler.py:
59-67); Welch power at 1e-9 relative of the spectrum's peak bin (FFT
rounding); moments at 1e-9 relative.
"""
import json
import math

import numpy as np
import pytest

from conftest import GOLDEN

from paper_1303_4994_b200 import profiler as P
from paper_1303_4994_b200.dtypes import Dtype
from paper_1303_4994_b200.errors import NoData

import sys
sys.path.insert(0, str(GOLDEN))
import profile_inputs as PI  # noqa: E402

GOLD = json.loads((GOLDEN / "profile_reports.json").read_text())


def unjson(v):
    if isinstance(v, dict) and set(v) == {"nonfinite"}:
        return float(v["nonfinite"])
    if isinstance(v, dict):
        return {k: unjson(w) for k, w in v.items()}
    if isinstance(v, list):
        return [unjson(w) for w in v]
    return v


# ---------------------------------------------------------------------------
# host logic (no GPU)
# ---------------------------------------------------------------------------
def test_hann_window_matches_scipy():
    from scipy.signal import get_window
    for m in (2, 4, 256, 1024, 4096):
        assert np.array_equal(P.hann_periodic(m), get_window("hann", m))


def test_constants_and_keys():
    assert P.FIVE_NINES == 0.99999 and len(P.DEFAULT_GRID) == 21
    assert P.DEFAULT_GRID[0] == 20.0 and P.DEFAULT_GRID[-1] == 120.0
    assert len(P.METRIC_KEYS) == 18 and P.TWO_SIGMA_COVERAGE == 0.955


def test_recommend_all_above_takes_max_ratio():
    pts = tuple(P.OperatingPoint(t, 10 - t / 20, 0.999999) for t in (40.0, 60.0))
    assert P.recommend_operating_point(P.RateCorrelationCurve(pts)) == pts[0]


def test_recommend_unreachable_flagged():
    pts = tuple(P.OperatingPoint(t, 5.0, 0.9 + t / 1000) for t in (40.0, 60.0))
    rec = P.recommend_operating_point(P.RateCorrelationCurve(pts))
    assert rec.target_unreachable and rec.r == pts[-1].r


def test_recommend_empty_curve():
    with pytest.raises(NoData):
        P.recommend_operating_point(P.RateCorrelationCurve(()))


def test_recommend_interpolation_and_bisection():
    pts = (P.OperatingPoint(40.0, 6.0, 0.9999), P.OperatingPoint(50.0, 5.0, 0.99999 + 5e-6),
           P.OperatingPoint(60.0, 4.0, 0.999999))
    curve = P.RateCorrelationCurve(pts)
    assert P.recommend_operating_point(curve) == pts[1]      # no re-encoder: upper bracket
    seen = []

    def reencode(t):   # r rises with the target; crosses the threshold at 49.5
        seen.append(t)
        return P.OperatingPoint(t, 5.5, 0.99999 + (t - 49.5) * 1e-6)
    rec = P.recommend_operating_point(curve, reencode)
    frac = (0.99999 - 0.9999) / (pts[1].r - 0.9999)
    assert seen[0] == pytest.approx(40.0 + frac * 10.0)
    assert rec.r >= P.FIVE_NINES
    for a, b in zip(seen, seen[1:]):   # bisection toward the upper bracket
        assert b == 0.5 * (a + 50.0)


@pytest.mark.parametrize("clear_at", list(range(0, 11)))
def test_recommend_bisection_call_sequence(clear_at):
    """Reference profiler.py:240-246: re-encode the interpolated target, up to
    8 bisection steps toward the upper bracket, and the point of the 8th step
    is never checked -- the loop falls through to reencode(upper).  The stub
    first clears the threshold on call number `clear_at` (0 = the
    interpolated point, 8 = the 8th bisection, 9+ = never)."""
    pts = (P.OperatingPoint(40.0, 6.0, 0.9999), P.OperatingPoint(50.0, 5.0, 0.999995))
    curve = P.RateCorrelationCurve(pts)
    calls = []

    def reencode(t):
        calls.append(t)
        ok = len(calls) - 1 >= clear_at or t == 50.0
        return P.OperatingPoint(t, 7.0 - len(calls) * 0.1, 0.999999 if ok else 0.99998)
    rec = P.recommend_operating_point(curve, reencode)
    if clear_at <= 7:
        assert len(calls) == clear_at + 1 and rec.srr_target == calls[-1]
    else:
        # the 8th bisection point (call 9) may clear the threshold: ignored
        assert len(calls) == 10 and calls[-1] == 50.0 and rec.srr_target == 50.0
    frac = (P.FIVE_NINES - pts[0].r) / (pts[1].r - pts[0].r)
    assert calls[0] == 40.0 + frac * 10.0
    for a, b in zip(calls[:9], calls[1:9]):
        assert b == 0.5 * (a + 50.0)


def test_recommend_non_monotone():
    above, below = 0.999995, 0.9999
    # no (below, above) neighbours: the first point at/above the threshold wins
    pts = (P.OperatingPoint(40.0, 6.0, above), P.OperatingPoint(50.0, 5.0, below))
    assert P.recommend_operating_point(P.RateCorrelationCurve(pts)) == pts[0]
    # otherwise the first (below, above) bracket decides, even after a dip
    pts = (P.OperatingPoint(40.0, 6.0, above), P.OperatingPoint(50.0, 5.0, below),
           P.OperatingPoint(60.0, 4.0, above))
    assert P.recommend_operating_point(P.RateCorrelationCurve(pts)) == pts[2]
    pts = (P.OperatingPoint(40.0, 6.0, below), P.OperatingPoint(50.0, 5.0, above),
           P.OperatingPoint(60.0, 4.0, below))
    assert P.recommend_operating_point(P.RateCorrelationCurve(pts)) == pts[1]


# ---------------------------------------------------------------------------
# GPU: statistics and the full report against the reference
# ---------------------------------------------------------------------------
gpu = pytest.mark.gpu


@gpu
@pytest.mark.parametrize("name", PI.NAMES)
def test_standalone_statistics_vs_reference(name):
    g = unjson(GOLD[name])
    x, code, grid, bs, seg = PI.make(name)
    xf = x.astype(np.float64)
    rng = np.random.default_rng(77)
    y = xf + 0.01 * rng.standard_normal(xf.size) * (np.std(xf) + 1.0)
    assert P.pearson_r(xf, y) == pytest.approx(g["pearson"], abs=1e-12)
    spec = P.welch_spectrum(xf, seg)
    ref_pow = np.array(g["welch"]["power"])
    assert spec.power.shape == ref_pow.shape
    assert np.allclose(spec.power, ref_pow, rtol=0, atol=1e-9 * ref_pow.max())
    assert spec.peak_db == pytest.approx(g["welch"]["peak_db"], abs=1e-6)
    d = xf - y
    d[::97] = 0.0
    dist = P.s2r_distribution(xf, d)
    assert dist.two_sigma_margin_db == g["s2r"]["margin"]                 # exact order statistic
    assert [list(p) for p in dist.cdf_points()] == g["s2r"]["cdf"]        # exact


def _close(a, b, rel=1e-9, abs_=1e-12):
    if isinstance(b, float) and math.isinf(b):
        return a == b
    return a == pytest.approx(b, rel=rel, abs=abs_)


@gpu
@pytest.mark.parametrize("name", PI.NAMES)
def test_profile_report_vs_reference(name):
    g = unjson(GOLD[name])["report"]
    x, code, grid, bs, seg = PI.make(name)
    rep = P.profile(x, Dtype.from_code(code), grid=grid, block_size=bs, name=name)
    assert set(rep) == {"dataset", "dtype", "curve", "recommended", "windows"}
    assert rep["dataset"] == name and rep["dtype"] == code
    # sweep: byte-exact encodes -> exact ratios; r to 1e-12
    assert len(rep["curve"]) == len(g["curve"])
    for a, b in zip(rep["curve"], g["curve"]):
        assert a["srr_target"] == b["srr_target"] and a["ratio"] == b["ratio"]
        assert a["r"] == pytest.approx(b["r"], abs=1e-12)
    ra, rb = rep["recommended"], g["recommended"]
    assert ra["target_unreachable"] == rb["target_unreachable"]
    assert ra["srr_target"] == pytest.approx(rb["srr_target"], abs=1e-9)
    assert ra["ratio"] == pytest.approx(rb["ratio"], rel=1e-12)
    assert ra["r"] == pytest.approx(rb["r"], abs=1e-12)
    wa, wb = rep["windows"], g["windows"]
    assert wa["ratio"] == pytest.approx(wb["ratio"], rel=1e-12)
    assert list(wa["metrics"]) == list(P.METRIC_KEYS)
    for k in P.METRIC_KEYS:
        va, vb = wa["metrics"][k], wb["metrics"][k]
        if "spectral" in k or k == "fft_s2r_margin_db":
            # a floor more than 150 dB under its peak is the transform's own
            # rounding noise (see the bins below): 1 dB there
            def is_noise(kk):
                f = wb["metrics"][kk]
                return isinstance(f, float) and np.isfinite(f) and f < wb["metrics"][kk.replace("floor", "peak")] - 150.0
            noise = is_noise(k) if "floor" in k else (
                k == "fft_s2r_margin_db" and any(is_noise(f"spectral_floor_{c}_db") for c in "xyd"))
            assert _close(va, vb, rel=0, abs_=1.0 if noise else 1e-6), k
        elif k == "two_sigma_s2r_margin_db":
            assert va == pytest.approx(vb, abs=1e-9), k
        else:
            scale = max(abs(wb["metrics"]["mean_x"]), wb["metrics"]["std_x"], 1.0)
            assert _close(va, vb, rel=1e-9, abs_=1e-12 * scale), k
    for sig in ("x", "d"):
        ba, bb = np.array(wa["spectra"][sig]["bins_db"]), np.array(wb["spectra"][sig]["bins_db"])
        assert ba.shape == bb.shape
        # bins within 150 dB of the spectrum's peak to 1e-6 dB; below that a bin
        # is the rounding noise of the transform itself (2^-50 of the peak in
        # power: a constant or a ramp has nothing else there) and cuFFT's noise
        # is not pocketfft's: those only have to be noise on both sides
        live = bb >= bb.max() - 150.0
        assert np.allclose(ba[live], bb[live], rtol=0, atol=1e-6)
        assert np.all(ba[~live] < bb.max() - 140.0)
        assert wa["spectra"][sig]["floor_db"] == pytest.approx(wb["spectra"][sig]["floor_db"],
                                                                abs=1e-6 if live.all() else 1.0)
    ca, cb = wa["s2r"]["cdf"], wb["s2r"]["cdf"]
    assert len(ca) == len(cb)
    assert np.allclose(np.array(ca), np.array(cb), rtol=1e-12, atol=1e-9)


@gpu
def test_session_cache_and_reencode_self_consistent():
    x, code, grid, bs, seg = PI.make("short_f32")
    s = P.ProfileSession(x, Dtype.from_code(code), grid=grid, block_size=bs)
    w1 = s.windows_at(50.0)
    assert s.windows_at(50.0) is w1
    rec = s.recommended
    again = s._reencode(rec.srr_target)
    assert again.ratio == rec.ratio and again.r == pytest.approx(rec.r, abs=1e-15)


@gpu
@pytest.mark.parametrize("seed", range(3))
def test_output_free_sweep_point_matches_full_encode_decode(seed):
    """apax_sweep_point (the chain's per-block (x, y) sums, the packer
    counting bytes) against a full encode + decode: container length exact,
    sums to 1e-12."""
    import torch
    from paper_1303_4994_b200 import Dtype
    from paper_1303_4994_b200.profiler import _Sums, _encode_decode, _sweep_points
    rng = np.random.default_rng(500 + seed)
    for dt in (Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64):
        n = int(rng.integers(1, 60000))
        x = np.cumsum(rng.standard_normal(n)) * 50.0
        x = x.astype(dt.np_dtype) if dt.is_float else np.clip(x, -30000, 30000).astype(dt.np_dtype)
        xd = torch.from_numpy(x).cuda()
        targets = [float(t) for t in rng.uniform(20, 120, 3)]
        fast = _sweep_points(xd, dt, targets, 4096)
        full = _encode_decode(xd, dt, targets, 4096)
        for (nb, sxx, sxy, syy), (nb2, y) in zip(fast, full):
            s = _Sums(xd, y, dt)
            assert nb == nb2, (dt, n)
            for a, b in ((sxx, s.sxx), (sxy, s.sxy), (syy, s.syy)):
                assert a == pytest.approx(b, rel=1e-12, abs=0.0), (dt, n)


@gpu
def test_profile_of_silence_raises_like_the_reference():
    """An all-zero array: the correlation is undefined at every grid point, the
    reference drops each with a warning and raises NoData("empty
    rate-correlation curve") (profiler.py:196, :228)."""
    x = np.zeros(8192 * 2, np.float32)
    with pytest.warns(UserWarning, match="correlation undefined at SRR target"):
        with pytest.raises(NoData, match="empty rate-correlation curve"):
            P.profile(x, Dtype.F32, grid=(2.0, 4.0), block_size=4096, name="zeros")
