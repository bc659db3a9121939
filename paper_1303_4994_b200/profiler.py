"""Dataset profiler on B200: the reference's profiler API
(pkg/src/apax/profiler.py) with every sample-level statistic computed by
the kernels in csrc/apax_profile.cu and every encode/decode by the codec
kernels.

Same names, arguments, constants, exceptions and report keys as the
reference:

* ``pearson_r`` (:40-48): fused sums of x*y, x^2, y^2;
* ``welch_spectrum`` (:61-74): batched fp64 FFT of periodic-Hann frames at
  50% overlap, "spectrum" scaling, mean over frames; host dB statistics
  over the <= 2049 bins;
* ``s2r_distribution`` (:105-124): the 95.5% margin and the CDF points are
  exact order statistics of |x|/|d| found by a radix multi-select on the
  GPU; numpy's log10 is applied to the selected ratios only (monotone);
* ``window2_metrics`` (:127-159): fused sums plus the two-pass std;
* ``rate_correlation_sweep`` (:184-199): whole-stream fixed-quality encodes
  (byte-identical to the reference) of all grid targets on concurrent CUDA
  streams, decoded on the GPU;
* ``recommend_operating_point`` (:202-246): host logic (scalar);
* ``ProfileSession`` / ``profile`` (:249-332).

Reductions are deterministic (fixed-order per-CTA partials); they differ
from numpy's pairwise / BLAS order by rounding only (the reference itself
is BLAS-thread-count sensitive).
"""
from __future__ import annotations

import ctypes
import math
import threading
import warnings
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .codec import Decoder, Encoder, _require_cuda, _stream_ptr, torch_dtype
from .dtypes import Dtype, Mode, StreamConfig
from .errors import NoData, UndefinedCorrelation, raise_status

FIVE_NINES = 0.99999
DEFAULT_GRID = tuple(float(t) for t in range(20, 121, 5))
DEFAULT_SEGMENT = 4096
_EPS_POWER = 1e-30
TWO_SIGMA_COVERAGE = 0.955

METRIC_KEYS = (
    "mean_x", "std_x", "spectral_peak_x_db", "spectral_floor_x_db",
    "mean_y", "std_y", "spectral_peak_y_db", "spectral_floor_y_db",
    "mean_d", "std_d", "spectral_peak_d_db", "spectral_floor_d_db",
    "rms_resid_pct", "rms_resid_db",
    "srr_db", "pearson_r",
    "fft_s2r_margin_db", "two_sigma_s2r_margin_db",
)

_F64 = Dtype.F64


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------
def _dev(arr, dtype: Dtype):
    """Host array -> contiguous CUDA tensor of the dtype (exact conversion)."""
    torch, _ = _require_cuda()
    if hasattr(arr, "is_cuda") and arr.is_cuda:
        return arr.reshape(-1).contiguous()
    a = np.ascontiguousarray(np.asarray(arr, dtype=dtype.np_dtype).reshape(-1))
    return torch.from_numpy(a).cuda()


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


class _Sums:
    """pass-0 and pass-1 sums of (x, y, d = x - y) on the device."""

    def __init__(self, xd, yd, dtype: Dtype, centred: bool = False, means=None):
        torch, L = _require_cuda()
        n = int(xd.numel())
        grid = int(L.apax_profile_grid())
        part = torch.empty(grid * 8, dtype=torch.float64, device=xd.device)
        cnt = torch.zeros(2, dtype=torch.int64, device=xd.device)
        raise_status(L.apax_profile_sums(_ptr(xd), _ptr(yd), n, dtype.wire_code, 0, 0.0, 0.0, 0.0,
                                         _ptr(part), _ptr(cnt), ctypes.c_void_p(_stream_ptr(None))))
        s = part.cpu().numpy().reshape(grid, 8).sum(axis=0)
        c = cnt.cpu().numpy()
        self.n = n
        self.sx, self.sy, self.sd, self.sxx, self.syy, self.sdd, self.sxy = (float(v) for v in s[:7])
        self.zero_x = int(c[0])     # x == 0 and d != 0
        self.zero_d = int(c[1])     # d == 0
        self.cxx = self.cyy = self.cdd = None
        if centred and n:
            # about the local means, or the global ones of a sharded array
            mx, my, md = means if means is not None else (self.sx / n, self.sy / n, self.sd / n)
            raise_status(L.apax_profile_sums(_ptr(xd), _ptr(yd), n, dtype.wire_code, 1, mx, my, md,
                                             _ptr(part), _ptr(cnt), ctypes.c_void_p(_stream_ptr(None))))
            s2 = part.cpu().numpy().reshape(grid, 8).sum(axis=0)
            self.cxx, self.cyy, self.cdd = float(s2[3]), float(s2[4]), float(s2[5])

    def pearson(self) -> float:
        if self.sxx == 0.0 or self.syy == 0.0:
            raise UndefinedCorrelation("a vector with zero energy has no correlation")
        return self.sxy / math.sqrt(self.sxx * self.syy)


def pearson_r(x, y) -> float:
    """Uncentered correlation sum(xy) / sqrt(sum(x^2) * sum(y^2))."""
    xd, yd = _dev(x, _F64), _dev(y, _F64)
    return _Sums(xd, yd, _F64).pearson()


# ---------------------------------------------------------------------------
# Welch spectrum
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class SpectrumStats:
    bins_db: np.ndarray
    peak_db: float
    floor_db: float  # median of the per-bin dB values
    mean_db: float
    dynamic_range_db: float
    power: np.ndarray  # linear per-bin power


_TABLES: Dict[Tuple[int, object], object] = {}


def hann_periodic(m: int) -> np.ndarray:
    """Periodic Hann window (scipy.signal.get_window('hann', m)): the
    symmetric m+1 point cosine window without its last point."""
    fac = np.linspace(-np.pi, np.pi, m + 1)
    w = np.zeros(m + 1)
    w += 0.5 * np.cos(0 * fac)
    w += 0.5 * np.cos(1 * fac)
    return w[:m]


def _welch_tables(seg: int, device):
    key = (seg, str(device))
    t = _TABLES.get(key)
    if t is None:
        torch, _ = _require_cuda()
        k = np.arange(seg // 2)
        ang = 2.0 * np.pi * k / seg
        tw = np.empty(seg, dtype=np.float64)
        tw[0::2] = np.cos(ang)
        tw[1::2] = -np.sin(ang)
        tab = np.concatenate([tw, hann_periodic(seg)])
        t = torch.from_numpy(tab).to(device)
        _TABLES[key] = t
    return t


def _welch_frame_sums(xd, yd, dtype: Dtype, which: int, n: int, seg: int):
    """Sum over the Hann-windowed frames (hop seg/2) of |rfft|^2 and the
    frame count (scipy.signal.welch before its scaling and mean)."""
    torch, L = _require_cuda()
    grid = int(L.apax_profile_grid())
    nb = seg // 2 + 1
    part = torch.empty(grid * nb, dtype=torch.float64, device=xd.device)
    tab = _welch_tables(seg, xd.device)
    raise_status(L.apax_profile_welch(_ptr(xd), _ptr(yd) if yd is not None else None, n, dtype.wire_code, which,
                                      seg, _ptr(tab), _ptr(part), ctypes.c_void_p(_stream_ptr(None))))
    return part.cpu().numpy().reshape(grid, nb).sum(axis=0), (n - seg) // (seg // 2) + 1


def _welch_scale(tot: np.ndarray, nframes: int, seg: int) -> np.ndarray:
    win = hann_periodic(seg)
    scale = 1.0 / win.sum() ** 2
    pxx = tot * scale
    pxx[1:-1] *= 2.0               # one-sided, even nfft: DC and Nyquist not doubled
    return pxx / nframes


def _welch_power(xd, yd, dtype: Dtype, which: int, n: int, seg: int) -> np.ndarray:
    tot, nframes = _welch_frame_sums(xd, yd, dtype, which, n, seg)
    return _welch_scale(tot, nframes, seg)


def _stats_from_power(pxx: np.ndarray) -> SpectrumStats:
    bins_db = 10.0 * np.log10(pxx + _EPS_POWER)
    peak = float(bins_db.max())
    floor = float(np.median(bins_db))
    return SpectrumStats(bins_db=bins_db, peak_db=peak, floor_db=floor, mean_db=float(bins_db.mean()),
                         dynamic_range_db=peak - floor, power=pxx)


def _segment(n: int, segment_length: int) -> int:
    seg = segment_length
    if n < seg:
        seg = 1 << max(int(n).bit_length() - 1, 1)
    return seg


def welch_spectrum(x, segment_length: int = DEFAULT_SEGMENT) -> SpectrumStats:
    """Averaged periodogram: Hann window, 50% overlap."""
    xd = _dev(x, _F64)
    n = int(xd.numel())
    seg = _segment(n, segment_length)
    return _stats_from_power(_welch_power(xd, None, _F64, 0, n, seg))


def spectral_flatness(power: np.ndarray) -> float:
    """Geometric mean over arithmetic mean of a power spectrum (host: <= 2049 bins)."""
    p = np.asarray(power, dtype=np.float64) + _EPS_POWER
    return float(np.exp(np.mean(np.log(p))) / np.mean(p))


def fft_s2r_margin(x_spec: SpectrumStats, d_spec: SpectrumStats) -> float:
    """Input spectral floor minus mean residual spectral level, in dB."""
    return x_spec.floor_db - d_spec.mean_db


# ---------------------------------------------------------------------------
# S2R distribution: exact order statistics by radix multi-select
# ---------------------------------------------------------------------------
_SEL_DIGITS = ((48, 15), (32, 16), (16, 16), (0, 16))   # (shift, width); the key's sign bit is 0


def _select_ratio_keys(xd, yd, dtype: Dtype, ranks: Sequence[int], y_is_output: bool,
                       reduce_hist=None) -> Dict[int, int]:
    """Ascending-rank order statistics (as uint64 bit patterns) of the
    ratio keys |x| / |d| over all n samples: a radix multi-select in 4
    passes over the keys (digits of 15, 16, 16, 16 bits; apax_profile_select).
    `reduce_hist` (multi-GPU) sums each pass's digit histograms over the
    ranks in place, so every rank picks the same digits and the ranks are
    global (distributed.sharded_window_stats)."""
    torch, L = _require_cuda()
    n = int(xd.numel())
    targets = sorted(set(int(r) for r in ranks))
    prefix = {r: 0 for r in targets}
    resid = {r: r for r in targets}
    sp = ctypes.c_void_p(_stream_ptr(None))
    for p, (sh, width) in enumerate(_SEL_DIGITS):
        uniq = sorted(set(prefix.values()))
        nb = 1 << width
        if p == 0:
            pre = torch.zeros(1, dtype=torch.int64, device=xd.device)
            hist = torch.zeros(nb, dtype=torch.int32, device=xd.device)
        else:
            pre = torch.tensor(np.array(uniq, dtype=np.uint64).view(np.int64), device=xd.device)
            hist = torch.zeros(len(uniq) * nb, dtype=torch.int32, device=xd.device)
        raise_status(L.apax_profile_select(_ptr(xd), _ptr(yd), n, dtype.wire_code, p, _ptr(pre), len(uniq),
                                           _ptr(hist), 1 if y_is_output else 0, sp))
        if reduce_hist is not None:
            reduce_hist(hist)
        h = hist.cpu().numpy().view(np.uint32).astype(np.int64).reshape(-1, nb)
        slot = {v: i for i, v in enumerate(uniq)}
        for r in targets:
            cum = np.cumsum(h[0 if p == 0 else slot[prefix[r]]])
            dg = int(np.searchsorted(cum, resid[r], side="right"))
            if dg >= nb:  # pragma: no cover - ranks are always < n
                raise RuntimeError("radix select lost its rank")
            resid[r] -= int(cum[dg - 1]) if dg else 0
            prefix[r] = (prefix[r] << width) | dg
    return prefix


def _key_to_ratio(k: int) -> np.float64:
    return np.array([k], dtype=np.uint64).view(np.float64)[0]


def _s2r_of_ratios(r: np.ndarray) -> np.ndarray:
    """20*log10(r) with the reference's +/-inf conventions, numpy's log10."""
    r = np.asarray(r, dtype=np.float64)
    out = np.empty(r.size, dtype=np.float64)
    inf = np.isinf(r)
    zero = r == 0.0
    rest = ~inf & ~zero
    out[inf] = math.inf
    out[zero] = -math.inf
    out[rest] = 20.0 * np.log10(r[rest])
    return out


class S2RDistribution:
    """Per-sample signal-to-residual ratios and their 2-sigma margin.  The
    margin and the CDF points come from GPU order statistics; ``s2r_db``
    (all n values) is materialised on demand."""

    def __init__(self, xd, yd, dtype: Dtype, y_is_output: bool, sums: Optional[_Sums] = None):
        self._xd, self._yd, self._dt, self._yo = xd, yd, dtype, y_is_output
        n = int(xd.numel())
        self._n = n
        if sums is None or not y_is_output:
            # counts of d == 0 and x == 0 != d
            if y_is_output:
                sums = _Sums(xd, yd, dtype)
                self._zero_x, self._zero_d = sums.zero_x, sums.zero_d
            else:
                ax = xd.double().abs()
                ad = yd.double().abs()
                self._zero_d = int((ad == 0).sum().item())
                self._zero_x = int(((ax == 0) & (ad != 0)).sum().item())
        else:
            self._zero_x, self._zero_d = sums.zero_x, sums.zero_d
        k = math.ceil(TWO_SIGMA_COVERAGE * n)
        self._margin_rank = n - k            # ascending rank of ordered_desc[k-1]
        nf = n - self._zero_x - self._zero_d
        self._nf = nf
        self._cdf_ranks = []
        if nf > 0:
            qs = np.linspace(0, nf - 1, min(201, nf)).astype(int)
            self._cdf_q = qs
            self._cdf_ranks = [self._zero_x + int(q) for q in qs]
        keys = _select_ratio_keys(xd, yd, dtype, [self._margin_rank] + self._cdf_ranks, y_is_output)
        self._keys = keys
        self.two_sigma_margin_db = float(_s2r_of_ratios([_key_to_ratio(keys[self._margin_rank])])[0])
        self._s2r = None

    @property
    def s2r_db(self) -> np.ndarray:
        if self._s2r is None:
            xf = self._xd.double()
            df = (xf - self._yd.double()) if self._yo else self._yd.double()
            ax, ad = xf.abs(), df.abs()
            r = ax / ad
            r[ad == 0] = math.inf
            self._s2r = _s2r_of_ratios(r.cpu().numpy())
        return self._s2r

    def cdf_points(self, n_points: int = 201) -> List[Tuple[float, float]]:
        """(s2r_db, fraction of samples <= s2r_db) on a quantile grid,
        finite values only (infinities are handled by count)."""
        if self._nf == 0:
            return []
        if n_points != 201:
            qs = np.linspace(0, self._nf - 1, min(n_points, self._nf)).astype(int)
            keys = _select_ratio_keys(self._xd, self._yd, self._dt, [self._zero_x + int(q) for q in qs], self._yo)
        else:
            qs, keys = self._cdf_q, self._keys
        vals = _s2r_of_ratios([_key_to_ratio(keys[self._zero_x + int(q)]) for q in qs])
        total = self._n
        return [(float(v), (self._zero_x + int(q) + 1) / total) for v, q in zip(vals, qs)]


def s2r_distribution(x, d) -> S2RDistribution:
    """Per-sample signal-to-residual ratios and their 2-sigma (95.5%) margin.

    d[i] = 0 gives +inf (always above any margin); x[i] = 0 with d[i] != 0
    gives -inf.  The margin is the largest level that at least 95.5% of
    samples meet or exceed."""
    return S2RDistribution(_dev(x, _F64), _dev(d, _F64), _F64, y_is_output=False)


# ---------------------------------------------------------------------------
# Window 2 metrics
# ---------------------------------------------------------------------------
def _metrics(s: _Sums, x_spec: SpectrumStats, y_spec: SpectrumStats, d_spec: SpectrumStats,
             two_sigma_margin_db: float) -> Dict[str, float]:
    n = s.n
    rms_x = math.sqrt(s.sxx / n)
    rms_d = math.sqrt(s.sdd / n)
    if rms_x > 0 and rms_d > 0:
        rms_resid_db = 20.0 * math.log10(rms_d / rms_x)
    elif rms_d == 0.0:
        rms_resid_db = -math.inf
    else:
        rms_resid_db = math.inf
    m = {
        "mean_x": s.sx / n, "std_x": math.sqrt(s.cxx / n),
        "spectral_peak_x_db": x_spec.peak_db, "spectral_floor_x_db": x_spec.floor_db,
        "mean_y": s.sy / n, "std_y": math.sqrt(s.cyy / n),
        "spectral_peak_y_db": y_spec.peak_db, "spectral_floor_y_db": y_spec.floor_db,
        "mean_d": s.sd / n, "std_d": math.sqrt(s.cdd / n),
        "spectral_peak_d_db": d_spec.peak_db, "spectral_floor_d_db": d_spec.floor_db,
        "rms_resid_pct": 100.0 * (rms_d / rms_x) if rms_x > 0 else math.inf,
        "rms_resid_db": rms_resid_db,
        "srr_db": -rms_resid_db,
        "pearson_r": s.pearson(),
        "fft_s2r_margin_db": fft_s2r_margin(x_spec, d_spec),
        "two_sigma_s2r_margin_db": two_sigma_margin_db,
    }
    assert tuple(m.keys()) == METRIC_KEYS
    return m


def window2_metrics(x, y, d, x_spec: SpectrumStats, y_spec: SpectrumStats, d_spec: SpectrumStats,
                    two_sigma_margin_db: float) -> Dict[str, float]:
    """The 18-entry comparison table for one operating point (d = x - y)."""
    xd, yd = _dev(x, _F64), _dev(y, _F64)
    return _metrics(_Sums(xd, yd, _F64, centred=True), x_spec, y_spec, d_spec, two_sigma_margin_db)


# ---------------------------------------------------------------------------
# sweep and recommendation
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class OperatingPoint:
    srr_target: float
    ratio: float
    r: float
    target_unreachable: bool = False


@dataclass(frozen=True)
class RateCorrelationCurve:
    points: Tuple[OperatingPoint, ...]
    recommended: Optional[OperatingPoint] = None


def _encode_decode(xd, dtype: Dtype, targets: Sequence[float], block_size: int):
    """Whole-stream fixed-quality encodes of xd at every target (concurrent
    CUDA streams), each decoded on the GPU.  Returns [(nbytes, y tensor)].
    Encoder + decoder plans of a target hold ~2.3x the input; targets run in
    groups that fit half of the free device memory."""
    torch, _ = _require_cuda()
    n = int(xd.numel())
    w = dtype.width_bytes
    per = 3 * n * max(w, 4) + (64 << 20)
    free, _total = torch.cuda.mem_get_info(xd.device)
    group = max(1, min(len(targets), int(0.5 * free // per)))
    out = []
    for g0 in range(0, len(targets), group):
        jobs = []
        for t in targets[g0:g0 + group]:
            cfg = StreamConfig(dtype=dtype, block_size=block_size, mode=Mode.FIXED_QUALITY, target=float(t))
            st = torch.cuda.Stream(device=xd.device)
            st.wait_stream(torch.cuda.current_stream(xd.device))
            enc = Encoder(n, cfg, device=xd.device)
            dec = Decoder(n, dtype, block_size, device=xd.device)
            with torch.cuda.stream(st):
                enc.encode(xd, stream=st)
                dec.decode(enc.out, enc.cap, enc.offsets, stream=st)
            jobs.append((enc, dec, st))
        for enc, dec, st in jobs:
            nbytes = enc.finish(stream=st)
            y = dec.finish(stream=st)
            torch.cuda.current_stream(xd.device).wait_stream(st)
            out.append((nbytes, y))
        del jobs
    return out


def _sweep_supported(xd, dtype: Dtype, block_size: int) -> bool:
    return (block_size == 4096 and dtype in (Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64)
            and xd.data_ptr() % 16 == 0)


def _sweep_points(xd, dtype: Dtype, targets: Sequence[float], block_size: int):
    """(container bytes, sum x^2, sum x*y, sum y*y) of the whole-stream
    fixed-quality encode at every target.  Output-free on the device
    (apax_sweep_point: the chain's per-block (x, y = decode) sums and the
    packer counting bytes; no container, no decoded array), all targets on
    concurrent CUDA streams; other block sizes / dtypes encode and decode."""
    torch, L = _require_cuda()
    n = int(xd.numel())
    if not _sweep_supported(xd, dtype, block_size):
        res = []
        for nbytes, y in _encode_decode(xd, dtype, targets, block_size):
            s = _Sums(xd, y, dtype)
            res.append((nbytes, s.sxx, s.sxy, s.syy))
        return res
    nb = (n + 4095) // 4096
    wsb = int(L.apax_sweep_point_workspace_bytes(n, dtype.wire_code))
    cur = torch.cuda.current_stream(xd.device)
    jobs = []
    for t in targets:
        st = torch.cuda.Stream(device=xd.device)
        st.wait_stream(cur)
        ws = torch.empty(wsb, dtype=torch.uint8, device=xd.device)
        stats = torch.empty(3 * nb, dtype=torch.float64, device=xd.device)
        status = torch.empty(4, dtype=torch.int64, device=xd.device)
        raise_status(L.apax_sweep_point(_ptr(xd), n, dtype.wire_code, float(t), _ptr(stats), _ptr(status), _ptr(ws),
                                        wsb, ctypes.c_void_p(int(st.cuda_stream))))
        jobs.append((st, stats, status, ws))
    out = []
    from .codec import _check_status
    for st, stats, status, _ws in jobs:
        st.synchronize()
        sv = status.cpu().numpy().view(np.uint64)
        _check_status(sv)
        tot = stats.cpu().numpy().reshape(nb, 3).sum(axis=0)
        out.append((int(sv[2]), float(tot[0]), float(tot[1]), float(tot[2])))
    cur.wait_stream(jobs[-1][0]) if jobs else None
    return out


def _point(t: float, n: int, dtype: Dtype, nbytes: int, sxx: float, sxy: float, syy: float) -> OperatingPoint:
    if sxx == 0.0 or syy == 0.0:
        raise UndefinedCorrelation("a vector with zero energy has no correlation")
    return OperatingPoint(t, n * dtype.width_bytes / nbytes, sxy / math.sqrt(sxx * syy))


def rate_correlation_sweep(x, dtype: Dtype, grid: Sequence[float] = DEFAULT_GRID,
                           block_size: int = 4096) -> RateCorrelationCurve:
    """Encode at every SRR target on the grid; each point is independent."""
    xd = _dev(x, dtype)
    n = int(xd.numel())
    targets = sorted(float(t) for t in grid)
    points: List[OperatingPoint] = []
    for t, (nbytes, sxx, sxy, syy) in zip(targets, _sweep_points(xd, dtype, targets, block_size)):
        try:
            points.append(_point(t, n, dtype, nbytes, sxx, sxy, syy))
        except UndefinedCorrelation:
            warnings.warn(f"correlation undefined at SRR target {t}; point dropped")
            continue
    return RateCorrelationCurve(points=tuple(points))


def recommend_operating_point(curve: RateCorrelationCurve,
                              reencode: Optional[Callable[[float], OperatingPoint]] = None,
                              threshold: float = FIVE_NINES) -> OperatingPoint:
    """Smallest SRR target whose correlation reaches the threshold
    (reference :202-246): linear interpolation between the bracketing grid
    points, then, given ``reencode``, up to 8 bisection steps toward the
    upper bracket; unreachable targets fall back to the max-r point."""
    pts = curve.points
    if not pts:
        raise NoData("empty rate-correlation curve")
    above = [p.r >= threshold for p in pts]
    if all(above):
        return max(pts, key=lambda p: p.ratio)
    if not any(above):
        best = max(pts, key=lambda p: p.r)
        return OperatingPoint(best.srr_target, best.ratio, best.r, target_unreachable=True)
    bracket = next(((pts[i], pts[i + 1]) for i in range(len(pts) - 1)
                    if not above[i] and above[i + 1]), None)
    if bracket is None:          # r not monotone: the first point over the line
        return pts[above.index(True)]
    lo, hi = bracket
    target = lo.srr_target + (threshold - lo.r) / (hi.r - lo.r) * (hi.srr_target - lo.srr_target)
    if reencode is None:
        return hi
    # reference :240-246: the point of the 8th bisection step is never
    # checked; the loop falls through to re-encoding the upper bracket
    upper = hi.srr_target
    point = reencode(target)
    for _ in range(8):
        if point.r >= threshold:
            return point
        target = 0.5 * (target + upper)
        point = reencode(target)
    return reencode(upper)


class ProfileSession:
    """Input samples plus a per-operating-point cache of decoded output,
    residual, and Window 2-4 results.  Single writer, many readers."""

    def __init__(self, x, dtype: Dtype, grid: Sequence[float] = DEFAULT_GRID, block_size: int = 4096,
                 segment_length: int = DEFAULT_SEGMENT, name: str = "") -> None:
        self.x = np.asarray(x, dtype=dtype.np_dtype) if not hasattr(x, "is_cuda") else x
        self._xd = _dev(x, dtype)
        self.dtype = dtype
        self.grid = tuple(sorted(float(t) for t in grid))
        self.block_size = block_size
        self.segment_length = segment_length
        self.name = name
        self._lock = threading.Lock()
        self._cache: Dict[float, dict] = {}
        self.curve = rate_correlation_sweep(self._xd, dtype, self.grid, block_size)
        self.recommended = recommend_operating_point(self.curve, self._reencode)
        self.current_point = self.recommended

    def _reencode(self, target: float) -> OperatingPoint:
        (nbytes, sxx, sxy, syy), = _sweep_points(self._xd, self.dtype, [target], self.block_size)
        return _point(target, int(self._xd.numel()), self.dtype, nbytes, sxx, sxy, syy)

    def windows_at(self, srr_target: float) -> dict:
        """Windows 2-4 for one operating point (cached)."""
        key = float(srr_target)
        with self._lock:
            if key in self._cache:
                return self._cache[key]
        (nbytes, y), = _encode_decode(self._xd, self.dtype, [key], self.block_size)
        xd, dt = self._xd, self.dtype
        n = int(xd.numel())
        seg = _segment(n, self.segment_length)
        x_spec = _stats_from_power(_welch_power(xd, y, dt, 0, n, seg))
        y_spec = _stats_from_power(_welch_power(xd, y, dt, 1, n, seg))
        d_spec = _stats_from_power(_welch_power(xd, y, dt, 2, n, seg))
        sums = _Sums(xd, y, dt, centred=True)
        dist = S2RDistribution(xd, y, dt, y_is_output=True, sums=sums)
        metrics = _metrics(sums, x_spec, y_spec, d_spec, dist.two_sigma_margin_db)
        result = {
            "srr_target": key,
            "ratio": n * dt.width_bytes / nbytes,
            "metrics": metrics,
            "spectra": {
                "x": {"bins_db": x_spec.bins_db.tolist(), "peak_db": x_spec.peak_db,
                      "floor_db": x_spec.floor_db, "mean_db": x_spec.mean_db,
                      "dynamic_range_db": x_spec.dynamic_range_db},
                "d": {"bins_db": d_spec.bins_db.tolist(), "peak_db": d_spec.peak_db,
                      "floor_db": d_spec.floor_db, "mean_db": d_spec.mean_db,
                      "dynamic_range_db": d_spec.dynamic_range_db},
            },
            "s2r": {
                "cdf": [[v, p] for v, p in dist.cdf_points()],
                "two_sigma_margin_db": dist.two_sigma_margin_db,
            },
        }
        with self._lock:
            self._cache[key] = result
        return result

    def report(self) -> dict:
        """Profiler report with the reference's keys
        (pkg/docs/schema/profile_report.schema.json)."""
        rec = self.recommended
        return {
            "dataset": self.name,
            "dtype": self.dtype.code,
            "curve": [{"srr_target": p.srr_target, "ratio": p.ratio, "r": p.r} for p in self.curve.points],
            "recommended": {"srr_target": rec.srr_target, "ratio": rec.ratio, "r": rec.r,
                            "target_unreachable": rec.target_unreachable},
            "windows": self.windows_at(rec.srr_target),
        }


def profile(x, dtype: Dtype, grid: Sequence[float] = DEFAULT_GRID, block_size: int = 4096,
            name: str = "") -> dict:
    """One-shot profiler report for a sample array."""
    return ProfileSession(x, dtype, grid, block_size, name=name).report()
