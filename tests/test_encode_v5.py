"""GPU parity of the v5 encoder (apax_encode_v5.cu: pack warps + a service
warp over segments of full 4096-sample blocks) against the CPU oracle, with
the cases its structure adds over the fused v3 kernel: several units per CTA
(APAX_ENC_V5=2 forces v5 past the one-wave launches), one-block units with
the warm_self pre-pass, blocks whose differences leave int32 (the 64-bit cold
paths), the exact monitor, error reports, the per-block trace, and equality
with the v3 kernel (APAX_ENC_V5=0).  Bit-exact for every byte."""
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig, decode_device, encode_device  # noqa: E402
from paper_1303_4994_b200 import _lib  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402
from paper_1303_4994_b200.errors import ApaxError  # noqa: E402


@pytest.fixture
def force_v5():
    old = os.environ.get("APAX_ENC_V5")
    os.environ["APAX_ENC_V5"] = "2"
    yield
    if old is None:
        os.environ.pop("APAX_ENC_V5", None)
    else:
        os.environ["APAX_ENC_V5"] = old


def _check(x, dt, mode, target, seg, pol="cold"):
    cfg = StreamConfig(dt, 4096, mode, target, segment_blocks=seg, segment_policy=pol)
    ref, offs, _ = O.encode(x, dt.wire_code, mode.value, target, 4096, segment_blocks=seg,
                            policy=1 if pol == "warm_self" else 0)
    res = encode_device(torch.from_numpy(x).cuda(), cfg)
    got = res.to_bytes()
    if got != ref:
        n = min(len(got), len(ref))
        a, b = np.frombuffer(got[:n], np.uint8), np.frombuffer(ref[:n], np.uint8)
        d = np.nonzero(a != b)[0]
        first = int(d[0]) if len(d) else n
        pytest.fail(f"{dt} {mode} T={target} P={seg} {pol}: first differing byte {first} "
                    f"(block {int(np.searchsorted(offs, first, side='right') - 1)}; len {len(got)} vs {len(ref)})")
    assert np.array_equal(res.block_offsets.cpu().numpy(), offs)
    y = decode_device(res.blob, res.nbytes, res.block_offsets, segment_blocks=seg).cpu().numpy()
    assert np.array_equal(y, O.decode(ref))


def test_kernel_name_reports_v5():
    name = _lib.lib().apax_encode_kernel_name(3, 2, 4096, 28).decode()
    assert name == "encode_v5_kernel"
    assert _lib.lib().apax_encode_kernel_name(4, 1, 4096, 28).decode() == "encode_v3_kernel"
    assert _lib.lib().apax_encode_kernel_name(3, 2, 1024, 28).decode() == "encode_v3_kernel"


@pytest.mark.parametrize("case", [
    ("f32", Mode.FIXED_QUALITY, 47.78, 28, "cold"),
    ("f32", Mode.FIXED_QUALITY, 90.0, 5, "cold"),
    ("f32", Mode.FIXED_RATE, 5.333, 28, "warm_self"),
    ("f32", Mode.FIXED_RATE, 12.0, 4, "cold"),
    ("i16", Mode.FIXED_RATE, 4.0, 7, "warm_self"),
    ("i16", Mode.FIXED_QUALITY, 35.0, 3, "cold"),
    ("i32", Mode.FIXED_RATE, 9.0, 6, "warm_self"),
    ("i32", Mode.FIXED_QUALITY, 120.0, 2, "cold"),
])
def test_one_wave_vs_oracle(case):
    dts, mode, target, seg, pol = case
    n = 4096 * 97 + 1234          # a partial last block: the generic v3 launch follows v5's
    if dts == "f32":
        _check(W.cfg2_ar2_f32(n), Dtype.F32, mode, target, seg, pol)
    elif dts == "i16":
        _check(W.cfg1_sines_i16(n), Dtype.I16, mode, target, seg, pol)
    else:
        _check(np.rint(W.cfg2_ar2_f32(n).astype(np.float64) * 3000).astype(np.int32), Dtype.I32, mode, target,
               seg, pol)


@pytest.mark.parametrize("case", [
    ("f32", Mode.FIXED_QUALITY, 47.78, 1, "cold"),
    ("f32", Mode.FIXED_RATE, 6.0, 1, "warm_self"),
    ("f32", Mode.FIXED_RATE, 6.0, 2, "warm_self"),
    ("i16", Mode.FIXED_RATE, 4.0, 1, "warm_self"),
    ("i16", Mode.FIXED_QUALITY, 30.0, 3, "cold"),
    ("i32", Mode.FIXED_QUALITY, 80.0, 2, "cold"),
])
def test_many_units_per_cta_vs_oracle(case, force_v5):
    """More units than resident CTAs: every CTA codes several units in turn
    (staging ring, barrier phases and the slot reused across units)."""
    dts, mode, target, seg, pol = case
    n = 4096 * 1500 + 17
    if dts == "f32":
        _check(W.cfg2_ar2_f32(n), Dtype.F32, mode, target, seg, pol)
    elif dts == "i16":
        _check(W.cfg1_sines_i16(n), Dtype.I16, mode, target, seg, pol)
    else:
        _check(np.rint(W.cfg2_ar2_f32(n).astype(np.float64) * 3000).astype(np.int32), Dtype.I32, mode, target,
               seg, pol)


def test_wide_blocks_vs_oracle():
    """i32 samples near the type's range at gain ~1 (differences leave int32:
    the 64-bit width / emission paths) next to small ones, and f32 blocks
    whose max |q| exceeds 2^30 (fixed quality far above the data's headroom)."""
    rng = np.random.default_rng(11)
    n = 4096 * 24
    x = rng.integers(-2 ** 31, 2 ** 31 - 1, n, dtype=np.int64).astype(np.int32)
    x[4096 * 5:4096 * 9] = rng.integers(-100, 100, 4096 * 4)
    x[4096 * 12:4096 * 13] = 0
    _check(x, Dtype.I32, Mode.FIXED_QUALITY, 180.0, 4)
    _check(x, Dtype.I32, Mode.FIXED_RATE, 30.0, 6, "warm_self")
    xf = (rng.standard_normal(n) * 1e3).astype(np.float32)
    xf[::7] *= -1.0
    _check(xf, Dtype.F32, Mode.FIXED_QUALITY, 200.0, 4)
    _check(xf, Dtype.F32, Mode.FIXED_RATE, 31.0, 3)


def test_exact_monitor_gate_vs_oracle():
    """Alternating-sign data: the sign-flip bound passes 1/3, the exact monitor
    runs and forces D0 (transform.py:67-83,107-113)."""
    rng = np.random.default_rng(12)
    n = 4096 * 16
    t = np.arange(n)
    for dt, scale in ((Dtype.I16, 9000.0), (Dtype.F32, 3.0), (Dtype.I32, 2.0e6)):
        x = scale * np.where(t % 2 == 0, 1.0, -1.0) * (1.0 + 0.3 * np.sin(t * 0.01)) + rng.normal(0, 0.05 * scale, n)
        x[4096 * 3:4096 * 5] = scale * np.sin(t[4096 * 3:4096 * 5] * 0.002)      # smooth blocks in between
        # zeros inside an oscillation: the monitor skips them (nonzero subsequence)
        x[4096 * 8:4096 * 9:3] = 0
        xa = x.astype(dt.np_dtype)
        _check(xa, dt, Mode.FIXED_RATE, 6.0, 4, "warm_self")
        _check(xa, dt, Mode.FIXED_QUALITY, 40.0, 8)


def test_zero_and_constant_blocks_vs_oracle():
    n = 4096 * 12
    x = np.zeros(n, np.float32)
    x[4096 * 2:4096 * 3] = 1.5
    x[4096 * 5:4096 * 6] = np.linspace(-1, 1, 4096, dtype=np.float32)
    x[4096 * 7] = 1e-30
    _check(x, Dtype.F32, Mode.FIXED_QUALITY, 60.0, 3)
    _check(x, Dtype.F32, Mode.FIXED_RATE, 4.0, 4, "warm_self")
    xi = np.zeros(n, np.int16)
    xi[4096 * 4:4096 * 5] = -32768
    xi[4096 * 9:] = 7
    _check(xi, Dtype.I16, Mode.FIXED_QUALITY, 20.0, 4)
    _check(xi, Dtype.I16, Mode.FIXED_RATE, 2.0, 2, "warm_self")


def test_nonfinite_is_reported_like_the_oracle():
    x = W.cfg2_ar2_f32(4096 * 8).copy()
    x[4096 * 5 + 123] = np.inf
    x[4096 * 6 + 7] = np.nan
    cfg = StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, 50.0, segment_blocks=4)
    with pytest.raises(ApaxError) as e_gpu:
        encode_device(torch.from_numpy(x).cuda(), cfg).to_bytes()
    with pytest.raises(O.OracleError) as e_ref:
        O.encode(x, 3, 2, 50.0, 4096, segment_blocks=4)
    assert str(4096 * 5 + 123) in str(e_gpu.value)          # the first non-finite index, as the reference reports it
    assert e_ref.value.detail == 4096 * 5 + 123


@pytest.mark.parametrize("mode,target,pol", [(Mode.FIXED_QUALITY, 47.78, "cold"), (Mode.FIXED_RATE, 5.0, "warm_self")])
def test_trace_vs_oracle(mode, target, pol):
    x = W.cfg2_ar2_f32(4096 * 20)
    cfg = StreamConfig(Dtype.F32, 4096, mode, target, segment_blocks=5, segment_policy=pol)
    enc = Encoder(x.size, cfg, trace=True)
    enc.encode(torch.from_numpy(x).cuda())
    nb = enc.finish()
    ref, _, tr = O.encode(x, 3, mode.value, target, 4096, segment_blocks=5, policy=1 if pol == "warm_self" else 0,
                          trace=True)
    assert enc.out[:nb].cpu().numpy().tobytes() == ref
    got = enc.trace.cpu().numpy()
    tr = np.asarray(tr).reshape(got.shape)
    assert np.allclose(got[:, 0], tr[:, 0], rtol=0, atol=1e-9)       # att_db
    assert np.allclose(got[:, 1], tr[:, 1], rtol=1e-12, atol=0)      # a
    assert np.array_equal(got[:, 2:], tr[:, 2:])                     # code, fbe, selector, costs, bytes, restart


def test_v5_equals_v3():
    x = W.cfg2_ar2_f32(4096 * 300)
    xd = torch.from_numpy(x).cuda()
    out = {}
    old = os.environ.get("APAX_ENC_V5")
    try:
        for v in ("0", "2"):
            os.environ["APAX_ENC_V5"] = v
            for mode, target, seg, pol in ((Mode.FIXED_QUALITY, 47.78, 28, "cold"), (Mode.FIXED_RATE, 5.3, 7, "warm_self")):
                res = encode_device(xd, StreamConfig(Dtype.F32, 4096, mode, target, segment_blocks=seg,
                                                      segment_policy=pol))
                out[(v, mode)] = (res.to_bytes(), res.block_offsets.cpu().numpy().copy())
    finally:
        if old is None:
            os.environ.pop("APAX_ENC_V5", None)
        else:
            os.environ["APAX_ENC_V5"] = old
    for mode in (Mode.FIXED_QUALITY, Mode.FIXED_RATE):
        assert out[("0", mode)][0] == out[("2", mode)][0]
        assert np.array_equal(out[("0", mode)][1], out[("2", mode)][1])
