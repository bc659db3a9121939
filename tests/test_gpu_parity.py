"""GPU parity: the sm_100a kernels (through the C ABI) against the reference's
frozen outputs (tests/golden, generated from the live reference) and the CPU
oracle.  Bit-exact for every byte and sample."""
import json

import numpy as np
import pytest

from conftest import GOLDEN, golden_containers, load_container
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_1303_4994_b200 import (Decoder, Dtype, Encoder, Mode, StreamConfig,  # noqa: E402
                                  decode_device, decode_stream, encode_device, encode_stream)
from paper_1303_4994_b200 import workloads as W  # noqa: E402

DT = {"i8": Dtype.I8, "i16": Dtype.I16, "i32": Dtype.I32, "f32": Dtype.F32, "f64": Dtype.F64}
POL = {0: "cold", 1: "warm_self"}


def _cfg(m):
    seg = m["segment_blocks"] or None
    return StreamConfig(DT[m["dtype"]], m["block_size"], Mode(m["mode"]),
                        float.fromhex(m["target_hex"]), segment_blocks=seg,
                        segment_policy=POL[m["policy"]])


@pytest.mark.parametrize("name", golden_containers())
def test_golden_container_encode(name):
    c = load_container(GOLDEN / "containers" / f"{name}.npz")
    cfg = _cfg(c["meta"])
    x = torch.from_numpy(np.ascontiguousarray(c["x"])).cuda()
    res = encode_device(x, cfg)
    got = res.to_bytes()
    if got != c["blob"]:
        n = min(len(got), len(c["blob"]))
        first = next((i for i in range(n) if got[i] != c["blob"][i]), n)
        pytest.fail(f"{name}: first differing byte {first} (len {len(got)} vs {len(c['blob'])})")
    assert np.array_equal(res.block_offsets.cpu().numpy(), c["offsets"])


@pytest.mark.parametrize("name", golden_containers())
def test_golden_container_decode(name):
    c = load_container(GOLDEN / "containers" / f"{name}.npz")
    blob = torch.from_numpy(np.frombuffer(c["blob"], np.uint8).copy()).cuda()
    # with the device block walk
    y = decode_device(blob, len(c["blob"])).cpu().numpy()
    assert y.dtype == c["y"].dtype and np.array_equal(y, c["y"])
    # with the side-band offsets
    offs = torch.from_numpy(c["offsets"]).cuda()
    y2 = decode_device(blob, len(c["blob"]), offs).cpu().numpy()
    assert np.array_equal(y2, c["y"])


@pytest.mark.parametrize("name", [n for n in golden_containers() if n.startswith(("seg_", "warm_"))])
def test_golden_container_decode_segments(name):
    """Segment-serial decoder (apax_decode_segments) on the golden
    segmented containers: bit-exact against the reference's decode."""
    c = load_container(GOLDEN / "containers" / f"{name}.npz")
    blob = torch.from_numpy(np.frombuffer(c["blob"], np.uint8).copy()).cuda()
    offs = torch.from_numpy(c["offsets"]).cuda()
    y = decode_device(blob, len(c["blob"]), offs, segment_blocks=c["meta"]["segment_blocks"]).cpu().numpy()
    assert y.dtype == c["y"].dtype and np.array_equal(y, c["y"])


@pytest.mark.parametrize("seed", range(6))
def test_segment_decoder_random_vs_oracle(seed):
    """Encoder containers of random segment length, dtype, mode and block
    size (powers of two, partial last blocks): the segment decoder is
    bit-exact against the oracle's decode."""
    rng = np.random.default_rng(4000 + seed)
    for _ in range(8):
        dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32][rng.integers(0, 4)]
        modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
        mode = modes[rng.integers(0, len(modes))]
        bs = int(rng.choice([128, 256, 1024, 2048, 4096, 4096]))
        target = float(rng.uniform(1, 12)) if mode is Mode.FIXED_RATE else float(rng.uniform(10, 100))
        seg = int(rng.choice([1, 2, 3, 8, 16]))
        x = _random_case(rng, dt)
        if rng.integers(0, 2):
            x = np.concatenate([x, x[: bs * 3]])
        cfg = StreamConfig(dt, bs, mode, target, segment_blocks=seg)
        res = encode_device(torch.from_numpy(x).cuda(), cfg)
        ref = O.decode(res.to_bytes())
        y = decode_device(res.blob, res.nbytes, res.block_offsets, segment_blocks=seg).cpu().numpy()
        assert np.array_equal(y, ref), (dt, mode, bs, seg, x.size)


def test_drop_in_bytes_api():
    c = load_container(GOLDEN / "containers" / "cfg1_i16_fr4.npz")
    cfg = _cfg(c["meta"])
    assert encode_stream(c["x"], cfg) == c["blob"]
    y = decode_stream(c["blob"])
    assert y.dtype == np.int16 and np.array_equal(y, c["y"])


def test_reference_entropy_golden_vectors_through_encoder():
    # A one-block LOSSLESS stream codes D0 = the samples themselves, so its
    # payload must equal the reference's pack_block golden payload.
    vecs = json.loads((GOLDEN / "entropy_vectors_ref.json").read_text())
    extra = json.loads((GOLDEN / "entropy_vectors_extra.json").read_text())["vectors"]
    n_checked = 0
    for vec in vecs + extra:
        v = np.asarray(vec["samples"], np.int64)
        if v.size > 4096 or np.abs(v).max(initial=0) >= 2 ** 31 - 1:
            continue
        blob = encode_stream(v.astype(np.int32), StreamConfig(Dtype.I32, 4096))
        assert blob[28 + 4:].hex() == vec["payload_hex"]
        assert np.array_equal(decode_stream(blob), v.astype(np.int32))
        n_checked += 1
    assert n_checked >= 10


def test_decode_errors_match_reference():
    d = json.loads((GOLDEN / "decode_errors.json").read_text())
    for case in d["cases"]:
        blob = bytes.fromhex(case["blob_hex"])
        if case["exc"] is None:
            y = decode_stream(blob)
            assert y.tobytes().hex() == case["y_hex"] and str(y.dtype) == case["y_dtype"]
            continue
        with pytest.raises(Exception) as ei:
            decode_stream(blob)
        assert type(ei.value).__name__ == case["exc"], case["name"]
        assert str(ei.value) == case["msg"], case["name"]


def test_encode_errors_match_reference():
    for case in json.loads((GOLDEN / "encode_errors.json").read_text()):
        if case["exc"] is None:
            continue
        dt = DT[case["dtype"]]
        x = np.frombuffer(bytes.fromhex(case["x_hex"]), dt.np_dtype)
        cfg = StreamConfig(dt, case["block_size"], Mode(case["mode"]), case["target"])
        with pytest.raises(Exception) as ei:
            encode_stream(x, cfg)
        assert type(ei.value).__name__ == case["exc"], case["name"]
        assert str(ei.value) == case["msg"], case["name"]


def _random_case(rng, dt):
    n = int(rng.integers(1, 20000))
    if dt is Dtype.F32:
        x = (np.cumsum(rng.standard_normal(n)) * 10.0 ** rng.uniform(-3, 3)).astype(np.float32)
    elif dt is Dtype.F64:
        x = np.cumsum(rng.standard_normal(n)) * 10.0 ** rng.uniform(-30, 30)
    else:
        info = np.iinfo(dt.np_dtype)
        kind = rng.integers(0, 3)
        if kind == 0:
            x = rng.integers(info.min, info.max + 1, n)
        else:
            x = np.clip(np.cumsum(rng.integers(-50, 51, n)) * (1 + (kind == 2) * 1000),
                        info.min, info.max)
        x = x.astype(dt.np_dtype)
    return x


@pytest.mark.parametrize("seed", range(12))
def test_random_configs_vs_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(8):
        dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64][rng.integers(0, 5)]
        modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
        mode = modes[rng.integers(0, len(modes))]
        bs = int(rng.choice([64, 100, 128, 256, 500, 1024, 2048, 4096, 6000, 8192, 16384]))
        target = float(rng.uniform(1, 12)) if mode is Mode.FIXED_RATE else float(rng.uniform(10, 100))
        seg = int(rng.choice([0, 0, 1, 2, 3, 8]))
        pol = "warm_self" if (mode is Mode.FIXED_RATE and rng.integers(0, 2)) else "cold"
        x = _random_case(rng, dt)
        cfg = StreamConfig(dt, bs, mode, target, segment_blocks=seg or None, segment_policy=pol)
        ref, offs, _ = O.encode(x, dt.wire_code, mode.value, target, bs, segment_blocks=seg,
                                policy=1 if pol == "warm_self" else 0, nthreads=4)
        res = encode_device(torch.from_numpy(x).cuda(), cfg)
        got = res.to_bytes()
        assert got == ref, (dt, mode, bs, target, seg, pol, x.size)
        y = decode_device(res.blob, res.nbytes).cpu().numpy()
        assert np.array_equal(y, O.decode(ref)), (dt, mode, bs, seg)


def test_bench_size_cfg2_segmented_vs_oracle():
    """Full BASELINE cfg2 size (2^26 f32, FQ at the profiler target, P=16):
    byte-exact container and bit-exact decode against the oracle."""
    x = W.cfg2_ar2_f32()
    cfg = StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=16)
    enc = Encoder(x.size, cfg)
    enc.encode(torch.from_numpy(x).cuda())
    res = enc.result()
    ref, offs, _ = O.encode(x, 3, 2, W.CFG2_TARGET_DB, 4096, segment_blocks=16, nthreads=0)
    assert res.to_bytes() == ref
    assert np.array_equal(res.block_offsets.cpu().numpy(), offs)
    dec = Decoder(x.size, Dtype.F32, 4096)
    dec.decode(res.blob, res.nbytes, res.block_offsets)
    y = dec.finish().cpu().numpy()
    yo = O.decode(ref, offs, nthreads=0)
    assert np.array_equal(y, yo)
    # the segment-serial decoder on the same container
    dec.decode(res.blob, res.nbytes, res.block_offsets, segment_blocks=16)
    assert np.array_equal(dec.finish().cpu().numpy(), yo)


def test_bench_size_cfg1_lossless_round_trip():
    x = W.cfg1_sines_i16()
    res = encode_device(torch.from_numpy(x).cuda(), StreamConfig(Dtype.I16, 4096))
    ref, offs, _ = O.encode(x, 1, 0, 0.0, 4096, nthreads=0)
    assert res.to_bytes() == ref
    y = decode_device(res.blob, res.nbytes, res.block_offsets).cpu().numpy()
    assert np.array_equal(y, x)


@pytest.mark.parametrize("n", [4096 * 3 + 3, 4096 + 1, 4096 * 3 + 4, 4096 * 2 + 29, 4096 * 5 + 100])
@pytest.mark.parametrize("dt,mode,target", [(Dtype.I16, Mode.LOSSLESS, 0.0), (Dtype.I32, Mode.LOSSLESS, 0.0),
                                            (Dtype.F32, Mode.FIXED_RATE, 8.0), (Dtype.I16, Mode.FIXED_QUALITY, 40.0)])
def test_short_partial_last_block(n, dt, mode, target):
    """A last block of a few groups (np not a multiple of a thread's 16
    samples): the exact centre-frequency monitor must look at the padded
    block only (a regression: stale q-buffer values past np fired the 1/3
    gate and forced D0 on cfg1's 3-sample tail)."""
    x = W.cfg1_sines_i16(n).astype(dt.np_dtype)
    res = encode_device(torch.from_numpy(x).cuda(), StreamConfig(dt, 4096, mode, target))
    ref, offs, _ = O.encode(x, dt.wire_code, mode.value, target, 4096)
    assert res.to_bytes() == ref
    assert np.array_equal(res.block_offsets.cpu().numpy(), offs)
    assert np.array_equal(decode_device(res.blob, res.nbytes).cpu().numpy(), O.decode(ref))


def _oscillating_case(rng, dt, n):
    """High-frequency sinusoid mixtures (centre frequency near the 1/3 gate
    of transform.py:107-113) plus noise and a random level."""
    t = np.arange(n, dtype=np.float64)
    f = rng.uniform(0.05, 0.5, 3)
    x = sum(rng.uniform(0.3, 1.0) * np.sin(2 * np.pi * fi * t + rng.uniform(0, 6.3)) for fi in f)
    x = x + rng.normal(0, rng.uniform(0.0, 0.5), n) + rng.uniform(-0.5, 0.5)
    if dt.is_float:
        return (x * 10.0 ** rng.uniform(-3, 5)).astype(dt.np_dtype)
    info = np.iinfo(dt.np_dtype)
    return np.clip(np.rint(x * 0.3 * info.max), info.min, info.max).astype(dt.np_dtype)


@pytest.mark.parametrize("seed", range(6))
def test_random_short_tails_vs_oracle(seed):
    """Random dtype / mode / block size / segments over oscillating data
    whose last block is a short tail (1..70 samples): the monitor gate, the
    partial-block paths and the d3 / v2 decoders, all against the oracle."""
    rng = np.random.default_rng(7000 + seed)
    for _ in range(8):
        dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64][rng.integers(0, 5)]
        modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
        mode = modes[rng.integers(0, len(modes))]
        bs = int(rng.choice([128, 256, 1000, 2048, 4096, 5000]))
        n = bs * int(rng.integers(1, 9)) + int(rng.integers(1, 71))
        target = float(rng.uniform(1, 12)) if mode is Mode.FIXED_RATE else float(rng.uniform(10, 100))
        seg = int(rng.choice([0, 0, 1, 2, 3]))
        pol = "warm_self" if (mode is Mode.FIXED_RATE and rng.integers(0, 2)) else "cold"
        x = _oscillating_case(rng, dt, n)
        cfg = StreamConfig(dt, bs, mode, target, segment_blocks=seg or None, segment_policy=pol)
        ref, offs, _ = O.encode(x, dt.wire_code, mode.value, target, bs, segment_blocks=seg,
                                policy=1 if pol == "warm_self" else 0)
        res = encode_device(torch.from_numpy(x).cuda(), cfg)
        assert res.to_bytes() == ref, (dt, mode, bs, target, seg, pol, n)
        yo = O.decode(ref)
        assert np.array_equal(decode_device(res.blob, res.nbytes).cpu().numpy(), yo), (dt, mode, bs, seg)
        if seg:
            y3 = decode_device(res.blob, res.nbytes, res.block_offsets, segment_blocks=seg).cpu().numpy()
            assert np.array_equal(y3, yo), (dt, mode, bs, seg, "d3")


@pytest.mark.parametrize("k", [10, 11, 12, 13, 14, 15])
def test_segment_decoder_width_boundaries(k):
    """The segment decoder's reconstruct scan switches arithmetic on the
    block's widest group (<= 14: 32-bit warp-level partial sums; <= 16:
    32-bit value sums; wider: 64-bit).  A 2^30 sine (D2 residual ~2^10) plus
    uniform noise of +-2^k gives D2 widths around k + 3, i.e. both sides of
    each switch: the LOSSLESS round trip is exact, the whole-stream and
    segmented decodes agree, and the container is the oracle's."""
    rng = np.random.default_rng(5000 + k)
    n = 4096 * 24 + 777
    i = np.arange(n)
    x = (np.round((2 ** 30) * np.sin(i * 2.0 ** -10)) +
         rng.integers(-(2 ** k), 2 ** k, n)).astype(np.int32)
    for seg in (4, None):
        cfg = StreamConfig(Dtype.I32, 4096, Mode.LOSSLESS, 0.0, segment_blocks=seg)
        res = encode_device(torch.from_numpy(x).cuda(), cfg)
        blob = res.to_bytes()
        assert blob == O.encode(x, Dtype.I32.wire_code, Mode.LOSSLESS.value, 0.0, 4096,
                                segment_blocks=seg or 0)[0]
        y = decode_device(res.blob, res.nbytes, res.block_offsets, segment_blocks=seg).cpu().numpy()
        assert np.array_equal(y, x), (k, seg)
        y2 = decode_device(res.blob, res.nbytes).cpu().numpy()
        assert np.array_equal(y2, x), (k, seg)


# ---------------------------------------------------------------------------
# encode_stream's input conversions (reference codec.py:266-272): inputs of
# other dtypes, coded by the container dtype path when it holds the widened
# values exactly, else by apax_encode_cast (generic kernel on int64 / f64)
# ---------------------------------------------------------------------------
def _cast_cases():
    return [m["name"] for m in json.loads((GOLDEN / "cast_manifest.json").read_text())]


@pytest.mark.parametrize("name", _cast_cases())
def test_cast_container_vs_reference(name):
    c = load_container(GOLDEN / "containers" / f"{name}.npz")
    m = c["meta"]
    cfg = StreamConfig(DT[m["dtype"]], m["block_size"], Mode(m["mode"]), float.fromhex(m["target_hex"]))
    got = encode_stream(c["x"], cfg)
    assert got == c["blob"], name
    y = decode_stream(c["blob"])
    assert y.dtype == c["y"].dtype and np.array_equal(y, c["y"])


def test_cast_errors_vs_reference():
    for case in json.loads((GOLDEN / "cast_errors.json").read_text()):
        x = np.frombuffer(bytes.fromhex(case["x_hex"]), np.dtype(case["x_dtype"]))
        cfg = StreamConfig(DT[case["dtype"]], case["block_size"], Mode(case["mode"]), case["target"])
        if case["exc"] is None:
            assert encode_stream(x, cfg).hex() == case["blob_hex"], case["name"]
            continue
        with pytest.raises(Exception) as ei:
            encode_stream(x, cfg)
        assert type(ei.value).__name__ == case["exc"], case["name"]
        assert str(ei.value) == case["msg"], case["name"]


@pytest.mark.parametrize("seed", range(4))
def test_cast_random_vs_oracle(seed):
    """f64 samples into f32 containers and int64 samples into narrower
    integer containers, every mode, random block sizes, against the oracle's
    restatement of the reference's widening."""
    rng = np.random.default_rng(3000 + seed)
    for _ in range(6):
        n = int(rng.integers(1, 30000))
        bs = int(rng.choice([64, 100, 512, 1000, 4096]))
        if rng.integers(0, 2):
            dt = Dtype.F32
            x = np.cumsum(rng.standard_normal(n)) * 10.0 ** rng.uniform(-3, 5)
            mode = Mode(int(rng.integers(1, 3)))
        else:
            dt = DT[str(rng.choice(["i8", "i16", "i32"]))]
            info = np.iinfo(dt.np_dtype)
            x = np.clip(np.cumsum(rng.standard_normal(n)) * float(info.max) * rng.uniform(0.01, 0.3),
                        -2.0 ** 32, 2.0 ** 32).astype(np.int64)
            mode = Mode(int(rng.integers(0, 3)))
        T = {Mode.LOSSLESS: 0.0, Mode.FIXED_RATE: float(rng.uniform(2, 12)),
             Mode.FIXED_QUALITY: float(rng.uniform(20, 90))}[mode]
        cfg = StreamConfig(dt, bs, mode, T)
        ref = O.encode(x, dt.wire_code, mode.value, T, bs)[0]
        assert encode_stream(x, cfg) == ref, (n, bs, dt, mode, T)
        assert np.array_equal(decode_stream(ref), O.decode(ref))


def test_cast_segmented_warm_self_vs_oracle():
    """Widened samples in segmented fixed-rate containers under warm_self: the
    preset's cost pass at gain 1 fails on samples beyond 34 bits exactly where
    the oracle's does (the first block of the first such segment), and codes
    the same bytes otherwise."""
    rng = np.random.default_rng(3100)
    t = np.arange(128 * 8 + 50)
    v = np.sin(t * 0.07) + rng.normal(0, 0.1, t.size)
    for scale, fails in ((0.3, False), (3.0, False), (50.0, True), (900.0, True)):
        x = np.rint(v * scale * (2 ** 31 - 1)).astype(np.int64)
        if fails:
            x[:128 * 3] //= 1000       # the first segment fits: the error is segment 1's
        cfg = StreamConfig(Dtype.I32, 128, Mode.FIXED_RATE, 6.0, segment_blocks=3, segment_policy="warm_self")
        try:
            ref = O.encode(x, 2, Mode.FIXED_RATE.value, 6.0, 128, segment_blocks=3, policy=1)[0]
        except O.OracleError as e:
            ref = e
        assert isinstance(ref, O.OracleError) == fails
        if fails:
            assert (ref.code, ref.detail) == (10, 3)
            with pytest.raises(Exception) as ei:
                encode_stream(x, cfg)
            assert "34-bit" in str(ei.value)
        else:
            assert encode_stream(x, cfg) == ref


# ---------------------------------------------------------------------------
# per-block traces against the reference stepping encode_block: scale code,
# block exponent, selector, costs, bytes and restart exact; the attenuation
# within 1e-9 dB and its gain within 1e-12 relative (the device's exp10 /
# log10 vs glibc's pow / log10)
# ---------------------------------------------------------------------------
def _trace_names():
    from trace_cases import traces
    return [t["name"] for t in traces()]


@pytest.mark.parametrize("name", _trace_names())
def test_trace_vs_reference(name):
    from trace_cases import trace_input, traces
    t = next(t for t in traces() if t["name"] == name)
    x = torch.from_numpy(trace_input(t)).cuda()
    cfg = StreamConfig(DT[t["dtype"]], 4096, Mode(t["mode"]), float.fromhex(t["target_hex"]),
                       segment_blocks=t["segment_blocks"] or None)
    res = encode_device(x, cfg, trace=True)
    tr = res.trace.cpu().numpy()
    ref = np.array(t["rows"], dtype=np.float64)
    assert tr.shape == ref.shape
    assert np.array_equal(tr[:, 2:], ref[:, 2:]), (name, np.argwhere(tr[:, 2:] != ref[:, 2:])[:5])
    assert np.allclose(tr[:, 0], ref[:, 0], rtol=0, atol=1e-9), name
    assert np.allclose(tr[:, 1], ref[:, 1], rtol=1e-12, atol=0), name


def test_floor_log2_quirk_containers():
    """glibc's floor(math.log2(s_des)) rounds up just below 2^32 and 2^-31:
    the device reproduces the reference's (code, fbe) and container."""
    for m in json.loads((GOLDEN / "quirk_manifest.json").read_text()):
        c = load_container(GOLDEN / "containers" / f"{m['name']}.npz")
        cfg = StreamConfig(DT[m["dtype"]], m["block_size"], Mode(m["mode"]), float.fromhex(m["target_hex"]))
        res = encode_device(torch.from_numpy(c["x"]).cuda(), cfg, trace=True)
        assert res.to_bytes() == c["blob"], m["name"]
        tr = res.trace.cpu().numpy()
        assert (int(tr[0][2]), int(tr[0][3])) == (m["first_block"]["code"], m["first_block"]["fbe"])
        assert np.array_equal(decode_stream(c["blob"]), c["y"])


@pytest.mark.parametrize("bs", [4096, 1000])
def test_whole_stream_ignores_segment_policy(bs):
    """segment_policy belongs to segments: a whole stream (segment_blocks=None)
    is the reference's encode_stream under either policy, on the split encoder
    (block size 4096) and the general one alike."""
    n = bs * 9 + 321
    for dt, x, target in ((Dtype.I16, W.cfg1_sines_i16(n), 4.0), (Dtype.F32, W.cfg2_ar2_f32(n), 6.0),
                          (Dtype.F64, W.cfg2_ar2_f32(n).astype(np.float64), 3.0)):
        ref, _, _ = O.encode(x, dt.wire_code, Mode.FIXED_RATE.value, target, bs, segment_blocks=0, policy=0)
        ref_w, _, _ = O.encode(x, dt.wire_code, Mode.FIXED_RATE.value, target, bs, segment_blocks=0, policy=1)
        assert ref == ref_w
        for pol in ("cold", "warm_self"):
            res = encode_device(torch.from_numpy(x).cuda(), StreamConfig(dt, bs, Mode.FIXED_RATE, target,
                                                                         segment_policy=pol))
            assert res.to_bytes() == ref, (dt, pol)


@pytest.mark.parametrize("bs,mode,target,seg,pol", [
    (8192, Mode.FIXED_QUALITY, 40.0, None, "cold"),        # the general encoder
    (4096, Mode.FIXED_RATE, 8.0, 2, "warm_self"),          # the fused segment encoder
    (4096, Mode.FIXED_RATE, 8.0, None, "cold"),            # the whole-stream chain + packer
    (4096, Mode.FIXED_QUALITY, 300.0, 4, "cold"),
    (128, Mode.FIXED_RATE, 16.0, None, "cold"),
])
def test_f64_beyond_block_exponent_range_vs_oracle(bs, mode, target, seg, pol):
    """f64 samples so large that the int8 block exponent stops at -127
    (|x| > 2^191): the quantized samples leave the 34-bit range and the
    reference raises InternalError for the first such block (entropy.py:53-54).
    The encoders report the same block, touch nothing outside their buffers,
    and the next encode on the same device is unaffected."""
    rng = np.random.default_rng(77)
    n = bs * 5 + 33
    x = np.cumsum(rng.standard_normal(n)) * 1e3
    x[bs * 2 + 7] = np.finfo(np.float64).max        # block 2
    x[bs * 3:bs * 3 + 50] = -1e200                  # block 3
    with pytest.raises(O.OracleError) as e_ref:
        O.encode(x, 4, mode.value, target, bs, segment_blocks=seg or 0, policy=1 if pol == "warm_self" else 0)
    assert e_ref.value.code == 10
    cfg = StreamConfig(Dtype.F64, bs, mode, target, segment_blocks=seg, segment_policy=pol)
    enc = Encoder(n, cfg)
    enc.encode(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    key = int(enc.status.cpu().numpy().view(np.uint64)[1])
    assert (key & 0xFF, key >> 8) == (10, e_ref.value.detail)
    x[bs * 2 + 7] = 1.0
    x[bs * 3:bs * 3 + 50] = 2.0
    ref = O.encode(x, 4, mode.value, target, bs, segment_blocks=seg or 0, policy=1 if pol == "warm_self" else 0)[0]
    assert encode_device(torch.from_numpy(x).cuda(), cfg).to_bytes() == ref
