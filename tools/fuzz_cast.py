"""Randomised parity search for encode_stream's input conversions (not a
test: a bug hunt): float64 samples into f32 / f64 containers, int64 samples
(in and out of range) and floats into integer containers, every mode, block
size and segment length, against the oracle's widened encode; then
decode_stream of the container against the oracle's decode.
Usage: python tools/fuzz_cast.py [cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, decode_stream, encode_stream  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 17)
bad = 0
for i in range(cases):
    dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64][rng.integers(0, 5)]
    modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
    mode = modes[rng.integers(0, len(modes))]
    bs = int(rng.choice([64, 128, 500, 1024, 4096, 4096, 8192]))
    n = bs * int(rng.integers(0, 12)) + int(rng.integers(1, 2 * bs))
    target = float(rng.uniform(0.5, 16)) if mode is Mode.FIXED_RATE else float(rng.uniform(5, 120))
    seg = int(rng.choice([0, 0, 1, 3, 6]))
    pol = "warm_self" if (mode is Mode.FIXED_RATE and rng.integers(0, 2)) else "cold"
    t = np.arange(n)
    v = np.sin(t * rng.uniform(1e-3, 0.5)) * rng.uniform(0.1, 1.0) + rng.normal(0, rng.uniform(0, 0.3), n)
    if dt.is_float:
        x = v * 10.0 ** rng.uniform(-8, 8)          # float64: not exactly representable in f32
        if os.environ.get("FUZZ_CAST_EXTREME") and rng.integers(0, 2):
            # beyond f32's range, up to f64's maximum, and below f32's denormals
            x = v * 10.0 ** float(rng.choice([-320, -300, -60, -40, 37, 39, 60, 190, 300, 307.5]))
        if rng.integers(0, 4) == 0:
            x = x.astype(np.float32).astype(np.float64)
        if rng.integers(0, 5) == 0:
            x = np.rint(v * 1000).astype(np.int64)  # integers into a float container
    else:
        info = np.iinfo(dt.np_dtype)
        scale = info.max * rng.choice([0.3, 1.0, 3.0, 50.0])   # beyond the container's range: clipped at decode
        if rng.integers(0, 2):
            x = np.rint(v * scale).astype(np.int64)
        else:
            x = v * scale                            # floats: astype(int64) truncates toward zero
    try:
        ref, _, _ = O.encode(x, dt.wire_code, mode.value, target, bs, segment_blocks=seg,
                             policy=1 if pol == "warm_self" else 0)
    except O.OracleError as e:
        ref = e
    cfg = StreamConfig(dt, bs, mode, target, segment_blocks=seg or None, segment_policy=pol)
    try:
        got = encode_stream(x, cfg)
    except Exception as e:  # noqa: BLE001
        got = e
    ok = (isinstance(ref, Exception) and isinstance(got, Exception)) or (got == ref)
    if ok and not isinstance(ref, Exception):
        ok = np.array_equal(decode_stream(got), O.decode(ref))
    if not ok:
        bad += 1
        print("MISMATCH", i, dt.code, mode.name, bs, n, round(target, 3), seg, pol, x.dtype,
              type(ref).__name__, type(got).__name__, flush=True)
print(f"{cases} cases, {bad} mismatches")
