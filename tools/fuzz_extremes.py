"""Randomised search at the edges of the value range (not a test: a bug
hunt): float arrays mixing denormals, signed zeros, values next to the
type's maximum, tiny and huge scales, silent blocks and single spikes;
integer arrays at the type's limits; extreme targets (rates from 0.01 to 40
bits per sample, qualities from -20 to 400 dB).  The encoder must give the
oracle's bytes or the oracle's error (code and block); the decode the
oracle's samples.  Usage: python tools/fuzz_extremes.py [cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig, decode_device  # noqa: E402

U64 = (1 << 64) - 1


def make_case(rng):
    dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64][rng.integers(0, 5)]
    modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
    mode = modes[rng.integers(0, len(modes))]
    bs = int(rng.choice([64, 128, 1000, 4096, 4096, 4096, 8192]))
    n = bs * int(rng.integers(0, 10)) + int(rng.integers(1, 2 * bs))
    if mode is Mode.FIXED_RATE:
        target = float(rng.choice([0.01, 0.1, 0.5, 1, 3, 8, 16, 31, 40]) * rng.uniform(0.9, 1.1))
    else:
        target = float(rng.choice([-20, 0, 1, 10, 60, 150, 300, 400]) + rng.uniform(-1, 1))
    seg = int(rng.choice([0, 0, 1, 2, 4]))
    pol = "warm_self" if (mode is Mode.FIXED_RATE and rng.integers(0, 2)) else "cold"
    t = np.arange(n)
    v = np.sin(t * rng.uniform(1e-3, 1.0)) + rng.normal(0, rng.uniform(0, 1.0), n)
    if dt.is_float:
        fi = np.finfo(dt.np_dtype)
        scale = float(rng.choice([fi.tiny * 1e-3, fi.tiny, 1e-20, 1.0, 1e20, fi.max / 8, fi.max / 2.5]))
        with np.errstate(over="ignore", under="ignore"):
            x = (v * scale).astype(dt.np_dtype)
        x[~np.isfinite(x)] = fi.max
        for _ in range(int(rng.integers(0, 4))):
            a = int(rng.integers(0, n)); x[a:a + int(rng.integers(1, 3 * bs))] = rng.choice([0.0, -0.0, fi.tiny, fi.max, -fi.max])
        for _ in range(int(rng.integers(0, 4))):
            x[int(rng.integers(0, n))] = rng.choice([fi.max, -fi.max, fi.tiny, fi.smallest_subnormal, 1.0])
    else:
        info = np.iinfo(dt.np_dtype)
        x = np.clip(np.rint(v * info.max * rng.choice([1e-3, 0.5, 1.0, 2.0])), info.min, info.max).astype(dt.np_dtype)
        for _ in range(int(rng.integers(0, 4))):
            a = int(rng.integers(0, n)); x[a:a + int(rng.integers(1, 3 * bs))] = rng.choice([0, info.min, info.max, -1, 1])
        if rng.integers(0, 3) == 0:
            x[::2] = info.max; x[1::2] = info.min          # the widest second differences
    return x, dt, mode, bs, n, target, seg, pol


if __name__ == "__main__":
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 37)
    bad = 0
    for i in range(cases):
        x, dt, mode, bs, n, target, seg, pol = make_case(rng)
        if os.environ.get("FUZZ_VERBOSE"):
            print("case", i, dt.code, mode.name, bs, n, round(target, 3), seg, pol, flush=True)
        try:
            ref = O.encode(x, dt.wire_code, mode.value, target, bs, segment_blocks=seg,
                           policy=1 if pol == "warm_self" else 0)[0]
        except O.OracleError as e:
            ref = e
        why = ""
        try:
            cfg = StreamConfig(dt, bs, mode, target, segment_blocks=seg or None, segment_policy=pol)
        except Exception as e:  # noqa: BLE001  (configs the package rejects: the oracle must reject them too)
            ok = isinstance(ref, O.OracleError)
            why = "config " + repr(e)[:60]
            cfg = None
        if cfg is not None:
            try:
                enc = Encoder(n, cfg)
                enc.encode(torch.from_numpy(np.ascontiguousarray(x)).cuda())
            except Exception as e:  # noqa: BLE001  (rejected at the call: the oracle must reject it too)
                ok = isinstance(ref, O.OracleError)
                why = "call " + repr(e)[:60]
                cfg = None
        if cfg is not None:
            torch.cuda.synchronize()
            st = enc.status.cpu().numpy().view(np.uint64)
            key, nonfin = int(st[1]), int(st[0])
            if isinstance(ref, O.OracleError):
                got = (key & 0xFF, key >> 8) if key != U64 else (9, nonfin) if nonfin != U64 else None
                ok = got == (ref.code, ref.detail)
                why = f"error: oracle {(ref.code, ref.detail)} gpu {got}"
            else:
                ok = key == U64 and nonfin == U64
                why = f"gpu error {key & 0xFF} at {key >> 8}"
                if ok:
                    nb = enc.finish()
                    ok = enc.out[:nb].cpu().numpy().tobytes() == ref
                    why = "bytes"
                if ok:
                    ok = np.array_equal(decode_device(enc.out, nb).cpu().numpy(), O.decode(ref), equal_nan=True)
                    why = "decode"
        if not ok:
            bad += 1
            print("MISMATCH", i, dt.code, mode.name, bs, n, round(target, 3), seg, pol, why, flush=True)
    print(f"{cases} cases, {bad} mismatches")
