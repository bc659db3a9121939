"""Randomised search over the block API (not a test: a bug hunt): stepping
encode_block with one CodecState / RateLoopState over the blocks of a random
stream (as the reference's encode_stream does, codec.py:274-285) must
rebuild the oracle's whole-stream container byte for byte, or stop at the
block where the oracle reports an error.
Usage: python tools/fuzz_block_api.py [cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1303_4994_b200 import Mode, StreamConfig  # noqa: E402
from paper_1303_4994_b200 import block as A  # noqa: E402
from paper_1303_4994_b200.block import CodecState, RateLoopState  # noqa: E402
from fuzz_extremes import make_case  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 43)
bad = 0
for i in range(cases):
    if rng.integers(0, 2):
        x, dt, mode, bs, n, target, _, _ = make_case(rng)
    else:
        from fuzz_extremes import Dtype
        dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64][rng.integers(0, 5)]
        modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
        mode = modes[rng.integers(0, len(modes))]
        bs = int(rng.choice([64, 256, 1000, 4096]))
        n = bs * int(rng.integers(0, 8)) + int(rng.integers(1, bs + 1))
        target = float(rng.uniform(1, 12)) if mode is Mode.FIXED_RATE else float(rng.uniform(10, 100))
        v = np.cumsum(rng.standard_normal(n))
        if dt.is_float:
            x = (v * 10.0 ** rng.uniform(-3, 3)).astype(dt.np_dtype)
        else:
            info = np.iinfo(dt.np_dtype)
            x = np.clip(np.rint(v * info.max * 0.02), info.min, info.max).astype(dt.np_dtype)
    x = x[:bs * 6]          # a few blocks: every step is a device round trip
    n = x.size
    try:
        ref = O.encode(x, dt.wire_code, mode.value, target, bs)[0]
    except O.OracleError as e:
        ref = e
    why = ""
    try:
        cfg = StreamConfig(dt, bs, mode, target)
        st = CodecState(cfg)
        loop = RateLoopState(cfg.target) if cfg.mode is Mode.FIXED_RATE else None
        parts = []
        err = None
        for b in range(0, n, bs):
            try:
                h, payload = A.encode_block(x[b:b + bs], st, loop)
            except Exception as e:  # noqa: BLE001
                err = (b // bs, type(e).__name__)
                break
            parts.append(h.serialize(dt) + payload)
        if isinstance(ref, O.OracleError):
            ok = err is not None and (ref.code == 9 or err[0] == ref.detail)
            why = f"oracle error {(ref.code, ref.detail)}, block API {err}"
        else:
            ok = err is None and b"".join(parts) == ref[28:]
            why = f"bytes (block API error {err})"
    except Exception as e:  # noqa: BLE001
        ok = isinstance(ref, O.OracleError)
        why = "config " + repr(e)[:80]
    if not ok:
        bad += 1
        print("MISMATCH", i, dt.code, mode.name, bs, n, round(target, 3), why, flush=True)
print(f"{cases} cases, {bad} mismatches")
