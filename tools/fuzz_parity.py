"""Randomised GPU-vs-oracle parity search (not a test: a bug hunt).
Usage: python tools/fuzz_parity.py [cases] [seed]"""
import sys
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, decode_device, encode_device  # noqa: E402
from test_gpu_parity import _oscillating_case, _random_case  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 99)
bad = 0
for i in range(cases):
    dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64][rng.integers(0, 5)]
    modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
    mode = modes[rng.integers(0, len(modes))]
    bs = int(rng.choice([64, 100, 128, 256, 512, 1000, 2048, 4096, 5000, 8192]))
    n = bs * int(rng.integers(0, int(os.environ.get("FUZZ_MAXBLK", "6")))) + int(rng.integers(1, 2 * bs))
    target = float(rng.uniform(0.5, 16)) if mode is Mode.FIXED_RATE else float(rng.uniform(5, 120))
    seg = int(rng.choice([0, 0, 1, 2, 3, 7]))
    pol = "warm_self" if (mode is Mode.FIXED_RATE and rng.integers(0, 2)) else "cold"
    x = _oscillating_case(rng, dt, n) if rng.integers(0, 2) else _random_case(rng, dt)[:n]
    if x.size == 0:
        continue
    try:
        ref, offs, _ = O.encode(x, dt.wire_code, mode.value, target, bs, segment_blocks=seg,
                                policy=1 if pol == "warm_self" else 0)
    except O.OracleError as e:
        ref = e
    cfg = StreamConfig(dt, bs, mode, target, segment_blocks=seg or None, segment_policy=pol)
    try:
        res = encode_device(torch.from_numpy(np.ascontiguousarray(x)).cuda(), cfg)
        got = res.to_bytes()
    except Exception as e:  # noqa: BLE001
        got = e
    ok = (isinstance(ref, Exception) and isinstance(got, Exception)) or (got == ref)
    if ok and not isinstance(ref, Exception):
        yo = O.decode(ref)
        ok = np.array_equal(decode_device(res.blob, res.nbytes).cpu().numpy(), yo)
        if ok:   # with the side-band index, segment structure not given (two-pass decode)
            ok = np.array_equal(decode_device(res.blob, res.nbytes, res.block_offsets).cpu().numpy(), yo)
        if ok and seg:
            ok = np.array_equal(decode_device(res.blob, res.nbytes, res.block_offsets,
                                              segment_blocks=seg).cpu().numpy(), yo)
    if not ok:
        bad += 1
        print("MISMATCH", i, dt.code, mode.name, bs, n, round(target, 3), seg, pol,
              type(ref).__name__ if isinstance(ref, Exception) else len(ref),
              type(got).__name__ if isinstance(got, Exception) else len(got), flush=True)
print(f"{cases} cases, {bad} mismatches")
