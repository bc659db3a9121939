"""Randomised search over the per-block trace (not a test: a bug hunt): the
GPU encoder's trace (att_db, a, code, fbe, selector, costs, bytes, restart per
block) against the oracle's for random dtypes, modes, block sizes, segment
lengths and policies.  att_db within 1e-9 dB, a within 1e-12 relative (the
device's exp10 against glibc's pow), everything else exact.
Usage: python tools/fuzz_trace.py [cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig  # noqa: E402
from test_gpu_parity import _oscillating_case, _random_case  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 23)
bad = 0
for i in range(cases):
    dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64][rng.integers(0, 5)]
    modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
    mode = modes[rng.integers(0, len(modes))]
    bs = int(rng.choice([64, 256, 1000, 4096, 4096, 4096, 8192]))
    n = bs * int(rng.integers(0, 40)) + int(rng.integers(1, 2 * bs))
    target = float(rng.uniform(0.5, 16)) if mode is Mode.FIXED_RATE else float(rng.uniform(5, 120))
    seg = int(rng.choice([0, 1, 2, 3, 5, 9]))
    pol = "warm_self" if (mode is Mode.FIXED_RATE and rng.integers(0, 2)) else "cold"
    x = _oscillating_case(rng, dt, n) if rng.integers(0, 2) else _random_case(rng, dt)[:n]
    if x.size == 0:
        continue
    n = x.size
    try:
        ref, _, tr = O.encode(x, dt.wire_code, mode.value, target, bs, segment_blocks=seg,
                              policy=1 if pol == "warm_self" else 0, trace=True)
    except O.OracleError:
        continue
    cfg = StreamConfig(dt, bs, mode, target, segment_blocks=seg or None, segment_policy=pol)
    try:
        enc = Encoder(n, cfg, trace=True)
        enc.encode(torch.from_numpy(np.ascontiguousarray(x)).cuda())
        nb = enc.finish()
        got = enc.trace.cpu().numpy()
        tr = np.asarray(tr).reshape(got.shape)
        ok = enc.out[:nb].cpu().numpy().tobytes() == ref
        why = "bytes"
        if ok:
            ok = np.array_equal(got[:, 2:], tr[:, 2:])
            why = "fields " + str(np.nonzero((got[:, 2:] != tr[:, 2:]).any(axis=1))[0][:4])
        if ok:
            ok = np.allclose(got[:, 0], tr[:, 0], rtol=0, atol=1e-9) and np.allclose(got[:, 1], tr[:, 1], rtol=1e-12, atol=0)
            why = "att/a"
    except Exception as e:  # noqa: BLE001
        ok, why = False, repr(e)[:80]
    if not ok:
        bad += 1
        print("MISMATCH", i, dt.code, mode.name, bs, n, round(target, 3), seg, pol, why, flush=True)
print(f"{cases} cases, {bad} mismatches")
