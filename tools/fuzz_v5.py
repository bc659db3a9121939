"""Randomised parity search for the v5 encoder (not a test: a bug hunt):
block size 4096, i16 / i32 / f32, fixed rate / fixed quality, cold and
warm_self, one-wave and several units per CTA (APAX_ENC_V5=2), against the
oracle.  FUZZ_NBLK_MIN / FUZZ_NBLK_MAX set the range of block counts (more
segments than resident CTAs: several units per CTA, the persistent v3 kernel).
Usage: python tools/fuzz_v5.py [cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, decode_device, encode_device  # noqa: E402
from test_gpu_parity import _oscillating_case  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
bad = 0
for i in range(cases):
    dt = [Dtype.I16, Dtype.I32, Dtype.F32][rng.integers(0, 3)]
    mode = [Mode.FIXED_RATE, Mode.FIXED_QUALITY][rng.integers(0, 2)]
    nblk = int(rng.integers(int(os.environ.get("FUZZ_NBLK_MIN", "1")), int(os.environ.get("FUZZ_NBLK_MAX", "60"))))
    n = 4096 * nblk + int(rng.integers(0, 2)) * int(rng.integers(1, 4096))
    seg = int(rng.choice([1, 2, 3, 5, 8, 13]))
    pol = "warm_self" if (mode is Mode.FIXED_RATE and rng.integers(0, 2)) else "cold"
    target = float(rng.uniform(0.5, 16)) if mode is Mode.FIXED_RATE else float(rng.uniform(5, 150))
    kind = int(rng.integers(0, 4))
    if kind == 0:
        x = _oscillating_case(rng, dt, n)
    elif kind == 1:   # smooth + noise + silent stretches + spikes
        t = np.arange(n)
        v = np.sin(t * rng.uniform(1e-4, 1e-2)) * rng.uniform(0.1, 1.0) + rng.normal(0, rng.uniform(0, 0.05), n)
        for _ in range(int(rng.integers(0, 4))):
            a = int(rng.integers(0, n)); v[a:a + int(rng.integers(1, 9000))] = 0.0
        for _ in range(int(rng.integers(0, 6))):
            v[int(rng.integers(0, n))] = rng.choice([-1.0, 1.0]) * rng.uniform(1, 50)
        if dt.is_float:
            x = (v * 10.0 ** rng.uniform(-20, 20)).astype(np.float32)
        else:
            info = np.iinfo(dt.np_dtype)
            x = np.clip(np.rint(v * rng.uniform(0.001, 1.0) * info.max), info.min, info.max).astype(dt.np_dtype)
    elif kind == 2:   # full-range noise (the 64-bit paths for i32)
        if dt.is_float:
            x = (rng.standard_normal(n) * 10.0 ** rng.uniform(-10, 30)).astype(np.float32)
        else:
            info = np.iinfo(dt.np_dtype)
            x = rng.integers(info.min, info.max, n, dtype=np.int64, endpoint=True).astype(dt.np_dtype)
    else:             # constant / tiny alphabets
        vals = rng.integers(-3, 4, int(rng.integers(1, 4)))
        x = rng.choice(vals, n).astype(dt.np_dtype)
    force = bool(rng.integers(0, 2))
    os.environ["APAX_ENC_V5"] = "2" if force else "1"
    try:
        ref, offs, _ = O.encode(x, dt.wire_code, mode.value, target, 4096, segment_blocks=seg,
                                policy=1 if pol == "warm_self" else 0)
    except O.OracleError as e:
        ref = e
    cfg = StreamConfig(dt, 4096, mode, target, segment_blocks=seg, segment_policy=pol)
    try:
        res = encode_device(torch.from_numpy(np.ascontiguousarray(x)).cuda(), cfg)
        got = res.to_bytes()
    except Exception as e:  # noqa: BLE001
        got = e
    ok = (isinstance(ref, Exception) and isinstance(got, Exception)) or (isinstance(ref, bytes) and got == ref)
    if ok and isinstance(ref, bytes):
        ok = np.array_equal(res.block_offsets.cpu().numpy(), offs)
        if ok:
            y = decode_device(res.blob, res.nbytes, res.block_offsets, segment_blocks=seg).cpu().numpy()
            ok = np.array_equal(y, O.decode(ref))
    if not ok:
        bad += 1
        print("MISMATCH", i, dt, mode, target, "P", seg, pol, "n", n, "kind", kind, "force", force,
              type(ref).__name__, type(got).__name__, flush=True)
print(f"{cases} cases, {bad} mismatches")
