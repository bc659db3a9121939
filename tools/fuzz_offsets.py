"""Robustness hunt for the decoders under a wrong side-band index (not a
test, and no oracle: a wrong index is the caller's error).  Random containers
are decoded with perturbed offset tables (negative, past the end, repeated,
swapped, shifted by a few bytes) and wrong segment lengths, through the
segment decoder, the two-pass decode and the block-range decode.  Nothing may
fault or hang: every call must end with samples or an error status, and a
decode with the true index afterwards must still give the oracle's samples.
Usage: python tools/fuzz_offsets.py [cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1303_4994_b200 import Decoder, Dtype, Mode, StreamConfig, decode_range, encode_device  # noqa: E402
from test_gpu_parity import _oscillating_case, _random_case  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 41)
bad = 0
for i in range(cases):
    dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64][rng.integers(0, 5)]
    modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
    mode = modes[rng.integers(0, len(modes))]
    bs = int(rng.choice([64, 256, 1000, 4096, 4096, 8192]))
    n = bs * int(rng.integers(1, 40)) + int(rng.integers(1, bs + 1))
    target = float(rng.uniform(1, 12)) if mode is Mode.FIXED_RATE else float(rng.uniform(10, 100))
    seg = int(rng.choice([0, 1, 3, 7]))
    x = _oscillating_case(rng, dt, n) if rng.integers(0, 2) else _random_case(rng, dt)[:n]
    if x.size < 2:
        continue
    n = x.size
    nb = (n + bs - 1) // bs
    res = encode_device(torch.from_numpy(np.ascontiguousarray(x)).cuda(),
                        StreamConfig(dt, bs, mode, target, segment_blocks=seg or None))
    blob = res.to_bytes()
    ref = O.decode(blob)
    offs = res.block_offsets.cpu().numpy().copy()
    dec = Decoder(n, dt, bs)
    why = ""
    try:
        for _ in range(4):
            o = offs.copy()
            for _ in range(int(rng.integers(1, 5))):
                k = int(rng.integers(0, nb + 1))
                kind = int(rng.integers(0, 7))
                if kind == 0: o[k] = -int(rng.integers(1, 1 << 40))
                elif kind == 1: o[k] = len(blob) + int(rng.integers(0, 1 << 20))
                elif kind == 2: o[k] = o[int(rng.integers(0, nb + 1))]
                elif kind == 3: o[k] += int(rng.integers(-9, 10))
                elif kind == 4: o[k:] = o[k:][::-1].copy()
                elif kind == 5: o[k] = int(rng.integers(0, len(blob)))
                else: o[k] = (1 << 62) + int(rng.integers(0, 1 << 20))
            od = torch.from_numpy(o).cuda()
            wrong_seg = int(rng.choice([seg or 1, 1, 2, 5, nb + 3]))
            why = f"segments offs P={wrong_seg}"
            dec.decode(res.blob, res.nbytes, od, segment_blocks=wrong_seg)
            torch.cuda.synchronize()
            why = "two-pass offs"
            dec.decode(res.blob, res.nbytes, od)
            torch.cuda.synchronize()
            b0 = int(rng.integers(0, nb)); b1 = int(rng.integers(b0 + 1, nb + 1))
            why = f"range {b0}:{b1}"
            try:
                decode_range(res.blob, res.nbytes, od, n, dt, bs, b0, b1, want_map=True)
            except Exception as e:  # noqa: BLE001  (an error status raised as an exception is fine)
                if "CUDA" in repr(e) or "illegal" in repr(e):
                    raise
            torch.cuda.synchronize()
        why = "true index after"
        dec.decode(res.blob, res.nbytes, res.block_offsets, segment_blocks=seg or None)
        ok = np.array_equal(dec.finish()[:n].cpu().numpy(), ref)
    except Exception as e:  # noqa: BLE001
        ok = False
        why += " " + repr(e)[:80]
    if not ok:
        bad += 1
        print("MISMATCH", i, dt.code, mode.name, bs, n, seg, why, flush=True)
        if "CUDA" in why or "illegal" in why:
            break
print(f"{cases} cases, {bad} mismatches")
