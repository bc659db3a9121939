"""Randomised search over the block-range decode (not a test: a bug hunt):
random containers (whole-stream and segmented, every dtype / mode / block
size) decoded by R random block ranges -- maps with a (0, 0) entry, entries
composed on the host (distributed.range_entries), ranges decoded again from
their entries -- against the oracle's decode of the whole container.
Usage: python tools/fuzz_range.py [cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, decode_range, encode_device  # noqa: E402
from paper_1303_4994_b200 import distributed as D  # noqa: E402
from test_gpu_parity import _oscillating_case, _random_case  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 29)
bad = 0
for i in range(cases):
    dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64][rng.integers(0, 5)]
    modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
    mode = modes[rng.integers(0, len(modes))]
    bs = int(rng.choice([64, 256, 1000, 2048, 4096, 4096, 8192]))
    n = bs * int(rng.integers(1, 50)) + int(rng.integers(1, bs + 1))
    target = float(rng.uniform(0.5, 16)) if mode is Mode.FIXED_RATE else float(rng.uniform(5, 120))
    seg = int(rng.choice([0, 0, 0, 2, 5]))
    x = _oscillating_case(rng, dt, n) if rng.integers(0, 2) else _random_case(rng, dt)[:n]
    if x.size < 2:
        continue
    n = x.size
    nb = (n + bs - 1) // bs
    try:
        res = encode_device(torch.from_numpy(np.ascontiguousarray(x)).cuda(),
                            StreamConfig(dt, bs, mode, target, segment_blocks=seg or None))
        blob = res.to_bytes()
    except Exception:  # noqa: BLE001
        continue
    try:
        ref = O.decode(blob)
        R = int(rng.integers(1, min(nb, 6) + 1))
        cuts = sorted(set([0, nb] + [int(c) for c in rng.integers(1, max(nb, 2), R - 1)])) if nb > 1 else [0, nb]
        ranges = list(zip(cuts[:-1], cuts[1:]))
        maps = [decode_range(res.blob, res.nbytes, res.block_offsets, n, dt, bs, b0, b1, want_map=True)[1]
                for b0, b1 in ranges]
        entries = D.range_entries(maps)
        parts = [decode_range(res.blob, res.nbytes, res.block_offsets, n, dt, bs, b0, b1, entry=e)[0].cpu().numpy()
                 for (b0, b1), e in zip(ranges, entries)]
        ok = np.array_equal(np.concatenate(parts), ref)
        why = "samples"
    except Exception as e:  # noqa: BLE001
        ok, why = False, repr(e)[:100]
    if not ok:
        bad += 1
        print("MISMATCH", i, dt.code, mode.name, bs, n, round(target, 3), seg, ranges if 'ranges' in dir() else "", why, flush=True)
print(f"{cases} cases, {bad} mismatches")
