"""Replays tests/test_gpu_parity.py::test_random_configs_vs_oracle cases one at
a time, printing each config before running it (hang / mismatch triage)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, encode_device  # noqa: E402
from test_gpu_parity import _random_case  # noqa: E402

bad = 0
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    rng = np.random.default_rng(1000 + seed)
    for it in range(8):
        dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64][rng.integers(0, 5)]
        modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
        mode = modes[rng.integers(0, len(modes))]
        bs = int(rng.choice([64, 100, 128, 256, 500, 1024, 2048, 4096, 6000, 8192, 16384]))
        target = float(rng.uniform(1, 12)) if mode is Mode.FIXED_RATE else float(rng.uniform(10, 100))
        seg = int(rng.choice([0, 0, 1, 2, 3, 8]))
        pol = "warm_self" if (mode is Mode.FIXED_RATE and rng.integers(0, 2)) else "cold"
        x = _random_case(rng, dt)
        print(f"seed {seed} it {it}: {dt.name} {mode.name} bs={bs} T={target:.3f} seg={seg} {pol} n={x.size}",
              end=" ", flush=True)
        cfg = StreamConfig(dt, bs, mode, target, segment_blocks=seg or None, segment_policy=pol)
        ref, offs, _ = O.encode(x, dt.wire_code, mode.value, target, bs, segment_blocks=seg,
                                policy=1 if pol == "warm_self" else 0, nthreads=4)
        res = encode_device(torch.from_numpy(x).cuda(), cfg)
        got = res.to_bytes()
        first = next((i for i in range(min(len(got), len(ref))) if got[i] != ref[i]), None)
        ok = got == ref
        bad += not ok
        print("ok" if ok else f"MISMATCH len {len(got)} vs {len(ref)} first {first}", flush=True)
print("bad", bad)
