"""Replays test_segment_decoder_random_vs_oracle cases one by one (triage)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, decode_device, encode_device  # noqa: E402
from test_gpu_parity import _random_case  # noqa: E402

seeds = [int(a) for a in sys.argv[1:]] or list(range(6))
for seed in seeds:
    rng = np.random.default_rng(4000 + seed)
    for it in range(8):
        dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32][rng.integers(0, 4)]
        modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
        mode = modes[rng.integers(0, len(modes))]
        bs = int(rng.choice([128, 256, 1024, 2048, 4096, 4096]))
        target = float(rng.uniform(1, 12)) if mode is Mode.FIXED_RATE else float(rng.uniform(10, 100))
        seg = int(rng.choice([1, 2, 3, 8, 16]))
        x = _random_case(rng, dt)
        if rng.integers(0, 2):
            x = np.concatenate([x, x[: bs * 3]])
        print(f"seed {seed} it {it}: {dt.name} {mode.name} bs={bs} seg={seg} n={x.size}", end=" ", flush=True)
        cfg = StreamConfig(dt, bs, mode, target, segment_blocks=seg)
        res = encode_device(torch.from_numpy(x).cuda(), cfg)
        torch.cuda.synchronize()
        print("enc ok", end=" ", flush=True)
        ref = O.decode(res.to_bytes())
        y = decode_device(res.blob, res.nbytes, res.block_offsets, segment_blocks=seg).cpu().numpy()
        print("ok" if np.array_equal(y, ref) else "MISMATCH", flush=True)
