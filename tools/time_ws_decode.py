"""Decode times of the reference's own (whole-stream) container of the cfg2
array: with the side-band index and without it (CUDA events, L2 flushed)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1303_4994_b200 import Decoder, Dtype, Encoder, Mode, StreamConfig  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402


def timed(fn, reps=8):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


x = W.cfg2_ar2_f32()
n = x.size
enc = Encoder(n, StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB))
enc.encode(torch.from_numpy(x).cuda())
nb = enc.finish()
dec = Decoder(n, Dtype.F32, 4096)
t_idx = timed(lambda: dec.decode(enc.out, nb, enc.offsets))
y1 = dec.finish().clone()
t_il = timed(lambda: dec.decode(enc.out, nb, None))
print(f"whole-stream cfg2 container ({nb} bytes): with index {t_idx:.4f} ms, index-less {t_il:.4f} ms, same={bool(torch.equal(dec.finish(), y1))}")
