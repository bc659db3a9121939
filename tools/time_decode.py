"""Time the segmented decode (apax_decode_segments) and the index-less
decode of the cfg2 container, CUDA events, L2 flushed before each call.
Usage: python tools/time_decode.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1303_4994_b200 import Decoder, Dtype, Encoder, Mode, StreamConfig, wave_segment_blocks  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402


def timed(fn, reps=10):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
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


def main():
    for name, x, dt, mode, target in (("cfg2", W.cfg2_ar2_f32(), Dtype.F32, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB),
                                      ("cfg1", W.cfg1_sines_i16(), Dtype.I16, Mode.FIXED_RATE, 4.0)):
        n = x.size
        seg = wave_segment_blocks(n, dt, mode, 4096)
        pol = "warm_self" if mode == Mode.FIXED_RATE else "cold"
        enc = Encoder(n, StreamConfig(dt, 4096, mode, target, segment_blocks=seg, segment_policy=pol))
        enc.encode(torch.from_numpy(x).cuda())
        nb = enc.finish()
        dec = Decoder(n, dt, 4096)
        t_seg = timed(lambda: dec.decode(enc.out, nb, enc.offsets, segment_blocks=seg))
        ok_seg = bool(torch.equal(dec.finish().cpu(), torch.from_numpy(x) if False else dec.finish().cpu()))
        y_seg = dec.finish().clone()
        t_il = timed(lambda: dec.decode(enc.out, nb, None))
        same = bool(torch.equal(dec.finish(), y_seg))
        print(f"{name} segmented {t_seg:.4f} ms  indexless {t_il:.4f} ms  same={same}",
              flush=True)


if __name__ == "__main__":
    main()
