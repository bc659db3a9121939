"""Encode timings of the fused (v3) and split (chain + packer) encoders on
BASELINE-shaped workloads, segmented and whole-stream (CUDA events, median
of 5 after 2 warm-ups).  Run on the GPU box:  python tools/time_encode.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402


def timed(enc, x, reps=5):
    ts = []
    for k in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        enc.encode(x)
        b.record()
        torch.cuda.synchronize()
        if k >= 2:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts)), enc.finish()


def main():
    cases = [
        ("cfg2 FQ P=28", W.cfg2_ar2_f32(1 << 26), Dtype.F32, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, 28, "cold"),
        ("cfg1 FR P=7", W.cfg1_sines_i16(1 << 24), Dtype.I16, Mode.FIXED_RATE, 4.0, 7, "warm_self"),
        ("cfg1 LOSSLESS whole", W.cfg1_sines_i16(1 << 24), Dtype.I16, Mode.LOSSLESS, 0.0, None, "cold"),
        ("cfg1 FR whole", W.cfg1_sines_i16(1 << 24), Dtype.I16, Mode.FIXED_RATE, 4.0, None, "cold"),
        ("cfg2/16 FQ whole", W.cfg2_ar2_f32(1 << 22), Dtype.F32, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, None, "cold"),
    ]
    if len(sys.argv) > 1:
        cases = [c for c in cases if any(s in c[0] for s in sys.argv[1:])]
    for name, xh, dt, mode, T, P, pol in cases:
        x = torch.from_numpy(xh).cuda()
        cfg = StreamConfig(dt, 4096, mode, T, segment_blocks=P, segment_policy=pol)
        out = {}
        blobs = {}
        for split in ("0", "1"):
            os.environ["APAX_ENC_SPLIT"] = split
            enc = Encoder(x.numel(), cfg)
            ms, nb = timed(enc, x)
            out[split] = ms
            blobs[split] = enc.out[:nb].cpu().numpy().tobytes()
        same = blobs["0"] == blobs["1"]
        print(f"{name:22s} fused {out['0']:8.3f} ms  split {out['1']:8.3f} ms  identical {same}  bytes {len(blobs['0'])}",
              flush=True)


if __name__ == "__main__":
    main()
