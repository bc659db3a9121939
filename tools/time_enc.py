"""Time the cfg2 device encode (and decode) only, with whatever library
APAX_LIB_PATH points at (tuning variants).  Usage: python tools/time_enc.py [P]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig, wave_segment_blocks  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402


def main():
    n = 1 << 26
    seg = int(sys.argv[1]) if len(sys.argv) > 1 else wave_segment_blocks(n, Dtype.F32, Mode.FIXED_QUALITY, 4096)
    x = torch.from_numpy(W.cfg2_ar2_f32(n)).cuda()
    enc = Encoder(n, StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=seg))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        enc.encode(x)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        enc.encode(x)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"P={seg} encode ms: median {ts[len(ts) // 2]:.4f} min {ts[0]:.4f}")


if __name__ == "__main__":
    main()
