"""cfg2 encode time and ratio against the segment length P: the one-wave v5
launch (P = 28) and ticketed launches with several units per CTA
(APAX_ENC_V5=2), v3 beside them (APAX_ENC_V5=0)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402


def timed(enc, x, reps=9):
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


x = torch.from_numpy(W.cfg2_ar2_f32(1 << 26)).cuda()
for P in (28, 19, 14, 10, 7, 4):
    cfg = StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=P)
    out = {}
    for v in ("0", "2"):
        os.environ["APAX_ENC_V5"] = v
        enc = Encoder(x.numel(), cfg)
        out[v] = timed(enc, x)
    print(f"P={P:3d} units {(16384 + P - 1) // P:5d}  v3 {out['0'][0]:.4f} ms  v5 {out['2'][0]:.4f} ms  ratio {4 * (1 << 26) / out['2'][1]:.4f}",
          flush=True)
