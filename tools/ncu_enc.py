"""One fused and one split cfg2 encode (2^26 f32 FQ, P = 28) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

x = torch.from_numpy(W.cfg2_ar2_f32(1 << 26)).cuda()
cfg = StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=28, segment_policy="cold")
for split in (sys.argv[1:] or ["0", "1"]):
    os.environ["APAX_ENC_SPLIT"] = split
    enc = Encoder(x.numel(), cfg)
    for _ in range(3):
        enc.encode(x)
    torch.cuda.synchronize()
    print(split, enc.finish())
