"""One index-less decode of the cfg2 container after warm-up (for an ncu
launch list: ncu --metrics gpu__time_duration.sum ... python tools/ncu_indexless.py)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig, decode_device, wave_segment_blocks  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

x = W.cfg2_ar2_f32()
n = x.size
seg = wave_segment_blocks(n, Dtype.F32, Mode.FIXED_QUALITY, 4096)
enc = Encoder(n, StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=seg))
enc.encode(torch.from_numpy(x).cuda())
nb = enc.finish()
for _ in range(3):
    decode_device(enc.out, nb)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("indexless")
y = decode_device(enc.out, nb)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
