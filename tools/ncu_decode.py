"""One segmented decode of the cfg2 container after warm-up (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1303_4994_b200 import Decoder, Dtype, Encoder, Mode, StreamConfig, wave_segment_blocks  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

x = W.cfg2_ar2_f32()
n = x.size
seg = wave_segment_blocks(n, Dtype.F32, Mode.FIXED_QUALITY, 4096)
enc = Encoder(n, StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=seg))
enc.encode(torch.from_numpy(x).cuda())
nb = enc.finish()
dec = Decoder(n, Dtype.F32, 4096)
for _ in range(3):
    dec.decode(enc.out, nb, enc.offsets, segment_blocks=seg)
torch.cuda.synchronize()
