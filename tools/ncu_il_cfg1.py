"""One index-less decode of the cfg1 container after warm-up (ncu launch list)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig, decode_device, wave_segment_blocks  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

x = W.cfg1_sines_i16()
n = x.size
seg = wave_segment_blocks(n, Dtype.I16, Mode.FIXED_RATE, 4096)
enc = Encoder(n, StreamConfig(Dtype.I16, 4096, Mode.FIXED_RATE, 4.0, segment_blocks=seg, segment_policy="warm_self"))
enc.encode(torch.from_numpy(x).cuda())
nb = enc.finish()
for _ in range(3):
    decode_device(enc.out, nb)
torch.cuda.synchronize()
