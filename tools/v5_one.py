import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig
from paper_1303_4994_b200 import workloads as W
x = torch.from_numpy(W.cfg2_ar2_f32(1 << 22)).cuda()
cfg = StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=28)
enc = Encoder(x.numel(), cfg)
print("ws bytes", enc.ws.numel(), flush=True)
for k in range(3):
    enc.encode(x)
    torch.cuda.synchronize()
    print("encode", k, "ok", enc.finish(), flush=True)
