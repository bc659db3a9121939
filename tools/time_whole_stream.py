import sys, time
sys.path.insert(0, ".")
import torch
from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig
from paper_1303_4994_b200 import workloads as W
x = torch.from_numpy(W.cfg1_sines_i16()).cuda()
for mode, tgt in ((Mode.FIXED_RATE, 4.0), (Mode.LOSSLESS, 0.0)):
    enc = Encoder(x.numel(), StreamConfig(Dtype.I16, 4096, mode, tgt))
    enc.encode(x); enc.finish()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); enc.encode(x); e1.record(); torch.cuda.synchronize()
    print(mode.name, "whole-stream cfg1 encode", round(e0.elapsed_time(e1), 3), "ms")
