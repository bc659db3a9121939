"""Encoder-only timing on cfg2 (2^26 f32, fixed quality, one-wave segments),
L2 flushed between launches; for comparing build variants
(APAX_LIB_PATH=build_variants/<v>/libapax_b200.so).  No parity check."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig, wave_segment_blocks  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

x = W.cfg2_ar2_f32()
n = x.size
seg = wave_segment_blocks(n, Dtype.F32, Mode.FIXED_QUALITY, 4096)
enc = Encoder(n, StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=seg))
xd = torch.from_numpy(x).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(23):
    flush.fill_(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    enc.encode(xd)
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
nb = enc.finish()
ts.sort()
print(f"{os.environ.get('APAX_LIB_PATH', 'product')}: encode median {ts[len(ts) // 2]:.4f} ms min {ts[0]:.4f} bytes {nb}")
