"""Timing of the secondary paths on cfg2 (2^26 f32): the general decoder
(apax_decode: any container, affine carry look-back) with and without the
side-band index, and the GPU profiler (profile(): 21-point sweep +
recommendation + window statistics)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1303_4994_b200 import Decoder, Dtype, Encoder, Mode, StreamConfig, profile, wave_segment_blocks  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

x = W.cfg2_ar2_f32()
n = x.size
seg = wave_segment_blocks(n, Dtype.F32, Mode.FQ if hasattr(Mode, "FQ") else Mode.FIXED_QUALITY, 4096)
enc = Encoder(n, StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=seg))
xd = torch.from_numpy(x).cuda()
enc.encode(xd)
nb = enc.finish()
dec = Decoder(n, Dtype.F32, 4096)
for name, kw in (("d3 segments+index", dict(offsets=enc.offsets, segment_blocks=seg)),
                 ("general decoder + index", dict(offsets=enc.offsets)),
                 ("general decoder, K5 discovery", dict(offsets=None))):
    for _ in range(3):
        dec.decode(enc.out, nb, kw["offsets"], segment_blocks=kw.get("segment_blocks"))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dec.decode(enc.out, nb, kw["offsets"], segment_blocks=kw.get("segment_blocks"))
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 10:.3f} ms")
for m in (1 << 20, 1 << 24):
    xs = x[:m]
    profile(xs, Dtype.F32)
    t = time.perf_counter()
    rep = profile(xs, Dtype.F32)
    print(f"profile 2^{m.bit_length() - 1} f32: {time.perf_counter() - t:.2f} s, recommended {rep['recommended']['srr_target']:.4f} dB")
