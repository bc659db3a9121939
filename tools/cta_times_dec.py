"""Per-CTA timeline of the one-wave segment decoder (variant built with
-DAPAX_D3_TIMES: tools/build_variant.sh timesd -DAPAX_D3_TIMES): the cfg2
container, distribution of the CTAs' exit times and their order within an SM."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("APAX_LIB_PATH", os.path.join(ROOT, "build_variants", "timesd", "libapax_b200.so"))
import torch  # noqa: E402

from paper_1303_4994_b200 import Decoder, Dtype, Encoder, Mode, StreamConfig, wave_segment_blocks  # noqa: E402
from paper_1303_4994_b200 import _lib  # noqa: E402
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
L = _lib.lib()
ng = (16384 + seg - 1) // seg
buf = np.zeros(ng * 4, np.uint64)
L.apax_debug_cta_times_d3(buf.ctypes.data_as(ctypes.c_void_p), ng)
t = buf.reshape(-1, 4).astype(np.int64)
t0 = t[:, 0].min()
st, ex = (t[:, 0] - t0) / 1e3, (t[:, 2] - t0) / 1e3
sm = t[:, 3]
print(f"cfg2 decode: P={seg} CTAs={ng}")
for name, v in (("start", st), ("exit", ex)):
    print(f"{name:8s} us: " + " ".join(f"{a:8.1f}" for a in np.percentile(v, [0, 10, 25, 50, 75, 90, 100])))
print("exit by CTA id, blocks of 32:", " ".join(f"{ex[i:i + 32].mean():.0f}" for i in range(0, ng, 32)))
agree = tot = 0
for k in range(148):
    ids = np.nonzero(sm == k)[0]
    if len(ids) < 2:
        continue
    tot += 1
    agree += int(np.array_equal(ids[np.argsort(ids)], ids[np.argsort(ex[ids])]))
print(f"SMs whose CTAs exit in blockIdx order: {agree} of {tot}")
print(f"mean exit {ex.mean():.1f} us, max {ex.max():.1f} us: perfect balance at the 4-CTA rate would end near the mean")
