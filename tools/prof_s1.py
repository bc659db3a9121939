"""S1 anatomy of the v3 encoder (variant built with -DAPAX_V3_PROF2):
mean cycles per block of thread 0's S1 chain, thread 32's wait for the
previous window's bulk store to read shared memory, and thread 0's wait at
B2.  Usage: tools/build_variant.sh prof2 -DAPAX_V3_PROF2; python tools/prof_s1.py"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("APAX_LIB_PATH", os.path.join(ROOT, "build_variants", "prof2", "libapax_b200.so"))
import torch  # noqa: E402

from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig, wave_segment_blocks  # noqa: E402
from paper_1303_4994_b200 import _lib  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

x = W.cfg2_ar2_f32()
seg = wave_segment_blocks(x.size, Dtype.F32, Mode.FIXED_QUALITY, 4096)
enc = Encoder(x.size, StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=seg))
xd = torch.from_numpy(x).cuda()
L = _lib.lib()
buf = np.zeros(4, np.uint64)
enc.encode(xd)
enc.finish()
L.apax_debug_prof2(buf.ctypes.data_as(ctypes.c_void_p))
b0 = buf.copy()
enc.encode(xd)
enc.finish()
L.apax_debug_prof2(buf.ctypes.data_as(ctypes.c_void_p))
d = (buf - b0).astype(np.float64)
print(f"blocks {d[3]:.0f}: S1 chain {d[0] / d[3]:.0f} cycles, store-read wait (thread 32) {d[1] / d[3]:.0f}, "
      f"B2 wait (thread 0) {d[2] / d[3]:.0f}")
