"""Phase cycles of the v5 encoder's pack thread 0 (variant built with
-DAPAX_V5_PROF: tools/build_variant.sh prof5 -DAPAX_V5_PROF), per block."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("APAX_LIB_PATH", os.path.join(ROOT, "build_variants", "prof5", "libapax_b200.so"))
import torch  # noqa: E402

from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig  # noqa: E402
from paper_1303_4994_b200 import _lib  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

names = ["emit", "wait S1", "stage+sums", "loadq+widths+peak", "wait B4", "totals+jee", "wait B4b", "chain"]
L = _lib.lib()
for lg in (22, 26):
    x = torch.from_numpy(W.cfg2_ar2_f32(1 << lg)).cuda()
    for mode, T, pol in ((Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, "cold"), (Mode.FIXED_RATE, 8.0, "warm_self")):
        enc = Encoder(x.numel(), StreamConfig(Dtype.F32, 4096, mode, T, segment_blocks=28, segment_policy=pol))
        enc.encode(x)
        enc.finish()
        L.apax_debug_prof5(None, 1)
        enc.encode(x)
        enc.finish()
        buf = np.zeros(16, np.uint64)
        L.apax_debug_prof5(buf.ctypes.data_as(ctypes.c_void_p), 0)
        nb = (1 << lg) // 4096
        per = buf[:8].astype(np.float64) / nb
        print(f"2^{lg} {mode.name} {pol}: cycles per block (thread 0): total {per.sum():.0f}")
        print("   " + "  ".join(f"{n} {v:.0f}" for n, v in zip(names, per)))
