"""Per-CTA timeline of the one-wave v3 encoder (variant built with
-DAPAX_V3_TIMES: tools/build_variant.sh times -DAPAX_V3_TIMES).  Runs the
cfg2 workload and prints the distribution of CTA coding-end and exit times."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("APAX_LIB_PATH", os.path.join(ROOT, "build_variants", os.environ.get("TIMES_VARIANT", "times"), "libapax_b200.so"))
import torch  # noqa: E402

from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig, wave_segment_blocks  # noqa: E402
from paper_1303_4994_b200 import _lib  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if wl == "cfg2":
    x = W.cfg2_ar2_f32()
    dt, mode, tgt, pol = Dtype.F32, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, "cold"
else:
    x = W.cfg3_grf_f32()
    dt, mode, tgt, pol = Dtype.F32, Mode.FIXED_RATE, 32 / 6, "warm_self"
seg = wave_segment_blocks(x.size, dt, mode, 4096)
enc = Encoder(x.size, StreamConfig(dt, 4096, mode, tgt, segment_blocks=seg, segment_policy=pol))
xd = torch.from_numpy(x).cuda()
for _ in range(3):
    enc.encode(xd)
enc.finish()
L = _lib.lib()
ng = (16384 + seg - 1) // seg
buf = np.zeros(ng * 4, np.uint64)
getattr(L, os.environ.get("TIMES_FN", "apax_debug_cta_times"))(buf.ctypes.data_as(ctypes.c_void_p), ng)
t = buf.reshape(-1, 4).astype(np.int64)
t0 = t[:, 0].min()
st, ce, ex = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
print(f"{wl}: P={seg} CTAs={ng}")
for name, v in (("start", st), ("coding end", ce), ("exit", ex), ("coding time", ce - st)):
    q = np.percentile(v, [0, 10, 50, 90, 99, 100])
    print(f"{name:12s} us: " + " ".join(f"{a:8.1f}" for a in q))
sm = t[:, 3]
per_sm = np.bincount(sm, minlength=148)
print("CTAs per SM histogram:", np.bincount(per_sm))
slow = np.argsort(ce - st)[-8:]
print("slowest CTAs (id, sm, coding us, ctas on that sm):",
      [(int(i), int(sm[i]), round(float(ce[i] - st[i]), 1), int(per_sm[sm[i]])) for i in slow])
ct = ce - st
sm_mean = np.array([ct[sm == k].mean() if (sm == k).any() else np.nan for k in range(148)])
print("per-SM mean coding time, SMs 0..147 (us):")
print(" ".join(f"{v:.0f}" for v in sm_mean))
print("coding time by CTA id, in blocks of 32 CTAs:", " ".join(f"{ct[i:i + 32].mean():.0f}" for i in range(0, len(ct), 32)))

if os.environ.get("TIMES_FN", "").endswith("5"):
    b2 = np.zeros(ng * 2, np.uint64)
    L.apax_debug_cta_times5b(b2.ctypes.data_as(ctypes.c_void_p), ng)
    t2 = b2.reshape(-1, 2).astype(np.int64)
    pk, cd = (t2[:, 0] - t0) / 1e3, (t2[:, 1] - t0) / 1e3
    for name, v in (("prefix known", pk), ("copy done", cd), ("prefix wait", pk - ce), ("copy time", cd - pk)):
        q = np.percentile(v, [0, 10, 50, 90, 99, 100])
        print(f"{name:12s} us: " + " ".join(f"{a:8.1f}" for a in q))
    print("id: coding end, prefix known, copy done, exit")
    for i in list(range(0, 12)) + list(range(140, 156)) + list(range(290, 300)) + list(range(576, ng)):
        print(f"  {i:4d} {ce[i]:8.1f} {pk[i]:8.1f} {cd[i]:8.1f} {ex[i]:8.1f}")

# within an SM: does blockIdx order predict the finishing order?
agree = tot = 0
inv = []
for k in range(148):
    ids = np.nonzero(sm == k)[0]
    if len(ids) < 2:
        continue
    order_id = ids[np.argsort(ids)]
    order_t = ids[np.argsort(ce[ids])]
    tot += 1
    agree += int(np.array_equal(order_id, order_t))
    if not np.array_equal(order_id, order_t) and len(inv) < 12:
        inv.append((k, [(int(i), round(float(ce[i]), 1)) for i in order_id]))
print(f"SMs whose CTAs finish in blockIdx order: {agree} of {tot}")
for k, v in inv:
    print("  SM", k, v)
