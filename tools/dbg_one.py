"""Encode one config on cuda:0 (timeout-friendly triage).  Args:
dtype mode bs target seg policy n [seed]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, encode_device  # noqa: E402

DTS = {"i8": (Dtype.I8, np.int8), "i16": (Dtype.I16, np.int16), "i32": (Dtype.I32, np.int32),
       "f32": (Dtype.F32, np.float32), "f64": (Dtype.F64, np.float64)}
dt, mode, bs, target, seg, pol, n = sys.argv[1:8]
seed = int(sys.argv[8]) if len(sys.argv) > 8 else 0
D, npd = DTS[dt]
mode, bs, target, seg, n = int(mode), int(bs), float(target), int(seg), int(n)
rng = np.random.default_rng(seed)
x = (np.cumsum(rng.standard_normal(n)) * 10.0).astype(npd)
print("oracle...", end=" ", flush=True)
ref, offs, _ = O.encode(x, D.wire_code, mode, target, bs, segment_blocks=seg, policy=1 if pol == "warm_self" else 0)
print("gpu...", end=" ", flush=True)
cfg = StreamConfig(D, bs, Mode(mode), target, segment_blocks=seg or None, segment_policy=pol)
res = encode_device(torch.from_numpy(x).cuda(), cfg)
got = res.to_bytes()
first = next((i for i in range(min(len(got), len(ref))) if got[i] != ref[i]), None)
print(sys.argv[1:], "ok" if got == ref else f"MISMATCH len {len(got)} vs {len(ref)} first {first}", flush=True)
