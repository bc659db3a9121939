"""Debug helper: encode one config on cuda:0 with a chosen encoder version
and compare with the CPU oracle (test infrastructure)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

DTS = {"i8": (Dtype.I8, np.int8), "i16": (Dtype.I16, np.int16), "i32": (Dtype.I32, np.int32),
       "f32": (Dtype.F32, np.float32), "f64": (Dtype.F64, np.float64)}


def run(dt, mode, target, bs, n, seg=None, policy="cold", seed=0):
    D, npd = DTS[dt]
    rng = np.random.default_rng(seed)
    if dt.startswith("f"):
        x = (np.cumsum(rng.normal(size=n)) * 10).astype(npd)
    else:
        info = np.iinfo(npd)
        x = np.clip(np.cumsum(rng.normal(size=n)) * 50, info.min, info.max).astype(npd)
    cfg = StreamConfig(D, bs, Mode(mode), target, segment_blocks=seg, segment_policy=policy)
    enc = Encoder(n, cfg)
    enc.encode(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    st = enc.status.cpu().numpy().view(np.uint64)
    ref, offs, _ = O.encode(x, D.wire_code, mode, target, bs, segment_blocks=seg or 0,
                            policy=0 if policy == "cold" else 1)
    nb = int(st[2])
    got = bytes(enc.out[:max(nb, 0) if nb < (1 << 40) else 0].cpu().numpy().tobytes())
    first = next((i for i in range(min(len(got), len(ref))) if got[i] != ref[i]), None)
    print(f"{dt} mode={mode} bs={bs} n={n} seg={seg}: status={[hex(int(v)) for v in st]} "
          f"len {len(got)} vs {len(ref)} first_diff={first} ok={got == ref}")
    return got == ref


if __name__ == "__main__":
    ok = True
    ok &= run("i16", 1, 4.0, 4096, 8192)
    ok &= run("i16", 0, 0.0, 4096, 3 * 4096 + 100)
    ok &= run("f32", 2, 47.77, 4096, 4 * 4096, seg=2)
    ok &= run("f32", 1, 5.33, 1024, 10 * 1024 + 7, seg=3)
    ok &= run("i32", 1, 3.2, 512, 20 * 512, seg=4, policy="warm_self")
    print("ALL OK" if ok else "FAIL")
