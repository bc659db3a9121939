"""profile() of the full-size cfg2 array (2^26 f32) on the GPU: wall time of
the sweep + recommendation (ProfileSession) and of the window statistics at
the recommended target; writes the recommended target (and its hex) next to
the timings.  Run on the GPU box:  python tools/time_profile.py [out.json]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1303_4994_b200 import Dtype  # noqa: E402
from paper_1303_4994_b200 import profiler as P  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402


def main():
    x = torch.from_numpy(W.cfg2_ar2_f32(1 << 26)).cuda()
    P.ProfileSession(x[:1 << 20], Dtype.F32)           # warm-up (plans, tables)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sess = P.ProfileSession(x, Dtype.F32)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rep = sess.report()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rec = sess.recommended
    out = {"workload": "cfg2 f32 AR(2) 2^26 samples, DEFAULT_GRID (21 targets), block 4096",
           "sweep_and_recommend_s": t1 - t0, "windows_at_recommended_s": t2 - t1, "profile_total_s": t2 - t0,
           "recommended": {"srr_target": rec.srr_target, "srr_target_hex": float(rec.srr_target).hex(),
                           "ratio": rec.ratio, "r": rec.r},
           "curve": [[p.srr_target, p.ratio, p.r] for p in sess.curve.points],
           "metrics": rep["windows"]["metrics"]}
    s = json.dumps(out, indent=1)
    print(s)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(s)


if __name__ == "__main__":
    main()
