"""v5 encoder against the fused v3 kernel (APAX_ENC_V5=0) on BASELINE-shaped
workloads: byte equality, block offsets, timing (CUDA events, median of 7)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402


def run(enc, x, reps=7):
    ts = []
    for k in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        enc.encode(x)
        b.record()
        torch.cuda.synchronize()
        if k >= 2:
            ts.append(a.elapsed_time(b))
    nb = enc.finish()
    return float(np.median(ts)), enc.out[:nb].cpu().numpy().tobytes(), enc.offsets.cpu().numpy().copy()


def main():
    small = len(sys.argv) > 1 and sys.argv[1] == "small"
    s = 4 if small else 0
    cases = [
        ("cfg2 FQ P=28", W.cfg2_ar2_f32(1 << (26 - s)), Dtype.F32, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, 28, "cold"),
        ("cfg2 FQ P=3", W.cfg2_ar2_f32((1 << 20) + 5), Dtype.F32, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, 3, "cold"),
        ("cfg2 FR cold P=5", W.cfg2_ar2_f32(1 << 21), Dtype.F32, Mode.FIXED_RATE, 8.0, 5, "cold"),
        ("cfg1 FR P=7 warm", W.cfg1_sines_i16(1 << (24 - s)), Dtype.I16, Mode.FIXED_RATE, 4.0, 7, "warm_self"),
        ("cfg1 FQ P=9", W.cfg1_sines_i16((1 << 20) + 4096 * 3 + 77), Dtype.I16, Mode.FIXED_QUALITY, 40.0, 9, "cold"),
        ("cfg3 FR P=28 warm", W.cfg2_ar2_f32(1 << (26 - s)), Dtype.F32, Mode.FIXED_RATE, 32.0 / 6.0, 28, "warm_self"),
        ("i32 FR P=4 warm", (W.cfg2_ar2_f32(1 << 21) * 1000).astype(np.int32), Dtype.I32, Mode.FIXED_RATE, 10.0, 4, "warm_self"),
        ("i32 FQ big P=6", (W.cfg2_ar2_f32(1 << 21) * 4e5).astype(np.int32), Dtype.I32, Mode.FIXED_QUALITY, 150.0, 6, "cold"),
    ]
    cases += [
        ("f32 FQ P=1 many units", W.cfg2_ar2_f32(1 << 22), Dtype.F32, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, 1, "cold"),
        ("i16 FR P=1 warm many", W.cfg1_sines_i16((1 << 22) + 100), Dtype.I16, Mode.FIXED_RATE, 4.0, 1, "warm_self"),
        ("f32 FR P=2 warm many", W.cfg2_ar2_f32((1 << 23) + 4096), Dtype.F32, Mode.FIXED_RATE, 6.0, 2, "warm_self"),
        ("i32 FQ P=3 many", (W.cfg2_ar2_f32(1 << 23) * 1000).astype(np.int32), Dtype.I32, Mode.FIXED_QUALITY, 60.0, 3, "cold"),
    ]
    ok = True
    for name, xh, dt, mode, T, P, pol in cases:
        x = torch.from_numpy(xh).cuda()
        cfg = StreamConfig(dt, 4096, mode, T, segment_blocks=P, segment_policy=pol)
        res = {}
        for v5 in ("0", "1"):
            os.environ["APAX_ENC_V5"] = "2" if v5 == "1" else "0"
            enc = Encoder(x.numel(), cfg)
            res[v5] = run(enc, x)
        same = res["0"][1] == res["1"][1]
        same_off = np.array_equal(res["0"][2], res["1"][2])
        ok = ok and same and same_off
        print(f"{name:20s} v3 {res['0'][0]:8.4f} ms  v5 {res['1'][0]:8.4f} ms  bytes {len(res['0'][1])} identical {same} offsets {same_off}",
              flush=True)
        if not same:
            a, b = np.frombuffer(res["0"][1], np.uint8), np.frombuffer(res["1"][1], np.uint8)
            m = min(len(a), len(b))
            d = np.nonzero(a[:m] != b[:m])[0]
            print("   len", len(a), len(b), "first diff", d[:8], "ndiff", len(d))
            offs = res["0"][2]
            if len(d):
                print("   block of first diff", int(np.searchsorted(offs, d[0], side="right") - 1))
    print("ALL OK" if ok else "MISMATCH")


if __name__ == "__main__":
    main()
