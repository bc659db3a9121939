"""Per-phase cycles of the whole-stream chain kernel (thread 0 clock64
deltas, -DAPAX_WS_PROF variant library under build_variants/).
  python tools/prof_ws.py --build      (here: compile the variant)
  python tools/prof_ws.py [fr|fq]      (GPU box: run cfg1 FR / 2^22 FQ whole stream)"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "build_variants")
SO = os.path.join(OUT, "libapax_wsprof.so")
NAMES = ["loop top", "S1", "B2", "phaseC/D2+JEE", "B3", "warp0 serial", "prep next", "B4", "-", "-"]
# (the marks' accumulators live in local memory in this variant: absolute
# numbers are inflated, use them for proportions)


def build():
    os.makedirs(OUT, exist_ok=True)
    src = os.path.join(ROOT, "paper_1303_4994_b200", "csrc")
    subprocess.run(["make", "-s", "-j8", "-C", src, f"OUT={SO}", f"BUILD={OUT}/obj_wsprof", "EXTRA=-DAPAX_WS_PROF"],
                   check=True)


def main():
    if "--build" in sys.argv:
        build()
        return
    os.environ["APAX_LIB_PATH"] = SO
    os.environ["APAX_WS_CHAIN"] = "1"
    sys.path.insert(0, ROOT)
    import torch
    from paper_1303_4994_b200 import Dtype, Encoder, Mode, StreamConfig, _lib
    from paper_1303_4994_b200 import workloads as W
    mode = sys.argv[1] if len(sys.argv) > 1 else "fr"
    if mode == "fr":
        x = torch.from_numpy(W.cfg1_sines_i16(1 << 24)).cuda()
        cfg = StreamConfig(Dtype.I16, 4096, Mode.FIXED_RATE, 4.0)
    else:
        x = torch.from_numpy(W.cfg2_ar2_f32(1 << 22)).cuda()
        cfg = StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB)
    enc = Encoder(x.numel(), cfg)
    enc.encode(x)
    enc.finish()
    L = _lib.lib()
    L.apax_debug_ws_prof.argtypes = [ctypes.c_void_p]
    buf = (ctypes.c_ulonglong * 15)()
    L.apax_debug_ws_prof(buf)
    nb = (x.numel() + 4095) // 4096
    tot = sum(buf[:8])
    for k, nm in enumerate(NAMES):
        print(f"{nm:12s} {buf[k] / nb:9.1f} cycles/block ({100 * buf[k] / max(tot, 1):5.1f}%)")
    print(f"total {tot / nb:.1f} cycles/block")


if __name__ == "__main__":
    main()
