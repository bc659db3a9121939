"""cfg5 sweep (BASELINE.json configs[4]): AR(1) rho=0.95 int32 / f32 arrays
over sizes and fixed rates, encode and decode GB/s (input bytes) on one GPU,
one JSON line per point.  Device-resident inputs; L2 flushed between legs;
CUDA events on the launching stream; one-wave cold segments."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1303_4994_b200 import Decoder, Dtype, Encoder, Mode, StreamConfig, wave_segment_blocks  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-bytes", default="20,22,24,26,28,30,32,34")
    ap.add_argument("--big-rates", default="2,4,10", help="rates at >= 4 GiB (generated on the GPU)")
    ap.add_argument("--rates", default="2,3,4,6,8,10")
    ap.add_argument("--dtypes", default="i32,f32")
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    for dts in a.dtypes.split(","):
        dt = Dtype.I32 if dts == "i32" else Dtype.F32
        for lb in [int(v) for v in a.log2_bytes.split(",")]:
            n = 1 << (lb - 2)
            big = lb >= 32
            x = (W.cfg5_ar1_device(n, dts, device=dev) if big else torch.from_numpy(W.cfg5_ar1(n, dts)).to(dev))
            for r in [float(v) for v in (a.big_rates if big else a.rates).split(",")]:
                seg = wave_segment_blocks(n, dt, Mode.FIXED_RATE, 4096)
                cfg = StreamConfig(dt, 4096, Mode.FIXED_RATE, 32.0 / r, segment_blocks=seg,
                                   segment_policy="warm_self")
                enc = Encoder(n, cfg, device=dev)
                dec = Decoder(n, dt, 4096, device=dev)
                ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(a.steps + 3)]
                for k in range(a.steps + 3):
                    flush.zero_()
                    ev[k][0].record(st)
                    enc.encode(x)
                    ev[k][1].record(st)
                    flush.zero_()
                    ev[k][2].record(st)
                    dec.decode(enc.out, enc.cap, enc.offsets, segment_blocks=seg)
                    ev[k][3].record(st)
                nb = enc.finish()
                y = dec.finish()
                torch.cuda.synchronize()
                te = sum(e[0].elapsed_time(e[1]) for e in ev[3:]) / a.steps
                td = sum(e[2].elapsed_time(e[3]) for e in ev[3:]) / a.steps
                ib = n * 4
                print(json.dumps({"workload": "cfg5", "dtype": dts, "bytes": ib, "rate": r,
                                  "generator": "cfg5_ar1_device" if big else "cfg5_ar1",
                                  "segment_blocks": seg, "segment_policy": "warm_self", "container_bytes": nb, "ratio": ib / nb,
                                  "encode_ms": te, "decode_ms": td,
                                  "encode_gbs": ib / te / 1e6, "decode_gbs": ib / td / 1e6,
                                  "encode_alg_gbs": (ib + nb) / te / 1e6,
                                  "decode_alg_gbs": (ib + nb) / td / 1e6}), flush=True)
                del enc, dec, y
            del x
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
