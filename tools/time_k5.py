"""Time index-less block discovery (K5 vs the serial walk) and the index-less
decode on the cfg2 container.  Usage: python tools/time_k5.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1303_4994_b200 import Decoder, Dtype, Mode, StreamConfig, encode_device  # noqa: E402
from paper_1303_4994_b200 import _lib  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    x = W.cfg2_ar2_f32()
    seg = int(os.environ.get("SEG", "37"))
    res = encode_device(torch.from_numpy(x).cuda(),
                        StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=seg))
    L = _lib.lib()
    n = x.size
    nb = (n + 4095) // 4096
    offs = torch.empty(nb + 1, dtype=torch.int64, device="cuda")
    status = torch.empty(4, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    out = {"nbytes": res.nbytes, "n_blocks": nb}
    for k5 in ("1", "0"):
        os.environ["APAX_K5"] = k5
        ms = timed(lambda: L.apax_find_blocks(res.blob.data_ptr(), res.nbytes, n, 3, 4096, offs.data_ptr(),
                                              status.data_ptr(), st), reps=10 if k5 == "1" else 2)
        ok = bool(torch.equal(offs, res.block_offsets))
        out[f"find_blocks_ms_k5={k5}"] = round(ms, 4)
        out[f"find_blocks_ok_k5={k5}"] = ok
    os.environ["APAX_K5"] = "1"
    dec = Decoder(n, Dtype.F32, 4096)
    out["decode_indexless_ms"] = round(timed(lambda: dec.decode(res.blob, res.nbytes)), 4)
    out["decode_index_ms"] = round(timed(lambda: dec.decode(res.blob, res.nbytes, res.block_offsets)), 4)
    out["decode_segments_ms"] = round(
        timed(lambda: dec.decode(res.blob, res.nbytes, res.block_offsets, segment_blocks=seg)), 4)
    out["indexless_GBps"] = round(n * 4 / out["decode_indexless_ms"] / 1e6, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
