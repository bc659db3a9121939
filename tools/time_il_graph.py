"""Host cost of the index-less decode's gated-fallback graph: the first call
(graph built) against later calls (graph cached), and against plain launches."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1303_4994_b200 import Decoder, Dtype, Encoder, Mode, StreamConfig  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

for lg in (26, 20):
    x = W.cfg2_ar2_f32(1 << lg)
    n = x.size
    enc = Encoder(n, StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=28 if lg == 26 else 2))
    enc.encode(torch.from_numpy(x).cuda())
    nb = enc.finish()
    for graph in ("1", "0"):
        os.environ["APAX_IL_GRAPH"] = graph
        dec = Decoder(n, Dtype.F32, 4096)
        torch.cuda.synchronize()
        ts = []
        for k in range(6):
            t0 = time.perf_counter()
            dec.decode(enc.out, nb, None)
            t1 = time.perf_counter()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            ts.append((round((t1 - t0) * 1e6), round((t2 - t0) * 1e6)))
        print(f"2^{lg} graph={graph}: (enqueue us, total us) per call: {ts}", flush=True)
