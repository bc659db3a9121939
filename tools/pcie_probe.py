"""PCIe probe: pinned H2D, D2H and both directions at once (GB/s), and the
pipelined e2e round trip of cfg2 at several chunk counts."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, wave_segment_blocks  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402
from paper_1303_4994_b200.pipeline import HostRoundTrip  # noqa: E402

nb = 256 << 20
h = torch.empty(nb, dtype=torch.uint8).pin_memory()
h2 = torch.empty(nb, dtype=torch.uint8).pin_memory()
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(f"{name}: {5 * nb / (time.perf_counter() - t) / 1e9:.1f} GB/s")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print(f"both directions: {2 * 5 * nb / (time.perf_counter() - t) / 1e9:.1f} GB/s total")
# chunk-sized copies (8.3 MB, a cfg2 container chunk) at aligned and odd offsets
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
m = 8_300_000
for off in (0, 28, 64, 4096 + 12):
    for name, fn in (("h2d", lambda: d[off:off + m].copy_(h[off:off + m], non_blocking=True)),
                     ("d2h", lambda: h[off:off + m].copy_(d[off:off + m], non_blocking=True)),
                     ("d2h-skew", lambda: h[off:off + m].copy_(d[28:28 + m], non_blocking=True))):
        fn()
        ev[0].record()
        for _ in range(10):
            fn()
        ev[1].record()
        torch.cuda.synchronize()
        print(f"{name} 8.3 MB at offset {off}: {10 * m / ev[0].elapsed_time(ev[1]) / 1e6:.1f} GB/s")
x = W.cfg2_ar2_f32()
n = x.size
seg = wave_segment_blocks(n, Dtype.F32, Mode.FIXED_QUALITY, 4096)
cfg = StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=seg)
xh = torch.from_numpy(x).pin_memory()
yh = torch.empty(n, dtype=torch.float32).pin_memory()
# PROBE_CFGS="chunks,depth,taper ..."; PROBE_TL="chunks,depth,taper" for the timeline
cfgs = [tuple(int(v) for v in c.split(",")) for c in os.environ.get("PROBE_CFGS", "4,3,1 8,3,1 8,4,1 16,3,1 16,4,1").split()]
for chunks, depth, taper in cfgs:
    rt = HostRoundTrip(n, cfg, chunks=chunks, depth=depth, taper=taper)
    blob_h = torch.empty(rt.blob_d.numel(), dtype=torch.uint8).pin_memory()
    offs_h = torch.empty(rt.n_blocks + 1, dtype=torch.int64).pin_memory()
    for _ in range(2):
        rt.run(xh, blob_h, offs_h, yh)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        rt.run(xh, blob_h, offs_h, yh)
    dt = (time.perf_counter() - t) / 5
    print(f"e2e chunks={chunks} depth={depth} taper={taper}: {dt * 1e3:.2f} ms/step, {n * 4 / dt / 1e9:.1f} GB/s, PCIe {(rt.h2d_bytes + rt.d2h_bytes) / dt / 1e9:.1f} GB/s both ways")
# timeline of one round trip
tc, td, tt = (int(v) for v in os.environ.get("PROBE_TL", "4,3,1").split(","))
rt = HostRoundTrip(n, cfg, chunks=tc, depth=td, taper=tt)
blob_h = torch.empty(rt.blob_d.numel(), dtype=torch.uint8).pin_memory()
offs_h = torch.empty(rt.n_blocks + 1, dtype=torch.int64).pin_memory()
rt.run(xh, blob_h, offs_h, yh)
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
rt.timeline = []
rt.run(xh, blob_h, offs_h, yh)
torch.cuda.synchronize()
for name, a, b in sorted(rt.timeline, key=lambda e: t0.elapsed_time(e[1])):
    print(f"{name:6s} {t0.elapsed_time(a):8.3f} -> {t0.elapsed_time(b):8.3f} ms ({a.elapsed_time(b):.3f})")
