import sys, time, ctypes; sys.path.insert(0, ".")
import torch, numpy as np
from paper_1303_4994_b200 import Dtype, Encoder, Decoder, Mode, StreamConfig, decode_device, wave_segment_blocks, _lib
from paper_1303_4994_b200 import workloads as W
x = W.cfg2_ar2_f32(); n = x.size
seg = wave_segment_blocks(n, Dtype.F32, Mode.FIXED_QUALITY, 4096)
enc = Encoder(n, StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=seg)); enc.encode(torch.from_numpy(x).cuda()); nb = enc.finish()
L = _lib.lib()
nbk = (n + 4095) // 4096
offs = torch.empty(nbk + 1, dtype=torch.int64, device="cuda"); st = torch.empty(4, dtype=torch.int64, device="cuda"); ps = torch.zeros(1, dtype=torch.int64, device="cuda")
def t(f, k=5):
    f(); torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / k * 1e3
print("find_blocks", t(lambda: L.apax_find_blocks(ctypes.c_void_p(enc.out.data_ptr()), nb, n, 3, 4096, ctypes.c_void_p(offs.data_ptr()), ctypes.c_void_p(st.data_ptr()), None)))
print("detect", t(lambda: L.apax_detect_segments(ctypes.c_void_p(enc.out.data_ptr()), nb, ctypes.c_void_p(offs.data_ptr()), nbk, ctypes.c_void_p(ps.data_ptr()), None)), "P", int(ps.item()), "status", st.cpu().numpy().view(np.uint64)[:2])
dec = Decoder(n, Dtype.F32, 4096)
print("d3", t(lambda: dec.decode(enc.out, nb, offs, segment_blocks=int(ps.item()))))
print("decode_device", t(lambda: decode_device(enc.out, nb)))
print("Decoder alloc", t(lambda: Decoder(n, Dtype.F32, 4096)))
ys = []
torch.cuda.synchronize(); a = time.perf_counter()
for _ in range(10):
    y = decode_device(enc.out, nb)
torch.cuda.synchronize(); print("decode_device loop (fresh y each call)", (time.perf_counter() - a) / 10 * 1e3, "ms")
