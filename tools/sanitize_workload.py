import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import oracle as O
from paper_1303_4994_b200 import Decoder, Dtype, Encoder, Mode, StreamConfig, encode_device, decode_device
from paper_1303_4994_b200 import workloads as W
# small segmented containers through the v3 encoder and the d3 decoder (full and partial blocks)
for dt, mode, tgt, n, seg, pol in ((Dtype.F32, Mode.FIXED_QUALITY, 45.0, 4096 * 19 + 77, 4, "cold"),
                                  (Dtype.I16, Mode.FIXED_RATE, 4.0, 4096 * 12, 3, "warm_self"),
                                  (Dtype.F64, Mode.FIXED_RATE, 21.3, 4096 * 9 + 5, 2, "warm_self"),
                                  (Dtype.I32, Mode.LOSSLESS, 0.0, 4096 * 10 + 3, None, "cold")):
    x = (W.cfg2_ar2_f32(n).astype(dt.np_dtype) if dt.is_float else W.cfg1_sines_i16(n).astype(dt.np_dtype))
    res = encode_device(torch.from_numpy(x).cuda(), StreamConfig(dt, 4096, mode, tgt, segment_blocks=seg, segment_policy=pol))
    y = decode_device(res.blob, res.nbytes, res.block_offsets, segment_blocks=seg).cpu().numpy()
    y2 = decode_device(res.blob, res.nbytes).cpu().numpy()
    ref, offs, _ = O.encode(x, dt.wire_code, mode.value, tgt, 4096, segment_blocks=seg or 0, policy=1 if pol == "warm_self" else 0)
    assert res.to_bytes() == ref and np.array_equal(y, O.decode(ref)) and np.array_equal(y2, y), dt
# whole-stream containers: the two-pass decode with the saved JEE parse, with and without the index,
# full and partial last blocks, a block size below 4096
for dt, mode, tgt, n, bs in ((Dtype.F32, Mode.FIXED_QUALITY, 45.0, 4096 * 11 + 77, 4096),
                            (Dtype.I16, Mode.FIXED_RATE, 4.0, 1024 * 21 + 5, 1024),
                            (Dtype.F64, Mode.FIXED_RATE, 21.3, 4096 * 9, 4096)):
    x = (W.cfg2_ar2_f32(n).astype(dt.np_dtype) if dt.is_float else W.cfg1_sines_i16(n).astype(dt.np_dtype))
    res = encode_device(torch.from_numpy(x).cuda(), StreamConfig(dt, bs, mode, tgt))
    ref = O.decode(res.to_bytes())
    assert np.array_equal(decode_device(res.blob, res.nbytes, res.block_offsets).cpu().numpy(), ref), dt
    assert np.array_equal(decode_device(res.blob, res.nbytes).cpu().numpy(), ref), dt
print("sanitizer workload ok")
