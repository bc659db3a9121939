"""Corrupted-container bug hunt for the index-less decode (decode_stream of
bytes: K5 block discovery + general decoder) against the oracle's serial
walk: same first failing (status, block) or the same samples.
Usage: python tools/fuzz_corrupt.py [cases] [seed]"""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1303_4994_b200 import Decoder, Dtype, Mode, StreamConfig, encode_device  # noqa: E402
from paper_1303_4994_b200.codec import parse_file_header  # noqa: E402
from test_gpu_parity import _oscillating_case  # noqa: E402

U64 = (1 << 64) - 1
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
bad = 0
for i in range(cases):
    dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64][rng.integers(0, 5)]
    modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
    mode = modes[rng.integers(0, len(modes))]
    bs = int(rng.choice([128, 256, 1000, 4096]))
    n = bs * int(rng.integers(1, 8)) + int(rng.integers(0, bs))
    target = float(rng.uniform(1, 12)) if mode is Mode.FIXED_RATE else float(rng.uniform(10, 100))
    x = _oscillating_case(rng, dt, n)
    res = encode_device(torch.from_numpy(x).cuda(), StreamConfig(dt, bs, mode, target))
    b = bytearray(res.to_bytes())
    kind = int(rng.integers(0, 3))
    if kind == 0:                                  # random byte edits in the body
        for _ in range(int(rng.integers(1, 4))):
            p = int(rng.integers(28, len(b)))
            b[p] = int(rng.integers(0, 256))
    elif kind == 1:                                # truncation
        b = b[:int(rng.integers(28, len(b)))]
    else:                                          # nibble-level edit near a block start
        offs = res.block_offsets.cpu().numpy()
        k = int(rng.integers(0, len(offs) - 1))
        p = int(offs[k]) + (6 if dt.is_float else 4) + int(rng.integers(0, 8))
        if p < len(b):
            b[p] ^= int(rng.integers(1, 256))
    blob = bytes(b)
    try:
        yo = O.decode(blob)
        r = ("ok", yo)
    except O.OracleError as e:
        r = ("err", e.code, e.detail)
    cfg, count = parse_file_header(blob[:28])
    d = torch.zeros(len(blob) + 64, dtype=torch.uint8, device="cuda")
    d[:len(blob)] = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).cuda()
    dec = Decoder(count, cfg.dtype, cfg.block_size)
    dec.decode(d, len(blob), None)
    torch.cuda.synchronize()
    st = dec.status.cpu().numpy().view(np.uint64)
    key = int(st[1])
    g = ("err", key & 0xFF, key >> 8) if key != U64 else ("ok", dec.y[:count].cpu().numpy())
    ok = g[0] == r[0] and (g[1:] == r[1:] if g[0] == "err" else np.array_equal(g[1], r[1]))
    if not ok:
        bad += 1
        print("MISMATCH", i, dt.code, mode.name, bs, n, kind, "gpu", g[:3] if g[0] == "err" else "ok",
              "oracle", r[:3] if r[0] == "err" else "ok", flush=True)
print(f"{cases} cases, {bad} mismatches")
