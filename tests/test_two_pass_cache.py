"""Two-pass decode of whole-stream containers (apax_decode): pass 2 loads the
JEE parse pass 1 saved in the workspace (DecParams::jee_cache) instead of
parsing the tokens again, and without a side-band index pass 1 loads the
parse the block discovery saved (DecParams::jee_k5, APAX_JEE_K5=0 to switch
it off).  The result must be the oracle's, and the same as
with the cache switched off (APAX_JEE_CACHE=0), for clean containers of every
sample type, ragged last blocks, other block sizes, and corrupted containers
(the reference's error code and position)."""
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_1303_4994_b200 import Decoder, Dtype, Mode, StreamConfig, encode_device  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

U64 = (1 << 64) - 1


def _decode(blob, offs, n, dt, bs, cache, k5=True):
    old = os.environ.get("APAX_JEE_CACHE")
    old5 = os.environ.get("APAX_JEE_K5")
    os.environ["APAX_JEE_CACHE"] = "1" if cache else "0"
    os.environ["APAX_JEE_K5"] = "1" if k5 else "0"
    try:
        d = torch.zeros(len(blob) + 64, dtype=torch.uint8, device="cuda")
        d[:len(blob)] = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).cuda()
        dec = Decoder(n, dt, bs)
        dec.decode(d, len(blob), offs)
        torch.cuda.synchronize()
        key = int(dec.status.cpu().numpy().view(np.uint64)[1])
        return ("err", key & 0xFF, key >> 8) if key != U64 else ("ok", dec.y[:n].cpu().numpy().copy())
    finally:
        for k, v in (("APAX_JEE_CACHE", old), ("APAX_JEE_K5", old5)):
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _oracle(blob):
    try:
        return ("ok", O.decode(blob))
    except O.OracleError as e:
        return ("err", e.code, e.detail)


def _same(a, b):
    if a[0] != b[0]:
        return False
    return np.array_equal(a[1], b[1]) if a[0] == "ok" else a[1:] == b[1:]


@pytest.mark.parametrize("case", [
    ("f32", 4096, 4096 * 70 + 1111, Mode.FIXED_QUALITY, 47.78),
    ("f32", 1024, 1024 * 200 + 3, Mode.FIXED_RATE, 6.0),
    ("i16", 4096, 4096 * 45, Mode.FIXED_RATE, 4.0),
    ("i32", 2048, 2048 * 90 + 500, Mode.FIXED_QUALITY, 100.0),
    ("f64", 4096, 4096 * 33 + 8, Mode.FIXED_RATE, 3.0),
    ("i8", 512, 512 * 300 + 77, Mode.FIXED_RATE, 2.0),
])
def test_whole_stream_cached_parse_vs_oracle(case):
    dts, bs, n, mode, target = case
    base = W.cfg2_ar2_f32(n).astype(np.float64)
    if dts == "f32":
        x, dt = base.astype(np.float32), Dtype.F32
    elif dts == "f64":
        x, dt = base * 1e3, Dtype.F64
    elif dts == "i16":
        x, dt = W.cfg1_sines_i16(n), Dtype.I16
    elif dts == "i32":
        x, dt = np.rint(base * 5000).astype(np.int32), Dtype.I32
    else:
        x, dt = np.clip(np.rint(base * 30), -128, 127).astype(np.int8), Dtype.I8
    res = encode_device(torch.from_numpy(x).cuda(), StreamConfig(dt, bs, mode, target))
    blob = res.to_bytes()
    ref = _oracle(blob)
    assert ref[0] == "ok"
    for offs in (res.block_offsets, None):
        on = _decode(blob, offs, n, dt, bs, True)
        off = _decode(blob, offs, n, dt, bs, False)
        assert _same(on, ref) and _same(off, ref), (case, "index" if offs is not None else "index-less")
        if offs is None:   # without the block discovery's records (pass 1 parses every block itself)
            assert _same(_decode(blob, None, n, dt, bs, True, k5=False), ref), (case, "index-less, no K5 records")


def test_whole_stream_cached_parse_errors():
    n = 4096 * 50
    x = W.cfg2_ar2_f32(n)
    res = encode_device(torch.from_numpy(x).cuda(), StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, 47.78))
    clean = res.to_bytes()
    offs = res.block_offsets.cpu().numpy()
    cases = []
    b = bytearray(clean); b[int(offs[23]) + 6] = 0xE0; cases.append(bytes(b))       # reserved JEE nibble
    b = bytearray(clean); b[int(offs[31])] |= 3; cases.append(bytes(b))             # reserved selector
    cases.append(clean[:int(offs[40]) + 20])                                         # truncated inside block 40
    for blob in cases:
        ref = _oracle(blob)
        assert ref[0] == "err"
        for o in (res.block_offsets, None):
            if o is not None and len(blob) < len(clean):
                continue    # the index of the full container does not describe the truncated one
            on = _decode(blob, o, n, Dtype.F32, 4096, True)
            off = _decode(blob, o, n, Dtype.F32, 4096, False)
            assert _same(on, ref) and _same(off, ref), (ref, on[0], on[1:] if on[0] == "err" else "")
            if o is None:
                assert _same(_decode(blob, None, n, Dtype.F32, 4096, True, k5=False), ref)
