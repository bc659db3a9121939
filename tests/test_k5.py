"""K5 index-less block discovery (apax_k5.cu) against the serial walk and the
oracle's offsets: the offsets must be exactly the walk's (the recurrence of
codec.py:317-323), and every failure -- corrupt, truncated or adversarial
streams, candidate overflow -- must give the walk's status and block index."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, decode_device, encode_device  # noqa: E402
from paper_1303_4994_b200 import _lib  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402


def _find_blocks(blob_bytes, n, dt, bs, k5=True):
    """apax_find_blocks through the C ABI -> (offsets int64[n_blocks+1], status u64[4])."""
    L = _lib.lib()
    nb = (n + bs - 1) // bs
    blob = torch.from_numpy(np.frombuffer(blob_bytes, np.uint8).copy()).cuda()
    offs = torch.empty(nb + 1, dtype=torch.int64, device="cuda")
    status = torch.empty(4, dtype=torch.int64, device="cuda")
    old = os.environ.get("APAX_K5")
    os.environ["APAX_K5"] = "1" if k5 else "0"
    try:
        st = L.apax_find_blocks(blob.data_ptr(), len(blob_bytes), n, dt, bs, offs.data_ptr(),
                                status.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
    finally:
        if old is None:
            del os.environ["APAX_K5"]
        else:
            os.environ["APAX_K5"] = old
    assert st == 0
    return offs.cpu().numpy(), status.cpu().numpy()


def _both(blob, n, dt, bs):
    a = _find_blocks(blob, n, dt, bs, True)
    b = _find_blocks(blob, n, dt, bs, False)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    return a


@pytest.mark.parametrize("seed", range(4))
def test_k5_offsets_random_containers(seed):
    rng = np.random.default_rng(9000 + seed)
    for _ in range(8):
        dt = [Dtype.I8, Dtype.I16, Dtype.I32, Dtype.F32, Dtype.F64][rng.integers(0, 5)]
        modes = [Mode.FIXED_RATE, Mode.FIXED_QUALITY] + ([] if dt.is_float else [Mode.LOSSLESS])
        mode = modes[rng.integers(0, len(modes))]
        bs = int(rng.choice([64, 128, 500, 1024, 4096, 16384]))
        target = float(rng.uniform(1, 12)) if mode is Mode.FIXED_RATE else float(rng.uniform(10, 100))
        n = int(rng.integers(bs, 40 * bs))
        if dt.is_float:
            x = (np.cumsum(rng.standard_normal(n)) * 10.0 ** rng.uniform(-3, 3)).astype(dt.np_dtype)
        else:
            info = np.iinfo(dt.np_dtype)
            x = rng.integers(info.min, info.max + 1, n).astype(dt.np_dtype)
        cfg = StreamConfig(dt, bs, mode, target, segment_blocks=int(rng.choice([0, 0, 3])) or None)
        res = encode_device(torch.from_numpy(x).cuda(), cfg)
        blob = res.to_bytes()
        offs, status = _both(blob, n, dt.wire_code, bs)
        assert np.array_equal(offs, res.block_offsets.cpu().numpy())
        assert status[1] == -1   # no error


def _decoy_i8(n_blocks, bs=4096):
    """int8 samples whose raw (selector 0, width 8) mantissa bytes spell
    block signatures: 04 00 00 00 F0 at many positions."""
    g = np.array([100, 4, 0, 0, 0, -16, 100, 100], np.int8)
    return np.tile(g, n_blocks * bs // g.size)


def test_k5_decoy_candidates_and_overflow():
    for nblk in (3, 12):   # 12 blocks x 512 decoys > cap -> overflow -> walk
        x = _decoy_i8(nblk)
        for mode, seg in ((Mode.LOSSLESS, 1), (Mode.LOSSLESS, None)):
            cfg = StreamConfig(Dtype.I8, 4096, mode, 0.0, segment_blocks=seg)
            res = encode_device(torch.from_numpy(x).cuda(), cfg)
            blob = res.to_bytes()
            # the decoys are really there
            assert blob.count(bytes([4, 0, 0, 0, 0xF0])) >= 256
            offs, status = _both(blob, x.size, Dtype.I8.wire_code, 4096)
            assert np.array_equal(offs, res.block_offsets.cpu().numpy())
            y = decode_device(res.blob, res.nbytes).cpu().numpy()
            assert np.array_equal(y, x)


def test_k5_errors_match_walk():
    """Corrupted / truncated streams: K5 falls back and reports the walk's
    status and block index."""
    rng = np.random.default_rng(5)
    x = W.cfg2_ar2_f32(4096 * 24)
    res = encode_device(torch.from_numpy(x).cuda(),
                        StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, 60.0, segment_blocks=4))
    blob = bytearray(res.to_bytes())
    offs = res.block_offsets.cpu().numpy()
    n = x.size
    cases = [bytes(blob[: len(blob) - 100]), bytes(blob[: int(offs[7]) + 3]), bytes(blob[: int(offs[23]) + 9])]
    for b in (2, 11, 23):   # reserved selector / broken JEE / header of the last block
        c = bytearray(blob)
        c[int(offs[b])] = 3
        cases.append(bytes(c))
        c = bytearray(blob)
        c[int(offs[b]) + 6] = 0xE0  # reserved JEE nibble 14
        cases.append(bytes(c))
    for _ in range(6):
        c = bytearray(blob)
        p = int(rng.integers(28, len(c)))
        c[p] ^= int(rng.integers(1, 256))
        cases.append(bytes(c))
    for i, c in enumerate(cases):
        o, s = _both(c, n, Dtype.F32.wire_code, 4096)
        if 3 <= i < 9 and i % 2 == 1:   # reserved selector at block b: reported at b
            b = (2, 11, 23)[(i - 3) // 2]
            assert s[1] != -1 and (int(s[1]) >> 8) == b


def test_k5_bench_size_cfg2_indexless_decode():
    """Full cfg2 size, whole-stream container: index-less decode equals the
    decode with the side-band index (and the oracle's offsets)."""
    x = W.cfg2_ar2_f32()
    cfg = StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, segment_blocks=16)
    res = encode_device(torch.from_numpy(x).cuda(), cfg)
    blob = res.to_bytes()
    offs, status = _find_blocks(blob, x.size, Dtype.F32.wire_code, 4096, True)
    assert status[1] == -1 and np.array_equal(offs, res.block_offsets.cpu().numpy())
    y = decode_device(res.blob, res.nbytes).cpu().numpy()
    y2 = decode_device(res.blob, res.nbytes, res.block_offsets).cpu().numpy()
    assert np.array_equal(y, y2)


def _gpu_indexless(blob: bytes, n, dt):
    """apax_decode without offsets (signature scan + speculative segment
    decode, full discovery + two-pass decode gated on the device)."""
    from paper_1303_4994_b200 import Decoder
    d = torch.zeros(len(blob) + 64, dtype=torch.uint8, device="cuda")
    d[:len(blob)] = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).cuda()
    dec = Decoder(n, dt, 4096)
    dec.decode(d, len(blob), None)
    torch.cuda.synchronize()
    key = int(dec.status.cpu().numpy().view(np.uint64)[1])
    if key != (1 << 64) - 1:
        return ("err", key & 0xFF, key >> 8)
    return ("ok", dec.y[:n].cpu().numpy())


def _oracle_indexless(blob: bytes):
    from oracle import oracle as O
    try:
        return ("ok", O.decode(blob, None, nthreads=0))
    except O.OracleError as e:
        return ("err", e.code, e.detail)


def _same(a, b):
    return a[0] == b[0] and (np.array_equal(a[1], b[1]) if a[0] == "ok" else a[1:] == b[1:])


def test_indexless_speculation_matches_oracle():
    """Containers that defeat the speculation (one candidate per block, the
    first at byte 28) in every way it can be defeated: the decode must equal
    the reference's walk-based decode (oracle), samples or first error."""
    x = W.cfg2_ar2_f32(4096 * 24 + 1000)
    n = x.size
    res = encode_device(torch.from_numpy(x).cuda(),
                        StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, 60.0, segment_blocks=4))
    blob = bytearray(res.to_bytes())
    offs = res.block_offsets.cpu().numpy()
    cases = {"clean": bytes(blob)}
    # a reserved header byte set: still a block for the reference, no longer
    # a candidate -> one candidate short
    c = bytearray(blob)
    c[int(offs[5]) + 3] = 1
    cases["reserved_byte"] = bytes(c)
    # ... plus a decoy signature in block 9's mantissas: one candidate per
    # block again, at the wrong places -> the decode's length check
    d = bytearray(c)
    p = int(offs[10]) - 40
    d[p:p + 7] = bytes([0, 0, 0, 0, 0, 0, 0xF0])
    cases["reserved_byte_and_decoy"] = bytes(d)
    # a segment head without its restart flag: the history runs on
    c = bytearray(blob)
    c[int(offs[8])] &= 0xFB
    cases["head_without_restart"] = bytes(c)
    # an extra restart inside a segment (the reference resets the history)
    c = bytearray(blob)
    c[int(offs[6])] |= 0x04
    cases["extra_restart"] = bytes(c)
    # errors: reserved selector, reserved JEE nibble, truncations
    for b in (0, 9, 24):
        c = bytearray(blob)
        c[int(offs[b])] = (c[int(offs[b])] & 0xFC) | 3
        cases[f"selector3_b{b}"] = bytes(c)
        c = bytearray(blob)
        c[int(offs[b]) + 6] = 0xE0
        cases[f"nibble14_b{b}"] = bytes(c)
    cases["truncated_mid"] = bytes(blob[: int(offs[13]) + 9])
    cases["truncated_tail"] = bytes(blob[: len(blob) - 5])
    for name, cb in cases.items():
        a, b = _gpu_indexless(cb, n, Dtype.F32), _oracle_indexless(cb)
        assert _same(a, b), (name, a[:1] + a[1:] if a[0] == "err" else "ok", b[:1] + b[1:] if b[0] == "err" else "ok")


@pytest.mark.parametrize("dt,mode,target,seg", [(Dtype.I16, Mode.FIXED_RATE, 4.0, 7), (Dtype.F64, Mode.FIXED_RATE, 20.0, 3),
                                                (Dtype.I32, Mode.FIXED_QUALITY, 40.0, 5), (Dtype.F32, Mode.LOSSLESS, 0.0, 0)])
def test_indexless_speculation_dtypes(dt, mode, target, seg):
    """Segmented (speculative path) and whole-stream (full discovery +
    two-pass) containers of other dtypes, partial last block included."""
    if dt is Dtype.F32 and mode is Mode.LOSSLESS:
        dt = Dtype.I8
    rng = np.random.default_rng(77)
    n = 4096 * 19 + 123
    xf = np.cumsum(rng.standard_normal(n)) * 30.0
    x = xf.astype(dt.np_dtype) if dt.is_float else np.clip(xf, np.iinfo(dt.np_dtype).min,
                                                             np.iinfo(dt.np_dtype).max).astype(dt.np_dtype)
    res = encode_device(torch.from_numpy(x).cuda(), StreamConfig(dt, 4096, mode, target, segment_blocks=seg or None))
    blob = res.to_bytes()
    a, b = _gpu_indexless(blob, n, dt), _oracle_indexless(blob)
    assert _same(a, b)
