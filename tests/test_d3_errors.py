"""Corrupted segmented containers through the segment-serial decoder
(apax_decode_segments: JEE parsed per warp in batches of 8 blocks) against
the oracle decoding at the same side-band offsets: the same first failing
(block, status) -- the lowest block wins, like the reference's serial walk
-- or, when a corruption still decodes, the same samples.  Corruptions hit
blocks at every position of a JEE batch.

One deliberate difference: when a corruption makes a block parse LONGER
than its span in the side-band index, the index no longer describes the
container (the reference's serial walk would now find a different next
block), and the GPU decoder reports "invalid argument" (42) for that block
instead of reading on into the next block as the oracle-with-offsets does;
the test checks that the walk indeed disagrees with the index there."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_1303_4994_b200 import Decoder, Dtype, Mode, StreamConfig, encode_device  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

U64 = (1 << 64) - 1


def _gpu(blob: bytes, offs, n, dt, seg):
    d = torch.zeros(len(blob) + 64, dtype=torch.uint8, device="cuda")
    d[:len(blob)] = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).cuda()
    dec = Decoder(n, dt, 4096)
    dec.decode(d, len(blob), torch.from_numpy(offs).cuda(), segment_blocks=seg)
    torch.cuda.synchronize()
    st = dec.status.cpu().numpy().view(np.uint64)
    key = int(st[1])
    if key != U64:
        return ("err", key & 0xFF, key >> 8)
    return ("ok", dec.y[:n].cpu().numpy())


def _walk_end(blob: bytes, k: int, bs: int = 4096) -> int:
    """End of block k by the reference's serial walk: the walk over a copy
    of the container whose header claims k + 1 blocks."""
    b = bytearray(blob)
    b[12:20] = int((k + 1) * bs).to_bytes(8, "little")
    return int(O.find_blocks(bytes(b))[k + 1])


def _oracle(blob: bytes, offs):
    try:
        return ("ok", O.decode(blob, offs, nthreads=0))
    except O.OracleError as e:
        return ("err", e.code, e.detail)


@pytest.mark.parametrize("dt,mode,target", [(Dtype.F32, Mode.FIXED_QUALITY, 45.0), (Dtype.I16, Mode.FIXED_RATE, 4.0)])
def test_corrupted_blocks_match_oracle(dt, mode, target):
    seg = 10
    n = 4096 * 37 + 500
    x = W.cfg2_ar2_f32(n) if dt == Dtype.F32 else W.cfg1_sines_i16(n)
    res = encode_device(torch.from_numpy(x).cuda(), StreamConfig(dt, 4096, mode, target, segment_blocks=seg))
    blob = res.to_bytes()
    offs = res.block_offsets.cpu().numpy()
    hs = 6 if dt.is_float else 4
    rng = np.random.default_rng(7)
    cases = 0
    for k in (0, 3, 7, 8, 9, 15, 23, 37):
        o = int(offs[k])
        variants = []
        b = bytearray(blob); b[o + hs] = 0x05; variants.append(bytes(b))                  # first token not an escape
        b = bytearray(blob); b[o] = (b[o] & ~3) | 3; variants.append(bytes(b))            # reserved selector
        b = bytearray(blob); b[o + hs + 1] = 0xE7; variants.append(bytes(b))              # escape value > 34 / nibble 14
        for _ in range(3):                                                                # random JEE nibble edits
            b = bytearray(blob)
            p = o + hs + int(rng.integers(0, 200))
            b[p] = int(rng.integers(0, 256))
            variants.append(bytes(b))
        variants.append(blob[:o + hs + 40])                                               # truncated inside block k
        for v in variants:
            g = _gpu(v, offs, n, dt, seg)
            r = _oracle(v, offs)
            if g[0] == "err" and g[1] == 42 and (r[0] == "ok" or r[2] > g[2]):
                kb = int(g[2])
                assert _walk_end(v, kb) > int(offs[kb + 1]), (k, kb)
                cases += 1
                continue
            assert g[0] == r[0], (k, g[:3] if g[0] == "err" else "ok", r[:3] if r[0] == "err" else "ok")
            if g[0] == "err":
                assert g[1:] == r[1:], (k, g, r)
            else:
                assert np.array_equal(g[1], r[1]), k
            cases += 1
    assert cases == 8 * 7
