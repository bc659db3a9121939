"""Whole-stream containers decoded by block ranges (apax_decode_range), the
per-rank step of the multi-GPU decode of SURVEY.md §8(e): every range is
decoded once with entry history (0, 0) for its affine history map, the maps
are composed in range order on the host (distributed.range_entries, the
function the ranks run after their all-gather), and every range is decoded
again from its exact entry.  The concatenated ranges must equal the
one-launch decode and the oracle bit for bit; for lossless integer streams
the composed entries must equal the input samples before each range."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, decode_device, decode_range, encode_device  # noqa: E402
from paper_1303_4994_b200 import distributed as D  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

M64 = (1 << 64) - 1


def _x(dt, n, seed):
    rng = np.random.default_rng(seed)
    if dt == Dtype.I16:
        return W.cfg1_sines_i16(n, seed=seed)
    if dt == Dtype.F32:
        return W.cfg2_ar2_f32(n, seed=seed)
    if dt == Dtype.I32:
        return np.clip(np.cumsum(rng.integers(-(1 << 24), 1 << 24, n)), -(1 << 31), (1 << 31) - 1).astype(np.int32)
    return W.cfg5_ar1(n, "f32", seed=seed).astype(np.float64) * 1e3


CASES = [
    # dtype, mode, target, block size, blocks, ranges
    (Dtype.I16, Mode.FIXED_RATE, 4.0, 4096, 37, 3),
    (Dtype.F32, Mode.FIXED_QUALITY, 47.77, 4096, 40, 4),
    (Dtype.I32, Mode.LOSSLESS, 0.0, 1024, 29, 3),
    (Dtype.F64, Mode.FIXED_RATE, 21.3, 2048, 25, 2),
    (Dtype.F32, Mode.FIXED_RATE, 5.33, 8192, 11, 3),       # bs > 4096: the v1 decoder
    (Dtype.I16, Mode.LOSSLESS, 0.0, 256, 64, 5),
]


@pytest.mark.parametrize("dt,mode,target,bs,nblk,R", CASES)
def test_range_decode_composes_to_whole_stream(dt, mode, target, bs, nblk, R):
    n = bs * nblk - 123          # partial last block
    x = _x(dt, n, nblk)
    res = encode_device(torch.from_numpy(x).cuda(), StreamConfig(dt, bs, mode, target))
    blob = res.to_bytes()
    ref = O.decode(blob)
    y_all = decode_device(res.blob, res.nbytes, res.block_offsets).cpu().numpy()
    assert np.array_equal(y_all, ref)
    nb = (n + bs - 1) // bs
    ranges = [D.shard_blocks(nb, R, r) for r in range(R)]
    maps = [decode_range(res.blob, res.nbytes, res.block_offsets, n, dt, bs, b0, b1, want_map=True)[1]
            for b0, b1 in ranges]
    entries = D.range_entries(maps)
    parts = [decode_range(res.blob, res.nbytes, res.block_offsets, n, dt, bs, b0, b1, entry=e)[0].cpu().numpy()
             for (b0, b1), e in zip(ranges, entries)]
    assert np.array_equal(np.concatenate(parts), ref)
    if mode == Mode.LOSSLESS:
        for (b0, _), e in zip(ranges[1:], entries[1:]):
            assert e == (int(x[b0 * bs - 1]) & M64, int(x[b0 * bs - 2]) & M64)
    # the composed map of every range applied to its entry is the next entry
    for r in range(R - 1):
        assert D.apply_map(maps[r], entries[r]) == entries[r + 1]
