"""Whole-stream LOSSLESS containers encoded by block ranges
(apax_encode_lossless_range), the per-rank step of the multi-GPU LOSSLESS
encode of SURVEY.md §8(e): each range gets the (bs + 2) samples before it
as its halo; the concatenated bodies must equal the one-call whole-stream
container (and the oracle's) byte for byte, with the same side-band index."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_1303_4994_b200 import Dtype, StreamConfig, encode_device, encode_lossless_range  # noqa: E402
from paper_1303_4994_b200 import distributed as D  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402


@pytest.mark.parametrize("dt,bs,nblk,R", [
    (Dtype.I16, 4096, 41, 3),
    (Dtype.I32, 1024, 33, 4),
    (Dtype.I8, 256, 70, 5),
    (Dtype.I16, 128, 9, 9),     # one block per range
])
def test_lossless_ranges_concatenate_to_whole_stream(dt, bs, nblk, R):
    n = bs * nblk - 77
    rng = np.random.default_rng(nblk)
    if dt == Dtype.I16:
        x = W.cfg1_sines_i16(n, seed=nblk)
    elif dt == Dtype.I32:
        x = np.cumsum(rng.integers(-5000, 5000, n)).astype(np.int32)
    else:
        x = rng.integers(-128, 128, n).astype(np.int8)
    xd = torch.from_numpy(x).cuda()
    whole = encode_device(xd, StreamConfig(dt, bs))
    wb = whole.to_bytes()
    ref, roffs, _ = O.encode(x, dt.wire_code, 0, 0.0, bs)
    assert wb == ref
    nb = (n + bs - 1) // bs
    body = b""
    offs = []
    for r in range(R):
        b0, b1 = D.shard_blocks(nb, R, r)
        s0, s1 = b0 * bs, min(n, b1 * bs)
        h = 0 if b0 == 0 else min(s0, bs + 2)
        res = encode_lossless_range(xd[s0 - h:s1], h, b0, dt, bs)
        part = res.to_bytes()
        assert part[:28] != b""           # its own header
        lo = res.block_offsets.cpu().numpy()
        offs.append(lo[:-1] - 28 + 28 + len(body))
        body += part[28:]
    assert wb[28:] == body
    assert np.array_equal(np.concatenate(offs + [[len(wb)]]), roffs)
