"""Pipelined host round trip (paper_1303_4994_b200/pipeline.py): the host
container assembled from per-chunk encodes equals the one-call encode of
the whole stream with the same segment length, byte for byte, with the
same side-band index; the decoded host samples equal the device decode."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, decode_device, encode_device  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402
from paper_1303_4994_b200.pipeline import HostRoundTrip  # noqa: E402


@pytest.mark.parametrize("dt,mode,target,bs,seg,n,chunks,taper", [
    (Dtype.F32, Mode.FIXED_QUALITY, 47.5, 4096, 5, 4096 * 5 * 13 + 1000, 4, 1),
    (Dtype.F32, Mode.FIXED_QUALITY, 60.0, 4096, 37, 4096 * 37 * 9, 8, 1),
    (Dtype.F32, Mode.FIXED_QUALITY, 47.5, 4096, 2, 4096 * 2 * 40 + 11, 9, 4),
    (Dtype.I16, Mode.FIXED_RATE, 4.0, 1024, 3, 1024 * 3 * 20 + 7, 5, 1),
    (Dtype.I32, Mode.LOSSLESS, 0.0, 512, 2, 512 * 2 * 3, 8, 1),
    (Dtype.F64, Mode.FIXED_RATE, 21.3, 2048, 4, 2048 * 4 * 6 + 3, 3, 1),
])
def test_host_round_trip_matches_whole_stream(dt, mode, target, bs, seg, n, chunks, taper):
    rng = np.random.default_rng(n)
    if dt.is_float:
        x = (np.cumsum(rng.standard_normal(n)) * 100).astype(dt.np_dtype)
    else:
        x = np.clip(np.cumsum(rng.integers(-40, 41, n)), -30000, 30000).astype(dt.np_dtype)
    cfg = StreamConfig(dt, bs, mode, target, segment_blocks=seg)
    ref = encode_device(torch.from_numpy(x).cuda(), cfg)
    ref_bytes = ref.to_bytes()
    rt = HostRoundTrip(n, cfg, chunks=chunks, taper=taper)
    xh = torch.from_numpy(x).pin_memory()
    blob_h = torch.zeros(len(ref_bytes) + 4096, dtype=torch.uint8).pin_memory()
    offs_h = torch.empty(rt.n_blocks + 1, dtype=torch.int64).pin_memory()
    yh = torch.empty(n, dtype=xh.dtype).pin_memory()
    for _ in range(2):   # buffers are reused across calls
        nb = rt.run(xh, blob_h, offs_h, yh)
        assert nb == len(ref_bytes)
        assert bytes(blob_h[:nb].numpy().tobytes()) == ref_bytes
        assert np.array_equal(offs_h.numpy(), ref.block_offsets.cpu().numpy())
        y = decode_device(ref.blob, ref.nbytes).cpu().numpy()
        assert np.array_equal(yh.numpy(), y)
    assert rt.h2d_bytes == x.nbytes + (nb - 28) + 8 * (rt.n_blocks + len(rt.ranges))
