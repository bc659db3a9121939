"""Index-less decode repeated on the same buffers: from the second decode on,
the fall-back behind the speculative segment decode (full discovery, second
chance, two-pass decode) runs inside a CUDA-graph IF node whose condition a
device kernel sets (apax_capi.cu, launch_gated_fallback).  Every repeat must
give the first decode's result and the oracle's: containers whose
speculation holds (the body is skipped), whole-stream containers and integer
containers with false candidates (the body runs), corrupted containers (the
body runs and reports the reference's error), and buffers re-used for a
different container of the same size."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_1303_4994_b200 import Decoder, Dtype, Mode, StreamConfig, encode_device  # noqa: E402
from paper_1303_4994_b200 import workloads as W  # noqa: E402

U64 = (1 << 64) - 1


def _repeat_decode(dec, d, nbytes, n, reps=4):
    out = []
    for _ in range(reps):
        dec.decode(d, nbytes, None)
        torch.cuda.synchronize()
        st = dec.status.cpu().numpy().view(np.uint64)
        key = int(st[1])
        out.append(("err", key & 0xFF, key >> 8) if key != U64 else ("ok", dec.y[:n].cpu().numpy().copy()))
    return out


def _oracle(blob):
    try:
        return ("ok", O.decode(blob))
    except O.OracleError as e:
        return ("err", e.code, e.detail)


def _same(a, b):
    if a[0] != b[0]:
        return False
    return np.array_equal(a[1], b[1]) if a[0] == "ok" else a[1:] == b[1:]


@pytest.mark.parametrize("case", ["f32_segments", "f32_whole_stream", "i16_segments", "i16_whole_stream"])
def test_repeated_indexless_decode(case):
    n = 4096 * 61 + 300
    if case.startswith("f32"):
        x, dt, mode, target = W.cfg2_ar2_f32(n), Dtype.F32, Mode.FIXED_QUALITY, 47.78
    else:
        x, dt, mode, target = W.cfg1_sines_i16(n), Dtype.I16, Mode.FIXED_RATE, 4.0
    seg = 7 if case.endswith("segments") else None
    res = encode_device(torch.from_numpy(x).cuda(), StreamConfig(dt, 4096, mode, target, segment_blocks=seg))
    blob = res.to_bytes()
    ref = _oracle(blob)
    assert ref[0] == "ok"
    d = torch.zeros(len(blob) + 64, dtype=torch.uint8, device="cuda")
    d[:len(blob)] = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).cuda()
    dec = Decoder(n, dt, 4096)
    for k, got in enumerate(_repeat_decode(dec, d, len(blob), n)):
        assert _same(got, ref), (case, "repeat", k)


def test_repeated_decode_of_corrupted_and_swapped_containers():
    """The same device buffers hold, in turn: a clean segmented container, a
    corrupted copy (an error through the graph body), the clean one again,
    and a whole-stream container of another array cut to the same length."""
    n = 4096 * 40
    x = W.cfg2_ar2_f32(n)
    res = encode_device(torch.from_numpy(x).cuda(), StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, 47.78,
                                                                 segment_blocks=5))
    clean = res.to_bytes()
    offs = res.block_offsets.cpu().numpy()
    bad = bytearray(clean)
    bad[int(offs[17]) + 6] = 0xE0            # a reserved JEE nibble in block 17
    bad2 = bytearray(clean)
    bad2[int(offs[9])] |= 3                  # reserved selector 3 in block 9
    d = torch.zeros(len(clean) + 64, dtype=torch.uint8, device="cuda")
    dec = Decoder(n, Dtype.F32, 4096)
    for blob in (clean, bytes(bad), clean, bytes(bad2), clean, bytes(bad), clean):
        d[:len(blob)] = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).cuda()
        ref = _oracle(blob)
        for k, got in enumerate(_repeat_decode(dec, d, len(blob), n, reps=3)):
            assert _same(got, ref), ("repeat", k, ref[0], got[0], got[1:] if got[0] == "err" else "")
