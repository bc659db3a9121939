"""Full-size whole-stream containers against the LIVE reference's SHA-256
pins (tests/golden/fullsize_pins.json, written by
tests/golden/make_fullsize_golden.py from the reference's own
`encode_stream`, pkg/src/apax/codec.py:258-285).

CPU: the oracle's whole-stream encode of cfg1 / cfg2 / cfg3 at their full
sizes hashes to the reference's container -- so the oracle, the checker of
every full-size GPU test, is pinned at full size, not only on the small
fixtures.  GPU: the device whole-stream encoders (the ws chain + packer for
fixed rate, the v3 chain + packer for fixed quality) hash to the same pins.
"""
import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN

from oracle import oracle as O
from paper_1303_4994_b200 import workloads as W

PINS = json.loads((GOLDEN / "fullsize_pins.json").read_text())
WIRE = {"I16": 1, "F32": 3}
MODE = {"FIXED_RATE": 1, "FIXED_QUALITY": 2}


def _case(name):
    p = PINS[name]
    x = np.ascontiguousarray(getattr(W, p["gen"])())
    assert hashlib.sha256(x.tobytes()).hexdigest() == p["x_sha256"], name
    return p, x


@pytest.mark.parametrize("name", sorted(PINS))
def test_oracle_whole_stream_matches_reference_pin(name):
    p, x = _case(name)
    blob, _, _ = O.encode(x, WIRE[p["dtype"]], MODE[p["mode"]], float.fromhex(p["target_hex"]), p["block_size"])
    assert len(blob) == p["container_bytes"]
    assert hashlib.sha256(blob).hexdigest() == p["container_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(PINS))
def test_gpu_whole_stream_matches_reference_pin(name):
    torch = pytest.importorskip("torch")
    from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, encode_device
    p, x = _case(name)
    cfg = StreamConfig(Dtype[p["dtype"]], p["block_size"], Mode[p["mode"]], float.fromhex(p["target_hex"]))
    res = encode_device(torch.from_numpy(x).cuda(), cfg)
    blob = res.to_bytes()
    assert len(blob) == p["container_bytes"]
    assert hashlib.sha256(blob).hexdigest() == p["container_sha256"]
