"""Inputs of the trace fixtures (tests/golden/trace_blocks.json), regenerated
from the seeded generators the fixture names and pinned by its SHA-256."""
import hashlib
import json

import numpy as np

from conftest import GOLDEN

GENS = {
    "cfg1_sines_i16(1 << 17)": lambda W: W.cfg1_sines_i16(1 << 17),
    "cfg2_ar2_f32(1 << 17)": lambda W: W.cfg2_ar2_f32(1 << 17),
    "cfg3_grf_f32(512)": lambda W: W.cfg3_grf_f32(512),
    "cfg4_modes_f64_np(48)": lambda W: W.cfg4_modes_f64_np(48),
    "cfg5_ar1(1 << 16, 'i32')": lambda W: W.cfg5_ar1(1 << 16, "i32"),
}


def traces():
    return json.loads((GOLDEN / "trace_blocks.json").read_text())["traces"]


def trace_input(t):
    from paper_1303_4994_b200 import workloads as W
    x = GENS[t["x_gen"]](W)
    assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == t["x_sha256"], t["name"]
    return x
