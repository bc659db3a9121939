"""SHA-256 pins of the LIVE reference's full-size whole-stream containers.

Runs the reference's own `encode_stream` (pkg/src/apax/codec.py:258-285) on
the BASELINE configs at their full sizes with no segments -- cfg1 (2^24
int16, fixed rate 4 bps), cfg2 (2^26 f32 AR(2), fixed quality at
workloads.CFG2_TARGET_DB) and cfg3 (8192^2 f32 field, fixed rate 32/6 bps)
-- and records the input's and the container's SHA-256 and length.  The
containers are too large to commit; tests/test_fullsize_pins.py checks the
oracle (CPU) and the GPU whole-stream encoder against these hashes.

Run in the build container (minutes: the reference is numpy):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_fullsize_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import pathlib
import sys
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF = os.environ.get("APAX_REF", "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)
sys.path.insert(0, str(REPO))

from apax import codec as rcodec  # noqa: E402  (the reference)
from apax.dtypes import Dtype, Mode, StreamConfig  # noqa: E402

from paper_1303_4994_b200 import workloads as W  # noqa: E402

CASES = {
    "cfg1_i16_fr4_whole": (W.cfg1_sines_i16, Dtype.I16, Mode.FIXED_RATE, 4.0),
    "cfg2_f32_fq_whole": (W.cfg2_ar2_f32, Dtype.F32, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB),
    "cfg3_f32_fr6_whole": (W.cfg3_grf_f32, Dtype.F32, Mode.FIXED_RATE, 32.0 / 6.0),
}


def sha(b) -> str:
    return hashlib.sha256(b).hexdigest()


def main():
    out = {}
    for name, (gen, dt, mode, target) in CASES.items():
        x = np.ascontiguousarray(gen())
        t0 = time.time()
        blob = rcodec.encode_stream(x, StreamConfig(dt, 4096, mode, target))
        out[name] = dict(gen=gen.__name__, dtype=dt.name, mode=mode.name, target_hex=float(target).hex(),
                         block_size=4096, n=int(x.size), x_sha256=sha(x.tobytes()),
                         container_sha256=sha(blob), container_bytes=len(blob),
                         reference_encode_s=round(time.time() - t0, 1))
        print(name, out[name], flush=True)
    (HERE / "fullsize_pins.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
