"""Fixtures for encode_stream's input conversions, from the LIVE reference.

The reference widens every input before quantizing it (pkg/src/apax/
codec.py:266-272): float configs take `x.astype(float64)`, integer configs
`x.astype(int64)` (floats truncate toward zero; values outside the
container's range are coded as they are and clipped at decode,
codec.py:143-145).  Run in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_cast_golden.py

Writes containers/cast_*.npz (input in its own dtype, config, reference
container and decode) plus cast_manifest.json, and cast_errors.json (inputs
whose widened values the reference rejects, with the exception it raises).
"""
from __future__ import annotations

import json
import os
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF = os.environ.get("APAX_REF", "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(HERE))

from apax import codec as rcodec  # noqa: E402  (the reference)
from apax.dtypes import Mode, StreamConfig  # noqa: E402
from make_golden import DT, OUT, save_case  # noqa: E402

from paper_1303_4994_b200 import workloads as W  # noqa: E402


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(20261021)
    x2 = W.cfg2_ar2_f32(1 << 15).astype(np.float64)
    f64 = x2 + rng.standard_normal(x2.size) * 1e-3          # not f32-representable
    ar = np.cumsum(rng.standard_normal(40000)) * 300.0
    cases = [
        # float64 samples into an f32 container (quantized from the f64 values)
        ("cast_f64_f32_fq120", f64, "f32", Mode.FIXED_QUALITY, 120.0, 4096),
        ("cast_f64_f32_fq48", f64, "f32", Mode.FIXED_QUALITY, 48.0, 4096),
        ("cast_f64_f32_fr30", f64, "f32", Mode.FIXED_RATE, 30.0, 4096),
        ("cast_f64_f32_fr6_bs1000", f64[:20000], "f32", Mode.FIXED_RATE, 6.0, 1000),
        ("cast_f64_f32_fr8_beyond_f32", np.concatenate([f64[:5000], [1e39, -3e38]]), "f32",
         Mode.FIXED_RATE, 8.0, 1024),
        # f32 / integer samples into float containers (exact widening)
        ("cast_f32_f64_fr20", x2.astype(np.float32), "f64", Mode.FIXED_RATE, 20.0, 4096),
        ("cast_i32_f32_fq70", rng.integers(-2 ** 30, 2 ** 30, 9000).astype(np.int32), "f32",
         Mode.FIXED_QUALITY, 70.0, 2048),
        ("cast_i64_f64_fr12", rng.integers(-2 ** 60, 2 ** 60, 7000), "f64", Mode.FIXED_RATE, 12.0,
         1024),
        # non-integer floats into integer containers (astype(int64) truncation)
        ("cast_f64_i16_fr6_trunc", np.clip(ar, -30000, 30000), "i16", Mode.FIXED_RATE, 6.0, 4096),
        ("cast_f32_i32_lossless_trunc", (ar * 7.3).astype(np.float32), "i32", Mode.LOSSLESS, 0.0,
         2048),
        ("cast_f64_i8_fq30_trunc", np.clip(ar / 100.0, -128, 127), "i8", Mode.FIXED_QUALITY, 30.0,
         512),
        # integers outside the container's range (coded as they are, clipped at decode)
        ("cast_i32_i16_lossless_oor", (ar * 4).astype(np.int32), "i16", Mode.LOSSLESS, 0.0, 4096),
        ("cast_i64_i8_fr4_oor", (ar / 5).astype(np.int64), "i8", Mode.FIXED_RATE, 4.0, 1024),
        ("cast_i64_i16_fq40_oor", (ar * 3).astype(np.int64), "i16", Mode.FIXED_QUALITY, 40.0, 4096),
        ("cast_i64_i32_fr8_oor", (ar * 5e4).astype(np.int64), "i32", Mode.FIXED_RATE, 8.0, 4096),
        ("cast_u16_i16_lossless", rng.integers(0, 65536, 9000).astype(np.uint16), "i16",
         Mode.LOSSLESS, 0.0, 4096),
        # in-range widening (the product codes these in the container dtype)
        ("cast_i16_i32_fr5", np.clip(ar, -30000, 30000).astype(np.int16), "i32", Mode.FIXED_RATE,
         5.0, 4096),
        ("cast_bool_i8_lossless", rng.integers(0, 2, 3000).astype(bool), "i8", Mode.LOSSLESS, 0.0,
         256),
    ]
    manifest = []
    for name, x, dt, mode, T, bs in cases:
        cfg = StreamConfig(DT[dt], bs, mode, T)
        blob = rcodec.encode_stream(x, cfg)
        meta = save_case(name, x, dt, mode, T, bs, blob)
        meta["x_dtype"] = str(np.asarray(x).dtype)
        manifest.append(meta)
    (HERE / "cast_manifest.json").write_text(json.dumps(manifest, indent=1))

    errs = []
    bad = [
        ("cast_i64_i32_beyond_34bit", np.concatenate([np.arange(5000), [2 ** 40]]).astype(np.int64),
         "i32", Mode.LOSSLESS, 0.0, 1024),
        ("cast_f64_i16_nonfinite_ok", np.where(np.arange(300) == 100, 1.5, 2.0), "i16",
         Mode.FIXED_RATE, 4.0, 64),
        ("cast_i32_f32_nan_free", np.arange(100, dtype=np.int32), "f32", Mode.FIXED_QUALITY, 60.0, 64),
        ("cast_f64_f32_nonfinite", np.where(np.arange(700) == 633, np.inf, 1.0), "f32",
         Mode.FIXED_QUALITY, 60.0, 256),
        # f32 y overflows to inf: pd = inf, math.log10(px / pd) = log10(0) raises
        ("cast_f64_f32_fq60_beyond_f32", np.concatenate([f64[:5000], [1e39, -3e38]]), "f32",
         Mode.FIXED_QUALITY, 60.0, 1024),
        # beyond the float block exponent's reach (fbe clamps at -127): q
        # overflows int64 on the second block
        ("f64_fq_beyond_fbe_internal", np.concatenate([np.ones(64), rng.standard_normal(64) * 1e200]),
         "f64", Mode.FIXED_QUALITY, 60.0, 64),
    ]
    for name, x, dt, mode, T, bs in bad:
        rec = dict(name=name, dtype=dt, mode=int(mode.value), target=T, block_size=bs,
                   x_dtype=str(x.dtype), x_hex=x.tobytes().hex())
        try:
            blob = rcodec.encode_stream(x, StreamConfig(DT[dt], bs, mode, T))
            rec.update(exc=None, blob_hex=blob.hex())
        except Exception as exc:  # noqa: BLE001
            rec.update(exc=type(exc).__name__, msg=str(exc))
        errs.append(rec)
    (HERE / "cast_errors.json").write_text(json.dumps(errs, indent=1))
    print(f"wrote {len(manifest)} cast containers, {len(errs)} cast error cases")


if __name__ == "__main__":
    main()
