"""Freeze the LIVE reference profiler's outputs for the GPU profiler tests.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_profile_golden.py

Writes tests/golden/profile_reports.json: for every input of
profile_inputs.py, the reference `profile(...)` report (curve, recommended,
windows: 18 metrics, spectra, S2R margin and CDF) plus stand-alone
`pearson_r`, `welch_spectrum` and `s2r_distribution` values.
"""
from __future__ import annotations

import json
import os
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REF = os.environ.get("APAX_REF", "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, REF)
sys.path.insert(0, str(HERE))

from apax import profiler as rp  # noqa: E402  (the reference)
from apax.dtypes import Dtype  # noqa: E402

import profile_inputs as PI  # noqa: E402


def jsonable(v):
    if isinstance(v, float) and not np.isfinite(v):
        return {"nonfinite": repr(v)}
    if isinstance(v, dict):
        return {k: jsonable(w) for k, w in v.items()}
    if isinstance(v, (list, tuple)):
        return [jsonable(w) for w in v]
    if isinstance(v, (np.floating,)):
        return jsonable(float(v))
    return v


def main():
    # inputs already frozen stay as they are (--all regenerates every one)
    path = HERE / "profile_reports.json"
    out = json.loads(path.read_text()) if path.exists() and "--all" not in sys.argv else {}
    for name in PI.NAMES:
        if name in out:
            continue
        x, code, grid, bs, seg = PI.make(name)
        dt = Dtype.from_code(code)
        rep = rp.profile(x, dt, grid=grid, block_size=bs, name=name)
        xf = x.astype(np.float64)
        rng = np.random.default_rng(77)
        y = xf + 0.01 * rng.standard_normal(xf.size) * (np.std(xf) + 1.0)
        spec = rp.welch_spectrum(xf, seg)
        d = xf - y
        d[::97] = 0.0
        dist = rp.s2r_distribution(xf, d)
        out[name] = {
            "report": rep,
            "pearson": rp.pearson_r(xf, y),
            "welch": {"power": spec.power.tolist(), "peak_db": spec.peak_db, "floor_db": spec.floor_db,
                      "mean_db": spec.mean_db},
            "s2r": {"margin": dist.two_sigma_margin_db, "cdf": dist.cdf_points()},
        }
        print(name, rep["recommended"], flush=True)
    (HERE / "profile_reports.json").write_text(json.dumps(jsonable(out)))


if __name__ == "__main__":
    main()
