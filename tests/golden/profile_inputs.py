"""Seeded inputs for the profiler parity fixtures (shared by
make_profile_golden.py, which runs the live reference, and the GPU tests).
Synthetic signals only (sines, AR processes, noise)."""
import numpy as np


def make(name: str) -> tuple:
    """Return (x, dtype code, grid, block_size, segment_length)."""
    if name == "ar2_f32":
        rng = np.random.default_rng(31)
        n = 32768
        e = rng.standard_normal(n)
        x = np.zeros(n)
        th = 0.3
        for t in range(2, n):
            x[t] = 2 * 0.98 * np.cos(th) * x[t - 1] - 0.98 ** 2 * x[t - 2] + e[t]
        return (x * 1e3).astype(np.float32), "f32", (20.0, 30.0, 40.0, 50.0, 60.0, 70.0), 4096, 4096
    if name == "sines_i16":
        rng = np.random.default_rng(32)
        n = 16384
        t = np.arange(n)
        f = rng.uniform(0.001, 0.2, 4)
        x = sum(2000 * np.sin(2 * np.pi * fi * t + rng.uniform(0, 6.28)) for fi in f)
        x = x + rng.normal(0, 20, n)
        return np.clip(np.rint(x), -32768, 32767).astype(np.int16), "i16", (40.0, 60.0, 80.0), 1024, 4096
    if name == "walk_f64":
        rng = np.random.default_rng(33)
        x = np.cumsum(rng.standard_normal(12000)) * 1e-3
        return x.astype(np.float64), "f64", (40.0, 60.0, 80.0, 100.0), 2048, 4096
    if name == "noise_i32_default_grid":
        rng = np.random.default_rng(34)
        x = np.cumsum(rng.integers(-40, 41, 20000)) * 100
        return x.astype(np.int32), "i32", tuple(float(t) for t in range(20, 121, 5)), 4096, 4096
    if name == "short_f32":
        rng = np.random.default_rng(35)
        x = (np.sin(0.05 * np.arange(3000)) * 50 + rng.normal(0, 0.5, 3000)).astype(np.float32)
        return x, "f32", (30.0, 50.0, 70.0), 512, 4096
    if name == "const_i16":
        # a constant: every difference stream is silent, the correlation of x
        # and y is undefined at most targets (points dropped with a warning)
        return np.full(16384, 7, np.int16), "i16", (2.0, 4.0, 20.0), 4096, 4096
    if name == "ramp_i32_unreachable":
        # no grid point reaches the correlation threshold: target_unreachable
        return np.arange(16384, dtype=np.int32), "i32", (2.0, 4.0), 4096, 4096
    raise KeyError(name)


NAMES = ("ar2_f32", "sines_i16", "walk_f64", "noise_i32_default_grid", "short_f32", "const_i16",
         "ramp_i32_unreachable")
