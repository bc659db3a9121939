"""Seeded synthetic workloads standing in for BASELINE.json's five configs.

No public dataset is involved (the paper's 25 datasets are confidential,
reference `SPEC.md:10,708`); these generators reproduce the shapes, sizes and
value distributions BASELINE.json names, per SURVEY.md §8(d).  Every
generator is numpy-seeded so the identical bytes feed the GPU path, the CPU
oracle and (in this container) the live reference.
"""
from __future__ import annotations

import numpy as np

__all__ = ["cfg1_sines_i16", "cfg2_ar2_f32", "cfg3_grf_f32", "cfg4_modes_f64",
           "cfg4_modes_f64_np", "cfg5_ar1", "CFG2_TARGET_DB"]

# FQ target for cfg2: the profiler's recommended SRR target
# (profile(x, Dtype.F32)["recommended"]["srr_target"]) of the full 2^26
# array.  The GPU profile() computes it in 0.55 s
# (profiles/r2_profile_cfg2_full.json: 47.781765928385084); the live CPU
# reference (OPENBLAS_NUM_THREADS=1, 474 s,
# profiles/r2_reference_profile_cfg2_full_cpu.json) gives 47.78176608065653
# -- 1.5e-7 dB apart, the reference's own BLAS-order sensitivity of r
# (SURVEY.md §8(a) A31).  The reference's value is the one stored, as hex, so
# the GPU path, the oracle and the reference arm use the identical f64
# (SURVEY.md §8(d) cfg2 note).
CFG2_TARGET_HEX = "0x1.7e410e932c55dp+5"  # 47.78176608065653 dB (full 2^26 array)
CFG2_TARGET_DB = float.fromhex(CFG2_TARGET_HEX)
# round 1's target, from the 2^20 analogue (still pinned by older fixtures)
CFG2_TARGET_2P20_HEX = "0x1.7e30c8e72cf90p+5"  # 47.77382069211956 dB


def cfg1_sines_i16(n: int = 1 << 24, seed: int = 1) -> np.ndarray:
    """int16: 8 sinusoids (f ~ U(0.001, 0.2) cycles/sample, amplitudes
    U(0.5, 1.5) rescaled to sum 8000, phases U(0, 2pi)) + N(0, 20^2)."""
    rng = np.random.default_rng(seed)
    f = rng.uniform(0.001, 0.2, 8)
    a = rng.uniform(0.5, 1.5, 8)
    a *= 8000.0 / a.sum()
    ph = rng.uniform(0, 2 * np.pi, 8)
    t = np.arange(n, dtype=np.float64)
    x = np.zeros(n, np.float64)
    for i in range(8):
        x += a[i] * np.sin(2 * np.pi * f[i] * t + ph[i])
    x += rng.normal(0.0, 20.0, n)
    return np.clip(np.rint(x), -32768, 32767).astype(np.int16)


def cfg2_ar2_f32(n: int = 1 << 26, seed: int = 2) -> np.ndarray:
    """float32 AR(2): x[t] = 2 r cos(th) x[t-1] - r^2 x[t-2] + e[t],
    r = 0.98, th ~ U(0, pi), e ~ N(0, 1), scaled by 1e3."""
    from scipy.signal import lfilter
    rng = np.random.default_rng(seed)
    th = rng.uniform(0, np.pi)
    r = 0.98
    e = rng.standard_normal(n)
    x = lfilter([1.0], [1.0, -2 * r * np.cos(th), r * r], e)
    return (x * 1e3).astype(np.float32)


def cfg3_grf_f32(side: int = 8192, seed: int = 3) -> np.ndarray:
    """float32 side x side row-major Gaussian random field, |F(k)|^2 ~ k^-3
    (rfft2 of white complex noise x |k|^-1.5, DC zeroed), plus uniform noise
    of +-1e-3 of the field's range."""
    rng = np.random.default_rng(seed)
    ky = np.fft.fftfreq(side)[:, None]
    kx = np.fft.rfftfreq(side)[None, :]
    k = np.sqrt(kx * kx + ky * ky)
    k[0, 0] = 1.0
    amp = k ** -1.5
    amp[0, 0] = 0.0
    spec = (rng.standard_normal(amp.shape) + 1j * rng.standard_normal(amp.shape)) * amp
    del amp, k
    img = np.fft.irfft2(spec, s=(side, side))
    del spec
    rngv = float(img.max() - img.min())
    img += rng.uniform(-1e-3 * rngv, 1e-3 * rngv, img.shape)
    return img.astype(np.float32).reshape(-1)


def cfg4_modes_f64(side: int = 1024, seed: int = 4, n_modes: int = 64, device=None, planes=None,
                   z0: int = 0):
    """float64 side^3 field: 64 modes A cos(2 pi k.r/side + phi), A ~ N(0,1),
    k in [-8, 8]^3, phi ~ U(0, 2 pi), plus N(0, sigma=1e-4) (read as sigma).

    Built as one f64 GEMM (cos(a + b) = cos a cos b - sin a sin b with a the
    x term and b the (y, z) terms), so the full 8 GiB field is generated on
    the GPU in milliseconds: returns a flat torch f64 tensor on `device`
    (default cuda:0 when available, else CPU).  Mode parameters are
    numpy-seeded; the noise comes in chunks of 2^26 samples, chunk c from a
    torch generator seeded (seed, c) on the same device, so the field is
    reproducible per device type and any slab can be generated on its own:
    `z0` / `planes` give the z planes [z0, z0 + planes) of the one field (a
    rank's shard of a sharded array, the CPU reference arm's sample)."""
    import torch
    if device is None:
        device = "cuda" if torch.cuda.is_available() else "cpu"
    dev = torch.device(device)
    rng = np.random.default_rng(seed)
    A = torch.from_numpy(rng.standard_normal(n_modes)).to(dev)
    K = torch.from_numpy(rng.integers(-8, 9, size=(n_modes, 3)).astype(np.float64)).to(dev)
    phi = torch.from_numpy(rng.uniform(0, 2 * np.pi, n_modes)).to(dev)
    r = torch.arange(side, dtype=torch.float64, device=dev) * (2 * np.pi / side)
    ax = K[:, 0, None] * r[None, :] + phi[:, None]                     # [m, x]
    C = torch.cat([torch.cos(ax), -torch.sin(ax)], 0)                 # [2m, x]
    del ax
    z0 = int(z0)
    nz = (side - z0) if planes is None else min(int(planes), side - z0)
    out = torch.empty(nz * side, side, dtype=torch.float64, device=dev)
    zc = max(1, min(nz, (1 << 26) // (side * side) or 1))            # z planes per GEMM chunk
    for za in range(0, nz, zc):
        zb = min(nz, za + zc)
        byz = (K[None, None, :, 1] * r[None, :, None] +
               K[None, None, :, 2] * r[z0 + za:z0 + zb, None, None])  # [z, y, m]
        B = torch.cat([A * torch.cos(byz), A * torch.sin(byz)], -1)   # [z, y, 2m]
        out[za * side:zb * side] = B.reshape(-1, 2 * n_modes) @ C
        del byz, B
    flat = out.reshape(-1)
    chunk = 1 << 26
    g0, g1 = z0 * side * side, (z0 + nz) * side * side                # global sample range
    g = torch.Generator(device=dev)
    for c in range(g0 // chunk, (g1 + chunk - 1) // chunk):
        a, b = max(g0, c * chunk), min(g1, (c + 1) * chunk)
        g.manual_seed(seed * 1000003 + c)
        noise = torch.randn(min(chunk, side ** 3 - c * chunk), dtype=torch.float64, device=dev, generator=g)
        flat[a - g0:b - g0] += noise[a - c * chunk:b - c * chunk] * 1e-4
        del noise
    return flat


def cfg4_modes_f64_np(side: int, seed: int = 4, n_modes: int = 64) -> np.ndarray:
    """numpy form of cfg4_modes_f64 for small sides (the golden fixtures in
    tests/golden were generated with it): direct cos of the summed phase,
    numpy N(0, 1e-4) noise."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal(n_modes)
    K = rng.integers(-8, 9, size=(n_modes, 3))
    phi = rng.uniform(0, 2 * np.pi, n_modes)
    r = np.arange(side, dtype=np.float64) * (2 * np.pi / side)
    out = np.empty((side, side, side), np.float64)
    for z in range(side):
        plane = np.zeros((side, side), np.float64)
        for m in range(n_modes):
            plane += A[m] * np.cos(K[m, 0] * r[None, :] + K[m, 1] * r[:, None]
                                   + K[m, 2] * r[z] + phi[m])
        out[z] = plane
    out += rng.normal(0.0, 1e-4, out.shape)
    return out.reshape(-1)


def cfg5_ar1(n: int, dtype: str = "i32", seed: int = 5, rho: float = 0.95) -> np.ndarray:
    """AR(1) rho=0.95 driven by N(0,1); int32 variant scaled by 1e6 and rint
    (the scale is not given by BASELINE.json: recorded choice), float32 as is."""
    from scipy.signal import lfilter
    rng = np.random.default_rng(seed)
    x = lfilter([1.0], [1.0, -rho], rng.standard_normal(n))
    if dtype == "i32":
        return np.clip(np.rint(x * 1e6), -2 ** 31, 2 ** 31 - 1).astype(np.int32)
    return x.astype(np.float32)


def cfg5_ar1_device(n: int, dtype: str = "i32", seed: int = 5, rho: float = 0.95, device=None):
    """cfg5 AR(1) generated on the GPU for the multi-GiB sweep points
    (host generation of 2^32 samples takes minutes): N(0,1) drive from a
    seeded torch generator; the recurrence x[t] = rho x[t-1] + e[t] is
    evaluated in rows of 64 samples as rho^t * cumsum(e * rho^-t) (f64), and
    the carry into a row is the truncated series sum_{k=1..12} rho^(64(k-1))
    * (last value of row r-k) -- the dropped terms are below rho^768 ~ 1e-17
    relative.  Same process as cfg5_ar1, different rounding and drive."""
    import torch
    if device is None:
        device = "cuda" if torch.cuda.is_available() else "cpu"
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    out_dt = torch.int32 if dtype == "i32" else torch.float32
    out = torch.empty(n, dtype=out_dt, device=dev)
    L, K = 64, 12
    t = torch.arange(L, dtype=torch.float64, device=dev)
    up, down = rho ** (-t), rho ** (t + 1)
    chunk = 1 << 26                       # samples per pass (multiple of L)
    prev_last = torch.zeros(K, dtype=torch.float64, device=dev)   # history rows (see below)
    for a in range(0, n, chunk):
        m = min(chunk, n - a)
        rows = (m + L - 1) // L
        e = torch.randn(rows * L, dtype=torch.float64, device=dev, generator=g).view(rows, L)
        loc = torch.cumsum(e * up, dim=1) * (rho ** t)     # each row's recurrence from 0
        last = torch.cat([prev_last, loc[:, -1]])            # local last values, K rows of history first
        c = torch.zeros(rows, dtype=torch.float64, device=dev)
        for k in range(1, K + 1):
            c += (rho ** (L * (k - 1))) * last[K - k:K - k + rows]
        x = loc + c[:, None] * down
        # the next pass sees the history as K-1 zero rows and one row whose
        # local last value is this pass's true last value (it carries the rest)
        prev_last = torch.zeros(K, dtype=torch.float64, device=dev)
        prev_last[-1] = x[-1, -1]
        x = x.reshape(-1)[:m]
        if dtype == "i32":
            out[a:a + m] = torch.clamp(torch.round(x * 1e6), -2 ** 31, 2 ** 31 - 1).to(torch.int32)
        else:
            out[a:a + m] = x.to(torch.float32)
    return out
