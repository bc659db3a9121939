"""Generate the committed parity fixtures from the LIVE reference package.

Run in the build container (where the reference is importable):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

The reference lives at $APAX_REF (default /root/reference/pkg/src).  It does
not exist on the GPU box, so everything the GPU tests need is frozen here:

* entropy_vectors_ref.json -- the reference's own golden entropy vectors
  (pkg/tests/golden/entropy_vectors.json), re-checked against the live
  reference and copied as data.
* containers/<name>.npz    -- (input, config, reference container, reference
  decode, reference block offsets) for whole-stream encodes (reference
  encode_stream), cold segmented containers (encode_stream per segment, as in
  SURVEY.md App. C E1), warm_self segments (reference CodecState/encode_block
  stepping, App. C E8) and corrupted containers with the exception the
  reference raises.
* pairwise.npz             -- np.mean / np.sum results for the pairwise-sum
  emulation (numpy 2.3.5 in this container).

Inputs come from paper_1303_4994_b200.workloads (seeded) plus small
hand-made edge cases; nothing is taken from any benchmark suite.
"""
from __future__ import annotations

import json
import os
import pathlib
import struct
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF = os.environ.get("APAX_REF", "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)
sys.path.insert(0, str(REPO))

import apax  # noqa: E402  (the reference)
from apax import codec as rcodec  # noqa: E402
from apax import dtypes as rdtypes  # noqa: E402
from apax import entropy as rentropy  # noqa: E402
from apax import errors as rerrors  # noqa: E402
from apax import transform as rtransform  # noqa: E402
from apax.dtypes import Dtype, Mode, StreamConfig  # noqa: E402

from paper_1303_4994_b200 import workloads as W  # noqa: E402

OUT = HERE / "containers"
DT = {"i8": Dtype.I8, "i16": Dtype.I16, "i32": Dtype.I32, "f32": Dtype.F32, "f64": Dtype.F64}


def block_walk(blob: bytes) -> np.ndarray:
    """Reference block walk (codec.py:310-328) recording offsets."""
    cfg, count = rcodec.parse_file_header(blob)
    hs = rdtypes.BlockHeader.size_for(cfg.dtype)
    pos, rem, offs = rcodec.FILE_HEADER_SIZE, count, []
    view = memoryview(blob)
    while rem > 0:
        n = min(cfg.block_size, rem)
        offs.append(pos)
        _, used = rentropy.unpack_block_counted(view[pos + hs:], (n + 3) // 4)
        pos += hs + used
        rem -= n
    offs.append(pos)
    return np.asarray(offs, np.int64)


def segmented_cold(x, cfg: StreamConfig, P: int) -> bytes:
    """header(full count) + per-segment encode_stream."""
    bs = cfg.block_size
    parts = [struct.pack(rcodec.FILE_HEADER_FMT, rcodec.MAGIC, rcodec.VERSION,
                         cfg.dtype.wire_code, cfg.mode.value, 0, bs, x.size,
                         float(cfg.target))]
    step = P * bs
    for s in range(0, x.size, step):
        parts.append(rcodec.encode_stream(x[s:s + step], cfg)[rcodec.FILE_HEADER_SIZE:])
    return b"".join(parts)


def segmented_warm_self(x, cfg: StreamConfig, P: int) -> bytes:
    """SURVEY.md App. C E8 warm_self, built from the reference's own
    CodecState / AttenuatorState / StreamCosts / encode_block."""
    assert cfg.mode is Mode.FIXED_RATE
    bs = cfg.block_size
    xs = x.astype(np.float64) if cfg.dtype.is_float else x.astype(np.int64)
    hs = rdtypes.BlockHeader.size_for(cfg.dtype)
    parts = [struct.pack(rcodec.FILE_HEADER_FMT, rcodec.MAGIC, rcodec.VERSION,
                         cfg.dtype.wire_code, cfg.mode.value, 0, bs, x.size,
                         float(cfg.target))]

    def costs_at(block, a):
        q, _, _ = rcodec.quantize_block(block, a, cfg.dtype)
        pad = (-q.size) % 4
        if pad:
            q = np.concatenate([q, np.zeros(pad, np.int64)])
        streams = rtransform.derive_streams(q, rtransform.DerivativeHistory())
        return rtransform.StreamCosts(*(rtransform.cost_from_exponents(
            rentropy.group_exponents(s)) for s in streams))

    step = P * bs
    for s in range(0, x.size, step):
        seg = xs[s:s + step]
        b0 = seg[:bs]
        c = costs_at(b0, 1.0)
        bps0 = (min(c.bits_d0, c.bits_d1, c.bits_d2) + hs * 8) / bs
        att0 = rdtypes.AttenuatorState(0.0).clamped(0.0 - 6.02 * (bps0 - cfg.target))
        st = rcodec.CodecState(cfg)
        st.attenuator = att0
        st.prev_costs = costs_at(b0, att0.a)
        loop = rcodec.RateLoopState(cfg.target)
        for b in range(0, seg.size, bs):
            h, payload = rcodec.encode_block(seg[b:b + bs], st, loop)
            parts.append(h.serialize(cfg.dtype))
            parts.append(payload)
    return b"".join(parts)


def save_case(name, x, dtype, mode, target, bs, blob, kind="whole", segment_blocks=0,
              policy=0):
    y = rcodec.decode_stream(blob)
    offs = block_walk(blob)
    meta = dict(name=name, dtype=dtype, mode=int(getattr(mode, "value", mode)), target=float(target),
                block_size=bs, kind=kind, segment_blocks=segment_blocks, policy=policy,
                target_hex=float(target).hex())
    np.savez_compressed(OUT / f"{name}.npz", x=np.asarray(x), blob=np.frombuffer(blob, np.uint8),
                        y=y, offsets=offs, meta=np.frombuffer(json.dumps(meta).encode(), np.uint8))
    return meta


def error_case(name, blob: bytes):
    try:
        y = rcodec.decode_stream(blob)
    except Exception as exc:  # noqa: BLE001
        return dict(name=name, blob_hex=blob.hex(), exc=type(exc).__name__, msg=str(exc))
    return dict(name=name, blob_hex=blob.hex(), exc=None, msg="", y_hex=y.tobytes().hex(),
                y_dtype=str(y.dtype))


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(20261020)
    manifest = []

    # ---- reference golden entropy vectors (data copy, verified live) ----
    ref_vec = json.loads((pathlib.Path(REF).parent / "tests" / "golden" /
                          "entropy_vectors.json").read_text())
    for vec in ref_vec:
        v = np.asarray(vec["samples"], np.int64)
        e = rentropy.group_exponents(v)
        assert e.tolist() == vec["exponents"]
        assert rentropy.pack_block(v, e).hex() == vec["payload_hex"]
    (HERE / "entropy_vectors_ref.json").write_text(json.dumps(ref_vec, indent=1))

    # ---- extra entropy vectors from the live reference ----
    extra = []
    for k in range(40):
        g = int(rng.integers(1, 64))
        w = int(rng.integers(0, 35))
        hi = 1 << max(w - 1, 0)
        v = rng.integers(-hi, hi, size=4 * g) if w else np.zeros(4 * g, np.int64)
        if k % 5 == 0:
            v[rng.integers(0, 4 * g, size=max(1, g // 2))] = 0
        e = rentropy.group_exponents(v)
        extra.append(dict(samples=v.tolist(), exponents=e.tolist(),
                          nibbles=rentropy.jee_encode(e.tolist()),
                          payload_hex=rentropy.pack_block(v, e).hex()))
    # JEE decode error statuses on crafted nibble streams
    jee_err = []
    for nibs, ng in ([15, 0], 1), ([15, 0, 8], 2), ([15, 0, 8, 14], 2), ([15, 2, 3], 1), \
                    ([4, 4], 3), ([15, 0, 8, 4], 2), ([15, 0, 1, 12, 12, 12], 4), \
                    ([15, 0, 34, 13], 2), ([15, 0, 14], 1), ([15, 0, 8, 0, 0], 5):
        try:
            out, used = rentropy._jee_decode_counted(nibs, ng)
            jee_err.append(dict(nibbles=nibs, n_groups=ng, exc=None, exps=out.tolist(),
                                used=used))
        except Exception as exc:  # noqa: BLE001
            jee_err.append(dict(nibbles=nibs, n_groups=ng, exc=type(exc).__name__,
                                msg=str(exc)))
    (HERE / "entropy_vectors_extra.json").write_text(
        json.dumps(dict(vectors=extra, jee_decode=jee_err), indent=0))

    # ---- pairwise summation pins (np.mean / np.sum on float64) ----
    sizes = [1, 2, 3, 7, 8, 9, 15, 16, 17, 63, 64, 65, 127, 128, 129, 130, 255, 256, 257,
             1000, 1023, 1024, 1025, 2047, 2048, 2049, 4095, 4096, 4097, 8191, 8192, 8193,
             12345, 16383, 16384, 16385]
    vals, sums, means = [], [], []
    for n in sizes:
        a = rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 6, n)
        vals.append(a)
        sums.append(float(np.sum(a)))
        means.append(float(np.mean(a)))
    np.savez_compressed(HERE / "pairwise.npz", sizes=np.asarray(sizes),
                        values=np.concatenate(vals), sums=np.asarray(sums),
                        means=np.asarray(means))

    # ---- whole-stream containers (reference encode_stream) ----
    x1 = W.cfg1_sines_i16(1 << 16)
    x2 = W.cfg2_ar2_f32(1 << 16)
    x3 = W.cfg3_grf_f32(256)
    x4 = W.cfg4_modes_f64_np(24)
    x5i = W.cfg5_ar1(1 << 15, "i32")
    x5f = W.cfg5_ar1(1 << 15, "f32")
    whole = [
        ("cfg1_i16_fr4", x1, "i16", Mode.FIXED_RATE, 4.0, 4096),
        ("cfg1_i16_lossless", x1, "i16", Mode.LOSSLESS, 0.0, 4096),
        ("cfg2_f32_fq", x2, "f32", Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, 4096),
        ("cfg3_f32_fr5333", x3, "f32", Mode.FIXED_RATE, 32 / 6, 4096),
        ("cfg4_f64_fr2133", x4, "f64", Mode.FIXED_RATE, 64 / 3, 4096),
        ("cfg5_i32_fr32", x5i, "i32", Mode.FIXED_RATE, 3.2, 4096),
        ("cfg5_f32_fr16", x5f, "f32", Mode.FIXED_RATE, 16.0, 4096),
        ("cfg5_i32_lossless_bs512", x5i[:30001], "i32", Mode.LOSSLESS, 0.0, 512),
        ("i16_fq60_bs1024", x1[:50000], "i16", Mode.FIXED_QUALITY, 60.0, 1024),
        ("i32_fq40_bs2048", x5i[:40000], "i32", Mode.FIXED_QUALITY, 40.0, 2048),
        ("f64_fq90", x4[:20000], "f64", Mode.FIXED_QUALITY, 90.0, 4096),
        ("f32_fq60_bs2048_sine", (np.sin(np.arange(20000) * 0.01) * 3).astype(np.float32),
         "f32", Mode.FIXED_QUALITY, 60.0, 2048),
        ("i8_lossless_bs64", rng.integers(-128, 128, 1001).astype(np.int8), "i8",
         Mode.LOSSLESS, 0.0, 64),
        ("i8_fr3_bs64", rng.integers(-128, 128, 1001).astype(np.int8), "i8",
         Mode.FIXED_RATE, 3.0, 64),
        ("i16_white_lossless_bs256", rng.integers(-32768, 32768, 10000).astype(np.int16),
         "i16", Mode.LOSSLESS, 0.0, 256),
        ("i32_white_lossless_bs1000", rng.integers(-2 ** 31, 2 ** 31, 7777).astype(np.int32),
         "i32", Mode.LOSSLESS, 0.0, 1000),
        ("i16_alternating_lossless", np.tile(np.array([32767, -32768], np.int16), 3000),
         "i16", Mode.LOSSLESS, 0.0, 4096),
        ("i16_alternating_fr2", np.tile(np.array([30000, -30000, 100, -100], np.int16), 3000),
         "i16", Mode.FIXED_RATE, 2.0, 1024),
        ("i16_partial_fr4", x1[:4096 + 37], "i16", Mode.FIXED_RATE, 4.0, 4096),
        ("i8_single", np.array([-42], np.int8), "i8", Mode.LOSSLESS, 0.0, 4096),
        ("i16_zeros_fr4", np.zeros(5000, np.int16), "i16", Mode.FIXED_RATE, 4.0, 1024),
        ("f32_zeros_fq", np.zeros(5000, np.float32), "f32", Mode.FIXED_QUALITY, 50.0, 1024),
        ("i16_constant_lossless", np.full(4096 * 4, 12345, np.int16), "i16", Mode.LOSSLESS,
         0.0, 4096),
        ("f32_tiny_fr8", (rng.standard_normal(9000) * 1e-38).astype(np.float32), "f32",
         Mode.FIXED_RATE, 8.0, 1024),
        ("f32_huge_fq", (rng.standard_normal(9000) * 1e37).astype(np.float32), "f32",
         Mode.FIXED_QUALITY, 70.0, 2048),
        ("f64_mixed_scale_fr12", rng.standard_normal(12000) * 10.0 ** rng.integers(-40, 40, 12000),
         "f64", Mode.FIXED_RATE, 12.0, 4096),
        ("f32_bs100_fq50", x2[:20000], "f32", Mode.FIXED_QUALITY, 50.0, 100),
        ("f32_bs16384_fr6", x2[:70000], "f32", Mode.FIXED_RATE, 6.0, 16384),
        ("i16_bs8192_lossless", x1[:50000], "i16", Mode.LOSSLESS, 0.0, 8192),
        ("i32_bs12000_fq70", x5i[:50000], "i32", Mode.FIXED_QUALITY, 70.0, 12000),
    ]
    for name, x, dt, mode, T, bs in whole:
        cfg = StreamConfig(DT[dt], bs, mode, T)
        blob = rcodec.encode_stream(x, cfg)
        manifest.append(save_case(name, x, dt, mode, T, bs, blob))

    # ---- cold segmented containers (App. C E1) ----
    seg = [
        ("seg_cfg1_fr4_P4", x1, "i16", Mode.FIXED_RATE, 4.0, 4096, 4),
        ("seg_cfg2_fq_P8", x2, "f32", Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, 4096, 8),
        ("seg_cfg2_fq_P1", x2[:40000], "f32", Mode.FIXED_QUALITY, W.CFG2_TARGET_DB, 4096, 1),
        ("seg_cfg5_i32_fr32_P3", x5i, "i32", Mode.FIXED_RATE, 3.2, 4096, 3),
        ("seg_lossless_i16_P2", x1[:40000], "i16", Mode.LOSSLESS, 0.0, 4096, 2),
        ("seg_f64_fr_P5_bs1024", x4[:30000], "f64", Mode.FIXED_RATE, 21.0, 1024, 5),
    ]
    for name, x, dt, mode, T, bs, P in seg:
        cfg = StreamConfig(DT[dt], bs, mode, T)
        blob = segmented_cold(x, cfg, P)
        manifest.append(save_case(name, x, dt, mode, T, bs, blob, "cold", P, 0))

    # ---- warm_self segments (App. C E8) ----
    warm = [
        ("warm_cfg1_fr4_P4", x1, "i16", 4.0, 4096, 4),
        ("warm_cfg3_fr5333_P4", x3, "f32", 32 / 6, 4096, 4),
        ("warm_cfg5_i32_fr32_P2", x5i, "i32", 3.2, 4096, 2),
    ]
    for name, x, dt, T, bs, P in warm:
        cfg = StreamConfig(DT[dt], bs, Mode.FIXED_RATE, T)
        blob = segmented_warm_self(x, cfg, P)
        manifest.append(save_case(name, x, dt, Mode.FIXED_RATE, T, bs, blob, "warm_self", P, 1))

    # ---- decode error cases (reference exception class + message) ----
    base = rcodec.encode_stream(np.arange(1000, dtype=np.int16), StreamConfig(Dtype.I16, 256))
    f32b = rcodec.encode_stream(x2[:3000], StreamConfig(Dtype.F32, 1024, Mode.FIXED_QUALITY, 50.0))
    errs = []
    errs.append(error_case("truncated_tail", base[:-3]))
    errs.append(error_case("truncated_file_header", base[:10]))
    errs.append(error_case("bad_magic", b"NOPE" + bytes(24)))
    b = bytearray(base); b[4] = 9
    errs.append(error_case("bad_version", bytes(b)))
    b = bytearray(base); b[5] = 7
    errs.append(error_case("bad_dtype_wire", bytes(b)))
    b = bytearray(base); b[6] = 5
    errs.append(error_case("bad_mode_wire", bytes(b)))
    b = bytearray(base); b[8:12] = struct.pack("<I", 60)
    errs.append(error_case("bad_block_size", bytes(b)))
    b = bytearray(base); b[8:12] = struct.pack("<I", 66)
    errs.append(error_case("block_size_not_mult4", bytes(b)))
    b = bytearray(f32b); b[6] = 0
    errs.append(error_case("lossless_float_header", bytes(b)))
    b = bytearray(f32b); b[6] = 1; b[20:28] = struct.pack("<d", 0.0)
    errs.append(error_case("fr_zero_target_header", bytes(b)))
    b = bytearray(base); b[28] |= 3
    errs.append(error_case("reserved_selector_block0", bytes(b)))
    offs = block_walk(base)
    b = bytearray(base); b[int(offs[2])] |= 3
    errs.append(error_case("reserved_selector_block2", bytes(b)))
    b = bytearray(base); b[int(offs[1]) + 4] = 0x4E
    errs.append(error_case("jee_no_abs_block1", bytes(b)))
    b = bytearray(base); b[int(offs[1]) + 4] = 0xF2; b[int(offs[1]) + 5] = 0x3F
    errs.append(error_case("jee_range_block1", bytes(b)))
    b = bytearray(base); b[int(offs[3]) + 5] = 0xEE
    errs.append(error_case("jee_reserved_block3", bytes(b)))
    errs.append(error_case("truncated_block_header", base[:int(offs[3]) + 2]))
    errs.append(error_case("truncated_mantissa_block3", base[:int(offs[4]) - 1]))
    errs.append(error_case("truncated_mantissa_f32_last", f32b[:-1]))
    errs.append(error_case("trailing_bytes_ok", base + b"\x01\x02\x03"))
    b = bytearray(base); b[12:20] = struct.pack("<Q", 0)
    errs.append(error_case("zero_count_ok", bytes(b)))
    b = bytearray(f32b); b[12:20] = struct.pack("<Q", 2000)
    errs.append(error_case("shorter_count_ok", bytes(b)))
    (HERE / "decode_errors.json").write_text(json.dumps(dict(
        base_hex=base.hex(), f32_hex=f32b.hex(), cases=errs), indent=1))

    # ---- encode error cases (reference exception class + message) ----
    enc_err = []
    cases = [
        ("nonfinite_index_77", np.where(np.arange(128) == 77, np.nan, 1.0), "f64",
         Mode.FIXED_QUALITY, 60.0, 64),
        ("nonfinite_inf_f32", np.where(np.arange(3000) == 2999, np.inf, 1.0).astype(np.float32),
         "f32", Mode.FIXED_RATE, 8.0, 1024),
        ("f64_huge_internal", rng.standard_normal(300) * 1e250, "f64", Mode.FIXED_RATE, 8.0, 64),
        ("f64_tiny_overflow", rng.standard_normal(300) * 1e-305, "f64", Mode.FIXED_QUALITY,
         60.0, 64),
        ("f64_huge_late_block", np.concatenate([np.ones(256), np.full(64, 1e300)]), "f64",
         Mode.FIXED_RATE, 8.0, 64),
    ]
    for name, x, dt, mode, T, bs in cases:
        try:
            rcodec.encode_stream(x, StreamConfig(DT[dt], bs, mode, T))
            enc_err.append(dict(name=name, exc=None))
        except Exception as exc:  # noqa: BLE001
            enc_err.append(dict(name=name, dtype=dt, mode=int(mode.value), target=T,
                                block_size=bs, x_hex=np.asarray(x, DT[dt].np_dtype).tobytes().hex(),
                                exc=type(exc).__name__, msg=str(exc)))
    (HERE / "encode_errors.json").write_text(json.dumps(enc_err, indent=1))

    (HERE / "manifest.json").write_text(json.dumps(manifest, indent=1))
    total = sum(p.stat().st_size for p in HERE.rglob("*") if p.is_file())
    print(f"wrote {len(manifest)} containers, {len(errs)} error cases, {total/1e6:.2f} MB")


if __name__ == "__main__":
    main()
