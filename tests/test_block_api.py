"""The reference's lower-level block API (pkg/src/apax/codec.py:66-255):
its loop-update KATs (pkg/tests/test_codec.py:91-119, restated) on the host
logic, its quantize KATs (:47-88, restated) and encode_block stepping
against containers the live reference produced, on the device."""
import numpy as np
import pytest

from conftest import GOLDEN, load_container

import paper_1303_4994_b200 as A
from paper_1303_4994_b200 import (AttenuatorState, BlockHeader, CodecState, Dtype, Mode, RateLoopState,
                                  StreamConfig, decode_scale_code)

# ---------------------------------------------------------------------------
# host: the adaptive loops (codec.py:171-189)
# ---------------------------------------------------------------------------


def test_rate_converged_fixpoint():
    att = AttenuatorState(-3.0)
    out = A.rate_loop_update(att, RateLoopState(4.0), actual_bits=4 * 1024, block_size=1024)
    assert out.att_db == att.att_db


def test_rate_error_step():
    out = A.rate_loop_update(AttenuatorState(-3.0), RateLoopState(4.0), 8 * 1024, 1024)
    assert out.att_db == pytest.approx(-3.0 - min(6, 0.75 * 4))


def test_rate_step_slew_limited_and_accumulates():
    loop = RateLoopState(1.0)
    out = A.rate_loop_update(AttenuatorState(-20.0), loop, 32 * 1024, 1024)
    assert out.att_db == pytest.approx(-26.0)
    assert loop.accumulated_error == 31.0


def test_quality_loop():
    assert A.quality_loop_update(AttenuatorState(-10.0), 60.0, 60.0).att_db == -10.0
    assert A.quality_loop_update(AttenuatorState(-10.0), 70.0, 60.0).att_db == pytest.approx(-15.0)
    assert A.quality_loop_update(AttenuatorState(-10.0), 100.0, 60.0).att_db == pytest.approx(-16.0)
    assert A.quality_loop_update(AttenuatorState(-10.0), float("inf"), 60.0).att_db == -10.0


def test_attenuator_clamps():
    lo = AttenuatorState(0.0).clamped(-1e9)
    assert lo.att_db == 20.0 * np.log10(2.0 ** -31) and lo.a == 2.0 ** -31
    assert AttenuatorState(0.0).clamped(5.0).att_db == 0.0 and AttenuatorState(0.0).a == 1.0


def test_derivative_history_and_costs():
    h = A.DerivativeHistory()
    h.advance(np.array([3, 7, 11]))
    assert (h.prev1, h.prev2) == (11, 7)
    h.reset()
    assert (h.prev1, h.prev2) == (0, 0)
    assert A.StreamCosts(30, 20, 20).argmin() == 1 and A.StreamCosts(5, 5, 5).argmin() == 0


# ---------------------------------------------------------------------------
# device: quantize / dequantize KATs and encode_block stepping
# ---------------------------------------------------------------------------
gpu = pytest.mark.gpu


@gpu
def test_quantize_kats():
    x = np.array([-7, 0, 12345, -32768])
    q, code, fbe = A.quantize_block(x, 1.0, Dtype.I16)
    assert q.tolist() == x.tolist() and decode_scale_code(code) == 1.0 and fbe is None
    x = np.array([0.5, -0.25, 0.75, 0.0])
    s = 2.0 ** 10
    q, code, fbe = A.quantize_block(x, s * 0.75 / 2 ** 30, Dtype.F32)
    assert decode_scale_code(code) * 2.0 ** fbe == s and q.tolist() == [512, -256, 768, 0]
    x = np.array([7, 8, 9, 10])
    q, code, _ = A.quantize_block(x, 0.5, Dtype.I16)
    assert q.tolist() == [4, 4, 4, 5]                      # round half to even
    y = A.dequantize_block(q, BlockHeader(0, False, code), Dtype.I16)
    assert y.tolist() == [8, 8, 8, 10]
    rng = np.random.default_rng(7)
    x = rng.uniform(-1000, 1000, size=4096)
    q, code, fbe = A.quantize_block(x, 1.0, Dtype.F64)
    s = decode_scale_code(code) * 2.0 ** fbe
    y = A.dequantize_block(q, BlockHeader(0, False, code, fbe), Dtype.F64)
    assert np.max(np.abs(y - x)) <= 0.5 / s
    for scale in (1e-30, 1.0, 1e30):
        q, _, _ = A.quantize_block(rng.uniform(-scale, scale, size=256), 1.0, Dtype.F64)
        assert np.max(np.abs(q)) < 2 ** 31
    from paper_1303_4994_b200.errors import RangeError, UnsupportedValue
    with pytest.raises(UnsupportedValue, match="non-finite float input"):
        A.quantize_block(np.array([1.0, np.inf]), 1.0, Dtype.F32)
    with pytest.raises(RangeError):
        A.quantize_block(np.array([1, 2]), 0.0, Dtype.I16)


@gpu
@pytest.mark.parametrize("name", ["cfg1_i16_fr4", "cfg2_f32_fq", "f64_fq90", "i16_partial_fr4", "i32_fq40_bs2048",
                                  "cfg5_i32_lossless_bs512", "f32_tiny_fr8", "i16_alternating_fr2"])
def test_encode_block_stepping_reproduces_reference_container(name):
    """Stepping encode_block with one CodecState / RateLoopState over the
    blocks (as the reference's encode_stream does, codec.py:274-285)
    rebuilds the reference's container byte for byte."""
    c = load_container(GOLDEN / "containers" / f"{name}.npz")
    m = c["meta"]
    dt = {"i8": Dtype.I8, "i16": Dtype.I16, "i32": Dtype.I32, "f32": Dtype.F32, "f64": Dtype.F64}[m["dtype"]]
    cfg = StreamConfig(dt, m["block_size"], Mode(m["mode"]), float.fromhex(m["target_hex"]))
    st = CodecState(cfg)
    loop = RateLoopState(cfg.target) if cfg.mode is Mode.FIXED_RATE else None
    parts = [c["blob"][:28]]
    x = c["x"]
    for b in range(0, x.size, cfg.block_size):
        h, payload = A.encode_block(x[b:b + cfg.block_size], st, loop)
        parts.append(h.serialize(dt) + payload)
    assert b"".join(parts) == c["blob"], name
    assert st.blocks_emitted == (x.size + cfg.block_size - 1) // cfg.block_size
