"""The reference's lower-level block API on the GPU.

Mirrors pkg/src/apax/codec.py:66-255 (``CodecState``, ``RateLoopState``,
``quantize_block``, ``dequantize_block``, ``encode_block``,
``rate_loop_update``, ``quality_loop_update``), pkg/src/apax/dtypes.py:183-205
(``AttenuatorState``) and pkg/src/apax/transform.py:31-64
(``DerivativeHistory``, ``StreamCosts``) with the same names, fields and
semantics, so the reference's block-level tests and demos
(pkg/tests/test_codec.py:47-119, pkg/demos/adaptive_loops.py) run against
this package.  Every sample-level operation runs on the device
(apax_quantize_block / apax_dequantize_block / apax_encode_block in
include/apax_b200.h); the scalar loop updates are host arithmetic, exactly
the reference's.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np

from . import _lib
from .codec import _check_status, _require_cuda, _stream_ptr
from .dtypes import BlockHeader, Dtype, Mode, StreamConfig, encode_scale_code
from .errors import raise_status

RATE_LOOP_GAIN_DB = 0.75     # codec.py:58
QUALITY_LOOP_GAIN = 0.5      # codec.py:59
MAX_STEP_DB = 6.0            # codec.py:60
SCALE_MIN = 2.0 ** -31       # dtypes.py:104

SELECTOR_D0, SELECTOR_D1, SELECTOR_D2 = 0, 1, 2


@dataclass(frozen=True)
class AttenuatorState:
    """Attenuation as a multiplier and its dB equivalent (dtypes.py:183-205)."""

    att_db: float
    a_min: float = SCALE_MIN
    a_max: float = 1.0
    loop_gain: float = 0.75

    @property
    def a(self) -> float:
        return min(max(10.0 ** (self.att_db / 20.0), self.a_min), self.a_max)

    def clamped(self, att_db: float) -> "AttenuatorState":
        lo = 20.0 * math.log10(self.a_min)
        hi = 20.0 * math.log10(self.a_max)
        return AttenuatorState(min(max(att_db, lo), hi), self.a_min, self.a_max, self.loop_gain)


@dataclass
class DerivativeHistory:
    """Trailing two quantized samples of the stream (transform.py:31-49)."""

    prev1: int = 0
    prev2: int = 0

    def reset(self) -> None:
        self.prev1 = 0
        self.prev2 = 0

    def advance(self, q: np.ndarray) -> None:
        n = q.size
        if n >= 2:
            self.prev2 = int(q[-2])
        elif n == 1:
            self.prev2 = self.prev1
        if n >= 1:
            self.prev1 = int(q[-1])


@dataclass(frozen=True)
class StreamCosts:
    """Estimated payload bits per candidate stream (transform.py:52-64)."""

    bits_d0: int
    bits_d1: int
    bits_d2: int

    def argmin(self) -> int:
        costs = (self.bits_d0, self.bits_d1, self.bits_d2)
        best = SELECTOR_D0
        for sel in (SELECTOR_D1, SELECTOR_D2):
            if costs[sel] < costs[best]:
                best = sel
        return best


@dataclass
class RateLoopState:
    target_bps: float
    accumulated_error: float = 0.0
    step_db: float = RATE_LOOP_GAIN_DB


@dataclass
class CodecState:
    """Mutable per-stream encoder state (codec.py:73-82)."""

    config: StreamConfig
    attenuator: AttenuatorState = field(default_factory=lambda: AttenuatorState(0.0))
    history: DerivativeHistory = field(default_factory=DerivativeHistory)
    prev_costs: Optional[StreamCosts] = None
    blocks_emitted: int = 0
    _initialized: bool = False


class _BlockState(ctypes.Structure):   # apax_block_state (include/apax_b200.h)
    _fields_ = [("att_db", ctypes.c_double), ("prev1", ctypes.c_int64), ("prev2", ctypes.c_int64),
                ("costs", ctypes.c_int64 * 3), ("has_costs", ctypes.c_int32), ("initialized", ctypes.c_int32),
                ("blocks_emitted", ctypes.c_int64)]


def _clamp_step(delta_db: float) -> float:
    return max(-MAX_STEP_DB, min(MAX_STEP_DB, delta_db))


def rate_loop_update(att: AttenuatorState, loop: RateLoopState, actual_bits: int,
                     block_size: int) -> AttenuatorState:
    """FIXED_RATE integrator (codec.py:171-176)."""
    error = actual_bits / block_size - loop.target_bps
    loop.accumulated_error += error
    return att.clamped(att.att_db - _clamp_step(loop.step_db * error))


def quality_loop_update(att: AttenuatorState, measured_srr_db: float,
                        target_srr_db: float) -> AttenuatorState:
    """FIXED_QUALITY integrator (codec.py:179-189)."""
    if not math.isfinite(measured_srr_db):
        return att
    delta = _clamp_step(QUALITY_LOOP_GAIN * (measured_srr_db - target_srr_db))
    return att.clamped(att.att_db - delta)


def _widen(x, dtype: Dtype) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64 if dtype.is_float else np.int64).reshape(-1))


def quantize_block(x, a: float, dtype: Dtype) -> Tuple[np.ndarray, int, Optional[int]]:
    """Quantize one block (codec.py:94-132) on the device; returns (q,
    scale_code, float_block_exp) with float_block_exp None for integers."""
    torch, L = _require_cuda()
    if not dtype.is_float:
        encode_scale_code(a)   # RangeError with the reference's message
    xw = _widen(x, dtype)
    n = xw.size
    xd = torch.from_numpy(xw).cuda() if n else torch.empty(1, dtype=torch.float64, device="cuda")
    q = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    hdr = torch.empty(2, dtype=torch.int32, device="cuda")
    status = torch.empty(4, dtype=torch.int64, device="cuda")
    raise_status(L.apax_quantize_block(ctypes.c_void_p(xd.data_ptr()), n, dtype.wire_code, float(a),
                                       ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(hdr.data_ptr()),
                                       ctypes.c_void_p(status.data_ptr()), ctypes.c_void_p(_stream_ptr(None))))
    torch.cuda.current_stream().synchronize()
    _check_status(status.cpu().numpy().view(np.uint64))
    h = hdr.cpu().numpy()
    return q[:n].cpu().numpy(), int(h[0]), (int(h[1]) if dtype.is_float else None)


def dequantize_block(q, header: BlockHeader, dtype: Dtype) -> np.ndarray:
    """Decoder dual of quantize_block (codec.py:135-146) on the device."""
    torch, L = _require_cuda()
    from .codec import torch_dtype
    qa = np.ascontiguousarray(np.asarray(q, dtype=np.int64).reshape(-1))
    n = qa.size
    if n == 0:
        return np.empty(0, dtype=dtype.np_dtype)
    qd = torch.from_numpy(qa).cuda()
    y = torch.empty(n, dtype=torch_dtype(dtype), device="cuda")
    fbe = header.float_block_exp or 0
    raise_status(L.apax_dequantize_block(ctypes.c_void_p(qd.data_ptr()), n, dtype.wire_code, int(header.scale_code),
                                         int(fbe), ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(_stream_ptr(None))))
    return y.cpu().numpy()


def encode_block(x, state: CodecState, rate_loop: Optional[RateLoopState] = None) -> Tuple[BlockHeader, bytes]:
    """Encode one block (codec.py:192-255) on the device, updating history,
    costs and the adaptive loop of `state` (and `rate_loop`) exactly as the
    reference does.  Blocks up to the configured block size."""
    torch, L = _require_cuda()
    cfg = state.config
    xw = _widen(x, cfg.dtype)
    n = xw.size
    if n < 1 or n > cfg.block_size:
        from .errors import InvalidConfig
        raise InvalidConfig(f"encode_block takes 1..{cfg.block_size} samples, got {n}")
    pc = state.prev_costs
    st = _BlockState(state.attenuator.att_db, state.history.prev1, state.history.prev2,
                     (ctypes.c_int64 * 3)(*((pc.bits_d0, pc.bits_d1, pc.bits_d2) if pc else (0, 0, 0))),
                     1 if pc else 0, 1 if state._initialized else 0, state.blocks_emitted)
    dst = torch.from_numpy(np.frombuffer(bytes(st), np.uint8).copy()).cuda()
    dt, bs, mode = cfg.dtype.wire_code, cfg.block_size, cfg.mode.value
    in_kind = 2 if cfg.dtype.is_float else 1
    cap = int(L.apax_max_encoded_bytes_cast(bs, in_kind, dt, bs))
    wsb = int(L.apax_encode_cast_workspace_bytes(bs, in_kind, dt, mode, bs, 0))
    xd = torch.from_numpy(xw).cuda()
    out = torch.empty(cap + 64, dtype=torch.uint8, device="cuda")
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    status = torch.empty(4, dtype=torch.int64, device="cuda")
    raise_status(L.apax_encode_block(ctypes.c_void_p(xd.data_ptr()), n, dt, mode, float(cfg.target), bs,
                                     ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(out.data_ptr()), cap,
                                     ctypes.c_void_p(status.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                     ctypes.c_void_p(_stream_ptr(None))))
    torch.cuda.current_stream().synchronize()
    s = status.cpu().numpy().view(np.uint64)
    _check_status(s)
    blob = bytes(out[:int(s[2])].cpu().numpy().tobytes())[28:]
    new = _BlockState.from_buffer_copy(bytes(dst.cpu().numpy().tobytes()))
    hs = BlockHeader.size_for(cfg.dtype)
    header = BlockHeader.parse(blob[:hs], cfg.dtype)
    if cfg.mode is Mode.FIXED_RATE and rate_loop is not None and state.blocks_emitted > 0:
        rate_loop.accumulated_error += len(blob) * 8 / cfg.block_size - rate_loop.target_bps
    att = new.att_db
    if cfg.mode is Mode.FIXED_RATE and rate_loop is None:
        att = state.attenuator.att_db   # no rate loop: the gain stays (codec.py:227)
    state.attenuator = AttenuatorState(att, state.attenuator.a_min, state.attenuator.a_max,
                                       state.attenuator.loop_gain)
    state.history = DerivativeHistory(int(new.prev1), int(new.prev2))
    state.prev_costs = StreamCosts(int(new.costs[0]), int(new.costs[1]), int(new.costs[2]))
    state.blocks_emitted = int(new.blocks_emitted)
    state._initialized = bool(new.initialized)
    return header, blob[hs:]
