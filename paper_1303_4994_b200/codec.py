"""Drop-in encode/decode API over the B200 C-ABI extension.

Reference interface mirrored (pkg/src/apax/codec.py):
  encode_stream(samples, config) -> bytes      codec.py:258-285
  decode_stream(data) -> np.ndarray            codec.py:308-329
  parse_file_header(data) -> (config, count)   codec.py:288-305
plus device-resident entry points for throughput work:
  encode_device / decode_device and the reusable Encoder / Decoder plans,
which keep inputs and outputs in HBM (torch CUDA tensors as buffers).

All arithmetic runs in libapax_b200.so kernels; this module only validates,
allocates device buffers, launches and maps status codes onto the
reference's exception classes.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from . import _lib
from .dtypes import Dtype, Mode, StreamConfig
from .errors import InvalidConfig, raise_status, status_exception

MAGIC = b"APAX"
VERSION = 1
FILE_HEADER_FMT = "<4sBBBBIQd"
FILE_HEADER_SIZE = struct.calcsize(FILE_HEADER_FMT)
_U64_MAX = (1 << 64) - 1
_POLICY = {"cold": 0, "warm_self": 1}


def _torch():
    import torch
    return torch


_TORCH_DT = {}


def torch_dtype(dt: Dtype):
    torch = _torch()
    if not _TORCH_DT:
        _TORCH_DT.update({Dtype.I8: torch.int8, Dtype.I16: torch.int16, Dtype.I32: torch.int32,
                          Dtype.F32: torch.float32, Dtype.F64: torch.float64})
    return _TORCH_DT[dt]


def _require_cuda():
    torch = _torch()
    L = _lib.lib()  # raises ExtensionMissing loudly
    if not torch.cuda.is_available():
        raise _lib.ExtensionMissing("no CUDA device: the B200 codec has no CPU fallback")
    return torch, L


def _stream_ptr(stream) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _check_status(status_host: np.ndarray) -> None:
    """Raise the reference exception for a device status buffer (4 x u64)."""
    nonfinite = int(status_host[0])
    if nonfinite != _U64_MAX:
        raise status_exception(9, nonfinite)
    key = int(status_host[1])
    if key != _U64_MAX:
        code = key & 0xFF
        raise status_exception(code, key >> 8)


# ---------------------------------------------------------------------------
# file header (codec.py:288-305)
# ---------------------------------------------------------------------------
def parse_file_header(data) -> Tuple[StreamConfig, int]:
    """Parse the container file header; returns (config, element_count)."""
    L = _lib.lib()
    buf = np.frombuffer(bytes(memoryview(data)[:FILE_HEADER_SIZE]), np.uint8)
    dt, mode, bs = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    count, target, detail = ctypes.c_int64(), ctypes.c_double(), ctypes.c_int64()
    st = L.apax_parse_file_header(buf.ctypes.data_as(ctypes.c_void_p), len(data),
                                  ctypes.byref(dt), ctypes.byref(mode), ctypes.byref(bs),
                                  ctypes.byref(count), ctypes.byref(target), ctypes.byref(detail))
    raise_status(st, detail.value)
    cfg = StreamConfig(dtype=Dtype.from_wire(dt.value), block_size=bs.value,
                       mode=Mode(mode.value), target=target.value)
    return cfg, int(count.value) & _U64_MAX


def wave_segment_blocks(n: int, dtype: Dtype, mode: Mode, block_size: int) -> int:
    """Segment length giving every resident encoder CTA of the current
    device one segment (apax_encode_wave_segment_blocks)."""
    _, L = _require_cuda()
    v = int(L.apax_encode_wave_segment_blocks(int(n), dtype.wire_code, mode.value, int(block_size)))
    if v < 1:
        raise InvalidConfig("invalid arguments")
    return v


def max_encoded_bytes(n: int, dtype: Dtype, block_size: int) -> int:
    return int(_lib.lib().apax_max_encoded_bytes(int(n), dtype.wire_code, int(block_size)))


# ---------------------------------------------------------------------------
# reusable device plans
# ---------------------------------------------------------------------------
@dataclass
class EncodedStream:
    """A container resident in HBM."""

    blob: "object"            # torch.uint8 CUDA tensor (capacity >= nbytes)
    nbytes: int
    block_offsets: "object"   # torch.int64 CUDA tensor, n_blocks + 1
    config: StreamConfig
    count: int

    def to_bytes(self) -> bytes:
        return bytes(self.blob[:self.nbytes].cpu().numpy().tobytes())


class Encoder:
    """Preallocated encode plan for (n, config) on one CUDA device.

    encode(x) enqueues one kernel launch on the current stream and returns
    immediately; `finish()` synchronises, checks the status buffer and
    returns the container length.
    """

    def __init__(self, n: int, config: StreamConfig, device=None, with_offsets: bool = True,
                 trace: bool = False):
        torch, L = _require_cuda()
        config.validate()
        if n < 1:
            raise InvalidConfig("element_count must be >= 1")
        self.n, self.config = int(n), config
        self.device = torch.device(device or "cuda")
        dt, bs = config.dtype.wire_code, config.block_size
        self.seg = int(config.segment_blocks or 0)
        self.policy = _POLICY[config.segment_policy]
        self.cap = int(L.apax_max_encoded_bytes(self.n, dt, bs))
        wsb = int(L.apax_encode_workspace_bytes(self.n, dt, config.mode.value, bs, self.seg))
        if wsb < 0:
            raise InvalidConfig("invalid encode arguments")
        self.n_blocks = (self.n + bs - 1) // bs
        self.out = torch.empty(self.cap + 64, dtype=torch.uint8, device=self.device)
        self.ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=self.device)
        self.status = torch.empty(4, dtype=torch.int64, device=self.device)
        self.offsets = (torch.empty(self.n_blocks + 1, dtype=torch.int64, device=self.device)
                        if with_offsets else None)
        self.trace = (torch.zeros(self.n_blocks, 10, dtype=torch.float64, device=self.device)
                      if trace else None)
        self._lib = L

    def encode(self, x, stream=None) -> None:
        torch = _torch()
        if x.device.type != "cuda" or x.dtype != torch_dtype(self.config.dtype) or x.numel() != self.n:
            raise InvalidConfig("input must be a CUDA tensor of the config dtype and length n")
        if not x.is_contiguous():
            x = x.contiguous()
        c = self.config
        st = self._lib.apax_encode(
            ctypes.c_void_p(x.data_ptr()), self.n, c.dtype.wire_code, c.mode.value,
            float(c.target), c.block_size, self.seg, self.policy,
            ctypes.c_void_p(self.out.data_ptr()), self.cap,
            ctypes.c_void_p(self.offsets.data_ptr()) if self.offsets is not None else None,
            ctypes.c_void_p(self.status.data_ptr()),
            ctypes.c_void_p(self.trace.data_ptr()) if self.trace is not None else None,
            ctypes.c_void_p(self.ws.data_ptr()), self.ws.numel(),
            ctypes.c_void_p(_stream_ptr(stream)))
        raise_status(st)

    def finish(self, stream=None) -> int:
        torch = _torch()
        (stream or torch.cuda.current_stream()).synchronize()
        s = self.status.cpu().numpy().view(np.uint64)
        _check_status(s)
        return int(s[2])

    def result(self) -> EncodedStream:
        nbytes = self.finish()
        return EncodedStream(self.out, nbytes, self.offsets, self.config, self.n)


class Decoder:
    """Preallocated decode plan for containers of (n, dtype, block_size)."""

    def __init__(self, n: int, dtype: Dtype, block_size: int, device=None, alloc_y: bool = True):
        torch, L = _require_cuda()
        self.n, self.dtype, self.bs = int(n), dtype, int(block_size)
        self.device = torch.device(device or "cuda")
        wsb = int(L.apax_decode_workspace_bytes(self.n, dtype.wire_code, self.bs))
        if wsb < 0:
            raise InvalidConfig("invalid decode arguments")
        self.ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=self.device)
        self.status = torch.empty(4, dtype=torch.int64, device=self.device)
        self.y = torch.empty(max(self.n, 1) if alloc_y else 1, dtype=torch_dtype(dtype), device=self.device)
        self._lib = L

    def decode(self, blob, nbytes: int, offsets=None, stream=None, out=None,
               segment_blocks: Optional[int] = None) -> None:
        """Enqueue a decode.  With the side-band `offsets` and the container's
        `segment_blocks` (the encoder's StreamConfig.segment_blocks), the
        segment-serial decoder runs (apax_decode_segments); otherwise the
        general decoder (apax_decode)."""
        y = self.y if out is None else out
        if y.numel() < self.n:
            raise InvalidConfig("decode output buffer smaller than the element count")
        offs = ctypes.c_void_p(offsets.data_ptr()) if offsets is not None else None
        if segment_blocks and offsets is not None:
            st = self._lib.apax_decode_segments(
                ctypes.c_void_p(blob.data_ptr()), int(nbytes), self.n, self.dtype.wire_code, self.bs,
                offs, int(segment_blocks), ctypes.c_void_p(y.data_ptr()),
                ctypes.c_void_p(self.status.data_ptr()), ctypes.c_void_p(self.ws.data_ptr()),
                self.ws.numel(), ctypes.c_void_p(_stream_ptr(stream)))
        else:
            st = self._lib.apax_decode(
                ctypes.c_void_p(blob.data_ptr()), int(nbytes), self.n, self.dtype.wire_code, self.bs,
                offs, ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(self.status.data_ptr()),
                ctypes.c_void_p(self.ws.data_ptr()), self.ws.numel(),
                ctypes.c_void_p(_stream_ptr(stream)))
        raise_status(st)

    def finish(self, stream=None):
        torch = _torch()
        (stream or torch.cuda.current_stream()).synchronize()
        _check_status(self.status.cpu().numpy().view(np.uint64))
        return self.y[:self.n]


# ---------------------------------------------------------------------------
# one-shot device API
# ---------------------------------------------------------------------------
def encode_device(x, config: StreamConfig, trace: bool = False) -> EncodedStream:
    """Encode a CUDA tensor; the container stays in HBM."""
    enc = Encoder(int(x.numel()), config, device=x.device, trace=trace)
    enc.encode(x.reshape(-1))
    res = enc.result()
    res.trace = enc.trace  # type: ignore[attr-defined]
    return res


def encode_lossless_range(x_ext, halo: int, first_block: int, dtype: Dtype, block_size: int) -> EncodedStream:
    """LOSSLESS whole-stream encode of the blocks from `first_block` on
    (apax_encode_lossless_range).  `x_ext` (CUDA tensor of the dtype) holds
    the `halo` samples before global sample first_block * block_size
    followed by the range's samples.  The result is a container of its own;
    its body (after the 28-byte header) is those blocks' bytes in the
    one-call whole-stream container, and its side-band index is relative to
    its own header."""
    torch, L = _require_cuda()
    x_ext = x_ext.reshape(-1).contiguous()
    if x_ext.dtype != torch_dtype(dtype):
        raise InvalidConfig("input dtype differs from the config dtype")
    n = int(x_ext.numel()) - int(halo)
    bs = int(block_size)
    cfg = StreamConfig(dtype, bs, Mode.LOSSLESS)
    cfg.validate()
    cap = int(L.apax_max_encoded_bytes(n, dtype.wire_code, bs))
    wsb = int(L.apax_encode_workspace_bytes(n, dtype.wire_code, 0, bs, 0))
    if cap < 0 or wsb < 0:
        raise InvalidConfig("invalid encode arguments")
    dev = x_ext.device
    out = torch.empty(cap + 64, dtype=torch.uint8, device=dev)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
    status = torch.empty(4, dtype=torch.int64, device=dev)
    nb = (n + bs - 1) // bs
    offs = torch.empty(nb + 1, dtype=torch.int64, device=dev)
    xp = x_ext.data_ptr() + int(halo) * x_ext.element_size()
    st = L.apax_encode_lossless_range(ctypes.c_void_p(xp), int(halo), n, dtype.wire_code, bs, int(first_block),
                                      ctypes.c_void_p(out.data_ptr()), cap, ctypes.c_void_p(offs.data_ptr()),
                                      ctypes.c_void_p(status.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                      ws.numel(), ctypes.c_void_p(_stream_ptr(None)))
    raise_status(st)
    torch.cuda.current_stream().synchronize()
    s = status.cpu().numpy().view(np.uint64)
    _check_status(s)
    return EncodedStream(out, int(s[2]), offs, cfg, n)


def decode_range(blob, nbytes: int, offsets, count: int, dtype: Dtype, block_size: int, b0: int, b1: int,
                 entry=(0, 0), want_map: bool = False):
    """Decode blocks [b0, b1) of a container held in HBM (apax_decode_range):
    `offsets` is the container's global side-band index (int64 CUDA tensor),
    `entry` the derivative history entering block b0 as two's-complement u64
    (q[-1], q[-2]).  Returns (y of the range, history map or None): the map
    (m11, m12, m21, m22, c1, c2) gives the history leaving block b1-1 as an
    affine function of `entry` (distributed.py composes them across ranks)."""
    torch, L = _require_cuda()
    bs = int(block_size)
    s0, s1 = b0 * bs, min(count, b1 * bs)
    m = s1 - s0
    wsb = int(L.apax_decode_workspace_bytes(m, dtype.wire_code, bs))
    if wsb < 0:
        raise InvalidConfig("invalid decode arguments")
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=blob.device)
    status = torch.empty(4, dtype=torch.int64, device=blob.device)
    y = torch.empty(max(m, 1), dtype=torch_dtype(dtype), device=blob.device)
    mp = torch.zeros(6, dtype=torch.int64, device=blob.device) if want_map else None
    st = L.apax_decode_range(ctypes.c_void_p(blob.data_ptr()), int(nbytes), int(count), dtype.wire_code, bs,
                             ctypes.c_void_p(offsets.data_ptr()), int(b0), int(b1),
                             ctypes.c_uint64(int(entry[0]) & 0xFFFFFFFFFFFFFFFF),
                             ctypes.c_uint64(int(entry[1]) & 0xFFFFFFFFFFFFFFFF),
                             ctypes.c_void_p(y.data_ptr()),
                             ctypes.c_void_p(mp.data_ptr()) if mp is not None else None,
                             ctypes.c_void_p(status.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                             ctypes.c_void_p(_stream_ptr(None)))
    raise_status(st)
    torch.cuda.current_stream().synchronize()
    _check_status(status.cpu().numpy().view(np.uint64))
    mv = [int(v) & 0xFFFFFFFFFFFFFFFF for v in mp.cpu().tolist()] if mp is not None else None
    return y[:m], mv


def _decodable_count(count: int, nbytes: int, cfg: StreamConfig) -> int:
    """Samples worth decoding: every block costs >= header + 2 bytes, so a
    count beyond what `nbytes` can hold is guaranteed to fail (truncated)
    within the first `limit + 1` blocks -- the same block the reference's
    serial walk stops at.  Caps the output allocation for crafted headers."""
    hs = 6 if cfg.dtype.is_float else 4
    limit_blocks = max(nbytes - FILE_HEADER_SIZE, 0) // (hs + 2) + 1
    return min(count, limit_blocks * cfg.block_size)


def decode_device(blob, nbytes: Optional[int] = None, offsets=None,
                  segment_blocks: Optional[int] = None):
    """Decode a container held in a CUDA uint8 tensor; returns a CUDA tensor.
    `segment_blocks` (with `offsets`) selects the segment-serial decoder."""
    torch = _torch()
    nbytes = int(blob.numel() if nbytes is None else nbytes)
    head = bytes(blob[:min(nbytes, FILE_HEADER_SIZE)].cpu().numpy().tobytes())
    if len(head) < FILE_HEADER_SIZE:
        raise_status(13)
    cfg, count = parse_file_header(head)
    if count == 0:
        return torch.empty(0, dtype=torch_dtype(cfg.dtype), device=blob.device)
    n = _decodable_count(count, nbytes, cfg)
    dec = Decoder(n, cfg.dtype, cfg.block_size, device=blob.device)
    ok = n == count
    # without offsets apax_decode discovers the blocks on the device (K5) and
    # decodes a segmented container (restart flags every P blocks) segment-
    # serially, anything else (whole stream, corruption) in two passes, with
    # no host round trip
    dec.decode(blob, nbytes, offsets if ok else None, segment_blocks=segment_blocks if ok else None)
    return dec.finish()


# ---------------------------------------------------------------------------
# drop-in host API (bytes / ndarray)
# ---------------------------------------------------------------------------
_IN_NATIVE, _IN_INT64, _IN_FLOAT64 = 0, 1, 2


def _reference_cast(x: np.ndarray, dt: Dtype):
    """The reference's input conversion (codec.py:266-272): float configs
    widen to float64 (non-finite values raise UnsupportedValue with the first
    index), integer configs to int64 (numpy astype: floats truncate toward
    zero).  Returns (array, in_kind): the container dtype itself whenever
    that holds the widened values exactly -- quantizing them from the
    narrower array gives the same bytes -- else the widened array, coded by
    apax_encode_cast."""
    if x.dtype == dt.np_dtype:
        return np.ascontiguousarray(x), _IN_NATIVE
    if dt.is_float:
        xf = np.ascontiguousarray(x.astype(np.float64))
        if dt is Dtype.F64:
            return xf, _IN_NATIVE
        with np.errstate(over="ignore", invalid="ignore"):   # values beyond f32: not representable, no warning
            x32 = xf.astype(np.float32)
        if np.array_equal(x32.astype(np.float64), xf, equal_nan=True):
            return x32, _IN_NATIVE
        return xf, _IN_FLOAT64
    xi = np.ascontiguousarray(x.astype(np.int64))
    info = np.iinfo(dt.np_dtype)
    if xi.size == 0 or (int(xi.min()) >= info.min and int(xi.max()) <= info.max):
        return xi.astype(dt.np_dtype), _IN_NATIVE
    return xi, _IN_INT64


def _encode_cast(xw: np.ndarray, in_kind: int, config: StreamConfig) -> bytes:
    """apax_encode_cast of a widened host array (int64 / float64)."""
    torch, L = _require_cuda()
    n = int(xw.size)
    dt, bs = config.dtype.wire_code, config.block_size
    seg = int(config.segment_blocks or 0)
    cap = int(L.apax_max_encoded_bytes_cast(n, in_kind, dt, bs))
    wsb = int(L.apax_encode_cast_workspace_bytes(n, in_kind, dt, config.mode.value, bs, seg))
    if cap < 0 or wsb < 0:
        raise InvalidConfig("invalid encode arguments")
    xd = torch.from_numpy(xw).to("cuda")
    out = torch.empty(cap + 64, dtype=torch.uint8, device="cuda")
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    status = torch.empty(4, dtype=torch.int64, device="cuda")
    st = L.apax_encode_cast(ctypes.c_void_p(xd.data_ptr()), in_kind, n, dt, config.mode.value,
                            float(config.target), bs, seg, _POLICY[config.segment_policy],
                            ctypes.c_void_p(out.data_ptr()), cap, None, ctypes.c_void_p(status.data_ptr()),
                            ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.c_void_p(_stream_ptr(None)))
    raise_status(st)
    torch.cuda.current_stream().synchronize()
    s = status.cpu().numpy().view(np.uint64)
    _check_status(s)
    return bytes(out[:int(s[2])].cpu().numpy().tobytes())


def encode_stream(samples, config: StreamConfig) -> bytes:
    """Encode a full sample stream into a standalone container (GPU)."""
    config.validate()
    x = np.asarray(samples)
    if x.ndim != 1:
        x = x.reshape(-1)
    if x.size < 1:
        raise InvalidConfig("element_count must be >= 1")
    torch, _ = _require_cuda()
    x, in_kind = _reference_cast(x, config.dtype)
    if in_kind != _IN_NATIVE:
        return _encode_cast(x, in_kind, config)
    if not x.flags.writeable:
        x = x.copy()
    xd = torch.from_numpy(x).to("cuda", non_blocking=False)
    enc = Encoder(x.size, config, with_offsets=False)
    enc.encode(xd)
    nbytes = enc.finish()
    return bytes(enc.out[:nbytes].cpu().numpy().tobytes())


def decode_stream(data) -> np.ndarray:
    """Decode a container back into a typed sample array (GPU)."""
    cfg, count = parse_file_header(data)
    if count == 0:
        return np.empty(0, dtype=cfg.dtype.np_dtype)
    torch, _ = _require_cuda()
    raw = np.frombuffer(bytes(data), np.uint8)
    blob = torch.empty(raw.size + 64, dtype=torch.uint8, device="cuda")
    blob[:raw.size].copy_(torch.from_numpy(raw.copy()))
    return decode_device(blob, raw.size).cpu().numpy()
