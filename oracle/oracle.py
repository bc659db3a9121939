"""ctypes front end of the CPU oracle (oracle/apax_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs as the checker.  The product package
(paper_1303_4994_b200) never imports this module.

Every function mirrors one reference function (file:line cited in
apax_oracle.c) with numpy arrays in and out; failures raise OracleError
carrying the shared status code (include/apax_status.h).
"""
from __future__ import annotations

import ctypes
import os
import pathlib
import struct
import subprocess

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libapax_oracle.so"

DTYPE_CODES = {"i8": 0, "i16": 1, "i32": 2, "f32": 3, "f64": 4}
NP_DTYPES = {0: np.int8, 1: np.int16, 2: np.int32, 3: np.float32, 4: np.float64}
HDR_SIZE = {0: 4, 1: 4, 2: 4, 3: 6, 4: 6}
FILE_HEADER_SIZE = 28


class OracleError(Exception):
    def __init__(self, code: int, detail: int):
        super().__init__(f"oracle status {code} (detail {detail})")
        self.code = code
        self.detail = detail


def build() -> pathlib.Path:
    """Compile the oracle with its Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.apax_oracle_encode.argtypes = [P, I64, I32, I32, D, I32, I64, I32, I32, P, I64,
                                         P, P, P, P]
        L.apax_oracle_encode.restype = I32
        L.apax_oracle_encode_src.argtypes = [P, I32, I64, I32, I32, D, I32, I64, I32, I32, P, I64,
                                             P, P, P, P]
        L.apax_oracle_encode_src.restype = I32
        L.apax_oracle_decode.argtypes = [P, I64, P, I64, P, I32, P]
        L.apax_oracle_decode.restype = I32
        L.apax_oracle_find_blocks.argtypes = [P, I64, P, P]
        L.apax_oracle_find_blocks.restype = I32
        L.apax_oracle_parse_header.argtypes = [P, I64, P, P, P, P, P, P]
        L.apax_oracle_parse_header.restype = I32
        L.apax_oracle_max_encoded_bytes.argtypes = [I64, I32, I32]
        L.apax_oracle_max_encoded_bytes.restype = I64
        L.apax_oracle_pairwise_sum.argtypes = [P, I64]
        L.apax_oracle_pairwise_sum.restype = D
        L.apax_oracle_group_exponents.argtypes = [P, I64, P]
        L.apax_oracle_group_exponents.restype = I32
        L.apax_oracle_jee_encode.argtypes = [P, I64, P]
        L.apax_oracle_jee_encode.restype = I64
        L.apax_oracle_jee_decode.argtypes = [P, I64, I64, P, P]
        L.apax_oracle_jee_decode.restype = I32
        L.apax_oracle_pack_block.argtypes = [P, P, I64, P, P]
        L.apax_oracle_pack_block.restype = I32
        L.apax_oracle_unpack_block.argtypes = [P, I64, I64, P, P]
        L.apax_oracle_unpack_block.restype = I32
        L.apax_oracle_encode_scale_code.argtypes = [D, P]
        L.apax_oracle_encode_scale_code.restype = I32
        L.apax_oracle_decode_scale_code.argtypes = [I32]
        L.apax_oracle_decode_scale_code.restype = D
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(st: int, detail: int = -1):
    if st:
        raise OracleError(st, detail)


# --------------------------------------------------------------------------
# codec
# --------------------------------------------------------------------------
TRACE_FIELDS = ("att_db", "a", "code", "fbe", "selector", "cost0", "cost1", "cost2",
                "nbytes", "restart")


def encode(x, dtype: int, mode: int, target: float = 0.0, block_size: int = 4096,
           segment_blocks: int = 0, policy: int = 0, nthreads: int = 1,
           trace: bool = False):
    """encode_stream (codec.py:258-285); segment_blocks>0 -> segmented container.

    Returns (blob bytes, block_offsets int64[n_blocks+1], trace or None)."""
    x = np.asarray(x).reshape(-1)
    src = 0
    if x.dtype != NP_DTYPES[dtype]:
        # encode_stream (codec.py:266-272) widens to float64 / int64 first
        src = 2 if dtype >= 3 else 1
        x = x.astype(np.float64 if src == 2 else np.int64)
    x = np.ascontiguousarray(x)
    n = x.size
    nb = (n + block_size - 1) // block_size
    cap = int(lib().apax_oracle_max_encoded_bytes(n, dtype, block_size)) + 64
    if src:
        cap = 28 + nb * ((6 if dtype >= 3 else 4) + (3 * (block_size // 4) + 1) // 2 + 17 * block_size) + 64
    out = np.zeros(cap, np.uint8)
    out_len = ctypes.c_int64(0)
    detail = ctypes.c_int64(-1)
    offs = np.zeros(nb + 1, np.int64)
    tr = np.zeros((max(nb, 1), len(TRACE_FIELDS)), np.float64) if trace else None
    st = lib().apax_oracle_encode_src(_ptr(x), src, n, dtype, mode, float(target), block_size,
                                      int(segment_blocks), int(policy), int(nthreads), _ptr(out),
                                      cap, ctypes.byref(out_len), _ptr(offs),
                                      _ptr(tr) if tr is not None else None, ctypes.byref(detail))
    _check(st, detail.value)
    return out[:out_len.value].tobytes(), offs, tr


def parse_header(blob: bytes):
    buf = np.frombuffer(blob, np.uint8)
    dt, mode, bs = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    count, target, detail = ctypes.c_int64(), ctypes.c_double(), ctypes.c_int64()
    st = lib().apax_oracle_parse_header(_ptr(buf), buf.size, ctypes.byref(dt),
                                        ctypes.byref(mode), ctypes.byref(bs),
                                        ctypes.byref(count), ctypes.byref(target),
                                        ctypes.byref(detail))
    _check(st, detail.value)
    return dt.value, mode.value, bs.value, count.value, target.value


def find_blocks(blob: bytes) -> np.ndarray:
    """The serial block walk of decode_stream (codec.py:317-323)."""
    dt, mode, bs, count, _ = parse_header(blob)
    nb = (count + bs - 1) // bs
    buf = np.frombuffer(blob, np.uint8)
    offs = np.zeros(nb + 1, np.int64)
    detail = ctypes.c_int64(-1)
    st = lib().apax_oracle_find_blocks(_ptr(buf), buf.size, _ptr(offs), ctypes.byref(detail))
    _check(st, detail.value)
    return offs


def decode(blob: bytes, block_offsets=None, nthreads: int = 1) -> np.ndarray:
    """decode_stream (codec.py:308-329)."""
    dt, mode, bs, count, _ = parse_header(blob)
    buf = np.frombuffer(blob, np.uint8)
    y = np.empty(count, NP_DTYPES[dt])
    detail = ctypes.c_int64(-1)
    offs = None
    if block_offsets is not None:
        offs = np.ascontiguousarray(block_offsets, np.int64)
    st = lib().apax_oracle_decode(_ptr(buf), buf.size, _ptr(y), count,
                                  _ptr(offs) if offs is not None else None, int(nthreads),
                                  ctypes.byref(detail))
    _check(st, detail.value)
    return y


def max_encoded_bytes(n: int, dtype: int, block_size: int) -> int:
    return int(lib().apax_oracle_max_encoded_bytes(n, dtype, block_size))


def file_header(dtype: int, mode: int, block_size: int, count: int, target: float) -> bytes:
    return struct.pack("<4sBBBBIQd", b"APAX", 1, dtype, mode, 0, block_size, count,
                       float(target))


# --------------------------------------------------------------------------
# entropy / dtypes primitives
# --------------------------------------------------------------------------
def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, np.float64)
    return float(lib().apax_oracle_pairwise_sum(_ptr(a), a.size))


def group_exponents(v) -> np.ndarray:
    v = np.ascontiguousarray(v, np.int64)
    e = np.zeros(max(v.size // 4, 1), np.int64)
    _check(lib().apax_oracle_group_exponents(_ptr(v), v.size, _ptr(e)))
    return e[:v.size // 4]


def jee_encode(e) -> list:
    e = np.ascontiguousarray(e, np.int64)
    out = np.zeros(3 * e.size + 3, np.uint8)
    k = lib().apax_oracle_jee_encode(_ptr(e), e.size, _ptr(out))
    return out[:k].tolist()


def jee_decode(nibbles, n_groups: int):
    nb = np.ascontiguousarray(nibbles, np.uint8)
    out = np.zeros(max(n_groups, 1), np.int64)
    used = ctypes.c_int64(0)
    st = lib().apax_oracle_jee_decode(_ptr(nb), nb.size, n_groups, _ptr(out),
                                      ctypes.byref(used))
    _check(st)
    return out[:n_groups], used.value


def pack_block(v, e) -> bytes:
    v = np.ascontiguousarray(v, np.int64)
    e = np.ascontiguousarray(e, np.int64)
    cap = 3 * e.size + 8 * v.size + 16
    out = np.zeros(cap, np.uint8)
    n = ctypes.c_int64(0)
    _check(lib().apax_oracle_pack_block(_ptr(v), _ptr(e), e.size, _ptr(out), ctypes.byref(n)))
    return out[:n.value].tobytes()


def unpack_block(payload: bytes, n_groups: int):
    buf = np.frombuffer(payload, np.uint8)
    v = np.zeros(4 * max(n_groups, 1), np.int64)
    used = ctypes.c_int64(0)
    _check(lib().apax_oracle_unpack_block(_ptr(buf), buf.size, n_groups, _ptr(v),
                                          ctypes.byref(used)))
    return v[:4 * n_groups], used.value


def encode_scale_code(a: float) -> int:
    c = ctypes.c_int(0)
    _check(lib().apax_oracle_encode_scale_code(float(a), ctypes.byref(c)))
    return c.value


def decode_scale_code(code: int) -> float:
    return float(lib().apax_oracle_decode_scale_code(int(code)))
