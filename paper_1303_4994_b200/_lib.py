"""Loader for the in-tree C-ABI extension libapax_b200.so (include/apax_b200.h).

There is no CPU fallback: every codec entry point calls `lib()`, which raises
ExtensionMissing when the .so is absent or fails to load, and DeviceMissing
when no CUDA device is present.
"""
from __future__ import annotations

import ctypes
import pathlib

_HERE = pathlib.Path(__file__).resolve().parent
import os as _os

# APAX_LIB_PATH overrides the in-tree library (tuning experiments only)
LIB_PATH = pathlib.Path(_os.environ.get("APAX_LIB_PATH", str(_HERE / "libapax_b200.so")))


class ExtensionMissing(ImportError):
    """libapax_b200.so is not built (run __graft_entry__.build())."""


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ExtensionMissing(f"{LIB_PATH} not found: build it with `python -c "
                               f"'import __graft_entry__ as g; g.build()'`")
    try:
        L = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:  # pragma: no cover
        raise ExtensionMissing(f"cannot load {LIB_PATH}: {exc}") from exc
    P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.apax_version.restype = ctypes.c_char_p
    L.apax_launch_count.argtypes = []
    L.apax_launch_count.restype = I64
    L.apax_status_string.argtypes = [I32]
    L.apax_status_string.restype = ctypes.c_char_p
    L.apax_max_encoded_bytes.argtypes = [I64, I32, I32]
    L.apax_max_encoded_bytes.restype = I64
    L.apax_encode_workspace_bytes.argtypes = [I64, I32, I32, I32, I64]
    L.apax_encode_workspace_bytes.restype = I64
    L.apax_encode.argtypes = [P, I64, I32, I32, D, I32, I64, I32, P, I64, P, P, P, P, I64, P]
    L.apax_encode.restype = I32
    L.apax_decode_workspace_bytes.argtypes = [I64, I32, I32]
    L.apax_decode_workspace_bytes.restype = I64
    L.apax_decode.argtypes = [P, I64, I64, I32, I32, P, P, P, P, I64, P]
    L.apax_decode.restype = I32
    L.apax_encode_wave_segment_blocks.argtypes = [I64, I32, I32, I32]
    L.apax_encode_wave_segment_blocks.restype = I64
    L.apax_encode_kernel_name.argtypes = [I32, I32, I32, I64]
    L.apax_encode_kernel_name.restype = ctypes.c_char_p
    # (bound only when present: APAX_LIB_PATH may point at an older tuning build)
    if hasattr(L, "apax_decode_range"):
        L.apax_decode_range.argtypes = [P, I64, I64, I32, I32, P, I64, I64, ctypes.c_uint64, ctypes.c_uint64,
                                        P, P, P, P, I64, P]
        L.apax_decode_range.restype = I32
    if hasattr(L, "apax_encode_lossless_range"):
        L.apax_encode_lossless_range.argtypes = [P, I64, I64, I32, I32, I64, P, I64, P, P, P, I64, P]
        L.apax_encode_lossless_range.restype = I32
    if hasattr(L, "apax_detect_segments"):
        L.apax_detect_segments.argtypes = [P, I64, P, I64, P, P]
        L.apax_detect_segments.restype = I32
    if hasattr(L, "apax_status_to_host"):
        L.apax_status_to_host.argtypes = [P, P, I32, P]
        L.apax_status_to_host.restype = I32
    L.apax_decode_segments_workspace_bytes.argtypes = [I64, I32, I32]
    L.apax_decode_segments_workspace_bytes.restype = I64
    L.apax_decode_segments.argtypes = [P, I64, I64, I32, I32, P, I64, P, P, P, I64, P]
    L.apax_decode_segments.restype = I32
    L.apax_profile_grid.argtypes = []
    L.apax_profile_grid.restype = I32
    L.apax_profile_sums.argtypes = [P, P, I64, I32, I32, D, D, D, P, P, P]
    L.apax_profile_sums.restype = I32
    L.apax_profile_welch.argtypes = [P, P, I64, I32, I32, I32, P, P, P]
    L.apax_profile_welch.restype = I32
    L.apax_profile_select.argtypes = [P, P, I64, I32, I32, P, I32, P, I32, P]
    L.apax_profile_select.restype = I32
    L.apax_max_encoded_bytes_cast.argtypes = [I64, I32, I32, I32]
    L.apax_max_encoded_bytes_cast.restype = I64
    L.apax_encode_cast_workspace_bytes.argtypes = [I64, I32, I32, I32, I32, I64]
    L.apax_encode_cast_workspace_bytes.restype = I64
    L.apax_encode_cast.argtypes = [P, I32, I64, I32, I32, D, I32, I64, I32, P, I64, P, P, P, I64, P]
    L.apax_encode_cast.restype = I32
    L.apax_quantize_block.argtypes = [P, I64, I32, D, P, P, P, P]
    L.apax_quantize_block.restype = I32
    L.apax_dequantize_block.argtypes = [P, I64, I32, I32, I32, P, P]
    L.apax_dequantize_block.restype = I32
    L.apax_encode_block.argtypes = [P, I64, I32, I32, D, I32, P, P, I64, P, P, I64, P]
    L.apax_encode_block.restype = I32
    L.apax_sweep_point_workspace_bytes.argtypes = [I64, I32]
    L.apax_sweep_point_workspace_bytes.restype = I64
    L.apax_sweep_point.argtypes = [P, I64, I32, D, P, P, P, I64, P]
    L.apax_sweep_point.restype = I32
    L.apax_find_blocks.argtypes = [P, I64, I64, I32, I32, P, P, P]
    L.apax_find_blocks.restype = I32
    L.apax_parse_file_header.argtypes = [P, I64, P, P, P, P, P, P]
    L.apax_parse_file_header.restype = I32
    _lib = L
    return L


EXPORTED_SYMBOLS = (
    "apax_version", "apax_status_string", "apax_max_encoded_bytes",
    "apax_encode_workspace_bytes", "apax_encode", "apax_decode_workspace_bytes",
    "apax_decode", "apax_find_blocks", "apax_parse_file_header",
    "apax_decode_segments_workspace_bytes", "apax_decode_segments",
    "apax_encode_wave_segment_blocks", "apax_profile_grid", "apax_profile_sums", "apax_profile_welch",
    "apax_profile_select", "apax_decode_range", "apax_status_to_host",
    "apax_encode_lossless_range", "apax_detect_segments",
    "apax_max_encoded_bytes_cast", "apax_launch_count", "apax_quantize_block", "apax_dequantize_block",
    "apax_encode_block", "apax_sweep_point", "apax_sweep_point_workspace_bytes", "apax_encode_cast_workspace_bytes", "apax_encode_cast",
    "apax_encode_kernel_name",
)
