"""CPU-side checks of the C-ABI library and the host logic (no compute calls
that need a GPU)."""
import ctypes
import json
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from oracle import oracle as O
from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, _lib, errors, parse_file_header
from paper_1303_4994_b200.dtypes import BlockHeader, decode_scale_code, encode_scale_code


def _declared_functions():
    text = (ROOT / "include" / "apax_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\**\s+\**(apax_[a-z_0-9]+)\(",
                                 text, re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _declared_functions()
    assert len(declared) >= 8
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(_lib.EXPORTED_SYMBOLS)
    assert L.apax_version().startswith(b"apax-b200")


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_max_encoded_bytes_matches_oracle():
    L = _lib.lib()
    for n, dt, bs in [(1, 0, 64), (1 << 26, 3, 4096), (12345, 4, 1000), (70000, 2, 16384)]:
        assert L.apax_max_encoded_bytes(n, dt, bs) == O.max_encoded_bytes(n, dt, bs)


def test_status_strings_cover_all_codes():
    L = _lib.lib()
    for code in list(range(0, 25)) + [40, 41, 42, 43, 44]:
        assert L.apax_status_string(code) != b"unknown status"


def test_parse_file_header_errors_match_reference():
    d = json.loads((GOLDEN / "decode_errors.json").read_text())
    header_cases = {"truncated_file_header", "bad_magic", "bad_version", "bad_dtype_wire",
                    "bad_mode_wire", "bad_block_size", "block_size_not_mult4",
                    "lossless_float_header", "fr_zero_target_header"}
    for case in d["cases"]:
        if case["name"] not in header_cases:
            continue
        blob = bytes.fromhex(case["blob_hex"])
        with pytest.raises(Exception) as ei:
            parse_file_header(blob)
        assert type(ei.value).__name__ == case["exc"], case["name"]
        assert str(ei.value) == case["msg"], case["name"]


def test_parse_file_header_fields():
    blob = O.file_header(1, 0, 64, 100, 0.0)
    cfg, count = parse_file_header(blob)
    assert cfg.dtype is Dtype.I16 and cfg.block_size == 64 and count == 100


def test_stream_config_validation_messages():
    with pytest.raises(errors.InvalidConfig, match="outside"):
        StreamConfig(Dtype.I16, 60).validate()
    with pytest.raises(errors.InvalidConfig, match="multiple of 4"):
        StreamConfig(Dtype.I16, 66).validate()
    with pytest.raises(errors.InvalidConfig, match="lossless unsupported"):
        StreamConfig(Dtype.F32).validate()
    with pytest.raises(errors.InvalidConfig, match="FixedRate target"):
        StreamConfig(Dtype.F32, mode=Mode.FIXED_RATE, target=0.0).validate()
    with pytest.raises(errors.InvalidConfig):
        StreamConfig(Dtype.I16, segment_blocks=0).validate()
    StreamConfig(Dtype.F32, mode=Mode.FIXED_QUALITY, target=60.0, segment_blocks=16).validate()


def test_exception_hierarchy_matches_reference():
    assert issubclass(errors.InternalError, RuntimeError)
    assert issubclass(errors.UnreadableFile, OSError)
    for name in ("RangeError", "InvalidConfig", "UnsupportedValue", "NotApaxFile",
                 "UnsupportedVersion", "TruncatedStream", "CorruptStream"):
        assert issubclass(getattr(errors, name), ValueError)
        assert issubclass(getattr(errors, name), errors.ApaxError)


def test_scale_code_host_utilities():
    for code in range(0, 1 << 16, 13):
        a = decode_scale_code(code)
        if 2.0 ** -31 <= a < 2.0 ** 33:
            assert encode_scale_code(a) == code == O.encode_scale_code(a)
    with pytest.raises(errors.RangeError):
        encode_scale_code(2.0 ** 33)


def test_block_header_round_trip():
    for sel in (0, 1, 2):
        for dt in (Dtype.I16, Dtype.F32):
            h = BlockHeader(sel, sel == 1, 12345, -5 if dt.is_float else None)
            assert BlockHeader.parse(h.serialize(dt), dt) == h
    with pytest.raises(errors.CorruptStream):
        BlockHeader.parse(bytes([3, 0, 0, 0]), Dtype.I16)
    with pytest.raises(errors.TruncatedStream):
        BlockHeader.parse(bytes([0, 0]), Dtype.I16)


def test_workspace_sizes_positive():
    L = _lib.lib()
    assert L.apax_decode_workspace_bytes(1 << 20, 3, 4096) > 0
    # encode workspace queries the device occupancy; without a GPU the
    # library falls back to a nominal 148-SM estimate
    assert L.apax_encode_workspace_bytes(1 << 20, 3, 2, 4096, 16) > 0


def test_product_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1303_4994_b200 import encode_stream
    with pytest.raises(_lib.ExtensionMissing):
        encode_stream(np.zeros(64, np.int16), StreamConfig(Dtype.I16, 64))
