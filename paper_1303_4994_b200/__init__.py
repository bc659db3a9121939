"""paper_1303_4994_b200: B200-native APAX universal numerical encoder/decoder.

Drop-in for the reference package's hot path (reference
`pkg/src/apax/__init__.py:9-21`): the same `encode_stream`, `decode_stream`,
`StreamConfig`, `Dtype`, `Mode` names, container bitstream and exceptions,
with every sample-level operation running in hand-written sm_100a kernels
behind the C ABI in include/apax_b200.h.  `profile` / `ProfileSession`
(reference profiler.py) run their statistics in csrc/apax_profile.cu.
"""
from .codec import (Decoder, EncodedStream, Encoder, decode_device, decode_range, decode_stream,
                    encode_lossless_range,
                    encode_device, encode_stream, max_encoded_bytes, parse_file_header,
                    wave_segment_blocks)
from .dtypes import BlockHeader, Dtype, Mode, StreamConfig, decode_scale_code, encode_scale_code
from . import errors
from .block import (AttenuatorState, CodecState, DerivativeHistory, RateLoopState, StreamCosts, dequantize_block,
                    encode_block, quality_loop_update, quantize_block, rate_loop_update)
from .profiler import ProfileSession, profile

__all__ = [
    "Dtype", "Mode", "StreamConfig", "BlockHeader", "encode_stream", "decode_stream",
    "parse_file_header", "encode_device", "decode_device", "decode_range", "encode_lossless_range", "Encoder", "Decoder",
    "EncodedStream", "max_encoded_bytes", "wave_segment_blocks", "profile", "ProfileSession", "encode_scale_code", "decode_scale_code", "errors",
    "AttenuatorState", "CodecState", "DerivativeHistory", "RateLoopState", "StreamCosts", "quantize_block",
    "dequantize_block", "encode_block", "rate_loop_update", "quality_loop_update",
]

__version__ = "0.2.0"
