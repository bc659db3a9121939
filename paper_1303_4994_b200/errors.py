"""Exception taxonomy of the reference (reference `pkg/src/apax/errors.py:4-61`),
plus the mapping from the C-ABI status codes (include/apax_status.h) onto
those classes with the reference's exact messages.

Class names, bases and messages are identical to the reference so callers'
`except` clauses and message matches keep working after the switch.
"""
from __future__ import annotations


class ApaxError(Exception):
    """Base class for all apax errors."""


class RangeError(ApaxError, ValueError):
    """A numeric argument is outside its documented domain."""


class InvalidConfig(ApaxError, ValueError):
    """A StreamConfig violates one of its invariants."""


class UnsupportedValue(ApaxError, ValueError):
    """Input contains values the codec cannot represent (NaN/Inf)."""


class NotApaxFile(ApaxError, ValueError):
    """Container magic does not match."""


class UnsupportedVersion(ApaxError, ValueError):
    """Container version is not understood by this decoder."""


class TruncatedStream(ApaxError, ValueError):
    """The encoded stream ends before the declared content does."""


class CorruptStream(ApaxError, ValueError):
    """The encoded stream contains an impossible token or field."""


class InternalError(ApaxError, RuntimeError):
    """An encoder-side consistency check failed (a bug, not bad input)."""


class UndefinedCorrelation(ApaxError, ValueError):
    """Pearson's r is undefined because one vector has zero energy."""


class NoData(ApaxError, ValueError):
    """An operation was asked to work on an empty curve or session."""


class SizeMismatch(ApaxError, ValueError):
    """A raw file's size is inconsistent with its declared element type."""


class UnreadableFile(ApaxError, OSError):
    """A raw dataset file could not be opened or read."""


class NonFiniteValue(ApaxError, ValueError):
    """A raw float dataset contains NaN or Inf (index reported)."""


class InvalidSpec(ApaxError, ValueError):
    """A synthetic-dataset spec has out-of-range parameters."""


class DeviceError(ApaxError, RuntimeError):
    """A CUDA launch or runtime failure inside the B200 extension (no
    reference counterpart: the reference never touches a device)."""


MAX_EXPONENT = 34

# status code -> (exception class, message template); `{d}` is the detail
# value reported by the device (index, wire code, block size, version).
_STATUS = {
    1: (TruncatedStream, "JEE nibble stream exhausted"),                      # entropy.py:175
    2: (CorruptStream, "reserved JEE nibble 14"),                             # entropy.py:176
    3: (CorruptStream, f"decoded exponent outside [0, {MAX_EXPONENT}]"),     # entropy.py:177
    4: (CorruptStream, "JEE token stream yields too many exponents"),         # entropy.py:178
    5: (CorruptStream, "JEE stream must start with an absolute exponent"),    # entropy.py:179
    6: (CorruptStream, "reserved selector value 3"),                          # dtypes.py:175
    7: (NotApaxFile, "bad magic"),                                            # codec.py:295
    8: (UnsupportedVersion, "container version {d}"),                         # codec.py:297
    9: (UnsupportedValue, "non-finite value at index {d}"),                   # codec.py:270
    10: (InternalError, "sample outside 34-bit range"),                       # entropy.py:54
    11: (TruncatedStream, "mantissa section truncated"),                      # entropy.py:266
    12: (TruncatedStream, "block header truncated"),                          # dtypes.py:171
    13: (TruncatedStream, "file header truncated"),                           # codec.py:291
    14: (CorruptStream, "unknown dtype wire code {d}"),                        # dtypes.py:52
    15: (CorruptStream, "unknown mode code {d}"),                              # codec.py:302
    16: (InvalidConfig, "block_size {d} outside [64, 16384]"),                 # dtypes.py:89-90
    17: (InvalidConfig, "block_size {d} not a multiple of 4"),                 # dtypes.py:92
    18: (InvalidConfig, "lossless unsupported for floats"),                    # dtypes.py:94
    19: (InvalidConfig, "FixedRate target must be > 0 bits/sample"),           # dtypes.py:96
    20: (InvalidConfig, "element_count must be >= 1"),                         # codec.py:265
    21: (OverflowError, "cannot convert float infinity to integer"),           # codec.py:120
    22: (RangeError, "attenuation outside [2^-31, 2^33)"),                     # dtypes.py:112
    23: (InternalError, "sample exceeds its group exponent width"),            # entropy.py:234
    24: (UnsupportedValue, "non-finite float input"),                          # codec.py:114
    25: (ValueError, "math domain error"),                                     # codec.py:251 log10(0)
    40: (ValueError, "output buffer too small"),
    41: (MemoryError, "allocation failure"),
    42: (ValueError, "invalid argument"),
    43: (DeviceError, "CUDA error"),
    44: (ValueError, "workspace too small"),
}


def status_exception(code: int, detail: int = -1) -> BaseException:
    """Exception instance for a non-zero status (reference class + message)."""
    cls, msg = _STATUS.get(int(code), (DeviceError, f"unknown status {code}"))
    return cls(msg.format(d=detail))


def raise_status(code: int, detail: int = -1) -> None:
    if code:
        raise status_exception(code, detail)
