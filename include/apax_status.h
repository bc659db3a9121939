/*
 * apax_status.h -- status codes shared by the B200 C-ABI (libapax_b200.so)
 * and the CPU oracle.  Each code maps 1:1 onto the reference exception class
 * and message (reference `pkg/src/apax/errors.py:4-61`); the Python layer
 * (paper_1303_4994_b200/errors.py) raises the identically named class.
 */
#ifndef APAX_STATUS_H
#define APAX_STATUS_H

enum apax_status {
    APAX_OK = 0,
    /* JEE decode statuses, entropy.py:174-180 (same numbering as the
     * reference's numba kernel return codes 1..5) */
    APAX_ERR_JEE_TRUNCATED = 1,      /* TruncatedStream "JEE nibble stream exhausted" */
    APAX_ERR_JEE_RESERVED = 2,       /* CorruptStream "reserved JEE nibble 14" */
    APAX_ERR_JEE_RANGE = 3,          /* CorruptStream "decoded exponent outside [0, 34]" */
    APAX_ERR_JEE_TOO_MANY = 4,       /* CorruptStream "JEE token stream yields too many exponents" */
    APAX_ERR_JEE_NO_ABS = 5,         /* CorruptStream "JEE stream must start with an absolute exponent" */
    APAX_ERR_SELECTOR = 6,           /* CorruptStream "reserved selector value 3" (dtypes.py:175) */
    APAX_ERR_NOT_APAX = 7,           /* NotApaxFile "bad magic" (codec.py:295) */
    APAX_ERR_VERSION = 8,            /* UnsupportedVersion "container version {v}" (codec.py:297) */
    APAX_ERR_NONFINITE = 9,          /* UnsupportedValue "non-finite value at index {i}" (codec.py:268-270) */
    APAX_ERR_INTERNAL = 10,          /* InternalError "sample outside 34-bit range" (entropy.py:53-54) */
    APAX_ERR_MANTISSA_TRUNCATED = 11,/* TruncatedStream "mantissa section truncated" (entropy.py:266) */
    APAX_ERR_BLOCK_HDR_TRUNCATED = 12,/* TruncatedStream "block header truncated" (dtypes.py:171) */
    APAX_ERR_FILE_HDR_TRUNCATED = 13,/* TruncatedStream "file header truncated" (codec.py:291) */
    APAX_ERR_DTYPE_WIRE = 14,        /* CorruptStream "unknown dtype wire code {w}" (dtypes.py:52) */
    APAX_ERR_MODE_WIRE = 15,         /* CorruptStream "unknown mode code {m}" (codec.py:302) */
    APAX_ERR_CFG_BLOCK_RANGE = 16,   /* InvalidConfig "block_size {bs} outside [64, 16384]" */
    APAX_ERR_CFG_BLOCK_MULT = 17,    /* InvalidConfig "block_size {bs} not a multiple of 4" */
    APAX_ERR_CFG_LOSSLESS_FLOAT = 18,/* InvalidConfig "lossless unsupported for floats" */
    APAX_ERR_CFG_FR_TARGET = 19,     /* InvalidConfig "FixedRate target must be > 0 bits/sample" */
    APAX_ERR_EMPTY = 20,             /* InvalidConfig "element_count must be >= 1" (codec.py:265) */
    APAX_ERR_OVERFLOW = 21,          /* OverflowError from math.floor(log2(inf)) (codec.py:120) */
    APAX_ERR_RANGE = 22,             /* RangeError "attenuation ... outside [2^-31, 2^33)" */
    APAX_ERR_INTERNAL_WIDTH = 23,    /* InternalError "sample exceeds its group exponent width" */
    APAX_ERR_NONFINITE_BLOCK = 24,   /* UnsupportedValue "non-finite float input" (codec.py:114) */
    APAX_ERR_MATH_DOMAIN = 25,       /* ValueError "math domain error": the quality loop's
                                        math.log10(px / pd) of an underflowed or overflowed
                                        ratio 0 (codec.py:251) */
    /* host-side / launch errors (no reference counterpart) */
    APAX_ERR_CAPACITY = 40,          /* output buffer too small */
    APAX_ERR_ALLOC = 41,             /* allocation failure */
    APAX_ERR_ARG = 42,               /* invalid argument */
    APAX_ERR_CUDA = 43,              /* CUDA launch/runtime error */
    APAX_ERR_WORKSPACE = 44          /* workspace too small */
};

#endif
