"""Pin the CPU oracle (oracle/apax_oracle.c) before trusting it.

Checks against (a) the reference's own golden entropy vectors
(pkg/tests/golden/entropy_vectors.json, copied by make_golden.py), (b) the
reference's known-answer tests restated (pkg/tests/test_entropy.py,
test_dtypes.py, test_codec.py), and (c) fixtures produced by the live
reference (tests/golden/make_golden.py).  CPU only.
"""
import json

import numpy as np
import pytest

from conftest import GOLDEN, golden_containers, load_container
from oracle import oracle as O
from paper_1303_4994_b200.errors import status_exception


def test_reference_entropy_golden_vectors():
    vecs = json.loads((GOLDEN / "entropy_vectors_ref.json").read_text())
    assert len(vecs) >= 6
    for vec in vecs:
        v = np.asarray(vec["samples"], np.int64)
        e = O.group_exponents(v)
        assert e.tolist() == vec["exponents"]
        payload = O.pack_block(v, e)
        assert payload.hex() == vec["payload_hex"]
        back, used = O.unpack_block(payload, e.size)
        assert back.tolist() == vec["samples"] and used == len(payload)


def test_extra_entropy_vectors():
    d = json.loads((GOLDEN / "entropy_vectors_extra.json").read_text())
    for vec in d["vectors"]:
        v = np.asarray(vec["samples"], np.int64)
        e = O.group_exponents(v)
        assert e.tolist() == vec["exponents"]
        assert O.jee_encode(e) == vec["nibbles"]
        assert O.pack_block(v, e).hex() == vec["payload_hex"]
    for case in d["jee_decode"]:
        if case["exc"] is None:
            out, used = O.jee_decode(case["nibbles"], case["n_groups"])
            assert out.tolist() == case["exps"] and used == case["used"]
        else:
            with pytest.raises(O.OracleError) as ei:
                O.jee_decode(case["nibbles"], case["n_groups"])
            exc = status_exception(ei.value.code)
            assert type(exc).__name__ == case["exc"] and str(exc) == case["msg"]


def test_entropy_kats():
    # pkg/tests/test_entropy.py:51-121 restated
    assert O.group_exponents([0, 0, 0, 0]).tolist() == [0]
    assert O.group_exponents([1, -1, 0, 0]).tolist() == [2]
    assert O.group_exponents([7, 7, 7, 7]).tolist() == [4]
    assert O.group_exponents([-8, 0, 0, 0]).tolist() == [4]
    assert O.jee_encode([8, 8, 8]) == [15, 0, 8, 4]
    assert O.jee_encode([8, 10]) == [15, 0, 8, 13]
    assert O.jee_encode([3, 12]) == [15, 0, 3, 15, 0, 12]
    assert O.jee_encode([14]) == [15, 0, 14]
    assert O.jee_decode([15, 0, 14], 1)[0].tolist() == [14]
    assert O.pack_block([0, 0, 0, 0], [0]) == bytes([0xF0, 0x00])
    assert O.pack_block([1, -1, 0, 0], [2]) == bytes([0xF0, 0x20, 0x70])
    with pytest.raises(O.OracleError):
        O.group_exponents([2 ** 34, 0, 0, 0])


def test_width_oracle_random(rng):
    for _ in range(200):
        g = rng.integers(-(2 ** 33), 2 ** 33, size=4)
        lo_hi = [(-(1 << (w - 1)), (1 << (w - 1)) - 1) for w in range(1, 35)]
        expect = 0 if not g.any() else next(w + 1 for w, (lo, hi) in enumerate(lo_hi)
                                            if all(lo <= v <= hi for v in g))
        assert O.group_exponents(g).tolist() == [expect]


def test_pack_round_trip_random(rng):
    for _ in range(100):
        n = 4 * int(rng.integers(1, 40))
        w = int(rng.integers(1, 35))
        v = rng.integers(-(1 << (w - 1)), 1 << (w - 1), size=n)
        e = O.group_exponents(v)
        p = O.pack_block(v, e)
        back, used = O.unpack_block(p + b"\xab\xcd", e.size)
        assert back.tolist() == v.tolist() and used == len(p)
        if e.sum():
            with pytest.raises(O.OracleError):
                O.unpack_block(p[:-1], e.size)


def test_scale_code_exhaustive():
    # pkg/tests/test_dtypes.py:52-72: round trip over all 2^16 codes
    for code in range(0, 1 << 16, 7):
        a = O.decode_scale_code(code)
        if 2.0 ** -31 <= a < 2.0 ** 33:
            assert O.encode_scale_code(a) == code
    assert O.encode_scale_code(1.0) == 31 << 10
    with pytest.raises(O.OracleError):
        O.encode_scale_code(2.0 ** 33)
    with pytest.raises(O.OracleError):
        O.encode_scale_code(2.0 ** -32)


def test_pairwise_sum_matches_numpy():
    z = np.load(GOLDEN / "pairwise.npz")
    off = 0
    for n, s, m in zip(z["sizes"], z["sums"], z["means"]):
        a = z["values"][off:off + n]
        off += n
        got = O.pairwise_sum(a)
        assert got == s, n
        assert got / n == m, n
        # and the live numpy on this machine
        assert got == float(np.sum(a))


@pytest.mark.parametrize("name", golden_containers())
def test_oracle_container_parity(name):
    c = load_container(GOLDEN / "containers" / f"{name}.npz")
    m = c["meta"]
    dt = O.DTYPE_CODES[m["dtype"]]
    target = float.fromhex(m["target_hex"])
    blob, offs, _ = O.encode(c["x"], dt, m["mode"], target, m["block_size"],
                             segment_blocks=m["segment_blocks"], policy=m["policy"],
                             nthreads=2)
    assert blob == c["blob"], name
    assert np.array_equal(offs, c["offsets"])
    y = O.decode(c["blob"])
    assert y.dtype == c["y"].dtype and np.array_equal(y, c["y"], equal_nan=True)
    assert np.array_equal(O.find_blocks(c["blob"]), c["offsets"])
    y2 = O.decode(c["blob"], block_offsets=c["offsets"], nthreads=3)
    assert np.array_equal(y2, c["y"], equal_nan=True)


def _hex_blob(d, case):
    return bytes.fromhex(case["blob_hex"])


def test_oracle_decode_errors():
    d = json.loads((GOLDEN / "decode_errors.json").read_text())
    for case in d["cases"]:
        blob = _hex_blob(d, case)
        if case["exc"] is None:
            y = O.decode(blob)
            assert y.tobytes().hex() == case["y_hex"] and str(y.dtype) == case["y_dtype"]
            continue
        with pytest.raises(O.OracleError) as ei:
            O.decode(blob)
        exc = status_exception(ei.value.code, ei.value.detail)
        assert type(exc).__name__ == case["exc"], case["name"]
        assert str(exc) == case["msg"], case["name"]


def test_oracle_encode_errors():
    cases = json.loads((GOLDEN / "encode_errors.json").read_text())
    for case in cases:
        if case["exc"] is None:
            continue
        x = np.frombuffer(bytes.fromhex(case["x_hex"]), O.NP_DTYPES[O.DTYPE_CODES[case["dtype"]]])
        with pytest.raises(O.OracleError) as ei:
            O.encode(x, O.DTYPE_CODES[case["dtype"]], case["mode"], case["target"],
                     case["block_size"])
        exc = status_exception(ei.value.code, ei.value.detail)
        assert type(exc).__name__ == case["exc"], case["name"]
        assert str(exc) == case["msg"], case["name"]


def test_segment_independence_property(rng):
    # a cold segmented container decodes to the input
    # (lossless) and each segment equals a standalone encode.
    x = rng.integers(-3000, 3000, 50000).astype(np.int16)
    blob, offs, _ = O.encode(x, 1, 0, 0.0, 1024, segment_blocks=5)
    assert np.array_equal(O.decode(blob), x)
    whole, _, _ = O.encode(x, 1, 0, 0.0, 1024)
    assert np.array_equal(O.decode(whole), x)
    seg0, _, _ = O.encode(x[:5 * 1024], 1, 0, 0.0, 1024)
    assert blob[28:int(offs[5])] == seg0[28:]


# ---------------------------------------------------------------------------
# encode_stream's input conversions (reference codec.py:266-272), pinned by
# containers the live reference produced from inputs of other dtypes
# (tests/golden/make_cast_golden.py)
# ---------------------------------------------------------------------------
def _cast_cases():
    return [m["name"] for m in json.loads((GOLDEN / "cast_manifest.json").read_text())]


_ORACLE_EXC = {"InternalError": 10, "UnsupportedValue": 9, "ValueError": 25}


@pytest.mark.parametrize("name", _cast_cases())
def test_oracle_cast_container_parity(name):
    c = load_container(GOLDEN / "containers" / f"{name}.npz")
    m = c["meta"]
    blob, offs, _ = O.encode(c["x"], O.DTYPE_CODES[m["dtype"]], m["mode"], float.fromhex(m["target_hex"]),
                             m["block_size"])
    assert blob == c["blob"], name
    assert np.array_equal(offs, c["offsets"])
    y = O.decode(c["blob"])
    assert y.dtype == c["y"].dtype and np.array_equal(y, c["y"])


def test_oracle_cast_errors():
    for case in json.loads((GOLDEN / "cast_errors.json").read_text()):
        x = np.frombuffer(bytes.fromhex(case["x_hex"]), np.dtype(case["x_dtype"]))
        args = (x, O.DTYPE_CODES[case["dtype"]], case["mode"], case["target"], case["block_size"])
        if case["exc"] is None:
            assert O.encode(*args)[0].hex() == case["blob_hex"], case["name"]
            continue
        with pytest.raises(O.OracleError) as ei:
            O.encode(*args)
        assert ei.value.code == _ORACLE_EXC[case["exc"]], case["name"]


def test_reference_cast_routing():
    """The product widens exactly like the reference and codes the widened
    values in the container dtype whenever that holds them exactly."""
    from paper_1303_4994_b200.codec import _IN_FLOAT64, _IN_INT64, _IN_NATIVE, _reference_cast
    from paper_1303_4994_b200.dtypes import Dtype
    for m in json.loads((GOLDEN / "cast_manifest.json").read_text()):
        c = load_container(GOLDEN / "containers" / f"{m['name']}.npz")
        dt = {"i8": Dtype.I8, "i16": Dtype.I16, "i32": Dtype.I32, "f32": Dtype.F32, "f64": Dtype.F64}[m["dtype"]]
        x = c["x"]
        xw, kind = _reference_cast(x, dt)
        wide = x.astype(np.float64 if dt.is_float else np.int64)
        if kind == _IN_NATIVE:
            assert xw.dtype == dt.np_dtype
            assert np.array_equal(xw.astype(wide.dtype), wide)
        else:
            assert kind == (_IN_FLOAT64 if dt.is_float else _IN_INT64)
            assert xw.dtype == wide.dtype and np.array_equal(xw, wide)
    x = np.array([1.5, -2.7, 3e9])
    xw, kind = _reference_cast(x, Dtype.I32)
    assert kind == _IN_INT64 and xw.tolist() == [1, -2, 3000000000]


# ---------------------------------------------------------------------------
# per-block traces (attenuation, code, block exponent, selector, costs,
# bytes, restart) against the reference stepping encode_block
# (tests/golden/make_trace_golden.py); the oracle calls the same glibc
# pow/log10 as the reference's CPython, so even att_db is exact
# ---------------------------------------------------------------------------
def _trace_names():
    from trace_cases import traces
    return [t["name"] for t in traces()]


@pytest.mark.parametrize("name", _trace_names())
def test_oracle_trace_vs_reference(name):
    from trace_cases import trace_input, traces
    t = next(t for t in traces() if t["name"] == name)
    x = trace_input(t)
    _, _, tr = O.encode(x, O.DTYPE_CODES[t["dtype"]], t["mode"], float.fromhex(t["target_hex"]), 4096,
                        segment_blocks=t["segment_blocks"], trace=True)
    ref = np.array(t["rows"], dtype=np.float64)
    assert tr.shape == ref.shape
    assert np.array_equal(tr, ref), (name, np.argwhere(tr != ref)[:5])


def test_oracle_floor_log2_quirk_containers():
    """glibc's floor(math.log2(s_des)) at the two boundaries where it changes
    the container (codec.py:120-122)."""
    for m in json.loads((GOLDEN / "quirk_manifest.json").read_text()):
        c = load_container(GOLDEN / "containers" / f"{m['name']}.npz")
        blob, _, tr = O.encode(c["x"], O.DTYPE_CODES[m["dtype"]], m["mode"], float.fromhex(m["target_hex"]),
                               m["block_size"], trace=True)
        assert blob == c["blob"], m["name"]
        assert (int(tr[0][2]), int(tr[0][3])) == (m["first_block"]["code"], m["first_block"]["fbe"])
        assert np.array_equal(O.decode(c["blob"]), c["y"])
