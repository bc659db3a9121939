"""`apax-b200` command line (paper_1303_4994_b200/cli.py): the reference
CLI's exit codes (pkg/src/apax/cli.py:161-177: 1 usage, 2 data, 3 internal)
and, on the GPU, file round trips checked against the CPU oracle."""
import json

import numpy as np
import pytest

from oracle import oracle as O
from paper_1303_4994_b200 import cli
from paper_1303_4994_b200 import workloads as W


def test_usage_errors_exit_1(tmp_path, capsys):
    raw = tmp_path / "x.f32"
    np.zeros(64, np.float32).tofile(raw)
    assert cli.main(["encode", str(raw), str(tmp_path / "o"), "--dtype", "f32"]) == 1   # lossless float
    assert "lossless unsupported for floats" in capsys.readouterr().err
    assert cli.main(["encode", str(raw), str(tmp_path / "o"), "--dtype", "f32", "--mode", "fixedrate"]) == 1
    assert cli.main(["encode", str(raw), str(tmp_path / "o"), "--dtype", "i16", "--block-size", "30"]) == 1
    assert cli.main(["profile", str(raw), "--dtype", "f32", "--grid", "50:20:5"]) == 1
    assert cli.main(["bogus"]) == 1
    assert cli.main([]) == 1


def test_data_errors_exit_2(tmp_path, capsys):
    assert cli.main(["encode", str(tmp_path / "missing"), str(tmp_path / "o"), "--dtype", "i16"]) == 2
    odd = tmp_path / "odd.i16"
    odd.write_bytes(b"\x01\x02\x03")
    assert cli.main(["encode", str(odd), str(tmp_path / "o"), "--dtype", "i16"]) == 2
    assert "not a multiple of 2" in capsys.readouterr().err
    nan = tmp_path / "nan.f32"
    np.array([1.0, np.nan, 2.0], np.float32).tofile(nan)
    assert cli.main(["encode", str(nan), str(tmp_path / "o"), "--dtype", "f32", "--mode", "fixedquality",
                     "--target", "40"]) == 2
    assert "non-finite value at element 1" in capsys.readouterr().err


def test_grid_text():
    assert cli.grid_from_text("20:120:5")[:3] == [20.0, 25.0, 30.0]
    assert cli.grid_from_text("20:120:5")[-1] == 120.0
    assert len(cli.grid_from_text("20:120:5")) == 21


@pytest.mark.gpu
@pytest.mark.parametrize("dt,np_dt,mode,target,seg", [
    ("i16", np.int16, "fixedrate", 4.0, None),
    ("f32", np.float32, "fixedquality", 45.0, 0),
    ("i32", np.int32, "lossless", 0.0, 3),
])
def test_gpu_file_round_trip(tmp_path, dt, np_dt, mode, target, seg, capsys):
    if dt == "i16":
        x = W.cfg1_sines_i16(4096 * 9 + 11)
    elif dt == "f32":
        x = W.cfg2_ar2_f32(4096 * 20)
    else:
        x = np.cumsum(np.random.default_rng(1).integers(-300, 300, 4096 * 7)).astype(np.int32)
    raw, cont, back = tmp_path / "x.raw", tmp_path / "x.apx", tmp_path / "y.raw"
    x.astype(np_dt).tofile(raw)
    args = ["encode", str(raw), str(cont), "--dtype", dt, "--mode", mode, "--target", str(target), "--sidecar"]
    if seg is not None:
        args += ["--segment-blocks", str(seg)]
    assert cli.main(args) == 0
    out = capsys.readouterr().out
    assert out.startswith("ratio: ")
    blob = cont.read_bytes()
    if seg is None:   # whole stream: the reference's container
        wire = {"i16": 1, "f32": 3, "i32": 2}[dt]
        assert blob == O.encode(x, wire, {"lossless": 0, "fixedrate": 1, "fixedquality": 2}[mode], target, 4096)[0]
    idx = np.fromfile(str(cont) + ".idx", dtype="<i8")
    assert np.array_equal(idx, O.find_blocks(blob))
    assert cli.main(["decode", str(cont), str(back)]) == 0
    y = np.fromfile(back, dtype=np_dt)
    assert np.array_equal(y, O.decode(blob))
    if mode == "lossless":
        assert np.array_equal(y, x)


@pytest.mark.gpu
def test_gpu_profile_json(tmp_path):
    x = W.cfg2_ar2_f32(1 << 16)
    raw = tmp_path / "x.f32"
    x.tofile(raw)
    rep = tmp_path / "r.json"
    assert cli.main(["profile", str(raw), "--dtype", "f32", "--json", str(rep), "--grid", "30:60:10"]) == 0
    d = json.loads(rep.read_text())
    assert "recommended" in d and "windows" in d
    assert rep.read_text() == cli.report_json(d)
