"""Profiler statistics of an array split over ranks
(distributed.sharded_window_stats): two processes (gloo; both on cuda:0 of
this one-GPU pool, which is fine for correctness: no kernel waits on another
rank) each hold half of (x, y = the GPU decode of x); the merged moments,
pearson r and SRR must match the one-process statistics of the whole array
to 1e-12 (the sums are added in a different order), and the 2-sigma S2R
margin -- an exact order statistic via all-reduced radix histograms --
must match exactly."""
import json
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data():
    from paper_1303_4994_b200 import Dtype, Mode, StreamConfig, decode_device, encode_device
    from paper_1303_4994_b200 import workloads as W
    x = W.cfg2_ar2_f32((1 << 18) + 12345)
    xd = torch.from_numpy(x).cuda()
    res = encode_device(xd, StreamConfig(Dtype.F32, 4096, Mode.FIXED_QUALITY, 45.0))
    y = decode_device(res.blob, res.nbytes, res.block_offsets)
    return xd, y


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1303_4994_b200 import Dtype
    from paper_1303_4994_b200 import distributed as D
    xd, y = _data()
    n = xd.numel()
    a, b = (n * rank) // world, (n * (rank + 1)) // world
    st = D.sharded_window_stats(xd[a:b].contiguous(), y[a:b].contiguous(), Dtype.F32)
    # Welch spectra: shards on hop (2048) boundaries
    hop = 2048
    cut = ((n // world) // hop) * hop
    a2, b2 = (0, cut) if rank == 0 else (cut, n)
    st["welch"] = [D.sharded_welch(xd[a2:b2], y[a2:b2], Dtype.F32, which=w).tolist() for w in (0, 1, 2)]
    with open(os.path.join(out_dir, f"s{rank}.json"), "w") as f:
        json.dump(st, f)
    dist.destroy_process_group()


def test_two_rank_window_stats_match_whole_array(tmp_path):
    import torch.multiprocessing as mp
    from paper_1303_4994_b200 import Dtype
    from paper_1303_4994_b200.profiler import S2RDistribution, _Sums
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    r0 = json.loads((tmp_path / "s0.json").read_text())
    r1 = json.loads((tmp_path / "s1.json").read_text())
    assert r0 == r1
    xd, y = _data()
    s = _Sums(xd, y, Dtype.F32, centred=True)
    n = s.n
    whole = {"mean_x": s.sx / n, "mean_y": s.sy / n, "mean_d": s.sd / n,
             "std_x": (s.cxx / n) ** 0.5, "std_y": (s.cyy / n) ** 0.5, "std_d": (s.cdd / n) ** 0.5,
             "pearson_r": s.pearson(), "srr_db": 10.0 * np.log10(s.sxx / s.sdd)}
    assert r0["n"] == n and r0["zero_x"] == s.zero_x and r0["zero_d"] == s.zero_d
    for k, v in whole.items():
        assert abs(r0[k] - v) <= 1e-12 * max(1.0, abs(v)), (k, r0[k], v)
    assert r0["two_sigma_s2r_margin_db"] == S2RDistribution(xd, y, Dtype.F32, True).two_sigma_margin_db
    from paper_1303_4994_b200.profiler import _welch_power
    for w in (0, 1, 2):
        ref = _welch_power(xd.double(), y.double(), Dtype.F64, w, n, 4096)
        got = np.array(r0["welch"][w])
        assert np.allclose(got, ref, rtol=1e-12, atol=0.0), w


# ---------------------------------------------------------------------------
# BASELINE cfg4 composition: ONE seeded field sharded by segment ranges, each
# rank generating only its own z planes, codec + global profiler statistics
# (distributed.sharded_round_trip), against the one-process results
# ---------------------------------------------------------------------------
SIDE, P = 128, 64            # 2^21 f64 samples, 512 blocks: 8 segments of 64 blocks


def _cfg4_cfg():
    from paper_1303_4994_b200 import Dtype, Mode, StreamConfig
    return StreamConfig(Dtype.F64, 4096, Mode.FIXED_RATE, 64.0 / 3.0, segment_blocks=P,
                        segment_policy="warm_self")


def _round_trip_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1303_4994_b200 import distributed as D
    from paper_1303_4994_b200 import workloads as W
    n = SIDE ** 3
    s0, s1 = D.shard_samples(n, 4096, P, world, rank)
    plane = SIDE * SIDE
    assert s0 % plane == 0 and s1 % plane == 0
    x = W.cfg4_modes_f64(SIDE, device="cuda", z0=s0 // plane, planes=(s1 - s0) // plane)
    r = D.sharded_round_trip(x, _cfg4_cfg())
    enc = r["encoder"]
    body = bytes(enc.out[28:28 + r["body_len"]].cpu().numpy().tobytes())
    np.save(os.path.join(out_dir, f"y{rank}.npy"), r["y"].cpu().numpy())
    with open(os.path.join(out_dir, f"b{rank}.bin"), "wb") as f:
        f.write(body)
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump({"offset": r["placement"].body_offset, "total": r["placement"].total_bytes,
                   "window": r["window"], "welch_x": r["welch_x"].tolist(),
                   "welch_d": r["welch_d"].tolist()}, f)
    dist.destroy_process_group()


def test_two_rank_cfg4_sharded_round_trip(tmp_path):
    import torch.multiprocessing as mp
    from paper_1303_4994_b200 import Dtype, decode_device, encode_device
    from paper_1303_4994_b200 import workloads as W
    from paper_1303_4994_b200.profiler import S2RDistribution, _Sums, _welch_power
    mp.spawn(_round_trip_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    x = W.cfg4_modes_f64(SIDE, device="cuda")
    res = encode_device(x, _cfg4_cfg())
    whole = res.to_bytes()
    r0 = json.loads((tmp_path / "r0.json").read_text())
    r1 = json.loads((tmp_path / "r1.json").read_text())
    b0, b1 = (tmp_path / "b0.bin").read_bytes(), (tmp_path / "b1.bin").read_bytes()
    # placement: rank 1's body starts where rank 0's ends; the concatenation
    # under the one-process header is the one-process container
    assert r0["offset"] == 28 and r1["offset"] == 28 + len(b0)
    assert r0["total"] == r1["total"] == len(whole)
    assert whole[:28] + b0 + b1 == whole
    y = decode_device(res.blob, res.nbytes, res.block_offsets)
    ycat = np.concatenate([np.load(tmp_path / "y0.npy"), np.load(tmp_path / "y1.npy")])
    assert np.array_equal(ycat, y.cpu().numpy())
    # global statistics = one-array statistics
    assert r0["window"] == r1["window"] and r0["welch_x"] == r1["welch_x"]
    s = _Sums(x, y, Dtype.F64, centred=True)
    n = s.n
    w = r0["window"]
    ref = {"mean_x": s.sx / n, "mean_d": s.sd / n, "std_x": (s.cxx / n) ** 0.5, "std_d": (s.cdd / n) ** 0.5,
           "pearson_r": s.pearson()}
    for k, v in ref.items():
        assert abs(w[k] - v) <= 1e-12 * max(1.0, abs(v)), (k, w[k], v)
    assert w["two_sigma_s2r_margin_db"] == S2RDistribution(x, y, Dtype.F64, True).two_sigma_margin_db
    for key, which in (("welch_x", 0), ("welch_d", 2)):
        refw = _welch_power(x, y, Dtype.F64, which, n, 4096)
        assert np.allclose(np.array(r0[key]), refw, rtol=1e-12, atol=0.0), key
