"""Multi-process (world size 2, gloo, CPU) tests of the sharding logic in
paper_1303_4994_b200.distributed: segment-aligned shard ranges, the
all-gather + exclusive scan that places every rank's body, the global
side-band index, and rank-ordered statistic merges.  The per-rank encoder
here is the CPU oracle (test infrastructure): the assembly is independent
of which encoder produced the bodies, and on GPUs `sharded_encode` feeds the
same functions from the B200 encoder."""
import json
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from paper_1303_4994_b200 import distributed as D
from paper_1303_4994_b200 import workloads as W


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [
    # (dtype wire, mode, target, block_size, segment_blocks, n)
    (3, 2, 45.0, 1024, 3, 1024 * 17 + 300),
    (1, 1, 4.0, 4096, 2, 4096 * 9),
    (2, 0, 0.0, 512, 5, 512 * 23 + 7),
    (3, 1, 5.33, 256, 1, 256 * 5),
]


def _inputs(dt, n):
    if dt == 3:
        return W.cfg2_ar2_f32(n)
    if dt == 1:
        return W.cfg1_sines_i16(n)
    rng = np.random.default_rng(7)
    return (np.cumsum(rng.integers(-100, 101, n)) * 1000).astype(np.int32)


def _worker(rank, world, port, outdir):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    results = []
    for (dt, mode, target, bs, seg, n) in CASES:
        x = _inputs(dt, n)
        s, e = D.shard_samples(n, bs, seg, world, rank)
        if e > s:
            blob, offs, _ = O.encode(x[s:e], dt, mode, target, bs, segment_blocks=seg)
            body, local_offs = blob[D.FILE_HEADER_SIZE:], offs
        else:
            body, local_offs = b"", np.array([D.FILE_HEADER_SIZE], np.int64)
        place = D.place_bodies(len(body))
        goffs = D.global_block_offsets(local_offs, place)
        header = D.file_header(dt, mode, bs, n, target)
        full = D.gather_container(body, header)
        parts = [None] * world
        dist.all_gather_object(parts, goffs[:-1].tolist())
        # statistics: rank-ordered merge of per-shard sums
        xs = x[s:e].astype(np.float64)
        merged = D.merge_sums([xs.sum(), (xs * xs).sum(), float(xs.size)])
        if rank == 0:
            ref, ref_offs, _ = O.encode(x, dt, mode, target, bs, segment_blocks=seg)
            all_offs = [o for p in parts for o in p] + [place.total_bytes]
            xf = x.astype(np.float64)
            results.append({
                "same_bytes": full == ref,
                "same_offsets": list(map(int, ref_offs)) == list(map(int, all_offs)),
                "total_ok": place.total_bytes == len(ref),
                "sum_ok": bool(np.allclose(merged, [xf.sum(), (xf * xf).sum(), xf.size], rtol=1e-12)),
            })
    if rank == 0:
        with open(os.path.join(outdir, "result.json"), "w") as f:
            json.dump(results, f)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_cover_segments():
    for n, bs, seg, world in [(10 ** 6, 4096, 16, 8), (4096 * 37 * 443, 4096, 37, 8), (1000, 128, 3, 4)]:
        ranges = [D.shard_samples(n, bs, seg, world, r) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        for (a, b), (c, d) in zip(ranges, ranges[1:]):
            assert b == c
        for a, b in ranges:
            assert a % (bs * seg) == 0   # every shard starts a segment (restart block)


def test_file_header_layout():
    h = D.file_header(3, 2, 4096, 1 << 26, 47.5)
    assert len(h) == 28 and h[:4] == b"APAX" and h[4] == 1 and h[5] == 3 and h[6] == 2


def test_two_rank_gloo_assembly(tmp_path):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    res = json.loads((tmp_path / "result.json").read_text())
    assert len(res) == len(CASES)
    for r in res:
        assert r == {"same_bytes": True, "same_offsets": True, "total_ok": True, "sum_ok": True}, r


def test_range_entries_compose_in_order():
    rng = np.random.default_rng(3)
    maps = [[int(v) for v in rng.integers(0, 1 << 63, 6)] for _ in range(5)]
    ent = D.range_entries(maps)
    assert ent[0] == (0, 0)
    h = (0, 0)
    for r, m in enumerate(maps):
        assert ent[r] == h
        m11, m12, m21, m22, c1, c2 = m
        h = ((m11 * h[0] + m12 * h[1] + c1) % (1 << 64), (m21 * h[0] + m22 * h[1] + c2) % (1 << 64))
    assert D.shard_blocks(10, 3, 0) == (0, 3) and D.shard_blocks(10, 3, 2) == (6, 10)


def _entry_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(11)
    maps = [[int(v) for v in rng.integers(0, 1 << 64, 6, dtype=np.uint64)] for _ in range(world)]
    e = D.whole_stream_entry(maps[rank])
    ok = e == D.range_entries(maps)[rank]
    with open(os.path.join(out_dir, f"entry{rank}.json"), "w") as f:
        json.dump({"ok": bool(ok)}, f)
    dist.destroy_process_group()


def test_two_rank_gloo_whole_stream_entries(tmp_path):
    """The all-gather of the ranks' history maps (u64 words through int64
    tensors) and their rank-ordered composition."""
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_entry_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert json.loads((tmp_path / f"entry{r}.json").read_text()) == {"ok": True}


def _halo_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bs, nb = 64, 11
    x = torch.arange(bs * nb - 5, dtype=torch.int32) * 7 - 300
    b0, b1 = D.shard_blocks(nb, world, rank)
    s0, s1 = b0 * bs, min(x.numel(), b1 * bs)
    halo = D.lossless_halo(x[s0:s1], bs)
    want = x[max(0, s0 - bs - 2):s0]
    ok = torch.equal(halo, want) if rank > 0 else halo.numel() == 0
    with open(os.path.join(out_dir, f"halo{rank}.json"), "w") as f:
        json.dump({"ok": bool(ok)}, f)
    dist.destroy_process_group()


def test_three_rank_gloo_lossless_halo(tmp_path):
    """Rank r's halo for a whole-stream LOSSLESS encode is the (bs + 2)
    samples before its block range (the all-gather of rank tails)."""
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_halo_worker, args=(3, port, str(tmp_path)), nprocs=3, join=True)
    for r in range(3):
        assert json.loads((tmp_path / f"halo{r}.json").read_text()) == {"ok": True}
