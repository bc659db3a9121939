"""Multi-GPU sharding of the codec and the profiler statistics
(SURVEY.md §8(e)): one process per GPU, torch.distributed for the plumbing.

Encode: the stream's segments (independent: every segment starts with a
restart block) are split into contiguous ranges, one per rank.
Each rank encodes its samples into a container body; the only data-path
exchange is an all-gather of the R body lengths (int64), whose exclusive
scan places every body after the 28-byte file header of the concatenated
stream.  Bodies stay sharded (gathering a multi-GB container would cost
more than the encode); `global_block_offsets` maps a rank's side-band index
into the concatenated stream.

Decode: a rank decodes its own body (a container of its segments).  A
whole-stream container (one restart block, no segments) shards by block
ranges instead: the history entering a range (the last two quantized values
of the previous block, transform.py:31-49) is an affine function of the
history entering the previous range, so every rank decodes its range once to
get that map (apax_decode_range with map_out), the R maps (6 words each) are
all-gathered and composed in rank order, and every rank re-decodes its range
from its exact entry history (App. B of SURVEY.md).

Whole-stream LOSSLESS encode: blocks depend on their predecessor only
through the previous block's costs and the last two samples, so ranks own
contiguous block ranges and each receives the (bs + 2)-sample halo before
its range from rank r-1 (one all-gather of R tails); the bodies then
concatenate into the one-GPU whole-stream container.

Profiler: per-rank sums are all-gathered and added in rank order, so the
result is deterministic and independent of the collective's reduction tree.

The byte-level assembly is independent of which encoder produced a body;
the CPU tests drive it with gloo and the oracle.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

FILE_HEADER_FMT = "<4sBBBBIQd"   # reference codec.py:53-56
FILE_HEADER_SIZE = 28


def shard_samples(n: int, block_size: int, segment_blocks: int, world: int, rank: int) -> Tuple[int, int]:
    """[start, end) samples of `rank`'s contiguous range of whole segments
    (segments split as evenly as possible; a rank may get none)."""
    if segment_blocks < 1:
        raise ValueError("sharding needs segment_blocks >= 1")
    n_blocks = (n + block_size - 1) // block_size
    n_seg = (n_blocks + segment_blocks - 1) // segment_blocks
    s0 = (n_seg * rank) // world
    s1 = (n_seg * (rank + 1)) // world
    seg_samples = segment_blocks * block_size
    return min(n, s0 * seg_samples), min(n, s1 * seg_samples)


def file_header(dtype_wire: int, mode: int, block_size: int, count: int, target: float) -> bytes:
    """The 28-byte container header of the concatenated stream."""
    return struct.pack(FILE_HEADER_FMT, b"APAX", 1, dtype_wire, mode, 0, block_size, count, float(target))


def _all_gather_i64(value: int, group=None, device=None):
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.tensor([int(value)], dtype=torch.int64, device=device)
    out = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, t, group=group)
    return [int(v) for v in out.cpu().tolist()]


@dataclass
class ShardPlacement:
    """Where a rank's body sits in the concatenated container."""

    rank: int
    body_offset: int              # byte offset of this rank's body in the stream
    total_bytes: int              # length of the concatenated container
    body_lengths: Tuple[int, ...]


def place_bodies(body_len: int, group=None, device=None) -> ShardPlacement:
    """All-gather of the body lengths + exclusive scan (the cross-GPU offset
    scan of SURVEY.md §8(e))."""
    import torch.distributed as dist
    lens = _all_gather_i64(body_len, group, device)
    rank = dist.get_rank(group)
    off = FILE_HEADER_SIZE + sum(lens[:rank])
    return ShardPlacement(rank, off, FILE_HEADER_SIZE + sum(lens), tuple(lens))


def global_block_offsets(local_offsets: np.ndarray, placement: ShardPlacement) -> np.ndarray:
    """Side-band index of a rank's blocks in the concatenated stream: local
    offsets (relative to the rank's own container, header included) shifted
    by the body's global position; the last entry is the body end."""
    lo = np.asarray(local_offsets, dtype=np.int64)
    return lo - FILE_HEADER_SIZE + placement.body_offset


def gather_container(body: bytes, header: bytes, group=None) -> Optional[bytes]:
    """Concatenated container on rank 0 (tests and small streams only)."""
    import torch.distributed as dist
    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, body, group=group)
    if dist.get_rank(group) != 0:
        return None
    return header + b"".join(parts)


def merge_sums(local: Sequence[float], group=None, device=None) -> np.ndarray:
    """Rank-ordered sum of per-rank statistic vectors (deterministic)."""
    import torch
    import torch.distributed as dist
    v = torch.tensor(np.asarray(local, dtype=np.float64), device=device)
    world = dist.get_world_size(group)
    out = torch.empty(world * v.numel(), dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(out, v, group=group)
    parts = out.cpu().numpy().reshape(world, -1)
    acc = np.zeros(parts.shape[1])
    for r in range(world):
        acc = acc + parts[r]
    return acc


def sharded_encode(x_local, config, group=None):
    """Encode this rank's contiguous whole-segment range on its GPU; returns
    (body bytes, ShardPlacement, global block offsets).  `config` must be
    segmented (StreamConfig.segment_blocks > 0) so every body starts with a
    restart block."""
    import torch
    from .codec import encode_device
    if not config.segment_blocks:
        raise ValueError("sharded_encode needs a segmented StreamConfig")
    res = encode_device(x_local, config)
    body_len = res.nbytes - FILE_HEADER_SIZE
    dev = x_local.device if isinstance(x_local, torch.Tensor) else None
    place = place_bodies(body_len, group, dev)
    body = bytes(res.blob[FILE_HEADER_SIZE:res.nbytes].cpu().numpy().tobytes())
    offs = global_block_offsets(res.block_offsets.cpu().numpy(), place)
    return body, place, offs


# ---------------------------------------------------------------------------
# whole-stream decode across ranks: affine history maps
# ---------------------------------------------------------------------------
_M64 = (1 << 64) - 1


def shard_blocks(n_blocks: int, world: int, rank: int) -> Tuple[int, int]:
    """[b0, b1) block range of `rank` for a whole-stream container."""
    return (n_blocks * rank) // world, (n_blocks * (rank + 1)) // world


def apply_map(m: Sequence[int], h: Tuple[int, int]) -> Tuple[int, int]:
    """History leaving a range whose map is m = (m11, m12, m21, m22, c1, c2),
    given the history h entering it (mod 2^64, two's complement)."""
    m11, m12, m21, m22, c1, c2 = (int(v) & _M64 for v in m)
    h1, h2 = h
    return ((m11 * h1 + m12 * h2 + c1) & _M64, (m21 * h1 + m22 * h2 + c2) & _M64)


def range_entries(maps: Sequence[Sequence[int]]) -> list:
    """Entry history of every range, in rank order: range 0 starts the stream
    (history (0, 0)), range r+1 enters with range r's map applied to range r's
    entry."""
    out = []
    h = (0, 0)
    for m in maps:
        out.append(h)
        h = apply_map(m, h)
    return out


def whole_stream_entry(my_map: Sequence[int], group=None, device=None) -> Tuple[int, int]:
    """All-gather of the R range maps (6 x int64 each) and the exclusive
    composition in rank order: the history entering this rank's range."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    v = torch.tensor([int(x) - (1 << 64) if int(x) >= (1 << 63) else int(x) for x in my_map],
                     dtype=torch.int64, device=device)
    out = torch.empty(world * 6, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, v, group=group)
    maps = [[int(x) & _M64 for x in row] for row in out.cpu().numpy().reshape(world, 6).tolist()]
    return range_entries(maps)[dist.get_rank(group)]


def sharded_decode_whole_stream(blob, nbytes: int, offsets, group=None):
    """Decode this rank's block range of a container resident on its GPU
    (`blob`, uint8 CUDA tensor; `offsets`, the global side-band index, int64
    CUDA tensor).  Returns (y of the range, (b0, b1))."""
    import torch.distributed as dist
    from .codec import decode_range, parse_file_header
    cfg, count = parse_file_header(bytes(blob[:FILE_HEADER_SIZE].cpu().numpy().tobytes()))
    nb = (count + cfg.block_size - 1) // cfg.block_size
    b0, b1 = shard_blocks(nb, dist.get_world_size(group), dist.get_rank(group))
    if b1 <= b0:
        import torch
        return torch.empty(0, device=blob.device), (b0, b1)
    _, m = decode_range(blob, nbytes, offsets, count, cfg.dtype, cfg.block_size, b0, b1, want_map=True)
    entry = whole_stream_entry(m, group, blob.device)
    y, _ = decode_range(blob, nbytes, offsets, count, cfg.dtype, cfg.block_size, b0, b1, entry=entry)
    return y, (b0, b1)



# ---------------------------------------------------------------------------
# whole-stream LOSSLESS encode across ranks: halo exchange
# ---------------------------------------------------------------------------
def lossless_halo(x_local, block_size: int, group=None):
    """The (bs + 2) samples before this rank's range, from rank r-1: one
    all-gather of every rank's tail (equal lengths; a rank whose range is
    shorter pads on the left).  Rank 0 receives an empty halo."""
    import torch
    import torch.distributed as dist
    h = block_size + 2
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    tail = x_local[-h:] if x_local.numel() >= h else x_local
    pad = torch.zeros(h, dtype=x_local.dtype, device=x_local.device)
    pad[h - tail.numel():] = tail
    out = torch.empty(world * h, dtype=x_local.dtype, device=x_local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    if rank == 0:
        return x_local[:0]
    return out[(rank - 1) * h: rank * h]


def sharded_encode_lossless_whole_stream(x_local, first_block: int, dtype, block_size: int, group=None):
    """Encode this rank's block range of a whole-stream LOSSLESS container:
    halo exchange, range encode on this rank's GPU, body placement.  Returns
    (body bytes, ShardPlacement, global block offsets).  Every rank's range
    must start on a block boundary (shard_blocks)."""
    import torch
    from .codec import encode_lossless_range
    halo = lossless_halo(x_local, block_size, group)
    x_ext = torch.cat([halo, x_local]) if halo.numel() else x_local
    res = encode_lossless_range(x_ext, halo.numel(), first_block, dtype, block_size)
    body_len = res.nbytes - FILE_HEADER_SIZE
    place = place_bodies(body_len, group, x_local.device)
    body = bytes(res.blob[FILE_HEADER_SIZE:res.nbytes].cpu().numpy().tobytes())
    offs = global_block_offsets(res.block_offsets.cpu().numpy(), place)
    return body, place, offs


# ---------------------------------------------------------------------------
# profiler statistics across ranks: global sums and
# S2R order statistics of a sharded (x, y)
# ---------------------------------------------------------------------------
def sharded_window_stats(x_local, y_local, dtype, group=None) -> dict:
    """Window statistics of (x, y, d = x - y) split over ranks (CUDA tensors
    of `dtype`, any shard sizes): the moments, uncentred pearson_r and SRR
    from rank-ordered merges of every rank's GPU sums (profiler.py:40-48,
    127-159), the std from a second pass about the global means, and the
    2-sigma S2R margin plus the zero counts from a radix multi-select whose
    per-pass digit histograms are all-reduced (profiler.py:105-124)."""
    import math

    import torch
    import torch.distributed as dist
    from .profiler import TWO_SIGMA_COVERAGE, _key_to_ratio, _s2r_of_ratios, _select_ratio_keys, _Sums
    # collectives on the GPU with NCCL; through host tensors with gloo
    dev = x_local.device if dist.get_backend(group) == "nccl" else None
    s = _Sums(x_local, y_local, dtype)
    tot = merge_sums([s.sx, s.sy, s.sd, s.sxx, s.syy, s.sdd, s.sxy, float(s.n), float(s.zero_x),
                      float(s.zero_d)], group, dev)
    sx, sy, sd, sxx, syy, sdd, sxy = (float(v) for v in tot[:7])
    n, zero_x, zero_d = int(tot[7]), int(tot[8]), int(tot[9])
    c = _Sums(x_local, y_local, dtype, centred=True, means=(sx / n, sy / n, sd / n))
    cen = merge_sums([c.cxx or 0.0, c.cyy or 0.0, c.cdd or 0.0], group, dev)

    def reduce_hist(h):
        if dev is None:
            hc = h.cpu()
            dist.all_reduce(hc, op=dist.ReduceOp.SUM, group=group)
            h.copy_(hc)
        else:
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)

    k = math.ceil(TWO_SIGMA_COVERAGE * n)
    rank = n - k
    keys = _select_ratio_keys(x_local, y_local, dtype, [rank], True, reduce_hist=reduce_hist)
    margin = float(_s2r_of_ratios([_key_to_ratio(keys[rank])])[0])
    rms_x, rms_d = math.sqrt(sxx / n), math.sqrt(sdd / n)
    return {
        "n": n, "mean_x": sx / n, "mean_y": sy / n, "mean_d": sd / n,
        "std_x": math.sqrt(cen[0] / n), "std_y": math.sqrt(cen[1] / n), "std_d": math.sqrt(cen[2] / n),
        "pearson_r": sxy / math.sqrt(sxx * syy),
        "srr_db": (20.0 * math.log10(rms_x / rms_d)) if rms_d > 0 else math.inf,
        "two_sigma_s2r_margin_db": margin, "zero_x": zero_x, "zero_d": zero_d,
    }


def sharded_welch(x_local, y_local, dtype, which: int = 0, seg: int = 4096, group=None):
    """Welch power spectrum (profiler.py:61-74: Hann frames of `seg`, hop
    seg/2) of x (which 0), y (1) or d = x - y (2) split over ranks.  Every
    rank's shard must start on a hop boundary of the global array (all but
    the last rank hold a multiple of seg/2 samples, at least seg/2).  A rank
    sums the frames inside its shard straight from its own array; the one
    frame that straddles its end is built from its last seg/2 samples and the
    first seg/2 of rank r+1 (an all-gather of every rank's head), so the
    union of the ranks' frames is exactly the one-array frame set.  Frame
    sums (seg/2 + 1 bins) and frame counts are all-gathered and added in
    rank order.  Collectives run on the GPU under NCCL, through host tensors
    under gloo.  Returns the power spectrum (numpy f64)."""
    import torch
    import torch.distributed as dist
    from .dtypes import Dtype
    from .profiler import _welch_frame_sums, _welch_scale
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dev = x_local.device if dist.get_backend(group) == "nccl" else None
    hop = seg // 2
    n_local = int(x_local.numel())
    if rank < world - 1 and (n_local % hop or n_local < hop):
        raise ValueError("sharded_welch: every shard but the last must hold a non-zero multiple of seg/2 samples")
    cdev = dev if dev is not None else torch.device("cpu")

    def _head(t):
        h = torch.zeros(hop, dtype=torch.float64, device=cdev)
        k = min(hop, n_local)
        if t is not None and k:
            h[:k] = t[:k].to(device=cdev, dtype=torch.float64)
        return h
    hx, hy = _head(x_local), _head(y_local)
    gx = torch.empty(world * hop, dtype=torch.float64, device=cdev)
    gy = torch.empty(world * hop, dtype=torch.float64, device=cdev)
    dist.all_gather_into_tensor(gx, hx, group=group)
    dist.all_gather_into_tensor(gy, hy, group=group)
    nb = hop + 1
    tot, nf = np.zeros(nb), 0
    if n_local >= seg:   # frames inside the shard, read in the shard's own dtype
        t, k = _welch_frame_sums(x_local, y_local, dtype, which, n_local, seg)
        tot, nf = tot + t, nf + k
    if rank < world - 1:  # the frame across the boundary with rank r + 1
        xs = x_local.device
        bx = torch.cat([x_local[n_local - hop:].double(), gx[(rank + 1) * hop:(rank + 2) * hop].to(xs)])
        by = (torch.cat([y_local[n_local - hop:].double(), gy[(rank + 1) * hop:(rank + 2) * hop].to(xs)])
              if y_local is not None else None)
        t, k = _welch_frame_sums(bx.contiguous(), by.contiguous() if by is not None else None, Dtype.F64,
                                 which, seg, seg)
        tot, nf = tot + t, nf + k
    parts = merge_sums(list(tot) + [float(nf)], group, dev)
    return _welch_scale(parts[:-1], int(parts[-1]), seg)


# ---------------------------------------------------------------------------
# one array sharded by segment ranges (BASELINE cfg4): codec + global
# profiler statistics
# ---------------------------------------------------------------------------
def sharded_round_trip(x_local, config, group=None, stats: bool = True, welch_seg: int = 4096) -> dict:
    """This rank's contiguous segment range of ONE array (x_local, CUDA
    tensor of the config dtype, starting on a segment boundary): encode the
    range on this GPU, place its body in the concatenated container (the
    all-gather of body lengths + exclusive scan), decode the body, and --
    with `stats` -- the global profiler statistics of (x, y = decode) over
    all ranks: moments, pearson r, SRR and the exact S2R margin
    (sharded_window_stats) and the Welch spectra of x and d
    (sharded_welch).  Returns a dict with the placement, this rank's body
    length, decoded range and the statistics."""
    from .codec import Decoder, Encoder
    if not config.segment_blocks:
        raise ValueError("sharded_round_trip needs a segmented StreamConfig")
    n_local = int(x_local.numel())
    enc = Encoder(n_local, config, device=x_local.device)
    enc.encode(x_local)
    nbytes = enc.finish()
    place = place_bodies(nbytes - FILE_HEADER_SIZE, group, x_local.device
                         if _backend(group) == "nccl" else None)
    dec = Decoder(n_local, config.dtype, config.block_size, device=x_local.device)
    dec.decode(enc.out, nbytes, enc.offsets, segment_blocks=config.segment_blocks)
    y = dec.finish()
    out = {"placement": place, "body_len": nbytes - FILE_HEADER_SIZE, "y": y, "encoder": enc}
    if stats:
        out["window"] = sharded_window_stats(x_local, y, config.dtype, group)
        out["welch_x"] = sharded_welch(x_local, y, config.dtype, 0, welch_seg, group)
        out["welch_d"] = sharded_welch(x_local, y, config.dtype, 2, welch_seg, group)
    return out


def _backend(group=None) -> str:
    import torch.distributed as dist
    return dist.get_backend(group)
