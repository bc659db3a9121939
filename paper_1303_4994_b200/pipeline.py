"""Copy/compute-overlapped host round trip: pinned host samples -> container
bytes + side-band block index in pinned host memory -> decoded samples in
pinned host memory, through the same C-ABI calls as the device API.

A whole-stream host round trip is PCIe-bound (the kernels take < 1 ms of a
~13 ms round trip for cfg2), so the stream is cut into chunks of whole
segments and each chunk flows through

    H2D samples -> apax_encode -> D2H container + index
                -> H2D container + index -> apax_decode_segments -> D2H samples

on one stream per copy direction (copies interleaved in the order that keeps
the other direction fed, see run()) plus one per kernel kind, so
host->device and device->host copies of different chunks run at the same
time on the two copy directions while the kernels run in between.  Segments are independent
(every segment starts with a restart block), so the chunk
containers' bodies concatenate into exactly the bytes of one encode of the
whole stream with the same segment length (the same property the multi-GPU
sharding uses, distributed.py); the host blob carries the whole-stream file
header.

The host must learn each chunk's container length before its D2H: one
event wait per chunk, issued after the next chunk's copy and encode are
already queued, so the GPU never idles on it.
"""
from __future__ import annotations

import ctypes
import struct
from typing import List, Optional

import numpy as np

from ._lib import lib as _native_lib
from .codec import FILE_HEADER_FMT, FILE_HEADER_SIZE, Decoder, Encoder, _check_status, torch_dtype
from .errors import raise_status
from .dtypes import StreamConfig
from .errors import InvalidConfig


def chunk_weights(k: int, taper: int = 1) -> List[int]:
    """Relative chunk sizes: all equal for taper <= 1, else min(2^i,
    2^(k-1-i), taper) (a geometric ramp up and down, capped)."""
    if taper <= 1:
        return [1] * k
    return [min(1 << min(i, 30), 1 << min(k - 1 - i, 30), int(taper)) for i in range(k)]


class HostRoundTrip:
    """Reusable pipelined host encode+decode plan for (n, config).

    `config.segment_blocks` must be set (chunks are whole segments).
    `chunks` is the number of pipeline chunks (rounded to segment
    boundaries).  `taper` > 1 shrinks the first and last chunks
    geometrically (weights 1, 2, 4, ... up to `taper`, mirrored): the
    pipeline fill (the first upload before any download can start) and
    drain (the last decode and download after the uploads end) then cost
    a small chunk each instead of a full one."""

    def __init__(self, n: int, config: StreamConfig, chunks: int = 8, device=None, depth: int = 3,
                 taper: int = 1):
        import torch
        if not config.segment_blocks:
            raise InvalidConfig("HostRoundTrip needs a segmented StreamConfig")
        config.validate()
        self.n, self.config = int(n), config
        self.device = torch.device(device or "cuda")
        bs, P = config.block_size, int(config.segment_blocks)
        seg_samples = bs * P
        n_seg = (self.n + seg_samples - 1) // seg_samples
        k = max(1, min(int(chunks), n_seg))
        wts = chunk_weights(k, taper)
        cw = np.concatenate([[0], np.cumsum(wts)])
        bounds = [min(self.n, int((n_seg * int(c)) // int(cw[-1])) * seg_samples) for c in cw]
        self.ranges = [(a, b) for a, b in zip(bounds, bounds[1:]) if b > a]
        self.depth = max(2, min(depth, len(self.ranges)))
        # one encoder / decoder per in-flight slot (buffers reused round-robin)
        lens = [b - a for a, b in self.ranges]
        nmax = max(lens)
        self.enc = [Encoder(nmax, config, device=self.device) for _ in range(self.depth)]
        self._enc_by_len = {}
        self.dec = {}
        for m in set(lens):
            self.dec[m] = Decoder(m, config.dtype, bs, device=self.device, alloc_y=False)
            if m != nmax:
                self._enc_by_len[m] = [Encoder(m, config, device=self.device) for _ in range(self.depth)]
        self.n_blocks = (self.n + bs - 1) // bs
        cap = sum(self.enc[0].cap for _ in self.ranges) + 64
        self.blob_d = torch.empty(cap, dtype=torch.uint8, device=self.device)   # decode-side container
        self.offs_d = torch.empty(self.n_blocks + len(self.ranges), dtype=torch.int64, device=self.device)
        self.status_log = torch.empty(len(self.ranges), 2, 4, dtype=torch.int64, device=self.device)
        self.nb_h = torch.empty(len(self.ranges), 4, dtype=torch.int64).pin_memory()
        self.offs_stage = torch.empty(self.n_blocks + len(self.ranges), dtype=torch.int64).pin_memory()
        self.s_h2d = torch.cuda.Stream(self.device)    # H2D samples and containers, interleaved
        self.s_enc = torch.cuda.Stream(self.device)    # encode kernels
        self.s_dec = torch.cuda.Stream(self.device)    # decode kernels
        self.s_d2h = torch.cuda.Stream(self.device)    # D2H containers and samples, interleaved
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self._lib = _native_lib()

    timeline = None   # set to a list to record (name, stream, start, end) CUDA events per op (tools)

    def _mark(self, stream, name):
        """Open a timeline entry on `stream`; returns a closer (no-op unless
        self.timeline is a list)."""
        import torch
        if self.timeline is None:
            return lambda: None
        a = torch.cuda.Event(enable_timing=True)
        a.record(stream)

        def close():
            b = torch.cuda.Event(enable_timing=True)
            b.record(stream)
            self.timeline.append((name, a, b))
        return close

    def _encoder(self, j: int, m: int) -> Encoder:
        pool = self.enc if m == self.enc[0].n else self._enc_by_len[m]
        return pool[j % self.depth]

    def header(self) -> bytes:
        c = self.config
        return struct.pack(FILE_HEADER_FMT, b"APAX", 1, c.dtype.wire_code, c.mode.value, 0, c.block_size,
                           self.n, float(c.target))

    def run(self, x_h, blob_h, offs_h, y_h) -> int:
        """One pipelined round trip.  x_h, y_h: pinned CPU tensors of the
        config dtype and length n; blob_h: pinned uint8 (>= container
        length); offs_h: pinned int64 (n_blocks + 1) receiving the global
        side-band index.  Returns the container length; raises the
        reference exception on any device status.

        A copy engine drains one stream's queue before it turns to another
        (measured: the container uploads waited behind every sample upload,
        so the first decoded samples left the device only after 5.8 ms of a
        10.7 ms step).  So each direction gets ONE stream with the copies in
        the order that keeps the other direction fed:
            H2D: x0, x1, c0, x2, c1, x3, ...      (c = container + index)
            D2H: c0, c1, y0, c2, y1, c3, ...
        Encode and decode kernels run on their own streams.  Chunk j + depth
        reuses chunk j's slot (device samples, encoder output, decoded
        samples) and waits on exactly the events that free it."""
        import torch
        P = int(self.config.segment_blocks)
        bs = self.config.block_size
        K = len(self.ranges)
        D = self.depth
        L = D - 1                          # sample chunks uploaded ahead of the container uploads
        ev_enc: List[Optional[torch.cuda.Event]] = [None] * K
        ev_cout: List[Optional[torch.cuda.Event]] = [None] * K
        ev_dec: List[Optional[torch.cuda.Event]] = [None] * K
        ev_y: List[Optional[torch.cuda.Event]] = [None] * K
        hdr = np.frombuffer(self.header(), np.uint8)
        blob_h[:FILE_HEADER_SIZE].copy_(torch.from_numpy(hdr.copy()))
        h2d = d2h = 0
        bodies = []
        spans = []

        def launch_encode(j):
            nonlocal h2d
            a, b = self.ranges[j]
            m = b - a
            e = self._encoder(j, m)
            slot = j % D
            xd = self._xbuf(slot, m)
            with torch.cuda.stream(self.s_h2d):
                if j >= D:
                    self.s_h2d.wait_event(ev_enc[j - D])    # encode j-D has read the slot's samples
                cl = self._mark(self.s_h2d, f"x{j}")
                xd.copy_(x_h[a:b], non_blocking=True)
                cl()
                ev_x = torch.cuda.Event()
                ev_x.record(self.s_h2d)
            h2d += m * x_h.element_size()
            self.s_enc.wait_event(ev_x)
            if j >= D:
                self.s_enc.wait_event(ev_cout[j - D])       # the slot's container has left the device
            cl = self._mark(self.s_enc, f"enc{j}")
            e.encode(xd, stream=self.s_enc)
            cl()
            # the container length reaches the host through SM stores into pinned
            # memory (apax_status_to_host): a copy-engine D2H would wait behind
            # the sample downloads queued on the D2H engine
            st = self._lib.apax_status_to_host(ctypes.c_void_p(e.status.data_ptr()),
                                               ctypes.c_void_p(self.nb_h[j].data_ptr()), 4,
                                               ctypes.c_void_p(self.s_enc.cuda_stream))
            if st:
                raise_status(st)
            with torch.cuda.stream(self.s_enc):
                ev = torch.cuda.Event()
                ev.record(self.s_enc)
            ev_enc[j] = ev

        def launch_y(j):
            nonlocal d2h
            a, b = self.ranges[j]
            m = b - a
            yd = self._ybuf(j % D, m)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(ev_dec[j])
                cl = self._mark(self.s_d2h, f"y{j}")
                y_h[a:b].copy_(yd[:m], non_blocking=True)
                cl()
                ev = torch.cuda.Event()
                ev.record(self.s_d2h)
            ev_y[j] = ev
            d2h += m * y_h.element_size()

        for j in range(min(L, K)):
            launch_encode(j)
        goff = FILE_HEADER_SIZE
        blk = 0
        for j in range(K):
            a, b = self.ranges[j]
            m = b - a
            e = self._encoder(j, m)
            slot = j % D
            ev_enc[j].synchronize()                         # the host needs the container length
            st = self.nb_h[j].numpy().view(np.uint64)
            _check_status(st)
            nb = int(st[2])
            body = nb - FILE_HEADER_SIZE
            nblk = (m + bs - 1) // bs
            # D2H container body + local index (device -> pinned host)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(ev_enc[j])
                cl = self._mark(self.s_d2h, f"cout{j}")
                blob_h[goff:goff + body].copy_(e.out[FILE_HEADER_SIZE:nb], non_blocking=True)
                stage = self.offs_stage[blk + j: blk + j + nblk + 1]
                stage.copy_(e.offsets[:nblk + 1], non_blocking=True)
                cl()
                ev_c = torch.cuda.Event()
                ev_c.record(self.s_d2h)
            ev_cout[j] = ev_c
            d2h += body + 8 * (nblk + 1)
            if j >= 1:
                launch_y(j - 1)
            # H2D container body + index back; decode from the host copy
            base = goff - FILE_HEADER_SIZE        # chunk's container view starts 28 B before its body
            with torch.cuda.stream(self.s_h2d):
                self.s_h2d.wait_event(ev_c)
                cl = self._mark(self.s_h2d, f"cin{j}")
                self.blob_d[goff:goff + body].copy_(blob_h[goff:goff + body], non_blocking=True)
                od = self.offs_d[blk + j: blk + j + nblk + 1]
                od.copy_(stage, non_blocking=True)
                cl()
                ev_ci = torch.cuda.Event()
                ev_ci.record(self.s_h2d)
            h2d += body + 8 * (nblk + 1)
            self.s_dec.wait_event(ev_ci)
            if j >= D:
                self.s_dec.wait_event(ev_y[j - D])           # the slot's decoded samples have left
            d = self.dec[m]
            yd = self._ybuf(slot, m)
            cl = self._mark(self.s_dec, f"dec{j}")
            d.decode(self.blob_d[base:], nb, od, stream=self.s_dec, out=yd, segment_blocks=P)
            cl()
            with torch.cuda.stream(self.s_dec):
                self.status_log[j, 1].copy_(d.status)
                ev_d = torch.cuda.Event()
                ev_d.record(self.s_dec)
            ev_dec[j] = ev_d
            bodies.append(body)
            goff += body
            blk += nblk
            if j + L < K:
                launch_encode(j + L)
        launch_y(K - 1)
        for ev in ev_y:
            ev.synchronize()
        # global side-band index: local offsets shifted to the body positions
        # (host arithmetic on the small index, after the copies landed)
        self._globalize(offs_h, bodies)
        for j in range(K):
            _check_status(self.status_log[j, 1].cpu().numpy().view(np.uint64))
        self.h2d_bytes, self.d2h_bytes = h2d, d2h
        return goff

    # ---- buffers ------------------------------------------------------
    def _xbuf(self, slot, m):
        import torch
        if not hasattr(self, "_xb"):
            nmax = max(b - a for a, b in self.ranges)
            self._xb = [torch.empty(nmax, dtype=torch_dtype(self.config.dtype), device=self.device)
                        for _ in range(self.depth)]
        return self._xb[slot][:m]

    def _ybuf(self, slot, m):
        import torch
        if not hasattr(self, "_yb"):
            nmax = max(b - a for a, b in self.ranges)
            self._yb = [torch.empty(nmax, dtype=torch_dtype(self.config.dtype), device=self.device)
                        for _ in range(self.depth)]
        return self._yb[slot][:m]

    def _globalize(self, offs_h, bodies) -> None:
        bs = self.config.block_size
        o = offs_h.numpy()
        st = self.offs_stage.numpy()
        goff = FILE_HEADER_SIZE
        blk = 0
        for j, (a, b) in enumerate(self.ranges):
            nblk = (b - a + bs - 1) // bs
            o[blk:blk + nblk + 1] = st[blk + j: blk + j + nblk + 1] + (goff - FILE_HEADER_SIZE)
            goff += bodies[j]
            blk += nblk
