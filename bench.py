"""Benchmark: APAX encode + decode on B200 (BASELINE.json metric
"encode & decode GB/s (input bytes) at 1/2/4/8 B200, % of HBM roofline").

Workload (N=1 line): BASELINE configs[1] = cfg2, float32 AR(2) 2^26 samples,
fixed-quality at the reference profiler's recommended SRR target, encoded as a
container of independent P-block segments (cold policy: every segment is
byte-identical to the reference encode_stream of that slice), then decoded.
P defaults to the one-wave length (every resident encoder CTA one segment:
37 blocks on a 148-SM B200); `--segment-blocks` fixes it.
One step = encode of the whole array + decode of the resulting container,
inputs resident in HBM.  `value` = input bytes / step time (GB/s).

Multi-GPU (torchrun): weak scaling, each rank encodes+decodes its own cfg2
shard (seeded per rank); the only collective is the allgather of container
byte counts that places the shards of a concatenated stream (NCCL).

`--impl reference` times the reference algorithm on the host cores: the C
oracle port (the reference is pure Python and cannot travel to the GPU box).
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "encode & decode GB/s (input bytes) at 1/2/4/8 B200, % of HBM roofline"
UNIT = "GB/s"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self._ok = True
        except Exception:  # noqa: BLE001
            pass

    def _run(self):
        N = self.N
        names = {
            0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, nm in names.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:  # noqa: BLE001
                break
            time.sleep(0.005)

    def __enter__(self):
        if self._ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._ok:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _ncu_traffic(kernel_prefix: str):
    """DRAM bytes per launch of the kernel from the committed ncu --set full
    summary (profiles/latest_ncu_summary.json), or None."""
    p = ROOT / "profiles" / "latest_ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
    except Exception:  # noqa: BLE001
        return None
    for k, v in d.items():
        if kernel_prefix in k:
            return {"bytes": v.get("dram_bytes_total"), "kernel": k,
                    "source": "profiles/latest_ncu_summary.json"}
    return None


def cpu_round_trip(x, target, seg, threads, budget_s=10.0, dt=3, mode=2, policy=0):
    """Oracle (C port of the reference) encode+decode on host cores."""
    from oracle import oracle as O
    O.lib()
    t0 = time.perf_counter()
    reps = 0
    enc_t = dec_t = 0.0
    while True:
        a = time.perf_counter()
        blob, offs, _ = O.encode(x, dt, mode, target, 4096, segment_blocks=seg, policy=policy,
                                 nthreads=threads)
        b = time.perf_counter()
        O.decode(blob, offs, nthreads=threads)
        c = time.perf_counter()
        enc_t += b - a
        dec_t += c - b
        reps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    nb = x.size * x.itemsize
    return {"gbs": nb * reps / (enc_t + dec_t) / 1e9, "enc_gbs": nb * reps / enc_t / 1e9,
            "dec_gbs": nb * reps / dec_t / 1e9, "reps": reps, "seconds": enc_t + dec_t}

# BASELINE.json configs; the N=1 headline is cfg2.
WORKLOADS = {
    "cfg1": "cfg1: int16 8 sinusoids + N(0,20^2), 2^24 samples/GPU, fixed rate 4:1 (4 bps)",
    "cfg2": "cfg2: f32 AR(2) r=0.98 x1e3, 2^26 samples/GPU, fixed-quality at the reference "
            "profiler's SRR target",
    "cfg3": "cfg3: f32 8192x8192 Gaussian random field k^-3 + U(+-1e-3 range), fixed rate 6:1",
    "cfg4": "cfg4: f64 1024^3 (8 GiB) 64 Fourier modes + N(0,1e-4), fixed rate 3:1",
    "cfg5": "cfg5: AR(1) rho=0.95 (int32 x1e6 or f32), fixed rate r:1 (bps = 32/r)",
}


def make_workload(args, rank, dev, world=1):
    """(x on the device, x on the host or None, StreamConfig, short name)."""
    import torch
    from paper_1303_4994_b200 import Dtype, Mode, StreamConfig
    from paper_1303_4994_b200 import workloads as W
    w = args.workload
    if w == "cfg1":
        xh = W.cfg1_sines_i16(1 << (args.n_log2 or 24), seed=1 + rank)
        dt, mode, target = Dtype.I16, Mode.FIXED_RATE, 4.0
    elif w == "cfg2":
        xh = W.cfg2_ar2_f32(1 << (args.n_log2 or 26), seed=2 + rank)
        dt, mode, target = Dtype.F32, Mode.FIXED_QUALITY, W.CFG2_TARGET_DB
    elif w == "cfg3":
        xh = W.cfg3_grf_f32(8192, seed=3 + rank)
        dt, mode, target = Dtype.F32, Mode.FIXED_RATE, 32.0 / 6.0
    elif w == "cfg4":
        dt, mode, target = Dtype.F64, Mode.FIXED_RATE, 64.0 / 3.0
        if args.shard_global:
            # this rank's contiguous segment range of ONE seeded 1024^3 field
            # (only its own z planes are generated)
            from paper_1303_4994_b200.distributed import shard_samples
            n_all, plane = 1 << 30, 1 << 20
            P = workload_segment_blocks(args, n_all, "f64")
            s0, s1 = shard_samples(n_all, 4096, P, world, rank)
            za, zb = s0 // plane, (s1 + plane - 1) // plane
            xd = W.cfg4_modes_f64(1024, seed=4, device=dev, z0=za, planes=zb - za)
            xd = xd[s0 - za * plane:s1 - za * plane].contiguous()
            return xd, None, dt, mode, target
        xd = W.cfg4_modes_f64(1024, seed=4 + rank, device=dev)
        return xd, None, dt, mode, target
    elif w == "cfg5":
        xh = W.cfg5_ar1(1 << (args.n_log2 or 26), args.cfg5_dtype, seed=5 + rank)
        dt = Dtype.I32 if args.cfg5_dtype == "i32" else Dtype.F32
        mode, target = Mode.FIXED_RATE, 32.0 / args.rate
    else:
        raise SystemExit(f"unknown workload {w}")
    return torch.from_numpy(xh).to(dev), xh, dt, mode, target



# One-wave segment length on B200: 148 SMs x 4 resident encoder CTAs (the
# v3 encoder's one-wave instantiation, apax_encode_wave_segment_blocks).  Both
# arms take P from this pure-Python rule so the reference arm never loads the
# GPU library; the GPU arm records the library's own answer beside it.
B200_SMS = 148
WAVE_CTAS_PER_SM = {"i8": 4, "i16": 4, "i32": 4, "f32": 4, "f64": 2}


def wave_p(n: int, dt: str = "f32") -> int:
    nb = (n + 4095) // 4096
    units = B200_SMS * WAVE_CTAS_PER_SM[dt]
    return max(1, (nb + units - 1) // units)


def workload_segment_blocks(args, n, dt: str = "f32"):
    """P of the workload: --segment-blocks, else the one-wave length (for
    --shard-global: of one eighth of the array, so the container is the same
    at every GPU count)."""
    if args.segment_blocks > 0:
        return args.segment_blocks
    if getattr(args, "shard_global", False):
        return wave_p(n // 8, dt)
    return wave_p(n, dt)


def _standalone_workloads():
    """paper_1303_4994_b200/workloads.py loaded as a module of its own (numpy
    only): the package's __init__ (and with it libapax_b200.so) is never
    imported by the reference arm."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "apax_bench_workloads", ROOT / "paper_1303_4994_b200" / "workloads.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def run_reference(args, rank):
    """--impl reference: the reference algorithm (C oracle port, a plain-C
    restatement of pkg/src/apax/codec.py + entropy.py + transform.py) on all
    host threads (OpenMP over segments), rank 0 only.  cfg1/cfg2/cfg3/cfg5:
    the GPU arm's full-size array and segment length (same config); cfg4
    (8 GiB): a 2^24-sample slab with the same P, extrapolated per block."""
    if rank != 0:
        return
    W = _standalone_workloads()
    threads = os.cpu_count() or 1
    w = args.workload
    wire = {"i16": 1, "i32": 2, "f32": 3, "f64": 4}
    same = True
    if w == "cfg1":
        x, dt, mode, target = W.cfg1_sines_i16(1 << (args.n_log2 or 24)), "i16", 1, 4.0
    elif w == "cfg3":
        x, dt, mode, target = W.cfg3_grf_f32(8192), "f32", 1, 32.0 / 6.0
    elif w == "cfg4":
        x = W.cfg4_modes_f64(1024, device="cpu", planes=16).numpy()   # 16 of the 1024 z planes
        dt, mode, target = "f64", 1, 64.0 / 3.0
        same = False
    elif w == "cfg5":
        x = W.cfg5_ar1(1 << (args.n_log2 or 26), args.cfg5_dtype)
        dt, mode, target = args.cfg5_dtype, 1, 32.0 / args.rate
    else:
        x, dt, mode, target = W.cfg2_ar2_f32(1 << (args.n_log2 or 26)), "f32", 2, W.CFG2_TARGET_DB
    full_n = (1 << 30) if w == "cfg4" else x.size
    seg = workload_segment_blocks(args, full_n, dt)
    pol = {"cold": 0, "warm_self": 1}.get(args.policy, 1 if mode == 1 else 0)
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as O
    for _ in range(max(1, min(args.warmup, 2))):
        blob, offs, _ = O.encode(x, wire[dt], mode, target, 4096, segment_blocks=seg, policy=pol,
                                 nthreads=threads)
    times = []
    for _ in range(args.steps):
        a = time.perf_counter()
        blob, offs, _ = O.encode(x, wire[dt], mode, target, 4096, segment_blocks=seg, policy=pol,
                                 nthreads=threads)
        O.decode(blob, offs, nthreads=threads)
        times.append(time.perf_counter() - a)
    t = sum(times) / len(times)
    v = x.size * x.itemsize / t / 1e9
    sample = (f"{w}: {x.size} samples ({x.nbytes >> 20} MiB {dt}) encode+decode per step, "
              f"{'the full workload' if same else 'a slab of the full array, GB/s extrapolated per block'}, "
              f"C oracle on {threads} host threads (OpenMP over segments)")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": dt, "data": "synthetic",
        "config": {"workload": WORKLOADS[w] + f"; {seg}-block {['cold', 'warm_self'][pol]} segments, "
                               "bs 4096; step = encode + decode",
                   "name": w, "n_samples": x.size, "segment_blocks": seg, "block_size": 4096,
                   "same_config": same},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--segment-blocks", type=int, default=0,
                    help="blocks per segment; 0 = one-wave (every resident encoder CTA one segment)")
    ap.add_argument("--n-log2", type=int, default=0, help="samples per GPU = 2^n (cfg1/2/5; 0 = config default)")
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS),
                    help="BASELINE config (the N=1 headline is cfg2; the others are reported beside it)")
    ap.add_argument("--cfg5-dtype", default="i32", choices=["i32", "f32"])
    ap.add_argument("--rate", type=float, default=4.0, help="cfg5 compression ratio r (bps = 32/r)")
    ap.add_argument("--policy", default="auto", choices=["auto", "cold", "warm_self"],
                    help="segment policy; auto = warm_self for fixed rate, cold for fixed quality")
    ap.add_argument("--shard-global", action="store_true",
                    help="cfg4: ranks hold contiguous segment ranges of ONE 1024^3 field (strong scaling); "
                         "the global profiler statistics are timed beside the codec step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=8, help="pipeline chunks of the e2e round trip")
    ap.add_argument("--e2e-taper", type=int, default=1,
                    help="> 1: geometric ramp of chunk sizes at both ends, capped at this weight")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: no e2e, no cpu baseline, no clocks")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1303_4994_b200 import Decoder, Dtype, Encoder, Mode, StreamConfig, decode_device
    from paper_1303_4994_b200 import workloads as W

    dev = torch.device("cuda", local)
    x, x_host, wdt, wmode, target = make_workload(args, rank, dev, world)
    n = x.numel()
    args.segment_blocks = workload_segment_blocks(args, (1 << 30) if args.shard_global else n, wdt.code)
    from paper_1303_4994_b200 import wave_segment_blocks
    lib_wave_p = wave_segment_blocks(n, wdt, wmode, 4096)
    policy = args.policy if args.policy != "auto" else (
        "warm_self" if wmode == Mode.FIXED_RATE else "cold")
    cfg = StreamConfig(wdt, 4096, wmode, target, segment_blocks=args.segment_blocks,
                       segment_policy=policy)
    width = wdt.width_bytes
    enc = Encoder(n, cfg, device=dev)
    dec = Decoder(n, wdt, 4096, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    nbytes_dev = enc.status[2:3]
    gathered = torch.zeros(world, dtype=torch.int64, device=dev)

    def step(record=None):
        if record:
            record[0].record(stream)
        enc.encode(x)
        if world > 1:  # cross-GPU offset scan: every rank's container length (inside the timed encode)
            dist.all_gather_into_tensor(gathered, nbytes_dev)
        if record:
            record[1].record(stream)
        flush.zero_()  # keep the container out of L2 for the decode timing
        if record:
            record[2].record(stream)
        dec.decode(enc.out, enc.cap, enc.offsets, segment_blocks=args.segment_blocks)
        if record:
            record[3].record(stream)
        flush.zero_()

    for _ in range(args.warmup):
        step()
    nbytes = enc.finish()
    y = dec.finish()
    # correctness of the measured output: decode(encode(x)) bit-matches a
    # second decode path (block walk) -- cheap self-consistency
    ok_roundtrip = bool(torch.isfinite(y).all().item())

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    from paper_1303_4994_b200 import _lib
    launches0 = int(_lib.lib().apax_launch_count())
    with sampler:
        t_wall0 = torch.cuda.Event(enable_timing=True)
        t_wall1 = torch.cuda.Event(enable_timing=True)
        t_wall0.record(stream)
        for k in range(args.steps):
            step(ev[k])
        t_wall1.record(stream)
        torch.cuda.synchronize()
    gpu_launches = int(_lib.lib().apax_launch_count()) - launches0
    if world > 1:
        dist.barrier()
    enc_ms = [e[0].elapsed_time(e[1]) for e in ev]
    dec_ms = [e[2].elapsed_time(e[3]) for e in ev]
    step_ms = [a + b for a, b in zip(enc_ms, dec_ms)]
    mean_step = sum(step_ms) / len(step_ms)
    mean_enc = sum(enc_ms) / len(enc_ms)
    mean_dec = sum(dec_ms) / len(dec_ms)
    if world > 1:
        t = torch.tensor([mean_step, mean_enc, mean_dec], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        mean_step, mean_enc, mean_dec = t.tolist()
        nb_all = torch.tensor([nbytes], dtype=torch.int64, device=dev)
        dist.all_reduce(nb_all)
        total_container = int(nb_all.item())
    else:
        total_container = nbytes

    in_bytes = n * width
    # whole-job input bytes: every rank's shard of one array (--shard-global)
    # or world independent arrays (weak scaling)
    job_bytes = (1 << 30) * width if args.shard_global else world * in_bytes
    value = job_bytes / (mean_step * 1e-3) / 1e9
    enc_gbs = job_bytes / world / (mean_enc * 1e-3) / 1e9
    dec_gbs = job_bytes / world / (mean_dec * 1e-3) / 1e9
    peak, peak_kind = _peaks()
    alg_enc = in_bytes + nbytes + 8 * (enc.n_blocks + 1)   # read x, write container + offsets
    alg_dec = nbytes + in_bytes + 8 * (enc.n_blocks + 1)   # read container + offsets, write y
    ach_enc = alg_enc / (mean_enc * 1e-3) / 1e9
    ach_dec = alg_dec / (mean_dec * 1e-3) / 1e9
    # the kernels bench's configs dispatch to (apax_capi.cu): v3 encoder and
    # segment-serial d3 decoder for every dtype at bs 4096
    enc_k = (_lib.lib().apax_encode_kernel_name(wdt.wire_code, cfg.mode.value, cfg.block_size,
                                                 int(cfg.segment_blocks or 0)).decode() + f"<{wdt.wire_code}")
    dec_k = f"decode_v3_kernel<{wdt.wire_code}"
    dominant = enc_k if mean_enc >= mean_dec else dec_k
    ach = ach_enc if mean_enc >= mean_dec else ach_dec  # noqa: E501

    # ---- e2e: host buffers through the C-ABI entry points ----
    # Pinned host samples -> H2D -> apax_encode -> D2H container + block index
    # -> H2D container + index -> apax_decode_segments -> D2H samples, every
    # step, pipelined over chunks of whole segments on copy-in / compute /
    # copy-out streams (paper_1303_4994_b200/pipeline.py).
    e2e = None
    if not args.no_e2e and not args.profile and x_host is not None:
        from paper_1303_4994_b200.pipeline import HostRoundTrip
        rt = HostRoundTrip(n, cfg, chunks=args.e2e_chunks, device=dev, taper=args.e2e_taper)
        xh = torch.from_numpy(x_host).pin_memory()
        blob_h = torch.empty(rt.blob_d.numel(), dtype=torch.uint8).pin_memory()
        offs_h = torch.empty(enc.n_blocks + 1, dtype=torch.int64).pin_memory()
        yh = torch.empty(n, dtype=x.dtype).pin_memory()
        e2e_steps = max(3, min(args.steps, 10))
        for _ in range(2):
            rt.run(xh, blob_h, offs_h, yh)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a = time.perf_counter()
        for _ in range(e2e_steps):
            nb = rt.run(xh, blob_h, offs_h, yh)
        e2e_s = (time.perf_counter() - a) / e2e_steps
        ok_e2e = bool(torch.equal(yh, dec.y[:n].cpu())) and \
            bool(torch.equal(blob_h[:nb], enc.out[:nb].cpu())) and \
            bool(torch.equal(offs_h, enc.offsets.cpu()))
        # index-less decode of the host container (like decode_stream(bytes)):
        # H2D container -> K5 block discovery -> decode -> D2H samples
        blob_d = torch.zeros(rt.blob_d.numel(), dtype=torch.uint8, device=dev)

        def indexless():   # the decode_stream(bytes) path: K5, segment detection, decode
            blob_d[:nb].copy_(blob_h[:nb], non_blocking=True)
            yd = decode_device(blob_d, nb)
            yh.copy_(yd, non_blocking=True)
            torch.cuda.synchronize()
        indexless()
        a = time.perf_counter()
        for _ in range(3):
            indexless()
        il_s = (time.perf_counter() - a) / 3
        ok_il = bool(torch.equal(yh, dec.y[:n].cpu()))
        # the same index-less decode with the container already in HBM:
        # apax_decode without offsets (signature scan, speculative offsets
        # checked block by block by the segment decode; the full discovery
        # and the two-pass decode gated off on the device).  CUDA events
        # around the C-ABI call on a plan made once (no host round trip)
        blob_d[:nb].copy_(blob_h[:nb])
        il_dec = Decoder(n, wdt, 4096, device=dev)
        il_dec.decode(blob_d, nb, None, stream=stream)
        il_dec.finish(stream)
        ild = []
        for _ in range(5):
            flush.zero_()   # the container out of L2, as in the timed step
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            il_dec.decode(blob_d, nb, None, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ild.append(e0.elapsed_time(e1))
        ok_il_dev = bool(torch.equal(il_dec.finish(stream)[:n].cpu(), dec.y[:n].cpu()))
        il_dev_ms = float(np.median(ild))
        if world > 1:
            t = torch.tensor([e2e_s, il_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s, il_s = t.tolist()
        e2e = {"value": world * in_bytes / e2e_s / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": rt.h2d_bytes,
               "d2h_bytes_per_step": rt.d2h_bytes,
               "ms_per_step": e2e_s * 1e3,
               "path": f"C-ABI apax_encode/apax_decode_segments with pinned host buffers, container + "
                       f"side-band block index round-tripped through the host, pipelined over "
                       f"{len(rt.ranges)} chunks of whole segments (taper {args.e2e_taper}; copy-in/compute/copy-out streams)",
               "bit_exact_vs_device_path": ok_e2e,
               "indexless_decode": {"value": world * in_bytes / il_s / 1e9, "unit": UNIT,
                                    "ms_per_step": il_s * 1e3,
                                    "path": "host container bytes only: H2D, K5 parallel block "
                                            "discovery, segment detection, decode, D2H samples",
                                    "device_ms": il_dev_ms,
                                    "device_bit_exact": ok_il_dev,
                                    "device_path": "container in HBM, no side-band index: apax_decode "
                                                   "(signature scan, speculative offsets checked by the "
                                                   "segment-serial decode; median of 5, L2 flushed)",
                                    "bit_exact_vs_device_path": ok_il}}

    # ---- --shard-global: the global profiler statistics of the one array ----
    prof = None
    if args.shard_global:
        from paper_1303_4994_b200 import distributed as D
        y_loc = dec.y[:n]
        grp = None
        if world == 1:   # a one-rank process group so the same collectives run
            import socket
            if not dist.is_initialized():
                with socket.socket() as so:
                    so.bind(("127.0.0.1", 0))
                    port = so.getsockname()[1]
                dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                        device_id=dev)
        D.sharded_window_stats(x, y_loc, wdt, grp)   # warm-up (tables, allocator)
        torch.cuda.synchronize()
        dist.barrier()
        a = time.perf_counter()
        wst = D.sharded_window_stats(x, y_loc, wdt, grp)
        wx = D.sharded_welch(x, y_loc, wdt, 0, 4096, grp)
        wd = D.sharded_welch(x, y_loc, wdt, 2, 4096, grp)
        torch.cuda.synchronize()
        t_prof = torch.tensor([time.perf_counter() - a], dtype=torch.float64, device=dev)
        dist.all_reduce(t_prof, op=dist.ReduceOp.MAX)
        prof = {"ms": float(t_prof.item()) * 1e3,
                "what": "global window statistics (rank-ordered merged sums, two-pass std, exact S2R margin by "
                        "all-reduced radix histograms) + Welch spectra of x and d over all ranks (NCCL)",
                "pearson_r": wst["pearson_r"], "srr_db": wst["srr_db"],
                "two_sigma_s2r_margin_db": wst["two_sigma_s2r_margin_db"],
                "welch_x_peak_db": float(10 * np.log10(wx.max() + 1e-30)),
                "welch_d_peak_db": float(10 * np.log10(wd.max() + 1e-30))}

    # ---- the reference's own container format: one whole stream, no segments ----
    # (encode_stream's output; what a user of the reference hands to
    # decode_stream).  Device times of its decode with and without the
    # side-band index: two passes over pseudo-segments (history maps, then the
    # samples from the composed entries).  N = 1, untimed encode.
    ref_container = None
    if world == 1 and not args.profile and not args.no_e2e and not args.shard_global and n <= (1 << 27):
        wenc = Encoder(n, StreamConfig(wdt, 4096, wmode, target), device=dev)
        wenc.encode(x)
        wnb = wenc.finish()
        wdec = Decoder(n, wdt, 4096, device=dev)

        def _timed_decode(offs):
            wdec.decode(wenc.out, wnb, offs, stream=stream)
            wdec.finish(stream)
            ts = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                wdec.decode(wenc.out, wnb, offs, stream=stream)
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            return float(np.median(ts)), wdec.finish(stream)[:n].clone()
        t_idx, y_idx = _timed_decode(wenc.offsets)
        t_il, y_il = _timed_decode(None)
        ref_container = {"what": "whole-stream container of the same array (byte-identical to the reference's "
                                 "encode_stream), decoded on the device; median of 5, L2 flushed",
                         "container_bytes": int(wnb),
                         "decode_with_index_ms": t_idx, "decode_indexless_ms": t_il,
                         "indexless_equals_indexed": bool(torch.equal(y_idx, y_il)),
                         "finite": bool(torch.isfinite(y_idx.double()).all()) if wdt.is_float else True}
        del wenc, wdec, y_idx, y_il

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        threads = os.cpu_count() or 1
        ns = max(1, (1 << 22) // (args.segment_blocks * 4096)) * args.segment_blocks * 4096
        xs = x[:ns].cpu().numpy()
        r = cpu_round_trip(xs, target, args.segment_blocks, threads, budget_s=12.0,
                           dt=wdt.wire_code, mode=wmode.value, policy=1 if policy == "warm_self" else 0)
        cpu = {"value": r["gbs"], "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{args.workload} first {xs.size} samples ({xs.nbytes >> 20} MiB, whole "
                         f"segments) encode+decode x{r['reps']}, "
                         f"C oracle (restatement of the reference), OpenMP over segments",
               "encode_gbs": r["enc_gbs"], "decode_gbs": r["dec_gbs"]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_step,
            "higher_is_better": True, "scaling": "strong" if args.shard_global else "weak",
            "vs_baseline": None, "dtype": wdt.code, "data": "synthetic",
            "config": {
                "workload": WORKLOADS[args.workload] +
                            (f" ({args.cfg5_dtype}, r={args.rate:g}, 2^{(n).bit_length() - 1} samples)"
                             if args.workload == "cfg5" else "") +
                            f"; {args.segment_blocks}-block {policy} segments, bs 4096; step = encode + "
                            "decode (device-resident)",
                "name": args.workload,
                "n_samples_per_gpu": n, "block_size": 4096,
                "segment_blocks": args.segment_blocks, "segment_policy": policy,
                "wave_segment_blocks_library": lib_wave_p,
                "mode": wmode.name, "target": target,
                "parallelism": (f"dp{world} (contiguous segment ranges of one array)" if args.shard_global
                                else f"dp{world} (segment shards)"),
                "l2": f"inputs ({in_bytes >> 20} MiB) {'larger' if in_bytes > (126 << 20) else 'smaller'} "
                      "than L2; L2 flushed (256 MiB write) between encode and decode and after decode",
            },
            "encode_gbs": enc_gbs * world, "decode_gbs": dec_gbs * world,
            "encode_ms": mean_enc, "decode_ms": mean_dec,
            "container_bytes": total_container, "ratio": job_bytes / total_container,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak,
                         "traffic": (_ncu_traffic(dominant) or {}).get("bytes"),
                         "traffic_source": (_ncu_traffic(dominant) or {}).get("source"),
                         "kernel": dominant,
                         "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": alg_enc if dominant == enc_k else alg_dec,
                         "encode": {"achieved": ach_enc, "frac": ach_enc / peak},
                         "decode": {"achieved": ach_dec, "frac": ach_dec / peak}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "profile_stats": prof,
            "reference_container": ref_container,
            "gpu_launches": gpu_launches,
            "clocks": sampler.summary(),
            "self_check": {"decoded_finite": ok_roundtrip},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
