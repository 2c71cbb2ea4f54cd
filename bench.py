"""bench.py — GPULZ compress/decompress throughput on B200 (the driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c5] [--no-cpu-baseline]

Workload (BASELINE.json's metric "... at 1/2/4/8 B200"): config c5, the 8 GiB
synthetic cuSZ-style u16 quant-code stream — 32 NYX-like 512^3 fields, seeds
42+k, one 256 MiB container each — S=2, W=255 ("window 256"
is capped at 255 by params.cpp:22-23), C=2048 symbols (4096-B chunks), I=2.
One step = one compress of the WHOLE 8 GiB stream with the input already in
HBM; the decompress of the produced image is timed the same way and
reported beside it.  Inputs (8 GiB) exceed the 126 MB L2: no flush needed.

N>1 (torchrun, NCCL): STRONG scaling — the same 8 GiB stream is split into
contiguous chunk ranges (dist.chunk_ranges), rank r holding only its range;
the timed step is the sharded compress of SURVEY.md §8e (dist.py): Kernels
I+II per rank, one NCCL all-gather of per-container sizes, rebased
table/stream segments per rank, P2P gather into ONE image on rank 0 that is
byte-identical to the single-GPU image.  value = 8 GiB / max-over-ranks time.

value        = compress GB/s of input bytes, whole job
e2e          = the same through the public C-ABI call (plzgpu_compress /
               plzgpu_decompress) with pinned HOST buffers, H2D + D2H inside
               the timed region; e2e.pageable = the same with pageable
               (malloc'd) buffers, the path a std::vector caller takes
roofline     = Kernel I (plz_bitmatch_kernel, ~98 % of a compress): its
               binding roof is the int32 ALU pipe, so `achieved` is the
               reference's matching work (one symbol compare per (aligned
               position, window candidate) pair) per second
               and `peak` the int32 lane-op rate measured in this run
               (plzgpu_int_peak, LOP3); the HBM view of the same kernel and
               the decode kernel's HBM roofline are reported beside it
cpu_baseline = oracle/_ref (the reference library, Release flags) on this
               host's cores over the stream's first container (256 MiB)
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

METRIC = "compress/decompress GB/s (input bytes) + compression ratio at 1/2/4/8 B200 vs CPU ref"
DATA = ("synthetic cuSZ-style quant codes (smooth field + halos, eb 1e-3, 3-D Lorenzo), "
        "generated on device; c5 = 32 fields, seeds 42+k")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pageable", action="store_true")
    ap.add_argument("--interval", type=int, default=0,
                    help="reference arm only: override the workload's interval I")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def config_of(w, world, interval=None):
    """The workload's config block — identical in both arms."""
    return {"workload": w.name, "S": w.S, "W": w.W, "C": w.C, "I": interval or w.I,
            "bytes": w.n_bytes, "containers": -(-w.n_bytes // (256 << 20)),
            "chunks": -(-w.n_bytes // (w.C * w.S)),
            "parallelism": (f"dp{world}: contiguous chunk-range shards of ONE stream "
                            "(strong scaling), NCCL size all-gather + P2P segment gather"
                            if world > 1 else "dp1"),
            "l2": "inputs exceed the 126 MB L2; no flush needed"}


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region.

    Polls NVML (nvidia_ml_py) from a thread every 2 ms, so even a timed region
    of a few tens of milliseconds gets samples; falls back to `nvidia-smi -lms`
    when NVML is unavailable.  __enter__ returns once the first sample is in."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons)
        self._stop = None

    def _poll_nvml(self, started):
        import pynvml as N

        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        bits = [(name, getattr(N, attr)) for name, attr in self.REASONS]
        while True:
            sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
            r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append((float(sm), float(mx), [n for n, b in bits if r & b]))
            started.set()
            if self._stop.wait(0.002):
                break
        N.nvmlShutdown()

    def _poll_smi(self, started):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={fields}",
                                 "--format=csv,noheader,nounits", "-lms", "20"],
                                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        names = [n for n, _ in self.REASONS]
        for line in proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            try:
                self.samples.append((float(parts[0]), float(parts[1]),
                                     [n for n, v in zip(names, parts[2:]) if v.lower().startswith("active")]))
            except (ValueError, IndexError):
                continue
            started.set()
            if self._stop.is_set():
                break
        proc.terminate()

    def __enter__(self):
        import threading

        self._stop = threading.Event()
        started = threading.Event()
        try:
            import pynvml  # noqa: F401
            target = self._poll_nvml
        except ImportError:
            target = self._poll_smi
        self._thread = threading.Thread(target=target, args=(started,), daemon=True)
        self._thread.start()
        started.wait(5.0)
        self.samples.clear()  # keep only samples taken inside the region
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._thread.join(timeout=5.0)

    def summary(self):
        sm = [s[0] for s in self.samples]
        mx = max((s[1] for s in self.samples), default=0)
        reasons = sorted({r for s in self.samples for r in s[2]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": reasons, "samples": len(sm)}


# ----------------------------------------------------------- reference arm
def first_container(w, device):
    """The stream's first container — a whole-container prefix of the very
    bytes the B200 arm compresses: c5's field 0 (seed 42), else the first
    256 MiB (the default block_bytes) of the workload."""
    from paper_2304_07342_b200 import datagen

    if w.fields > 1:
        return datagen.quant_codes(w, 42, device, fields=(0, 1))
    d = datagen.quant_codes(w, 42, device)
    return d[: min(d.numel(), 256 << 20)].clone()


def cpu_reference(w, steps, warmup, interval=None):
    """The reference library (oracle/_ref: its own sources, Release flags) on
    every host core over the stream's first container."""
    import numpy as np
    import torch

    import oracle as O

    dev = "cuda" if torch.cuda.is_available() else "cpu"
    host = np.ascontiguousarray(first_container(w, dev).cpu().numpy())
    n = host.size
    cores = os.cpu_count() or 1
    p = O.make_params(w.S, w.W, w.C, interval or w.I)
    kind = "reference" if O.ref_available() else "port"
    ptr = host.ctypes.data
    if kind == "reference":
        comp = lambda: O.ref_compress_into(ptr, n, p, cores)  # noqa: E731
    else:
        comp = lambda: len(O.compress(host.tobytes(), p))  # noqa: E731
        cores = 1
    for _ in range(warmup):
        img_len = comp()
    t = []
    for _ in range(steps):
        t0 = time.perf_counter()
        img_len = comp()
        t.append(time.perf_counter() - t0)
    img = O.ref_compress(host.tobytes(), p, cores) if kind == "reference" else O.compress(host.tobytes(), p)
    buf = np.frombuffer(img, dtype=np.uint8).copy()
    d = []
    for _ in range(max(1, min(steps, 3))):
        t0 = time.perf_counter()
        if kind == "reference":
            O.ref_decompress_into(buf.ctypes.data, len(img), cores)
        else:
            O.decompress(img)
        d.append(time.perf_counter() - t0)
    return {"compress_gbs": n * len(t) / sum(t) / 1e9, "decompress_gbs": n * len(d) / sum(d) / 1e9,
            "ratio": n / img_len, "cores": cores, "kind": kind, "sample_bytes": n,
            "ms_per_step": 1e3 * sum(t) / len(t),
            "sample": (f"the stream's first container: {n >> 20} MiB of {w.name} "
                       f"({'field 0, ' if w.fields > 1 else ''}seed 42), mean of {len(t)} "
                       f"compress calls after {warmup} warm-up")}


def run_reference_arm(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    from paper_2304_07342_b200 import datagen

    w = datagen.WORKLOADS[args.workload]
    try:
        r = cpu_reference(w, max(1, args.steps), max(0, args.warmup), interval=args.interval or None)
    except FileNotFoundError as e:
        print(json.dumps({"impl": "reference", "unavailable": str(e)}))
        return 0
    line = {
        "metric": METRIC, "value": r["compress_gbs"], "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": f"u{8 * w.S}",
        "data": DATA, "impl": "reference",
        "config": config_of(w, args.gpus, args.interval or None),
        "ratio": r["ratio"],
        "decompress": {"value": r["decompress_gbs"], "unit": "GB/s"},
        "cpu_baseline": {"value": r["compress_gbs"], "unit": "GB/s", "cores": r["cores"],
                         "kind": r["kind"], "sample": r["sample"],
                         "sample_bytes": r["sample_bytes"], "decompress_gbs": r["decompress_gbs"],
                         "ratio_on_sample": r["ratio"]},
        "e2e": {"value": r["compress_gbs"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- B200 arm
def local_slice(w, params, rank, world, dev):
    """This rank's contiguous chunk range of the workload stream, generated
    on its own GPU (only the fields it overlaps); the final range also
    returns the stream's raw tail (< S bytes)."""
    from paper_2304_07342_b200 import datagen
    from paper_2304_07342_b200 import dist as D

    n_total = w.n_bytes
    n_chunks, _ = D.geometry(n_total, params)
    cb, ce = D.chunk_ranges(n_chunks, world)[rank]
    lo = cb * w.C * w.S
    hi = n_total if ce == n_chunks else ce * w.C * w.S
    if w.fields > 1:
        fb = w.field_bytes
        k0, k1 = lo // fb, -(-hi // fb)
        d = datagen.quant_codes(w, 42, dev, fields=(k0, k1))
        d_local = d[lo - k0 * fb:hi - k0 * fb]
        if d_local.numel() != d.numel():
            d_local = d_local.clone()
    else:
        d = datagen.quant_codes(w, 42, dev)
        d_local = d[lo:hi].clone() if world > 1 else d
    tl = n_total % w.S if ce == n_chunks else 0
    tail = bytes(d_local[d_local.numel() - tl:].cpu().tolist()) if tl else b""
    return d_local, (cb, ce), tail, n_chunks


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2304_07342_b200 import _lib, datagen, plz
    from paper_2304_07342_b200 import dist as D

    rank, world, local = dist_env()
    gloo = os.environ.get("BENCH_DIST_BACKEND", "nccl") == "gloo"
    if gloo:
        local = 0  # every rank on cuda:0, exchanges staged through the host
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            # the rank count is visible in NCCL's init log (driver check)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
    w = datagen.WORKLOADS[args.workload]
    params = plz.validate(plz.Params(w.S, w.W, w.C, w.I))
    ctx = plz.context(local)
    stream = torch.cuda.Stream(dev)
    sh = stream.cuda_stream
    n_total = w.n_bytes
    d_in, (cb, ce), tail, n_chunks = local_slice(w, params, rank, world, dev)
    n = d_in.numel()
    cpb = (256 << 20) // (w.C * w.S)
    aligned = cb % cpb == 0 and (ce % cpb == 0 or ce == n_chunks)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    cdev = "cpu" if gloo else dev

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def reduce(x: float, op) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    def timed(fn, steps):
        """CUDA-event ms per step on `stream`, barrier + sync both sides, max over ranks."""
        barrier()
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            for _ in range(steps):
                fn()
            ev[1].record(stream)
        torch.cuda.synchronize()
        barrier()
        return reduce(ev[0].elapsed_time(ev[1]) / steps, dist.ReduceOp.MAX if world > 1 else None)

    # ---- compress (device-resident): one image of the whole stream
    if world == 1:
        cap = plz.compress_bound(n, params)
        img = torch.empty(cap, dtype=torch.uint8, device=dev)
        lens = torch.zeros(4, dtype=torch.int64, device=dev)

        def compress_step():
            ctx.compress_async(params, d_in.data_ptr(), n, img.data_ptr(), cap, lens.data_ptr(), sh)
    else:
        backend = D.GpuBackend(params, local, ctx)
        comm = D.TorchComm(cdev)
        shard_out = {}

        def compress_step():
            shard_out["img"], shard_out["len"] = D.compress_sharded(backend, comm, params, n_total,
                                                                    d_in, tail, sh)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            compress_step()
    torch.cuda.synchronize()
    if world == 1:
        ptr_tok, lit_tok = ctx.finish(sh)
        img_len = int(lens[0].item())
        launches_per_step = ctx.last_launches
    else:
        img_len = int(reduce(float(shard_out["len"]), dist.ReduceOp.MAX))
        ctx.shard_encode(params, d_in.data_ptr(), n_total, cb, ce, sh)  # its launch count
        launches_per_step = ctx.last_launches + 1 + (1 if rank == 0 else 0)
        st = ctx.finish(sh)
        ptr_tok = int(reduce(float(st[0]), dist.ReduceOp.SUM))
        lit_tok = int(reduce(float(st[1]), dist.ReduceOp.SUM))
    with ClockSampler(local) as clk:
        c_ms = timed(compress_step, args.steps)

    # ---- Kernel I alone (the roofline numerator) on this rank's bytes
    enc_ms = reduce(encode_kernel_ms(ctx, params, d_in, n, stream, args.steps),
                    dist.ReduceOp.MAX if world > 1 else None)
    # ---- per-stage CUDA-event times (Kernels I, II, III + headers) of the
    # same compress, for the scan and deflate rooflines (north_star)
    stage_ms = (ctx.profile_stages(params, d_in.data_ptr(), n, img.data_ptr(), img.numel(),
                                   max(3, min(args.steps, 5)), sh) if world == 1 else None)

    # ---- decompress (device-resident)
    if world == 1:
        out = torch.empty(n + 16, dtype=torch.uint8, device=dev)
        ctx_img = img

        def decompress_step():
            ctx.decompress_async(img.data_ptr(), img_len, out.data_ptr(), out.numel(),
                                 lens.data_ptr() + 8, sh)
    else:
        # every rank holds the one image; rank r decodes chunk range r
        if rank == 0:
            ctx_img = shard_out["img"][:img_len].contiguous()
        else:
            ctx_img = torch.empty(img_len, dtype=torch.uint8, device=dev)
        if gloo:
            buf = ctx_img.cpu()
            dist.broadcast(buf, 0)
            ctx_img = buf.to(dev)
        else:
            dist.broadcast(ctx_img, 0)
        shard_out.clear()
        dec = {}

        def decompress_step():
            dec["r"] = D.decompress_sharded(backend, comm, ctx_img, False, sh)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            decompress_step()
    if world == 1:
        ctx.finish(sh)
    d_ms = timed(decompress_step, args.steps)
    if world == 1:
        ctx.finish(sh)
        roundtrip_ok = bool(torch.equal(out[:n], d_in))
    else:
        _, dslice, dbegin = dec["r"]
        roundtrip_ok = bool(torch.equal(dslice, d_in)) and dbegin == cb * w.C * w.S
        roundtrip_ok = bool(reduce(float(roundtrip_ok), dist.ReduceOp.MIN))
        del dec
    del ctx_img
    if world == 1:
        del out

    # ---- end to end through the public call with pinned HOST buffers: at
    # N>1 each rank compresses its host shard — whole containers when the
    # ranges align with them (c5 at 1/2/4/8), so the parts concatenate to
    # the one image
    e2e = None
    if world == 1 or aligned:
        h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h_in.copy_(d_in)
        hcap = plz.compress_bound(n, params)
        h_img = torch.empty(hcap, dtype=torch.uint8, pin_memory=True)
        h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        part = {}

        def e2e_compress():
            part["len"] = ctx.compress_ptr(params, h_in.data_ptr(), n, h_img.data_ptr(), hcap, sh)[0]

        def e2e_decompress():
            ctx.decompress_ptr(h_img.data_ptr(), part["len"], h_out.data_ptr(), n, sh)

        for _ in range(max(1, args.warmup)):
            e2e_compress()
            e2e_decompress()
        e2e_c_ms = timed(e2e_compress, args.steps)
        h_out.zero_()
        e2e_d_ms = timed(e2e_decompress, args.steps)
        part_len = part["len"]
        e2e_dec_ok = bool(reduce(float(torch.equal(h_out, h_in)), dist.ReduceOp.MIN if world > 1 else None))
        if world == 1:
            same = bool(torch.equal(h_img[:part_len].to(dev), img[:img_len]))
        else:
            same = int(reduce(float(part_len), dist.ReduceOp.SUM)) == img_len
        # the link's own ceiling: plain pinned copies of the same n bytes
        link = {}
        for name, fn in (("h2d_gbs", lambda: d_in.copy_(h_in, non_blocking=True)),
                         ("d2h_gbs", lambda: h_out.copy_(d_in, non_blocking=True))):
            link[name] = n_total / (timed(fn, 3) * 1e-3) / 1e9
        e2e = {"value": n_total / (e2e_c_ms * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": n_total, "d2h_bytes_per_step": img_len,
               "matches_device_image": same,
               "decompress": {"value": n_total / (e2e_d_ms * 1e-3) / 1e9, "unit": "GB/s",
                              "h2d_bytes_per_step": img_len, "d2h_bytes_per_step": n_total,
                              "roundtrip_ok": e2e_dec_ok},
               "link": {**link, "note": "plain pinned cudaMemcpy of the same bytes: "
                                        "the PCIe ceiling e2e runs against"},
               "api": "plzgpu_compress / plzgpu_decompress (C-ABI) with pinned host buffers"
                      + ("; one call per rank on its host shard of whole containers" if world > 1 else "")}
        del h_in, h_img, h_out
        # pageable buffers (the std::vector path of plz::compress callers)
        if world == 1 and not args.no_pageable:
            e2e["pageable"] = pageable_e2e(ctx, params, d_in, n, img_len, stream, sh, timed,
                                           max(1, min(args.steps, 3)))
    else:
        e2e = {"value": None, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "note": "rank ranges do not align with containers at this N"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---- rooflines
    peak, peak_kind = load_peaks()
    int_peaks = {}
    for op, name in ((0, "lop3"), (1, "iadd3"), (2, "shf"), (3, "popc_iadd")):
        v, e = ctypes.c_double(), _lib.Error()
        if _lib.lib().plzgpu_int_peak(local, op, ctypes.byref(v), ctypes.byref(e)) == 0:
            int_peaks[name] = v.value
    nw = [1, 2, 4, 8][(w.W > 32) + (w.W > 64) + (w.W > 128)]
    prof = ncu_profile_facts(f"plz_bitmatch_kernel<{w.S}, {nw}, 12>")
    dprof = ncu_profile_facts("plz_decode_kernel<0, 1>")  # the S = 2 instance (c5)
    pairs = match_pairs(n, w)
    pairs_s = pairs / (enc_ms * 1e-3)
    lane_peak = int_peaks.get("lop3")
    enc_bytes = n + img_len / world  # input read + staged tokens written (~ image share)
    dec_bytes = img_len + n_total    # image read + output written
    dec_gbs = dec_bytes / (d_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC,
        "value": n_total / (c_ms * 1e-3) / 1e9,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": c_ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": f"u{8 * w.S}",
        "data": DATA,
        "config": config_of(w, world),
        "ratio": n_total / img_len,
        "image_bytes": img_len,
        "decompress": {"value": n_total / (d_ms * 1e-3) / 1e9, "unit": "GB/s",
                       "ms_per_step": d_ms, "roundtrip_ok": roundtrip_ok},
        "e2e": e2e,
        "roofline": {
            "kernel": f"plz_bitmatch_kernel<{w.S},{nw},12> (Kernel I: match + greedy walk + encode)",
            "bound": "int32-alu",
            "achieved": pairs_s / 1e9,
            "peak": lane_peak / 1e9 if lane_peak else None,
            "unit": "G pair-compares/s vs G int32 lane-ops/s",
            "frac": pairs_s / lane_peak if lane_peak else None,
            "traffic": prof["dram_bytes"] if prof else None,
            "peak_kind": "measured in this run (plzgpu_int_peak: LOP3 lane-ops/s)",
            "pairs_per_launch": pairs, "ms_per_launch": enc_ms,
            "note": ("achieved = the reference matcher's work (one symbol compare per aligned "
                     "position x window candidate, SURVEY.md §8d) per second; Kernel I does it "
                     "with W/32 bitmap word-ops per step, so frac may exceed 1"),
            "int_peaks_lane_ops_per_s": int_peaks,
            "alu_pipe": ({"frac": prof["alu_pipe_pct"] / 100,
                          "issue_active": prof["issue_active_pct"] / 100,
                          "source": prof["source"]} if prof and prof.get("alu_pipe_pct") else None),
            "hbm": {"achieved": enc_bytes / (enc_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                    "frac": enc_bytes / (enc_ms * 1e-3) / 1e9 / peak, "peak_kind": peak_kind,
                    "bytes_per_launch": enc_bytes},
        },
        "roofline_decompress": {
            "kernel": "plz_parse_kernel + plz_decode_kernel (decode ~98 % of the step)",
            "bound": "hbm", "achieved": dec_gbs, "peak": peak, "unit": "GB/s",
            "frac": dec_gbs / peak, "peak_kind": peak_kind, "bytes_per_step": dec_bytes,
            "traffic": dprof["dram_bytes"] if dprof else None,
            "source": dprof["source"] if dprof else None},
        "stages": stage_rooflines(stage_ms, n_chunks, img_len, peak, peak_kind),
        "tokens": {"pointer": ptr_tok, "literal": lit_tok},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            r = cpu_reference(w, 2, 0)
            line["cpu_baseline"] = {"value": r["compress_gbs"], "unit": "GB/s", "cores": r["cores"],
                                    "kind": r["kind"], "sample": r["sample"],
                                    "sample_bytes": r["sample_bytes"],
                                    "decompress_gbs": r["decompress_gbs"],
                                    "ratio_on_sample": r["ratio"]}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"unavailable": str(e)}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    print(json.dumps(line), flush=True)
    return 0


def stage_rooflines(stage_ms, n_chunks, img_len, peak, peak_kind):
    """HBM rooflines of Kernel II (global scan: psize/fsize read, P64/F64
    written — 24 B per chunk) and Kernel III + headers (staged slices read,
    image written, 24 B of prefixes/sizes per chunk read) from the live
    per-stage CUDA-event times (plzgpu_profile_stages), with the ncu DRAM
    traffic of the committed capture beside each."""
    if not stage_ms:
        return None
    out = {"source": "plzgpu_profile_stages (CUDA events on the launch stream, mean of the steps)",
           "kernel_I_ms": stage_ms[0]}
    for key, ms, name, nbytes, pat in (
            ("kernel_II", stage_ms[1], "plz_scan_kernel (decoupled look-back scan)",
             24 * n_chunks, "plz_scan_kernel"),
            ("kernel_III", stage_ms[2], "plz_assemble_batch_kernel + plz_headers_kernel (deflate)",
             2 * img_len + 24 * n_chunks, "plz_assemble")):
        prof = ncu_profile_facts(pat)
        gbs = nbytes / (ms * 1e-3) / 1e9 if ms > 0 else None
        out[key] = {"kernel": name, "ms": ms, "bound": "hbm", "bytes": nbytes, "achieved": gbs,
                    "peak": peak, "unit": "GB/s", "frac": gbs / peak if gbs else None,
                    "peak_kind": peak_kind,
                    "traffic": prof["dram_bytes"] if prof else None,
                    "source": prof["source"] if prof else None}
    return out


def pageable_e2e(ctx, params, d_in, n, img_len, stream, sh, timed, steps):
    """e2e through plzgpu_compress / plzgpu_decompress with pageable host
    buffers (what plz::compress(std::span) / std::vector callers pass)."""
    import torch

    from paper_2304_07342_b200 import plz

    cap = plz.compress_bound(n, params)
    p_in = torch.empty(n, dtype=torch.uint8)
    p_in.copy_(d_in)
    p_img = torch.empty(cap, dtype=torch.uint8)
    p_out = torch.empty(n, dtype=torch.uint8)
    part = {}

    def comp():
        part["len"] = ctx.compress_ptr(params, p_in.data_ptr(), n, p_img.data_ptr(), cap, sh)[0]

    def decomp():
        ctx.decompress_ptr(p_img.data_ptr(), part["len"], p_out.data_ptr(), n, sh)

    comp()
    decomp()
    c_ms = timed(comp, steps)
    p_out.zero_()
    d_ms = timed(decomp, steps)
    ok = part["len"] == img_len and bool(torch.equal(p_out, p_in))
    return {"value": n / (c_ms * 1e-3) / 1e9, "unit": "GB/s",
            "decompress": n / (d_ms * 1e-3) / 1e9, "steps": steps, "roundtrip_ok": ok,
            "h2d_bytes_per_step": n, "d2h_bytes_per_step": img_len}


def match_pairs(n_bytes: int, w) -> int:
    """Σ over chunks Σ over positions p ≡ 0 (mod I) of min(W, p): the
    candidate pairs the reference's find_match examines."""
    def per_chunk(m):
        k = (m + w.I - 1) // w.I                  # aligned positions 0, I, ..., < m
        full = min(k, w.W // w.I + 1)             # p = j*I <= W: min(W, p) = p
        s = w.I * full * (full - 1) // 2
        return s + (k - full) * w.W
    nsym = n_bytes // w.S
    chunks, last = divmod(nsym, w.C)
    return chunks * per_chunk(w.C) + (per_chunk(last) if last else 0)


def ncu_profile_facts(kernel: str):
    """DRAM traffic per launch and pipe utilisation of `kernel` from the newest
    committed ncu capture of this code (profiles/<round>/kernel_metrics.csv,
    tools/profile_round.sh on a B200) — not measured inside this run."""
    import csv
    import glob

    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "kernel_metrics.csv"))):
        with open(path) as fh:
            for row in csv.DictReader(fh):
                if kernel in row.get("kernel", ""):
                    best = (path, row)
    if not best:
        return None
    path, row = best
    f = lambda k: float(row[k]) if row.get(k) not in (None, "") else None  # noqa: E731
    return {"source": os.path.relpath(path, ROOT), "dram_bytes": (f("dram_read_B") or 0) +
            (f("dram_write_B") or 0), "alu_pipe_pct": f("alu_pipe_pct"),
            "issue_active_pct": f("issue_active_pct"), "sm_throughput_pct": f("sm_throughput_pct")}


def encode_kernel_ms(ctx, params, d_in, n, stream, steps):
    """CUDA-event time of Kernel I alone via the library's encode-only entry."""
    import torch

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    sh = stream.cuda_stream
    for _ in range(2):
        ctx.encode_only(params, d_in.data_ptr(), n, sh)
    ev[0].record(stream)
    for _ in range(steps):
        ctx.encode_only(params, d_in.data_ptr(), n, sh)
    ev[1].record(stream)
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / steps


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
