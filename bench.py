#!/usr/bin/env python
"""Benchmark: VGG16 conv stack through the B200 RNS-Winograd path.

Workload (BASELINE.json config 4; config 2 at --batch 1): the 13 3x3 conv
layers of VGG16 on 224x224x3 int8 images, every layer an exact int32
RNS-Winograd convolution F(14x14,3x3) over RNS(4001,4331) plus the device
glue (relu, >> shift, clip, 2x2 max-pool).  Strong scaling by default: the
256-image batch of config 4 is split over the N ranks (one process per GPU,
256/N images each); ``--weak`` gives every rank --batch images instead.  The
only collective is one all-gather of the final (B,7,7,512) int8 maps.

Metric: direct-conv-equivalent INT8 TOPS = sum over layers of
2*B*Ho*Wo*C*K*9 divided by the stack latency (whole job, all ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--weak] [--impl reference]

With --gpus N > 1 and no torchrun environment, bench.py launches itself
under torch.distributed.run with N ranks (NCCL, 127.0.0.1).  One JSON line on
rank 0.  ``--impl reference`` times the CPU reference arm: the numpy
restatement of the reference's winograd_layer_conv (oracle/ref_port.py), on
the host cores, one image per worker process.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "direct-conv-equivalent INT8 TOPS and layer latency (VGG16 3x3), 1/2/4/8 B200"
UNIT = "TOPS"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=256,
                    help="global batch (strong scaling, split over the ranks); with --weak, images per GPU")
    ap.add_argument("--weak", action="store_true", help="weak scaling: every rank serves --batch images")
    ap.add_argument("--no-layer-configs", action="store_true",
                    help="skip the per-layer latency lines of BASELINE configs 1, 3 and 5")
    ap.add_argument("--impl", default="rnsw", choices=["rnsw", "reference"])
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU-only check of the multi-rank plumbing (launcher, gloo, shards, gather, max-over-ranks)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-images", type=int, default=1)
    ap.add_argument("--no-graph", action="store_true", help="launch the 39 kernels per step eagerly")
    ap.add_argument("--unfused", action="store_true",
                    help="materialise every layer's int32 output and run the glue as a separate kernel")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# CPU reference arm (oracle port of rw/layer.py:301-389; bench convention of
# rw/cli.py:445-472: filters precomputed outside the timed region)

_REF_STATE = {}


def _ref_worker_init(moduli, tile_m):
    _REF_STATE["moduli"] = moduli
    _REF_STATE["tile_m"] = tile_m


def _ref_one_image(idx):
    import numpy as np
    from oracle import ref_port
    from oracle.vgg_ref import requant_pool
    from paper_2007_12216_b200 import workloads as W

    x = W.vgg16_images(1, start=idx)
    banks, mats = _REF_STATE["banks"], _REF_STATE["mats"]
    t0 = time.perf_counter()
    for i, (name, side, c, k, pool) in enumerate(W.VGG16_LAYERS):
        y = ref_port.winograd_layer(x, _REF_STATE["weights"][i], 1, _REF_STATE["tile_m"], _REF_STATE["moduli"],
                                    mats=mats, filters=banks[i])
        x = requant_pool(y, W.VGG16_SHIFTS[i], pool)
    return time.perf_counter() - t0, int(np.asarray(x, dtype=np.int64).sum())


def _prepare_reference(moduli=(4001, 4331), tile_m=14):
    """Filter banks for the CPU path (excluded from timing, as the reference
    bench does).  Exact einsum formulation of G g G^T mod m, checked equal
    to the reference-order computation in tests/test_oracle.py."""
    from oracle import ref_port
    from paper_2007_12216_b200 import workloads as W

    weights = W.vgg16_weights()
    mats = {m: ref_port.modular_matrices(tile_m, 3, m) for m in moduli}
    banks = [ref_port.filter_bank_fast(w, mats) for w in weights]
    _REF_STATE.update(weights=weights, mats=mats, banks=banks, moduli=tuple(moduli), tile_m=tile_m)


def cpu_reference_throughput(images: int, procs: int, moduli=(4001, 4331)):
    """Time `images` images through the CPU port with `procs` worker
    processes (fork after the filter banks are built); returns
    (TOPS, seconds, per-image seconds)."""
    import multiprocessing as mp

    from paper_2007_12216_b200 import workloads as W

    if "banks" not in _REF_STATE:
        _prepare_reference(moduli)
    ops_per_image = W.VGGConfig(batch=1).direct_ops()
    t0 = time.perf_counter()
    if procs <= 1:
        res = [_ref_one_image(i) for i in range(images)]
    else:
        ctx = mp.get_context("fork")
        with ctx.Pool(procs) as pool:
            res = pool.map(_ref_one_image, range(images))
    wall = time.perf_counter() - t0
    return ops_per_image * images / wall / 1e12, wall, [r[0] for r in res]


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2007_12216_b200 import workloads as W

    n_res = 2
    cores = len(os.sched_getaffinity(0))
    procs = max(1, cores // n_res)
    _prepare_reference()
    vals = []
    for step in range(args.warmup + args.steps):
        tops, wall, per = cpu_reference_throughput(procs, procs)
        if step >= args.warmup:
            vals.append((tops, wall))
    value = statistics.median(v[0] for v in vals)
    ms = statistics.median(v[1] for v in vals) * 1e3
    sample = (f"{procs} images per step (one per worker process, {n_res} threads each: the reference's "
              f"one-thread-per-modulus pool), all 13 VGG16 layers, F(14x14,3x3) RNS(4001,4331), numpy port of "
              f"rw/layer.py winograd_layer_conv, filters precomputed")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (seeded PCG64, rw/cli.py:82-94 convention)",
        "config": {"workload": "VGG16 13x conv3x3 stack, 224x224x3, F(14x14,3x3), RNS(4001,4331), CPU sample",
                   "images_per_step": procs},
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": procs * n_res, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.out = out
        else:
            self.out = ""

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for line in self.out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measure_int8_peak(torch):
    """Dense INT8 tensor throughput on this GPU: torch._int_mm (cuBLASLt
    s8 x s8 -> s32) at 8192^3, best of 10 (burst)."""
    n = 8192
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t()
    for _ in range(3):
        torch._int_mm(a, b)
    best = float("inf")
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2 * n**3 / (best * 1e-3) / 1e12


def load_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    capture (profiles/*traffic*.json): an EARLIER capture of this build's
    kernels (ncu cannot run inside the timed bench), labelled as such."""
    for p in sorted((ROOT / "profiles").glob("*traffic*.json"), reverse=True):
        try:
            return json.loads(p.read_text()), str(p.relative_to(ROOT))
        except (OSError, ValueError):
            continue
    return {}, None


def _device_latency(torch, fn, reps: int):
    """Device time of one call of `fn` (its kernel chain), best of `reps`:
    the call is captured once as a CUDA graph and the replays are timed with
    CUDA events, so the host-side Python / ctypes work between the kernels
    (plan lookup, range check, tensor-map encoding) is not counted as device
    latency.  Falls back to events around the eager call if capture fails."""
    try:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()  # warm the plan / workspace caches on the capture stream
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        call, how = g.replay, "cuda-graph replay of the call's kernel chain, CUDA events"
    except Exception as exc:  # capture not possible: time the eager call
        torch.cuda.synchronize()
        call, how = fn, f"eager call, CUDA events ({type(exc).__name__} during graph capture)"
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, how


def layer_config_latencies(torch, reps: int = 10):
    """BASELINE configs 1, 3 and 5 as single layers through the reference
    entry point winograd_layer_conv (filters precomputed, as rw/cli.py:458-472
    does): device latency with resident torch tensors (CUDA events, best of
    `reps`), end-to-end latency with numpy host buffers in and out (the H2D
    copy, the kernels and the D2H copy, wall clock, best of `reps`), and the
    device tcgen05 direct conv beside it.  Returns {name: {...}}."""
    import numpy as np

    import paper_2007_12216_b200 as rnsw
    from paper_2007_12216_b200 import workloads as W

    cases = []
    c1, w1, x1 = W.config1()
    cases.append((c1, w1, x1))
    c3, w3, x3 = W.config3()
    cases.append((c3, w3, x3))
    w5, x5 = W.config5_operands()
    for c5 in W.config5_cases():
        cases.append((c5, w5, x5))
    out = {}
    direct_done = {}
    for case, w, x in cases:
        spec = rnsw.LayerSpec(h=case.h, w=case.w, c=case.c, k=case.k, r=case.r, padding=case.pad,
                              batch=case.batch, tile_m=case.tile_m)
        system = rnsw.RnsSystem(case.moduli)
        mts = rnsw.reduce_for_system(rnsw.cached_transforms(case.tile_m, case.r), system)
        bank = rnsw.precompute_filter_transforms(w, mts)
        xd = torch.from_numpy(x).cuda()
        wd = torch.from_numpy(w).cuda()

        def dev_call():
            return rnsw.winograd_layer_conv(spec, wd, xd, system, declared_bound=case.declared_bound, filters=bank)

        for _ in range(3):
            dev_call()
        torch.cuda.synchronize()
        best, how = _device_latency(torch, dev_call, reps)
        host_best = float("inf")
        for _ in range(max(3, reps // 2)):
            t0 = time.perf_counter()
            y = rnsw.winograd_layer_conv(spec, w, x, system, declared_bound=case.declared_bound, filters=bank)
            host_best = min(host_best, time.perf_counter() - t0)
        assert isinstance(y, np.ndarray) and y.dtype == np.int32
        rec = {"ms": round(best, 4), "timing": how, "TOPS": round(case.direct_ops() / (best * 1e-3) / 1e12, 2),
               "e2e_host_ms": round(host_best * 1e3, 4),
               "tile": f"F({case.tile_m}x{case.tile_m},{case.r}x{case.r})", "moduli": list(case.moduli)}
        dkey = (case.batch, case.h, case.c, case.k, case.r)
        if dkey not in direct_done:
            packed = rnsw.DirectWeights(wd)
            for _ in range(3):
                rnsw.direct_conv(spec, wd, xd, packed)
            torch.cuda.synchronize()
            dbest, _ = _device_latency(torch, lambda: rnsw.direct_conv(spec, wd, xd, packed), reps)
            direct_done[dkey] = round(dbest, 4)
        rec["direct_tcgen05_ms"] = direct_done[dkey]
        out[case.name] = rec
    return out


def _roofline_bound(ops: float, nbytes: float, tensor_peak_tops: float, hbm_gbs: float) -> str:
    """Which roof binds a kernel: its arithmetic intensity (int8 ops per
    algorithmic DRAM byte) against the ridge point of the two peaks."""
    ridge = tensor_peak_tops * 1e12 / (hbm_gbs * 1e9)
    return "tensor" if nbytes > 0 and ops / nbytes > ridge else "hbm"


def run_gpu_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2007_12216_b200 import _native, parallel
    from paper_2007_12216_b200 import workloads as W
    from paper_2007_12216_b200.vgg import VGG16Rns

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    # RNSW_BENCH_FORCE_DIST=1: initialise NCCL and run the gather / max-over-ranks
    # collectives even with one rank (the multi-rank code path on a one-GPU box)
    force = os.environ.get("RNSW_BENCH_FORCE_DIST") == "1" and "RANK" in os.environ
    multi = world > 1 or force
    if multi:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # strong scaling (default): config 4's batch is split over the ranks;
    # weak: every rank serves its own --batch images.  The ranks meet once,
    # in the final all-gather.
    global_batch = args.batch * world if args.weak else args.batch
    start, shard = parallel.shard_range(global_batch, world, rank)
    net = VGG16Rns()
    x_host = W.vgg16_images(shard, start=start)
    x_pinned = torch.from_numpy(x_host).pin_memory()
    x_dev = x_pinned.cuda()
    gathered = torch.empty((global_batch, 7, 7, 512), dtype=torch.int8, device="cuda") if multi else None
    out_pinned = torch.empty((global_batch if rank == 0 else shard, 7, 7, 512), dtype=torch.int8).pin_memory()

    fwd = net.forward if args.unfused else net.forward_fused
    if not args.unfused and not args.no_graph:
        # one CUDA graph per step (the same kernels, launched by the driver
        # instead of 39 ctypes calls); capture does two eager passes first
        fwd = net.graph(x_dev)
    fwd_staged = net.forward_staged if args.unfused else net.forward_fused_staged

    def step(x):
        return parallel.gather_maps(fwd(x), world, out=gathered, force=force)

    graph_used = not args.unfused and not args.no_graph

    def barrier():
        if multi:
            dist.barrier()

    # clocks are sampled from before the warm-up (nvidia-smi needs ~0.5 s to
    # produce its first sample) until the timed region ends
    gpu_index = local
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        gpu_index = vis.split(",")[local]
    with ClockSampler(gpu_index) as clocks:
        for _ in range(args.warmup):  # exactly W untimed warm-up steps
            step(x_dev)
        torch.cuda.synchronize()
        barrier()
        # -------- timed region: K steps, inputs resident in HBM --------
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step(x_dev)
        e1.record()
        torch.cuda.synchronize()
        barrier()
    elapsed = parallel.max_over_ranks(e0.elapsed_time(e1) / 1e3, world, device="cuda", force=force)
    total_ops = W.VGGConfig(batch=global_batch).direct_ops() * args.steps
    value = total_ops / elapsed / 1e12
    ms_per_step = elapsed / args.steps * 1e3

    # -------- per-kernel device times over a second timed pass --------
    rec = []
    torch.cuda.synchronize()
    for _ in range(args.steps):
        fwd_staged(x_dev, lambda kind, i, a, b: rec.append((kind, i, a, b)))
    torch.cuda.synchronize()
    per_kind, per_layer = {}, {}
    for kind, i, a, b in rec:
        dt = a.elapsed_time(b) / 1e3 / args.steps
        per_kind[kind] = per_kind.get(kind, 0.0) + dt
        per_layer.setdefault(i, {}).setdefault(kind, 0.0)
        per_layer[i][kind] += dt
    work = net.layer_work(shard, fused=not args.unfused)
    stage_sum = sum(per_kind.values())
    dominant = max(per_kind, key=per_kind.get)

    # -------- e2e: host buffers through the public API, copies timed --------
    # VGG16Rns.run_stream: every step H2D-copies its input batch from pinned
    # host memory and D2H-copies its result, on a copy stream that overlaps
    # the neighbouring steps' compute (the fused graph path; the unfused /
    # eager variants keep the serial loop)
    barrier()
    torch.cuda.synchronize()
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if graph_used:
        host_in = [x_pinned] * args.steps
        host_out = [out_pinned if rank == 0 else None] * args.steps
        post = (lambda y: parallel.gather_maps(y, world, out=gathered, force=force)) if multi else None
        net.run_stream(host_in[:2], host_out[:2], post=post)  # warm-up: graphs, buffers, streams
        torch.cuda.synchronize()
        barrier()
        h0.record()
        net.run_stream(host_in, host_out, post=post)
        h1.record()
    else:
        h0.record()
        for _ in range(args.steps):
            xd = x_pinned.to("cuda", non_blocking=True)
            y = step(xd)
            if rank == 0:
                out_pinned.copy_(y, non_blocking=True)
        h1.record()
    torch.cuda.synchronize()
    e2e_elapsed = parallel.max_over_ranks(h0.elapsed_time(h1) / 1e3, world, device="cuda", force=force)
    e2e_value = total_ops / e2e_elapsed / 1e12
    h2d = x_host.nbytes * world
    d2h = out_pinned.numel()

    if rank != 0:
        if multi:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6.65 TB/s (B200_PROFILING.md)"
    work_key = {"gemm": "gemm_bytes", "input_transform": "input_transform_bytes", "product": "product_bytes",
                "output_transform": "output_transform_bytes", "glue": "glue_bytes"}

    def kind_work(kind, key=None):
        # algorithmic work of the layers that ran this kind of kernel
        key = key or work_key[kind]
        return sum(work[i][key] for i, v in per_layer.items() if kind in v)

    int8_peak = measure_int8_peak(torch)
    dom_bytes = kind_work(dominant)
    dom_ops = kind_work(dominant, "gemm_ops") if dominant == "gemm" else 0
    bound = _roofline_bound(dom_ops, dom_bytes, int8_peak, hbm_peak)
    if bound == "tensor":
        roof = {"bound": "tensor", "achieved": round(dom_ops / per_kind[dominant] / 1e12, 3),
                "peak": round(int8_peak, 1), "unit": "TFLOP/s",
                "peak_source": "measured this run: torch._int_mm int8 8192^3 burst (MEASURED_PEAKS.json has no int8)"}
    else:
        roof = {"bound": "hbm", "achieved": round(dom_bytes / per_kind[dominant] / 1e9, 1), "peak": hbm_peak,
                "unit": "GB/s", "peak_source": hbm_src}
    roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
    roof["kernel"] = dominant
    roof["algorithmic_bytes_per_step"] = dom_bytes
    if dom_ops:
        roof["intensity_ops_per_byte"] = round(dom_ops / dom_bytes, 1)
    roof["ridge_ops_per_byte"] = round(int8_peak * 1e12 / (hbm_peak * 1e9), 1)
    traffic_tab, traffic_src = load_traffic()
    roof["traffic"] = traffic_tab.get(f"{dominant}:b{shard}")
    roof["traffic_source"] = (f"{traffic_src}: ncu dram__bytes_read.sum + dram__bytes_write.sum of this kernel's "
                              f"launches in one step, from an earlier capture (not measured in this run)"
                              if roof["traffic"] is not None else None)

    stages = {}
    for kind, sec in per_kind.items():
        st = {"ms": round(sec * 1e3, 3), "share": round(sec / stage_sum, 4),
              "GB_s": round(kind_work(kind) / sec / 1e9, 1)}
        st["frac_hbm"] = round(st["GB_s"] / hbm_peak, 4)
        if kind == "gemm":
            st["TOPS"] = round(kind_work(kind, "gemm_ops") / sec / 1e12, 2)
            st["frac_int8_peak"] = round(st["TOPS"] / int8_peak, 4)
        stages[kind] = st
    layer_ms = {work[i]["name"]: round(sum(v.values()) * 1e3, 3) for i, v in sorted(per_layer.items())}
    layer_stage_ms = {work[i]["name"]: {k: round(t * 1e3, 3) for k, t in v.items()} for i, v in sorted(per_layer.items())}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "int8",
        "dtype_note": "int8 operands on tcgen05 kind::i8 with int32 accumulation; every layer exact in int32 "
                      "(RNS residues), int8 maps between layers (BASELINE glue)",
        "data": "synthetic (seeded PCG64 images U{0..127}, weights round(N(0,20^2)) clipped; no dataset)",
        "config": {"workload": f"BASELINE config 4: VGG16 13x conv3x3 stack, 224x224x3, batch {global_batch} "
                               f"({shard} images per GPU), F(14x14,3x3), RNS(4001,4331), relu/shift/maxpool glue "
                               + ("as a separate kernel (int32 outputs materialised)" if args.unfused else
                                  "fused into each layer's output stage"),
                   "global_batch": global_batch, "per_rank_batch": shard, "tile": "F(14x14,3x3)",
                   "moduli": [4001, 4331], "parallelism": f"image-sharded x{world}, one all-gather at the end",
                   "l2": "inputs and intermediates larger than L2 (126 MB); no flush needed",
                   "layer_ms": layer_ms, "layer_stage_ms": layer_stage_ms,
                   "launch": "CUDA graph per step" if graph_used else "eager"},
        "stages": stages,
        "gpu_launches": (net.launches_per_forward() if args.unfused else net.launches_fused()) * args.steps,
        "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": round(e2e_elapsed / args.steps * 1e3, 3),
                "path": "VGG16Rns.run_stream: pinned host batch -> H2D -> 13 layers (CUDA graph) -> D2H, copies "
                        "overlapped with the neighbouring steps on a copy stream"},
        "roofline": roof,
        "int8_peak_tops_measured": round(int8_peak, 1),
        "clocks": clocks.summary(),
    }
    if _native.library_path() != _native._PRODUCT_LIB:
        line["diagnostic_library"] = str(_native.library_path())

    if world == 1 and not args.no_layer_configs:
        try:
            line["layer_configs"] = layer_config_latencies(torch)
        except Exception as exc:  # reported, never silently dropped
            line["layer_configs"] = {"error": repr(exc)}

    if world == 1 and not args.no_cpu_baseline:
        n_res = 2
        tops, wall, per = cpu_reference_throughput(args.cpu_sample_images, 1)
        line["cpu_baseline"] = {
            "value": round(tops, 6), "unit": UNIT, "cores": n_res, "kind": "port",
            "sample": f"{args.cpu_sample_images} image(s) through all 13 layers on the host, numpy port of the "
                      f"reference winograd_layer_conv (one thread per modulus, as shipped), filters precomputed; "
                      f"{wall:.1f} s",
        }
    if force:
        line["forced_collectives"] = "NCCL initialised with one rank; gather and max-over-ranks ran as collectives"
    print(json.dumps(line), flush=True)
    if multi:
        dist.barrier()
        dist.destroy_process_group()


def run_dry_arm(args):
    """The N-rank plumbing of the GPU arm without a GPU: same launcher, shard
    split, final all-gather and max-over-ranks, over gloo on CPU tensors."""
    import torch
    import torch.distributed as dist

    from paper_2007_12216_b200 import parallel

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    global_batch = args.batch * world if args.weak else args.batch
    start, shard = parallel.shard_range(global_batch, world, rank)
    local = torch.full((shard, 7, 7, 512), rank + 1, dtype=torch.int8)
    local[:, 0, 0, 0] = torch.arange(start, start + shard, dtype=torch.int64).remainder(127).to(torch.int8)
    maps = parallel.gather_maps(local, world)
    elapsed = parallel.max_over_ranks(0.001 * (rank + 1), world)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "global_batch": global_batch, "per_rank_batch": shard,
                          "scaling": "weak" if args.weak else "strong", "gathered_shape": list(maps.shape),
                          "gathered_ranks": sorted({int(v) for v in maps[:, 1, 1, 1].tolist()}),
                          "image_tags_ok": bool((maps[:, 0, 0, 0].to(torch.int64) ==
                                                 torch.arange(global_batch).remainder(127)).all()),
                          "max_elapsed_s": elapsed}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def spawn_ranks(args) -> int:
    """--gpus N without a torchrun environment: relaunch this script under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.dry_run:
        run_dry_arm(args)
    elif args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
