#!/usr/bin/env python
"""Benchmark of the B200 quantized SFC 3x3 convolution (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--workload 2]

One JSON line on rank 0.  Metric: direct-equivalent int8 TOPS (18*N*Cout*Cin*HO*WO ops of
the direct 3x3 conv each SFC conv replaces) summed over the step, whole job.  A "step" is
one pass of the hot path over the workload's batch: for the default workload (BASELINE.json
configs[1] = config 2) that is the sweep of all three 3x3 SFC variants on
x[8,128,28,28] ~ U[0,127], w ~ per-oc int8 N(0,1), with int32 y_int and fp32 outputs.

Timing: W untimed warm-up steps, then K steps between barrier + synchronize brackets;
each step is timed with CUDA events on the launching stream and an L2 flush (256 MB
write) runs between steps outside the events (the inputs are smaller than L2).
Multi-GPU (torchrun): weak scaling, every rank runs the full per-rank batch of a global
batch N times larger; the per-tensor activation scale is made global by an all-reduce(MAX)
of one int32 (quant.cpp:171-172) inside the step; time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2407_02913_b200 import workloads as wl  # noqa: E402

METRIC = "SFC int8 3x3 conv direct-equivalent TOPS/GPU and % of int8/HBM roofline"
UNIT = "TOPS"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", type=int, default=2, choices=sorted(wl.WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax = float(p[2])
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- CPU baselines
def reference_call_seconds(x, w, variant, threads=1):
    """Wall time of the reference's quantized_fast_conv2d (oracle/_ref) or, if that was not
    built, of the C oracle port.  Returns (seconds, kind)."""
    from oracle import bindings as ob
    t = time.perf_counter()
    if ob.ref_available():
        ob.ref_quantized_fast_conv2d(x, w, variant, 1)
        kind = "reference"
    else:
        ob.quantized_conv(x, w, variant, threads=threads, want=("out",), report=True)
        kind = "port"
    return time.perf_counter() - t, kind


def cpu_baseline(work: wl.Workload, budget_s: float = 12.0):
    """Single-threaded reference on a bounded sample: one image per call, cycling over the
    workload's layers and variants until ~budget_s of CPU work."""
    ops, secs, calls, kind = 0, 0.0, 0, "reference"
    li = 0
    items = [(i, L, v) for i, L in enumerate(work.layers) for v in work.variants]
    while secs < budget_s and calls < 64:
        i, L, v = items[li % len(items)]
        x = wl.activations(work.config, i, L, batch=1)
        w = wl.weights(work.config, i, L)
        dt, kind = reference_call_seconds(x, w, v)
        secs += dt
        ops += wl.direct_equivalent_ops(L, batch=1)
        calls += 1
        li += 1
    return {"value": ops / secs / 1e12, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{calls} single-image quantized_fast_conv2d calls ({work.name}, per-image scales), "
                      f"{secs:.1f} s, 1 thread (the reference hot path is single-threaded)"}


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path on the host cores."""
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor
    work = wl.WORKLOADS[args.workload]
    nthreads = os.cpu_count() or 1
    # One task = one image of one (layer, variant); ctypes releases the GIL during the call.
    tasks = []
    for i, L in enumerate(work.layers):
        w = wl.weights(work.config, i, L)
        x = wl.activations(work.config, i, L)
        for v in work.variants:
            for b in range(L.batch):
                tasks.append((x[b:b + 1], w, v, wl.direct_equivalent_ops(L, batch=1)))
    # Bound the step so the whole run ends within a few minutes.
    dt1, kind = reference_call_seconds(tasks[0][0], tasks[0][1], tasks[0][2])
    per_step_budget = 150.0 / max(1, args.steps + args.warmup)
    max_tasks = max(1, int(per_step_budget * nthreads / max(dt1, 1e-3)))
    sample = tasks if len(tasks) <= max_tasks else tasks[:: max(1, len(tasks) // max_tasks)][:max_tasks]
    step_ops = sum(t[3] for t in sample)

    def one(t):
        return reference_call_seconds(t[0], t[1], t[2])[0]

    times = []
    with ThreadPoolExecutor(max_workers=nthreads) as pool:
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            list(pool.map(one, sample))
            if s >= args.warmup:
                times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = step_ops / (ms / 1e3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": work.name, "variants": list(work.variants),
                   "sample_fraction": len(sample) / len(tasks)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": kind,
                         "sample": f"{len(sample)} of {len(tasks)} single-image quantized_fast_conv2d calls per step "
                                   f"on {nthreads} threads (reference API, per-image scales)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- peaks
def measured_peaks(torch):
    peaks = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        peaks["hbm_gbs"] = float(mp["hbm_gbs"])
        peaks["hbm_src"] = "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        pass
    # int8 tensor peak is not in MEASURED_PEAKS.json: measure cuBLASLt int8 (torch._int_mm) live.
    try:
        n = 8192
        a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t()
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        peaks["int8_tops"] = 2 * n ** 3 / (best / 1e3) / 1e12
        peaks["int8_src"] = "measured live: torch._int_mm 8192^3 best of 10"
        del a, b
    except Exception as e:  # pragma: no cover
        peaks["int8_tops"] = 4500.0
        peaks["int8_src"] = f"nominal dense int8 (measurement failed: {type(e).__name__})"
    return peaks


# --------------------------------------------------------------------------- B200 arm
def run_b200(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2407_02913_b200 import sfconv as sc
    from paper_2407_02913_b200._lib import SFC_OK  # noqa: F401  (loads fail loudly below)
    from paper_2407_02913_b200._lib import lib

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    lib()  # raise now if libsfc_b200.so is missing
    work = wl.WORKLOADS[args.workload]
    out_kind = "i8" if work.requant else ("y32" if work.config == 5 else "y32+f32")

    # ---- setup (offline filter stage is per layer, outside the timed region)
    calls = []
    rq = wl.requant_scales(work.config, len(work.layers))
    h2d_bytes = d2h_bytes = 0
    for i, L in enumerate(work.layers):
        xg = wl.activations(work.config, i, L, batch=L.batch * world)
        x_host = torch.from_numpy(np.ascontiguousarray(xg[rank * L.batch:(rank + 1) * L.batch])).pin_memory()
        x = x_host.to(dev)
        w = torch.from_numpy(wl.weights(work.config, i, L)).to(dev)
        ho = L.hw + 2 * L.pad - L.r + 1
        for v in work.variants:
            layer = sc.SfcLayer(v, w)
            ws = layer.workspace(L.batch, L.hw, L.hw, L.pad)
            oshape = (L.batch, L.cout, ho, ho)
            outs = {}
            if out_kind == "i8":
                outs["out_i8"] = torch.empty(oshape, dtype=torch.int8, device=dev)
            else:
                outs["y_int32"] = torch.empty(oshape, dtype=torch.int32, device=dev)
                if out_kind == "y32+f32":
                    outs["out_f32"] = torch.empty(oshape, dtype=torch.float32, device=dev)
            host_outs = {k: torch.empty(t.shape, dtype=t.dtype).pin_memory() for k, t in outs.items()}
            calls.append(dict(L=L, v=v, layer=layer, ws=ws, x=x, x_host=x_host, outs=outs, host_outs=host_outs,
                              vmax=torch.zeros(1, dtype=torch.int32, device=dev), rq=float(rq[i]),
                              spec=layer.spec,
                              sched_rec=layer.schedule(L.batch, L.hw, L.hw, L.pad)["recompute"],
                              p_layout=layer.schedule(L.batch, L.hw, L.hw, L.pad)["p_layout"]))
            h2d_bytes += x_host.numel()
            d2h_bytes += sum(t.numel() * t.element_size() for t in host_outs.values())
    # inputs are shared between variants of one layer: H2D once per layer
    h2d_bytes = sum(c["x_host"].numel() for c in calls if c["v"] == work.variants[0])
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    group = dist.group.WORLD if world > 1 else None

    def run_call(c):
        if world == 1:  # absmax -> act -> gemm -> output, chained with programmatic dependent launch
            c["layer"].forward(c["x"], c["ws"], c["L"].pad, requant_scale=c["rq"], **c["outs"])
            return
        # the single-GPU forward's schedule: absmax (+ V kept), all-reduce(MAX) of vmax, then
        # the quantize / contract / transform kernels
        c["vmax"].zero_()
        if c["sched_rec"]:
            c["layer"].absmax(c["x"], c["vmax"], c["L"].pad)
        else:
            c["layer"].transform(c["x"], c["vmax"], c["ws"], c["L"].pad)  # absmax, V kept in ws
        dist.all_reduce(c["vmax"], op=dist.ReduceOp.MAX, group=group)
        if c["sched_rec"]:
            c["layer"].conv(c["x"], c["vmax"], c["ws"], c["L"].pad, requant_scale=c["rq"], **c["outs"])
        else:
            c["layer"].conv_kept(tuple(c["x"].shape), c["vmax"], c["ws"], c["L"].pad, requant_scale=c["rq"],
                                 **c["outs"])

    def step():
        for c in calls:
            run_call(c)

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    # ---- warm-up
    for _ in range(args.warmup):
        step()
    sync_all()

    # ---- timed region (device time; L2 flushed between steps outside the events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local_rank)
    sync_all()
    with clocks:
        for s in range(args.steps):
            flush.zero_()
            ev[s][0].record(stream)
            step()
            ev[s][1].record(stream)
        sync_all()
    ms_local = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    step_ops = sum(wl.direct_equivalent_ops(c["L"]) for c in calls) * world
    value = step_ops / (ms / 1e3) / 1e12
    # N=1: workspace reset, absmax (+V kept), [quantizing transform,] gemm, output (per the
    # call's schedule); N>1: the reset is a torch zero_() of vmax, not one of ours
    # (the Cin <= 4 path has no GEMM launch: its contraction runs inside the output kernel)
    launches_per_step = sum((5 if c["sched_rec"] else 4) - (0 if world == 1 else 1) - (1 if c["p_layout"] == 3 else 0)
                            for c in calls)

    # ---- end to end through the public API: pinned host input -> device -> outputs -> pinned host
    # outputs go back on a copy stream as soon as their call is done, so the device-to-host
    # transfer of call i overlaps the kernels of call i+1 (the step ends when the last copy has
    # landed: the compute stream waits for the copy stream before the closing event)
    # inputs come in on an upload stream, all enqueued at the start of the step; each call waits
    # only for its own input (PCIe is full duplex: uploads overlap downloads and kernels)
    copy_stream = torch.cuda.Stream(device=dev)
    up_stream = torch.cuda.Stream(device=dev)

    def e2e_step():
        ready = {}
        up_stream.wait_stream(stream)  # (the previous step's kernels are done with the inputs)
        with torch.cuda.stream(up_stream):
            for c in calls:
                if id(c["x"]) not in ready:
                    c["x"].copy_(c["x_host"], non_blocking=True)
                    ready[id(c["x"])] = torch.cuda.Event()
                    ready[id(c["x"])].record(up_stream)
        for c in calls:
            stream.wait_event(ready[id(c["x"])])
            run_call(c)
            ev_done = torch.cuda.Event()
            ev_done.record(stream)
            copy_stream.wait_event(ev_done)
            with torch.cuda.stream(copy_stream):
                for k, t_dev in c["outs"].items():
                    c["host_outs"][k].copy_(t_dev, non_blocking=True)
                    t_dev.record_stream(copy_stream)
        stream.wait_stream(copy_stream)

    for _ in range(2):
        e2e_step()
    sync_all()
    e2e_ms = []
    for s in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_step()
        b.record(stream)
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    t = torch.tensor([sum(e2e_ms) / len(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = step_ops / (float(t.item()) / 1e3) / 1e12

    # ---- per-kernel live timing (same stream, CUDA events between the stage launches), in
    # the schedule forward() picks per call (sfc_conv_schedule): kept V = absmax (+V kept),
    # the saturation reset, the GEMM quantizing the kept V in its converter warps, the output
    # transform; recompute = absmax, reset, quantizing transform -> vq, TMA-fed GEMM, output
    stage_names = ["absmax", "sat_reset", "quantize", "gemm", "output"]
    stage_ms = {n: 0.0 for n in stage_names}
    per_call_stage = []
    L_ = lib()
    import ctypes
    reps = max(3, args.steps // 2)
    for c in calls:
        acc = {n: 0.0 for n in stage_names}
        x, ws, pad = c["x"], c["ws"], c["L"].pad
        n, _, h, w_ = x.shape
        rec = c["sched_rec"]  # the schedule forward() (N=1) and the sharded steps (N>1) run
        c["recompute"] = rec
        masks = ((1, "sat_reset"), (2, "quantize"), (4, "gemm"), (8, "output")) if rec else \
            ((1, "sat_reset"), (4 | 16, "gemm"), (8 | 16, "output"))  # 16: the kept-V path
        for _ in range(reps):
            flush.zero_()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(len(masks) + 2)]
            o = sc.Outputs(*(sc._ptr(c["outs"].get(k)) for k in ("y_int32", "y_int64", "out_f32", "out_f64", "out_i8")),
                           c["rq"])
            c["vmax"].zero_()
            e[0].record(stream)
            if rec:
                c["layer"].absmax(x, c["vmax"], pad)  # absmax only (as in forward)
            else:
                c["layer"].transform(x, c["vmax"], ws, pad)  # absmax + V kept (as in forward)
            e[1].record(stream)
            for si, (mask, _) in enumerate(masks):
                sc.check(L_.sfc_conv_int8_stages(c["layer"]._h, sc._ptr(x), n, h, w_, pad, sc._ptr(c["vmax"]),
                                                 sc._ptr(ws), ws.numel(), ctypes.byref(o), mask,
                                                 ctypes.c_void_p(stream.cuda_stream)))
                e[2 + si].record(stream)
            e[-1].synchronize()
            acc["absmax"] += e[0].elapsed_time(e[1]) / reps
            for si, (_, nme) in enumerate(masks):
                acc[nme] += e[1 + si].elapsed_time(e[2 + si]) / reps
        per_call_stage.append(acc)
        for k in stage_names:
            stage_ms[k] += acc[k]

    result = None
    if rank == 0:
        peaks = measured_peaks(torch)
        dom = max(stage_names, key=lambda k: stage_ms[k])
        # algorithmic units of the dominant kernel, summed over the step's launches
        alg_bytes = alg_ops = 0
        for c in calls:
            L, sp = c["L"], c["spec"]
            F = sp.K * sp.K
            T, _, ho = wl.tile_grid(L, sp.M)
            xb = L.batch * L.cin * L.hw * L.hw
            outb = sum(t.numel() * t.element_size() for t in c["outs"].values())
            rec = c["recompute"]
            pb = {0: 4, 1: 3, 3: 0}.get(c["p_layout"], 4)  # P bytes per value: int32, 24-bit planar, none
            if dom == "absmax":
                alg_bytes += xb + (0 if rec else 2 * F * T * L.cin)  # read x (+ keep int16 V)
            elif dom == "quantize":
                alg_bytes += xb + F * T * L.cin  # read x, write int8 vq
            elif dom == "gemm":  # reads vq (int8) or the kept V (int16) and uq, writes P
                alg_ops += 2 * F * T * L.cin * L.cout
                alg_bytes += (1 if rec else 2) * F * T * L.cin + F * L.cin * L.cout + pb * F * T * L.cout
            elif dom == "output":  # P in (or, Cin <= 4, vq words and uq: the fused dp4a contraction)
                alg_bytes += (pb * F * T * L.cout if pb else 4 * F * T + F * L.cout * 4) + outb
            else:
                alg_bytes += 64
        kms = stage_ms[dom]
        if dom == "gemm" and alg_ops / (peaks["int8_tops"] * 1e12) >= alg_bytes / (peaks["hbm_gbs"] * 1e9):
            roof = {"bound": "tensor", "achieved": alg_ops / (kms / 1e3) / 1e12, "peak": peaks["int8_tops"],
                    "unit": "TOPS", "peak_src": peaks["int8_src"]}
        else:
            roof = {"bound": "hbm", "achieved": alg_bytes / (kms / 1e3) / 1e9, "peak": peaks["hbm_gbs"],
                    "unit": "GB/s", "peak_src": peaks["hbm_src"]}
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["kernel"] = dom
        roof["kernel_share_of_step"] = kms / sum(stage_ms.values())
        roof["alg_bytes_per_launch"] = alg_bytes / len(calls)
        roof["traffic"] = None  # dram bytes per launch of this kernel (ncu --set full, profiles/)
        tr_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tr_path):
            try:
                with open(tr_path) as f:
                    tr = json.load(f)
                roof["traffic"] = tr.get(f"{work.name}:{dom}")
                if roof["traffic"]:
                    roof["traffic_src"] = tr.get("_note", "")
            except Exception:
                pass
        # whole-step roofline: sum over calls of max(ops/P, bytes/BW), algorithmic
        t_roof = 0.0
        for c in calls:
            L, sp = c["L"], c["spec"]
            F = sp.K * sp.K
            T, _, ho = wl.tile_grid(L, sp.M)
            ops = 2 * F * T * L.cin * L.cout
            b = L.batch * L.cin * L.hw * L.hw + F * L.cin * L.cout + sum(
                t.numel() * t.element_size() for t in c["outs"].values())
            t_roof += max(ops / (peaks["int8_tops"] * 1e12), b / (peaks["hbm_gbs"] * 1e9))
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "s8", "data": "synthetic (seeded numpy PCG64, SURVEY §8d seed scheme)",
            "config": {"workload": work.name, "variants": list(work.variants), "batch_per_gpu": work.layers[0].batch,
                       "layers": len(work.layers), "outputs": out_kind, "l2": "flushed between steps (256 MB write)",
                       "parallelism": f"batch-shard dp{world}"},
            "roofline": roof,
            "step_roofline": {"t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms,
                              "note": "sum over convs of max(2*K^2*T*Cin*Cout/P_int8, alg bytes/BW_hbm)"},
            "stage_ms_per_step": stage_ms,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d_bytes,
                    "d2h_bytes_per_step": d2h_bytes},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks.summary(),
            "peaks": peaks,
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                result["cpu_baseline"] = cpu_baseline(work)
            except Exception as e:  # the baseline is reported, never required
                result["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                          "sample": f"unavailable: {type(e).__name__}: {e}"}
    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps(result), flush=True)


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if world > 1 and args.impl == "b200":
        import torch.distributed as dist
        if True:
            import torch
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.impl == "reference":
            run_reference_arm(args, rank, world)
        else:
            run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            if dist.is_initialized():
                dist.destroy_process_group()


if __name__ == "__main__":
    main()
