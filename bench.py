#!/usr/bin/env python
"""Benchmark of the B200 quantized SFC 3x3 convolution (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--workload 4]
                    [--scaling strong|weak]

One JSON line on rank 0.  Metric: direct-equivalent int8 TOPS (18*N*Cout*Cin*HO*WO ops of the
direct 3x3 conv each SFC conv replaces) summed over the step, whole job.  A "step" is one pass
of the hot path over the workload's batch.  Default workload: config 4 (VGG-16's 13 convs at
batch 128, int8 requant outputs), the largest single-GPU BASELINE configuration.

Timing: W untimed warm-up steps, then K steps between barrier + synchronize brackets; each step
is timed with CUDA events on the launching stream and an L2 flush (256 MB write) runs between
steps outside the events.

Multi-GPU: `--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N local ranks (127.0.0.1).  Default scaling is strong: the global
batch of every layer is split into contiguous shards (distributed.shard_bounds), every rank
runs the absmax pass on its shard, one all-reduce(MAX) of an int32 makes the activation scale
global (quant.cpp:171-172), then the quantize / contract / transform kernels run on the shard.
Time = max over ranks.  After timing, every layer's sharded output is gathered to rank 0 and
compared byte for byte with a single-GPU forward of the whole batch.  `--scaling weak` keeps
the per-rank batch fixed instead.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2407_02913_b200 import workloads as wl  # noqa: E402

METRIC = "SFC int8 3x3 conv direct-equivalent TOPS/GPU and % of int8/HBM roofline"
UNIT = "TOPS"
# int8 dense tensor peak for the roofline denominator (not in MEASURED_PEAKS.json): cuBLASLt
# int8 (torch._int_mm 8192^3, best of 10) measured on this pool's B200s in round 1, pinned so
# the denominator does not move between runs; `--measure-int8-peak` re-measures it live.
INT8_PEAK_TOPS = 2943.0
INT8_PEAK_SRC = "pinned: torch._int_mm 8192^3 best of 10 on B200, round 1 (nominal dense 4500)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", type=int, default=4, choices=sorted(wl.WORKLOADS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the multi-GPU gather check")
    ap.add_argument("--no-graph", action="store_true", help="time direct launches instead of a captured step graph")
    ap.add_argument("--measure-int8-peak", action="store_true")
    ap.add_argument("--stages", action="store_true", help="per-kernel stage timing (always on at N=1)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` outside torchrun: run N local ranks through torch.distributed.run."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # communicator init lines show the rank count
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


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


def arm_config(work: wl.Workload, world: int, scaling: str) -> dict:
    """The `config` object both arms print (identical, so the two lines compare like for like)."""
    return {"workload": work.name, "variants": list(work.variants), "layers": len(work.layers),
            "global_batch": work.layers[0].batch * (world if scaling == "weak" else 1),
            "outputs": "i8" if work.requant else ("y32" if work.config == 5 else "y32+f32"),
            "l2": "flushed between steps (256 MB write)",
            "parallelism": f"batch-shard dp{world}", "scaling": scaling}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


# --------------------------------------------------------------------------- CPU baselines
def _best_of(fn, reps=3):
    best = 1e300
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t)
    return best


def cpu_baseline(work: wl.Workload, budget_s: float = 25.0):
    """SURVEY §8(d)'s three CPU legs, best of 3 each (as proj/tools/sfconv_cli.cpp:387-397 times
    its bench), on a bounded sample: single images of the workload's layers, cheapest first,
    until ~budget_s of CPU work.  Legs: (1) the reference's quantized_fast_conv2d as shipped
    (single-threaded; its QuantReport fills mse/snr with an fp64 direct_conv2d, quant.cpp:282);
    (2) SFC-only = (1) minus a separately timed direct_conv2d of the same shape; (3)
    fast_conv2d(threads = nproc, reduced_products = true), the reference's only multi-core path
    (fp64, not quantized; conv.cpp:532-544) on enough images to give every thread tiles."""
    from oracle import bindings as ob
    if not ob.ref_available():
        raise RuntimeError("oracle/_ref (the compiled reference) is not built")
    nproc = os.cpu_count() or 1
    order = sorted(range(len(work.layers)), key=lambda i: wl.direct_equivalent_ops(work.layers[i], batch=1))
    ops1 = t_q = t_d = 0.0
    ops3 = t_f = 0.0
    used, spent = [], 0.0
    for i in order:
        L = work.layers[i]
        v = work.variants[0]
        x1 = wl.activations(work.config, i, L, batch=1)
        w = wl.weights(work.config, i, L)
        tq = _best_of(lambda: ob.ref_quantized_fast_conv2d(x1, w, v, L.pad))
        td = _best_of(lambda: ob.ref_direct_conv2d(x1, w, L.pad))
        tiles1, _, _ = wl.tile_grid(L, 6)
        nb = min(L.batch, max(1, -(-4 * nproc // tiles1)))
        xb = wl.activations(work.config, i, L, batch=nb)
        tf = _best_of(lambda: ob.ref_fast_conv2d(xb, w, v, L.pad, threads=nproc, reduced=True))
        ops1 += wl.direct_equivalent_ops(L, batch=1)
        ops3 += wl.direct_equivalent_ops(L, batch=nb)
        t_q, t_d, t_f = t_q + tq, t_d + td, t_f + tf
        used.append(i)
        spent += 4 * (tq + td + tf)
        if spent > budget_s:
            break
    sfc_only = max(t_q - t_d, 1e-9)
    legs = {
        "quantized_fast_conv2d": {"value": ops1 / t_q / 1e12, "cores": 1,
                                  "note": "as shipped: includes the report's fp64 direct_conv2d"},
        "sfc_only": {"value": ops1 / sfc_only / 1e12, "cores": 1,
                     "note": f"quantized_fast_conv2d minus direct_conv2d ({100 * t_d / t_q:.0f}% of it)"},
        "fast_conv2d_nproc": {"value": ops3 / t_f / 1e12, "cores": nproc,
                              "note": "fp64 fast_conv2d, reduced_products, threads=nproc (not quantized)"},
    }
    return {"value": legs["sfc_only"]["value"], "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"layers {used} of {work.name}, one image each (legs 1-2) / enough images for "
                      f"{nproc} threads (leg 3), best of 3, {spent / 4:.1f} s per pass; value = leg 2 (SFC-only)",
            "legs": legs, "cpu_model": cpu_model(), "nproc": nproc}


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path (oracle/_ref, compiled
    from /root/reference/proj/src) on all host threads, SFC-only: each step runs a bounded sample
    of the workload's (layer, image) calls of quantized_fast_conv2d in a thread pool and, on the
    same pool, the direct_conv2d its QuantReport embeds (quant.cpp:282); step time = the
    difference of the two wall times."""
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor

    from oracle import bindings as ob
    work = wl.WORKLOADS[args.workload]
    nthreads = os.cpu_count() or 1
    kind = "reference" if ob.ref_available() else "port"
    if kind != "reference":
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}), flush=True)
        return
    tasks = []  # (x one image, w, variant, pad, ops)
    per_layer = max(1, nthreads // 2)
    for i, L in enumerate(work.layers):
        w = wl.weights(work.config, i, L)
        x = wl.activations(work.config, i, L, batch=min(L.batch, per_layer))
        for v in work.variants:
            for b in range(x.shape[0]):
                tasks.append((x[b:b + 1], w, v, L.pad, wl.direct_equivalent_ops(L, batch=1)))
    # bound one step to ~150 s / (steps + warmup) of wall time on the pool
    t0 = time.perf_counter()
    ob.ref_quantized_fast_conv2d(tasks[0][0], tasks[0][1], tasks[0][2], tasks[0][3])
    dt1 = time.perf_counter() - t0
    mean_ops = sum(t[4] for t in tasks) / len(tasks)
    dt_mean = dt1 * mean_ops / tasks[0][4]
    per_step_budget = 150.0 / max(1, args.steps + args.warmup)
    max_tasks = max(1, int(per_step_budget * nthreads / max(dt_mean, 1e-3)))
    sample = tasks if len(tasks) <= max_tasks else tasks[:: max(1, len(tasks) // max_tasks)][:max_tasks]
    step_ops = sum(t[4] for t in sample)

    def q(t):
        ob.ref_quantized_fast_conv2d(t[0], t[1], t[2], t[3])

    def d(t):
        ob.ref_direct_conv2d(t[0], t[1], t[3])

    times = []
    with ThreadPoolExecutor(max_workers=nthreads) as pool:
        for s in range(args.warmup + args.steps):
            a = time.perf_counter()
            list(pool.map(q, sample))
            b = time.perf_counter()
            list(pool.map(d, sample))
            c = time.perf_counter()
            if s >= args.warmup:
                times.append(max((b - a) - (c - b), 1e-9))
    ms = 1e3 * sum(times) / len(times)
    value = step_ops / (ms / 1e3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded numpy PCG64, SURVEY §8d seed scheme)",
        "impl": "reference", "config": arm_config(work, world, args.scaling),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": kind,
                         "sample": f"{len(sample)} of the workload's single-image calls per step "
                                   f"({step_ops / 1e12:.4f} TOP direct-equivalent), SFC-only = "
                                   f"quantized_fast_conv2d wall minus direct_conv2d wall on {nthreads} threads "
                                   f"(reference API; per-image activation scales)",
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- peaks
def measured_peaks(torch, live_int8: bool):
    peaks = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)",
             "int8_tops": INT8_PEAK_TOPS, "int8_src": INT8_PEAK_SRC}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        peaks["hbm_gbs"] = float(mp["hbm_gbs"])
        peaks["hbm_src"] = "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        pass
    if live_int8:
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
        peaks["int8_tops_live"] = 2 * n ** 3 / (best / 1e3) / 1e12
    return peaks


def conv_roofline(L, spec, out_bytes, peaks, batch):
    """SURVEY §8(d) per conv: ops = 2 K^2 T Cin Cout (the full schedule executed), algorithmic
    bytes = x (int8) + uq (int8, K^2 Cin Cout) + the outputs written; t_roof = max of the two."""
    F = spec.K * spec.K
    T, _, _ = wl.tile_grid(L, spec.M, batch=batch)
    ops = 2 * F * T * L.cin * L.cout
    byts = batch * L.cin * L.hw * L.hw + F * L.cin * L.cout + out_bytes
    t_t, t_h = ops / (peaks["int8_tops"] * 1e12), byts / (peaks["hbm_gbs"] * 1e9)
    return ops, byts, t_t, t_h


# --------------------------------------------------------------------------- B200 arm
def run_b200(args, rank, world, local_rank):
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2407_02913_b200 import sfconv as sc
    from paper_2407_02913_b200._lib import lib
    from paper_2407_02913_b200.distributed import ShardedConv, shard_bounds

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L_ = lib()  # raises now if libsfc_b200.so is missing: there is no fallback path
    work = wl.WORKLOADS[args.workload]
    cfg = arm_config(work, world, args.scaling)
    out_kind = cfg["outputs"]
    strong = args.scaling == "strong"

    # ---- setup (the offline filter stage is per layer, outside the timed region)
    calls = []
    rq = wl.requant_scales(work.config, len(work.layers))
    for i, L in enumerate(work.layers):
        gb = L.batch if strong else L.batch * world
        lo, hi = shard_bounds(gb, rank, world)
        xg = wl.activations(work.config, i, L, batch=gb)
        x_host = torch.from_numpy(np.ascontiguousarray(xg[lo:hi])).pin_memory()
        x = x_host.to(dev)
        w = torch.from_numpy(wl.weights(work.config, i, L)).to(dev)
        ho = L.hw + 2 * L.pad - L.r + 1
        nb = hi - lo
        for v in work.variants:
            layer = sc.SfcLayer(v, w)
            ws = layer.workspace(max(nb, 1), L.hw, L.hw, L.pad)
            oshape = (nb, L.cout, ho, ho)
            outs = {}
            if out_kind == "i8":
                outs["out_i8"] = torch.empty(oshape, dtype=torch.int8, device=dev)
            else:
                outs["y_int32"] = torch.empty(oshape, dtype=torch.int32, device=dev)
                if out_kind == "y32+f32":
                    outs["out_f32"] = torch.empty(oshape, dtype=torch.float32, device=dev)
            host_outs = {k: torch.empty(t.shape, dtype=t.dtype).pin_memory() for k, t in outs.items()}
            sched = layer.schedule(max(nb, 1), L.hw, L.hw, L.pad)
            calls.append(dict(i=i, L=L, v=v, layer=layer, ws=ws, x=x, x_host=x_host, outs=outs,
                              host_outs=host_outs, vmax=torch.zeros(1, dtype=torch.int32, device=dev),
                              rq=float(rq[i]), spec=layer.spec, nb=nb, gb=gb, lo=lo,
                              sched_rec=sched["recompute"], p_layout=sched["p_layout"], w=w))
    h2d_bytes = sum(c["x_host"].numel() for c in calls if c["v"] == work.variants[0])
    d2h_bytes = sum(t.numel() * t.element_size() for c in calls for t in c["host_outs"].values())
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    group = dist.group.WORLD if world > 1 else None

    def run_call(c):
        if world == 1:  # one forward: every kernel of the conv chained with programmatic dependent launch
            c["layer"].forward(c["x"], c["ws"], c["L"].pad, requant_scale=c["rq"], **c["outs"])
            return
        # sharded: the single-GPU schedule split at the exchange -- absmax (+ V kept) on the
        # shard, all-reduce(MAX) of the int32 vmax, then quantize / contract / transform
        c["vmax"].zero_()
        if c["nb"] > 0:
            if c["sched_rec"]:
                c["layer"].absmax(c["x"], c["vmax"], c["L"].pad)
            else:
                c["layer"].transform(c["x"], c["vmax"], c["ws"], c["L"].pad)
        dist.all_reduce(c["vmax"], op=dist.ReduceOp.MAX, group=group)
        if c["nb"] == 0:
            return
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

    # One step's launches as a CUDA graph (single GPU): the same kernels with their programmatic
    # dependent-launch edges, replayed without the per-launch host cost (ctypes, tensor-map
    # encoding), which otherwise starves the GPU between the short kernels of small layers.
    graph = None
    if world == 1 and not args.no_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):  # (captured on torch's side stream; replays on `stream`)
                step()
            sync_all()
            for _ in range(2):
                graph.replay()
            sync_all()
        except Exception as exc:  # capture unsupported here: time the launches directly
            print(f"[bench] CUDA graph capture failed ({exc}); timing direct launches", file=sys.stderr)
            graph = None
            torch.cuda.synchronize()

    # ---- timed region (device time; L2 flushed between steps outside the events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local_rank)
    sync_all()
    with clocks:
        for s in range(args.steps):
            flush.zero_()
            ev[s][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step()
            ev[s][1].record(stream)
        sync_all()
    ms_local = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    step_ops = sum(wl.direct_equivalent_ops(c["L"], batch=c["gb"]) for c in calls)
    value = step_ops / (ms / 1e3) / 1e12
    # kernels of ours per step (sfc_conv_schedule): the workspace reset, absmax (+V kept),
    # [quantizing transform,] gemm, output; Cin <= 4 has no GEMM launch; N>1 replaces the
    # reset kernel by a torch zero_() of vmax
    launches_per_step = sum((5 if c["sched_rec"] else 4) - (0 if world == 1 else 1) - (1 if c["p_layout"] == 3 else 0)
                            for c in calls if c["nb"] > 0)

    # ---- end to end through the public API: pinned host input -> device -> outputs -> pinned host
    # inputs come in on an upload stream (all enqueued at the start of the step; each call waits
    # only for its own input), outputs go back on a copy stream as soon as their call is done
    copy_stream = torch.cuda.Stream(device=dev)
    up_stream = torch.cuda.Stream(device=dev)

    def e2e_step():
        ready = {}
        up_stream.wait_stream(stream)
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

    # ---- multi-GPU: gather every layer's shards to rank 0, compare with a 1-GPU forward
    mcheck = None
    if world > 1 and not args.no_check:
        step()
        torch.cuda.synchronize()
        ok = total = 0
        for c in calls:
            k = next(iter(c["outs"]))
            full = ShardedConv.gather_to_rank0(c["outs"][k], c["gb"])
            if rank == 0:
                xg = torch.from_numpy(wl.activations(work.config, c["i"], c["L"], batch=c["gb"])).to(dev)
                ref = torch.empty_like(full)
                ws = c["layer"].workspace(c["gb"], c["L"].hw, c["L"].hw, c["L"].pad)
                c["layer"].forward(xg, ws, c["L"].pad, requant_scale=c["rq"], **{k: ref})
                torch.cuda.synchronize()
                ok += int(torch.equal(full, ref))
                total += 1
                del ws, xg, ref
        if rank == 0:
            mcheck = {"layers_bit_exact": ok, "layers": total,
                      "what": "gathered sharded outputs vs a single-GPU forward of the whole batch"}

    # ---- per-kernel live timing on the launching stream (CUDA events between the stage
    # launches), in the schedule forward() picks per call (sfc_conv_schedule)
    stage_names = ["absmax", "sat_reset", "quantize", "gemm", "output"]
    stage_ms = {n: 0.0 for n in stage_names}
    if world == 1 or args.stages:
        reps = max(3, args.steps // 2)
        for c in calls:
            if c["nb"] == 0:
                continue
            x, ws, pad = c["x"], c["ws"], c["L"].pad
            n, _, h, w_ = x.shape
            rec = c["sched_rec"]
            masks = ((1, "sat_reset"), (2, "quantize"), (4, "gemm"), (8, "output")) if rec else \
                ((1, "sat_reset"), (4 | 16, "gemm"), (8 | 16, "output"))  # 16: the kept-V path
            for _ in range(reps):
                flush.zero_()
                e = [torch.cuda.Event(enable_timing=True) for _ in range(len(masks) + 2)]
                o = sc.Outputs(*(sc._ptr(c["outs"].get(k)) for k in ("y_int32", "y_int64", "out_f32", "out_f64",
                                                                      "out_i8")), c["rq"])
                c["vmax"].zero_()
                e[0].record(stream)
                if rec:
                    c["layer"].absmax(x, c["vmax"], pad)
                else:
                    c["layer"].transform(x, c["vmax"], ws, pad)
                e[1].record(stream)
                for si, (mask, _) in enumerate(masks):
                    sc.check(L_.sfc_conv_int8_stages(c["layer"]._h, sc._ptr(x), n, h, w_, pad, sc._ptr(c["vmax"]),
                                                     sc._ptr(ws), ws.numel(), ctypes.byref(o), mask,
                                                     ctypes.c_void_p(stream.cuda_stream)))
                    e[2 + si].record(stream)
                e[-1].synchronize()
                stage_ms["absmax"] += e[0].elapsed_time(e[1]) / reps
                for si, (_, nme) in enumerate(masks):
                    stage_ms[nme] += e[1 + si].elapsed_time(e[2 + si]) / reps

    result = None
    if rank == 0:
        peaks = measured_peaks(torch, args.measure_int8_peak)
        # SURVEY §8(d) roofline of the whole step: sum over convs of max(ops / P_int8, alg bytes / BW)
        t_roof = t_ten = t_hbm = 0.0
        tot_ops = tot_bytes = 0
        for c in calls:  # per GPU: rank 0's shard (the largest one under shard_bounds)
            if c["nb"] == 0:
                continue
            ob_ = sum(tt.numel() * tt.element_size() for tt in c["outs"].values())
            ops, byts, tt_, th_ = conv_roofline(c["L"], c["spec"], ob_, peaks, c["nb"])
            tot_ops += ops
            tot_bytes += byts
            t_roof += max(tt_, th_)
            t_ten += tt_ if tt_ >= th_ else 0.0
            t_hbm += th_ if th_ > tt_ else 0.0
        frac = t_roof * 1e3 / ms
        bound = "hbm" if t_hbm >= t_ten else "tensor"
        peak = peaks["hbm_gbs"] if bound == "hbm" else peaks["int8_tops"]
        dom = max(stage_names, key=lambda k: stage_ms[k]) if any(stage_ms.values()) else None
        roof = {"bound": bound, "achieved": frac * peak, "peak": peak, "unit": "GB/s" if bound == "hbm" else "TOPS",
                "frac": frac, "peak_src": peaks["hbm_src"] if bound == "hbm" else peaks["int8_src"],
                "kernel": "whole SFC conv (all launches of each conv, summed over the step)",
                "alg_bytes_per_step": tot_bytes, "alg_ops_per_step": tot_ops,
                "t_roof_ms": t_roof * 1e3,
                "definition": "SURVEY §8(d): t_roof = sum over convs of max(2*K^2*T*Cin*Cout / P_int8, "
                              "(x + uq + outputs) bytes / BW_hbm); frac = t_roof / measured step time; "
                              "achieved = frac * peak",
                "traffic": None}
        tr_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tr_path):
            try:
                with open(tr_path) as f:
                    tr = json.load(f)
                roof["traffic"] = tr.get(f"{work.name}:step")
                if roof["traffic"]:
                    roof["traffic_src"] = tr.get("_note", "")
            except Exception:
                pass
        if dom is not None:
            tot_stage = sum(stage_ms.values())
            roof["dominant_kernel"] = {"stage": dom, "ms_per_step": stage_ms[dom],
                                       "share_of_step": stage_ms[dom] / tot_stage if tot_stage else None}
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "s8", "data": "synthetic (seeded numpy PCG64, SURVEY §8d seed scheme)",
            "config": cfg,
            "roofline": roof,
            "stage_ms_per_step": stage_ms,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d_bytes * world,
                    "d2h_bytes_per_step": d2h_bytes * world},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks.summary(),
            "peaks": peaks,
        }
        if mcheck is not None:
            result["multi_gpu_check"] = mcheck
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
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if world > 1 and args.impl == "b200":
        import torch
        import torch.distributed as dist
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
