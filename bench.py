#!/usr/bin/env python
"""Benchmark of the fused operation-chain path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5|c1|c2|c3|c4] [--impl fk|reference]

One "step" = one execute_fused of the workload's whole pipeline (one fused
launch). Default workload: configs[4] (C5), the cvGS preprocessing chain
(crop -> bilinear resize -> cast -> normalise -> split) at 8192 crops of
224x224x3 per GPU — configs[1]'s pipeline sized for a B200 (C2's 4.9 MB step
is below launch latency; it stays a parity case). Multi-GPU: one process per
GPU (torchrun), each shards its own 8192 crops (weak scaling), no collective
on the data path; time = max over ranks of device time.

Prints ONE JSON line (rank 0). `value` = whole-job Mpixel/s with inputs
resident in HBM; `e2e` = the same through the C-ABI with host buffers (H2D of
the frames and D2H of every output plane inside the timed region);
`roofline` = algorithmic bytes / kernel time vs the measured HBM copy peak;
`cpu_baseline` = the unmodified reference (oracle/_ref) on this host's cores.
`--impl reference` times only the reference CPU implementation.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2508_07071_b200.shard import shard_range, sum_over_ranks  # noqa: E402

METRIC = "Mpixel/s and achieved HBM GB/s (% of 8 TB/s) per fused pipeline vs unfused and CPU"
UNIT = "Mpixel/s"
L2_FLUSH_BYTES = 512 << 20      # > 126 MB L2: written between timed steps
SPEC_HBM_GBS = 8000.0


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str):
    """dram read+write bytes per launch of the fused kernel from the committed ncu capture."""
    for name in sorted(os.listdir(os.path.join(ROOT, "profiles")), reverse=True) if os.path.isdir(
            os.path.join(ROOT, "profiles")) else []:
        if name.startswith("ncu_summary") and name.endswith(".json"):
            try:
                with open(os.path.join(ROOT, "profiles", name)) as f:
                    d = json.load(f)
                if workload in d and d[workload].get("dram_bytes") is not None:
                    return int(d[workload]["dram_bytes"]), name
            except Exception:
                pass
    return None, None


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
               0x2: "applications_clocks_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            # warm the query path so the first in-region sample is not a slow one
            pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# --------------------------------------------------------------- workloads --
def build(lib, workload: str, rank: int, crops: int, n_ops: int, world: int = 1, strong: bool = False):
    """The workload's pipeline for this rank: weak scaling gives every rank `crops`
    crops of its own; strong scaling splits `crops` into contiguous shards."""
    from paper_2508_07071_b200 import workloads as wl
    if workload == "c1":
        return wl.c1(lib, sets=4)      # 4 x 41.5 MB rotated sets > L2: no flush needed
    if workload == "c2":
        return wl.c2(lib)
    if workload == "c3":
        return wl.c3(lib, n_ops, sets=2)  # 2 x 134 MB rotated sets > L2
    if workload == "c4":
        lo, hi = shard_range(crops, rank, world) if strong else (rank * crops, (rank + 1) * crops)
        return wl.crops_224(lib, hi - lo, per_crop_norm=True, name="C4", first=lo)
    lo, hi = shard_range(crops, rank, world) if strong else (rank * crops, (rank + 1) * crops)
    return wl.crops_224(lib, hi - lo, per_crop_norm=False, name="C5", first=lo)


def workload_name(workload, crops, n_ops):
    return {"c1": "configs[0] C1: 3840x2160 f32 -> mul,add,sub,div,cast -> u8 (vertical fusion)",
            "c2": "configs[1] C2: cvGS 50 crops of 1920x1080 u8x3 -> bilinear 64x128 -> SwapRB -> f32 -> "
                  "normalize -> split",
            "c3": f"configs[2] C3: {n_ops} chained f32 ops on 4096x4096",
            "c4": f"configs[3] C4: {crops} crops 224x224x3 per GPU, per-crop resize + per-crop normalize, split",
            "c5": f"configs[4] C5: {crops} crops 224x224x3 per GPU, crop->bilinear resize->cast f32->normalize"
                  "->split (cvGS chain at B200 scale)"}[workload]


def describe(w, workload, crops, n_ops, world):
    d = workload_name(workload, crops, n_ops)
    cfg = {"workload": d, "points_per_gpu": w.points, "alg_bytes_per_gpu": w.alg_bytes,
           "out_bytes_per_gpu": w.out_bytes, "in_bytes_per_gpu": w.in_bytes,
           "parallelism": f"batch-sharded x{world}, no collective" if world > 1 else "1 GPU",
           "l2": (f"{1 + len(w.rotate)} input/output sets rotated between steps "
                  f"({(1 + len(w.rotate)) * w.alg_bytes / 1e6:.0f} MB > 126 MB L2), no flush") if w.rotate else
                 "512 MiB L2 flush (buffer write) between timed steps, outside the step events"}
    for k in ("frames", "out", "crops", "shape", "n_ops", "per_crop_normalize"):
        if k in w.info:
            cfg[k] = w.info[k]
    return cfg


# -------------------------------------------------------------- reference --
def run_reference(args, workload, sample_crops, budget_s, steps=None, warmup=1):
    """The unmodified reference (oracle/_ref/libfk_ref.so) on this host's cores."""
    from paper_2508_07071_b200.opfuse import ExecConfig, Library
    kind = "reference"
    try:
        lib = Library("reference")
    except FileNotFoundError:
        lib, kind = Library("oracle"), "port"
    cores = len(os.sched_getaffinity(0))
    w = build(lib, workload, 0, sample_crops, args.n_ops)
    cfg = ExecConfig(workers=cores)
    times = []
    for _ in range(warmup):
        lib.execute_fused(w.pipeline, cfg)
    t_start = time.time()
    while True:
        rep = lib.execute_fused(w.pipeline, cfg)
        times.append(rep.wall_time_ns / 1e9)
        if steps is not None:
            if len(times) >= steps:
                break
        elif time.time() - t_start > budget_s or len(times) >= 50:
            break
    mean = sum(times) / len(times)
    sample = (f"{sample_crops} crops ({w.points} px) per call" if workload in ("c4", "c5") else
              f"full {workload.upper()} ({w.points} px) per call")
    return {"value": w.points / mean / 1e6, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": sample + f", {len(times)} timed calls, mean {mean * 1e3:.1f} ms, reference execute_fused "
                               f"(OpenMP, workers={cores}, -O2)"}, mean


# ------------------------------------------------------------------- main --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="fk", choices=["fk", "reference"])
    ap.add_argument("--crops", type=int, default=8192, help="crops per GPU (weak) or in total (strong)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--n-ops", type=int, default=64)
    ap.add_argument("--cpu-sample-crops", type=int, default=256)
    ap.add_argument("--cpu-budget-s", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-unfused", action="store_true")
    ap.add_argument("--force-generic", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        cpu, mean = run_reference(args, args.workload, args.cpu_sample_crops, 1e9, steps=args.steps,
                                  warmup=args.warmup)
        line = {"metric": METRIC, "value": cpu["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": mean * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": workload_name(args.workload, args.crops, args.n_ops),
                           "sample": cpu["sample"], "parallelism": "host cores (OpenMP), rank 0 only"},
                "impl": "reference", "cpu_baseline": cpu,
                "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist
    from paper_2508_07071_b200.opfuse import ExecConfig, Library

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = Library("cuda")
    w = build(lib, args.workload, rank, args.crops, args.n_ops, world, args.scaling == "strong")
    job_points = sum_over_ranks(w.points, "cuda") if world > 1 else w.points
    stream = torch.cuda.current_stream()
    cfg = ExecConfig(stream=stream.cuda_stream, force_generic=args.force_generic)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")

    pipes = [w.pipeline] + list(w.rotate)   # rotated sets (C1/C3) need no flush

    def step_events(fn, k):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        # Hold the stream on a device-side spin while the host enqueues the k steps,
        # so the per-step events time the GPU, not the Python/ctypes launch rate
        # (a 41 MB step runs faster than the host can issue it).
        torch.cuda._sleep(int(2e6 + 1e5 * k))
        for i, (a, b) in enumerate(evs):
            if not w.rotate:
                flush.fill_(1)
            a.record(stream)
            fn(i)
            b.record(stream)
        return evs

    for i in range(max(args.warmup, len(pipes))):
        if not w.rotate:
            flush.fill_(1)
        lib.execute_fused(pipes[i % len(pipes)], cfg)
    torch.cuda.synchronize()

    # ---- timed region: EXACTLY K fused steps
    launches0 = lib._c.fk_cuda_kernel_launch_count()
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        evs = step_events(lambda i: lib.execute_fused(pipes[i % len(pipes)], cfg), args.steps)
        kernel = lib.last_kernel()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = lib._c.fk_cuda_kernel_launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = job_points * args.steps / (total_ms / 1e3) / 1e6

    # ---- unfused comparator (same workload, one launch per op)
    unfused = None
    if not args.no_unfused:
        for i in range(2):
            lib.execute_unfused(pipes[i % len(pipes)], cfg)
        torch.cuda.synchronize()
        uev = step_events(lambda i: lib.execute_unfused(pipes[i % len(pipes)], cfg), 3)
        torch.cuda.synchronize()
        ums = statistics.mean(a.elapsed_time(b) for a, b in uev)
        unfused = {"ms_per_step": ums, "mpix_s": w.points / ums / 1e3, "speedup_fused_vs_unfused": ums / ms_per_step,
                   "kernels_per_step": w.pipeline.n_compute + 1}

    # ---- e2e through the C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        srcs = [(p.storage, torch.empty(p.storage.numel(), dtype=torch.uint8, pin_memory=True)) for p in w.sources]
        for dev_t, host_t in srcs:
            host_t.copy_(dev_t)
        outs = [(o, torch.empty(o.numel(), dtype=torch.uint8, pin_memory=True)) for o in w.outputs]
        h2d = sum(d.numel() for d, _ in srcs)
        d2h = sum(o.numel() for o, _ in outs)

        def e2e_step():
            for dev_t, host_t in srcs:
                dev_t.copy_(host_t, non_blocking=True)
            lib.execute_fused(w.pipeline, cfg)
            for o, host_t in outs:
                host_t.copy_(o, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        k = max(1, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(stream)
        for _ in range(k):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        ems = a.elapsed_time(b) / k
        if world > 1:
            t = torch.tensor([ems], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": job_points / (ems / 1e3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems}

    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = measured_peak()
    achieved = w.alg_bytes / (ms_per_step / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(w.name)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": peak_src, "frac_of_8tbs": achieved / SPEC_HBM_GBS,
                "alg_bytes_per_launch": w.alg_bytes, "kernel": kernel,
                "traffic_source": traffic_src}
    cpu = None
    if not args.no_cpu and world == 1:
        cpu, _ = run_reference(args, args.workload, args.cpu_sample_crops, args.cpu_budget_s)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": describe(w, args.workload, args.crops, args.n_ops, world),
            "gbs": achieved, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "unfused": unfused,
            "gpu_launches": int(launches), "clocks": clocks.summary(),
            "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)}}
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
