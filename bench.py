#!/usr/bin/env python
"""Benchmark of the fused operation-chain path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5|c1|c2|c3|c4]
                    [--impl fk|reference] [--scaling strong|weak] [--no-sub]

One "step" = one execute_fused of the workload's whole pipeline (one fused
launch). Default workload: configs[4] (C5), 8192 crops of 224x224x3 in total —
crop -> bilinear resize -> cast f32 -> normalise -> split — partitioned across
the N GPUs by batch index (strong scaling): one process per
GPU (torchrun), each builds and runs its own contiguous shard, no collective on
the data path; time = max over ranks of device time.

Before anything is timed, the timed pipeline's complete output is compared bit
for bit with the C oracle's (oracle/, the checker pinned to the reference in
tests/test_oracle.py) on the same seeded inputs — the reference bench's
require_equal gate (bench.cpp:93-96). On a mismatch the line carries no value
and the process exits 2.

Prints ONE JSON line (rank 0): `value` = whole-job Mpixel/s with inputs resident
in HBM; `e2e` = the same through the C-ABI with host buffers (H2D of the frames
and D2H of every output plane inside the timed region); `roofline` =
algorithmic bytes / kernel time vs the measured HBM peak; `unfused` = the
one-kernel-per-op comparator; `cpu_baseline` = the unmodified reference
(oracle/_ref) on this host's cores; `sub` (N = 1) = the other BASELINE configs
(C1, C2, C3 sweep, C4 sweep), each gated, timed, with its roofline, unfused and
CPU figures. `--impl reference` times only the reference CPU implementation on
the same workload (all 8192 crops per step).
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
C3_SWEEP = (1, 16, 64, 256, 1000)
C4_SWEEP = (1, 8, 64, 256, 1024)


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
    d = os.path.join(ROOT, "profiles")
    for name in sorted(os.listdir(d), reverse=True) if os.path.isdir(d) else []:
        if name.startswith("ncu_summary") and name.endswith(".json"):
            try:
                with open(os.path.join(d, name)) as f:
                    s = json.load(f)
                if workload in s and s[workload].get("dram_bytes") is not None:
                    return int(s[workload]["dram_bytes"]), name
            except Exception:
                pass
    return None, None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


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
def build(lib, workload: str, n_ops: int = 64, crops: int = 8192, first: int = 0, sets: int = 1):
    """The workload's pipeline on `lib` (same seeded inputs on every backend)."""
    from paper_2508_07071_b200 import workloads as wl
    if workload == "c1":
        return wl.c1(lib, sets=sets)
    if workload == "c2":
        return wl.c2(lib)
    if workload == "c3":
        return wl.c3(lib, n_ops, sets=sets)
    return wl.crops_224(lib, crops, per_crop_norm=workload == "c4", name=workload.upper(), first=first)


def workload_name(workload, crops, n_ops, scaling="strong"):
    per = "in total, sharded by batch index" if scaling == "strong" else "per GPU"
    return {"c1": "configs[0] C1: 3840x2160 f32 -> mul,add,sub,div,cast -> u8 (vertical fusion)",
            "c2": "configs[1] C2: cvGS 50 crops of 1920x1080 u8x3 -> bilinear 64x128 -> SwapRB -> f32 -> "
                  "normalize -> split",
            "c3": f"configs[2] C3: {n_ops} chained f32 ops on 4096x4096",
            "c4": f"configs[3] C4: {crops} crops 224x224x3 {per}, per-crop resize + per-crop normalize, split",
            "c5": f"configs[4] C5: {crops} crops 224x224x3 {per}, crop->bilinear resize->cast f32->normalize"
                  "->split (cvGS chain at B200 scale)"}[workload]


# ------------------------------------------------------------- parity gate --
def parity_gate(w, workload, n_ops, crops, first):
    """The timed pipeline's complete output vs the C oracle's on the same inputs
    (bench.cpp:93-96 require_equal). Compared on the GPU, byte for byte."""
    import torch
    from paper_2508_07071_b200.opfuse import ExecConfig, Library
    oracle = Library("oracle")
    wo = build(oracle, workload, n_ops, crops, first)
    oracle.execute_fused(wo.pipeline, ExecConfig(workers=len(os.sched_getaffinity(0))))
    nbytes, bad = 0, 0
    for got, want in zip(w.outputs, wo.outputs):
        wt = want.to(got.device)
        nbytes += got.numel()
        bad += int((got != wt).sum().item())
    return {"passed": bad == 0, "compared_bytes": nbytes, "mismatched_bytes": bad,
            "against": "oracle/fk_oracle.c (pinned to the reference, tests/test_oracle.py)"}


# ------------------------------------------------------------------ timing --
def time_steps(lib, pipes, cfg, steps, flush, stream, run=None):
    """Per-step device times (ms) of `steps` executes, CUDA events on the launching
    stream. Without rotation (one pipeline) L2 is flushed between steps, outside
    the events; the stream is held on a device spin while the host enqueues, so
    the events time the GPU and not the Python launch rate."""
    import torch
    run = run or lib.execute_fused
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda._sleep(int(2e6 + 1e5 * steps))
    for i, (a, b) in enumerate(evs):
        if len(pipes) == 1:
            flush.fill_(1)
        a.record(stream)
        run(pipes[i % len(pipes)], cfg)
        b.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def cpu_reference(workload, n_ops, sample_crops, budget_s, threads=None, steps=None, warmup=1, rows=None):
    """The unmodified reference (oracle/_ref/libfk_ref.so) on this host's cores
    (the C oracle port when the reference was not built)."""
    from paper_2508_07071_b200.opfuse import ExecConfig, Library
    kind = "reference"
    try:
        lib = Library("reference")
    except FileNotFoundError:
        lib, kind = Library("oracle"), "port"
    cores = threads or len(os.sched_getaffinity(0))
    from paper_2508_07071_b200 import workloads as wl
    if workload == "c3" and rows:
        w = wl.c3(lib, n_ops, H=rows)
    else:
        w = build(lib, workload, n_ops, sample_crops) if not (workload == "c4" and kind == "reference") else \
            build(Library("oracle"), workload, n_ops, sample_crops)  # only its pixel count is used
    cfg = ExecConfig(workers=cores)
    run = lambda: lib.execute_fused(w.pipeline, cfg).wall_time_ns / 1e9  # noqa: E731
    if workload == "c4" and kind == "reference":
        # per-crop constants: one single-plane pipeline per crop (bench.cpp:199-202)
        planes, keep = wl.c4_reference_planes(lib, sample_crops)
        run = lambda: sum(lib.execute_fused(p, cfg).wall_time_ns for p, _ in planes) / 1e9  # noqa: E731
    for _ in range(warmup):
        run()
    times, t0 = [], time.time()
    while True:
        times.append(run())
        if steps is not None:
            if len(times) >= steps:
                break
        elif time.time() - t0 > budget_s or len(times) >= 30:
            break
    mean = sum(times) / len(times)
    sample = (f"{sample_crops} crops ({w.points} px)" if workload in ("c4", "c5") else
              f"{w.points} px of {workload.upper()}" + (f" ({rows} of 4096 rows)" if rows else ""))
    how = ("one single-plane pipeline per crop (per-crop constants), " if workload == "c4" and kind == "reference"
           else "")
    return {"value": w.points / mean / 1e6, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{sample} per call, {how}{len(times)} timed calls, mean {mean * 1e3:.2f} ms, reference "
                      f"execute_fused (OpenMP, workers={cores}, -O2)", "cpu_model": cpu_model()}, mean


# -------------------------------------------------------------- sub-results --
def sub_result(lib, cfg, stream, flush, workload, n_ops=64, crops=8192, steps=10, cpu_budget=2.0):
    """One BASELINE config: gated, timed (fused + unfused), roofline, CPU figure."""
    import torch
    sets = 4 if workload == "c1" else 2 if workload == "c3" else 1
    w = build(lib, workload, n_ops, crops, 0, sets)
    lib.execute_fused(w.pipeline, cfg)
    torch.cuda.synchronize()
    gate = parity_gate(w, workload, n_ops, crops, 0)
    pipes = [w.pipeline] + list(w.rotate)
    for i in range(3):
        lib.execute_fused(pipes[i % len(pipes)], cfg)
    ms = statistics.mean(time_steps(lib, pipes, cfg, steps, flush, stream))
    kernel = lib.last_kernel()
    # back-to-back: 20 launches between two events (the launches overlap their
    # ramp and tail; rotating sets or a flush-free run over > L2 inputs)
    b2b = None
    if len(pipes) > 1:
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(4e6))
        a.record(stream)
        for i in range(20):
            lib.execute_fused(pipes[i % len(pipes)], cfg)
        e.record(stream)
        torch.cuda.synchronize()
        b2b = a.elapsed_time(e) / 20
    lib.execute_unfused(w.pipeline, cfg)
    ums = statistics.mean(time_steps(lib, pipes, cfg, 3, flush, stream, lib.execute_unfused))
    peak, _ = measured_peak()
    gbs = w.alg_bytes / (ms / 1e3) / 1e9
    mpix = w.points / (ms / 1e3) / 1e6
    sample = min(crops, 64) if workload in ("c4", "c5") else crops
    rows = 256 if workload == "c3" and n_ops >= 64 else None
    cpu, _ = cpu_reference(workload, n_ops, sample, cpu_budget, rows=rows)
    out = {"workload": workload_name(workload, crops, n_ops), "ms_per_step": ms, "mpix_s": mpix, "gbs": gbs,
           "frac_of_measured_peak": gbs / peak, "frac_of_8tbs": gbs / SPEC_HBM_GBS, "kernel": kernel,
           "alg_bytes": w.alg_bytes, "points": w.points, "gate": gate["passed"],
           "unfused": {"ms_per_step": ums, "speedup_fused_vs_unfused": ums / ms,
                       "kernels_per_step": w.pipeline.n_compute + 1},
           "cpu_baseline": cpu, "speedup_vs_cpu": mpix / cpu["value"]}
    if b2b is not None:
        out["back_to_back_ms_per_step"] = b2b
        out["back_to_back_frac_of_measured_peak"] = w.alg_bytes / (b2b / 1e3) / 1e9 / peak
    if workload == "c1":
        # the same traffic through one PyTorch kernel (33.2 MB f32 read, 8.3 MB u8 write):
        # what a single 41 MB launch costs on this GPU, launch and ramp included
        src = torch.rand(2160, 3840, device="cuda")
        srcs = [src, torch.rand_like(src), torch.rand_like(src), torch.rand_like(src)]
        for s in srcs:
            s.to(torch.uint8)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda._sleep(int(2e6))
        for i, (a, e) in enumerate(evs):
            a.record(stream)
            srcs[i % 4].to(torch.uint8)
            e.record(stream)
        torch.cuda.synchronize()
        out["torch_same_traffic_ms"] = statistics.mean(a.elapsed_time(e) for a, e in evs)
    if workload == "c3":
        # FP32 roofline above N ~ 45: N * P ops at the FMA pipe's packed rate
        out["fp32_ops"] = n_ops * w.points
    del w
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------- main --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="fk", choices=["fk", "reference"])
    ap.add_argument("--crops", type=int, default=8192, help="crops in total (strong) or per GPU (weak)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"])
    ap.add_argument("--n-ops", type=int, default=64)
    ap.add_argument("--cpu-sample-crops", type=int, default=256)
    ap.add_argument("--cpu-budget-s", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-unfused", action="store_true")
    ap.add_argument("--no-gate", action="store_true", help="skip the parity gate (profiling runs only)")
    ap.add_argument("--no-sub", action="store_true", help="skip the C1-C4 sub-results")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and "WORLD_SIZE" in os.environ:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    strong = args.scaling == "strong" and args.workload in ("c4", "c5")
    scaling = "strong" if strong else "weak"

    if args.impl == "reference":
        if rank != 0:
            return
        # the same workload as the fk arm: all crops of the job (strong) on the host cores
        crops = args.crops if (strong or world == 1) else args.crops * world
        cpu, mean = cpu_reference(args.workload, args.n_ops, crops, 1e9, steps=args.steps, warmup=args.warmup)
        one, _ = cpu_reference(args.workload, args.n_ops, 32, 5.0, threads=1, warmup=0)
        cpu["single_thread"] = {"value": one["value"], "sample": one["sample"]}
        line = {"metric": METRIC, "value": cpu["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": mean * 1e3, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": workload_name(args.workload, crops, args.n_ops, scaling),
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
    if strong:
        lo, hi = shard_range(args.crops, rank, world)
    else:
        lo, hi = rank * args.crops, (rank + 1) * args.crops
    w = build(lib, args.workload, args.n_ops, hi - lo, lo, 4 if args.workload == "c1" else 2 if args.workload == "c3" else 1)
    job_points = sum_over_ranks(w.points, "cuda") if world > 1 else w.points
    stream = torch.cuda.current_stream()
    cfg = ExecConfig(stream=stream.cuda_stream)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    pipes = [w.pipeline] + list(w.rotate)   # rotated sets (C1/C3) need no flush

    # ---- parity gate: the timed pipeline's whole output vs the oracle (bench.cpp:93-96)
    lib.execute_fused(w.pipeline, cfg)
    torch.cuda.synchronize()
    gate = None if args.no_gate else parity_gate(w, args.workload, args.n_ops, hi - lo, lo)
    ok = gate is None or gate["passed"]
    if world > 1:
        t = torch.tensor([0 if ok else 1], device="cuda")
        dist.all_reduce(t)
        ok = int(t.item()) == 0
    if not ok:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "unit": UNIT, "n_gpus": world, "impl": "fk",
                              "gate": gate or {"passed": False, "rank": "other"},
                              "error": "parity gate failed: output differs from the oracle; not timed"}))
        sys.exit(2)

    for i in range(max(args.warmup, len(pipes))):
        if len(pipes) == 1:
            flush.fill_(1)
        lib.execute_fused(pipes[i % len(pipes)], cfg)
    torch.cuda.synchronize()

    # ---- timed region: EXACTLY K fused steps
    launches0 = lib._c.fk_cuda_kernel_launch_count()
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        step_ms = time_steps(lib, pipes, cfg, args.steps, flush, stream)
        kernel = lib.last_kernel()
        if world > 1:
            dist.barrier()
    launches = lib._c.fk_cuda_kernel_launch_count() - launches0
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
        ums = statistics.mean(time_steps(lib, pipes, cfg, 3, flush, stream, lib.execute_unfused))
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
        del srcs, outs

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
                "alg_bytes_per_launch": w.alg_bytes, "kernel": kernel, "traffic_source": traffic_src}
    cpu = None
    if not args.no_cpu and world == 1:
        cpu, _ = cpu_reference(args.workload, args.n_ops, args.cpu_sample_crops, args.cpu_budget_s)
    cfgd = {"workload": workload_name(args.workload, args.crops, args.n_ops, scaling),
            "points_per_gpu": w.points, "alg_bytes_per_gpu": w.alg_bytes, "out_bytes_per_gpu": w.out_bytes,
            "in_bytes_per_gpu": w.in_bytes,
            "parallelism": f"batch-sharded x{world} (crops [{lo}, {hi}) on rank 0), no collective" if world > 1
            else "1 GPU",
            "l2": (f"{len(pipes)} input/output sets rotated between steps "
                   f"({len(pipes) * w.alg_bytes / 1e6:.0f} MB > 126 MB L2), no flush") if len(pipes) > 1 else
                  "512 MiB L2 flush (buffer write) between timed steps, outside the step events"}
    for key in ("frames", "out", "crops", "shape", "n_ops", "per_crop_normalize"):
        if key in w.info:
            cfgd[key] = w.info[key]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfgd,
            "gbs": achieved, "roofline": roofline, "gate": gate, "cpu_baseline": cpu, "e2e": e2e,
            "unfused": unfused, "gpu_launches": int(launches), "clocks": clocks.summary(),
            "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)}}
    if world == 1 and not args.no_sub and args.workload == "c5":
        del w, pipes
        torch.cuda.empty_cache()
        sub = {"C1": sub_result(lib, cfg, stream, flush, "c1", steps=20),
               "C2": sub_result(lib, cfg, stream, flush, "c2", steps=50)}
        for n in C3_SWEEP:
            sub[f"C3[N={n}]"] = sub_result(lib, cfg, stream, flush, "c3", n_ops=n, steps=10)
        for b in C4_SWEEP:
            sub[f"C4[B={b}]"] = sub_result(lib, cfg, stream, flush, "c4", crops=b, steps=20 if b < 256 else 10)
        line["sub"] = sub
        line["sub_gates_passed"] = all(s["gate"] for s in sub.values())
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
