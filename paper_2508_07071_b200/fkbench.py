"""The reference's benchmark CLI on B200 (bench.hpp, bench.cpp:127-514).

    python -m paper_2508_07071_b200.fkbench <vf|hf|vf-hf|ipo|datasize|datatype|memory>
        [--repeats N] [--warmup N] [--threads N] [--coarsen B] [--csv PATH] [--seed S]
        [--backend cuda|oracle|reference]

Each experiment builds the reference's workload (same extents, ops, constants
and sweeps), runs the fused strategy and the reference's baseline strategy
once, requires their outputs to be bit-identical (the equality gate,
bench.cpp:93-96: exit 2 on failure), then times `repeats` runs of each after
`warmup` untimed ones and writes the reference's CSV schema
(experiment,param,fused_ns,unfused_ns,speedup,rsd_pct; bench.cpp:497-514).
Usage errors exit 1. On the CUDA backend a run is timed on the device (CUDA
events around the call, or around the whole baseline loop); on the CPU
backends by the wall clock, as the reference does. Inputs are seeded
(`--seed`); the reference's own generator is not reproduced (the gate compares
the two strategies on identical inputs within one run).

Differences from the reference, by necessity: `memory` uses a 256x512 source
(the reference's 256x256 makes its own crop 10,20,120,240 out of bounds);
vf-hf's per-op baseline (2 pairs passes per plane) is run with fewer repeats
when one baseline run exceeds 0.5 s.
"""
from __future__ import annotations

import argparse
import math
import sys
import time
from dataclasses import dataclass, field

import numpy as np

from . import api
from ._ffi import BILINEAR, F32, F32X3, F64, SWAP_RB, U8
from .opfuse import ExecConfig, Library, OpfuseError, const_of, f32, f32x3, u8

EXPERIMENTS = ("vf", "hf", "vf-hf", "ipo", "datasize", "datatype", "memory")
KIND_NAME = {U8: "u8", F32: "f32", F64: "f64"}
STATIC_LOOP_THRESHOLD = 64  # bench.cpp:100-108


class GateFailure(RuntimeError):
    """The two strategies disagreed bit-wise (bench.hpp:34-37); exit 2."""


@dataclass
class Options:
    repeats: int = 30
    warmup: int = 2
    threads: int = 0
    coarsen: int = 8
    chunk_rows: int = 8
    seed: int = 42
    backend: str = "cuda"
    quick: bool = False       # trimmed sweeps (tests): vf-hf <= 1000 pairs, datasize <= 1e6, ipo step 55


@dataclass
class Record:  # bench.hpp:22-29
    experiment: str
    param: str
    fused_ns: float
    unfused_ns: float
    rsd_pct: float

    @property
    def speedup(self) -> float:
        return self.unfused_ns / self.fused_ns


@dataclass
class Bench:
    opt: Options
    lib: Library = field(init=False)

    def __post_init__(self):
        self.lib = Library(self.opt.backend)
        self.rng = np.random.default_rng(self.opt.seed)
        self.cuda = self.opt.backend == "cuda"
        self.cfg = ExecConfig(workers=self.opt.threads, coarsening=self.opt.coarsen, chunk_rows=self.opt.chunk_rows)
        if self.cuda:
            import torch
            self.torch = torch
            self.cfg.stream = torch.cuda.current_stream().cuda_stream

    # -- inputs
    def plane(self, w, h, kind):
        return self.lib.plane_alloc(w, h, kind)

    def random_plane(self, w, h, kind):  # fill_random, bench.cpp:26-49
        shape = (h, w, 3) if kind >= 3 else (h, w)
        base = kind - 3 if kind >= 3 else kind
        if base == U8:
            a = self.rng.integers(0, 256, shape, dtype=np.uint8)
        else:
            a = self.rng.random(shape).astype(np.float32 if base == F32 else np.float64)
        return self.lib.plane_from_numpy(a)

    # -- timing (time_repeats, bench.cpp:68-79)
    def series(self, fn, repeats=None):
        repeats = repeats or self.opt.repeats
        out = []
        for i in range(self.opt.warmup + repeats):
            if self.cuda:
                a, b = self.torch.cuda.Event(enable_timing=True), self.torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                b.synchronize()
                dt = a.elapsed_time(b) * 1e6
            else:
                t0 = time.perf_counter_ns()
                fn()
                dt = float(time.perf_counter_ns() - t0)
            if i >= self.opt.warmup:
                out.append(dt)
        return out

    @staticmethod
    def stats(s):
        m = sum(s) / len(s)
        rsd = 0.0 if m == 0 else math.sqrt(sum((v - m) ** 2 for v in s) / len(s)) / m * 100.0
        return m, rsd

    def record(self, exp, param, fused, unfused):
        fm, fr = self.stats(fused)
        um, ur = self.stats(unfused)
        return Record(exp, str(param), fm, um, max(fr, ur))

    def sync(self):
        if self.cuda:
            self.torch.cuda.synchronize()

    def require_equal(self, a, b, where):  # bench.cpp:93-96
        self.sync()
        if a.kind != b.kind or not np.array_equal(a.to_numpy().view(np.uint8), b.to_numpy().view(np.uint8)):
            raise GateFailure(f"equality gate failed: {where}")

    def compressed(self, chain, op, n):  # append_compressed, bench.cpp:100-108
        if n == 0:
            return
        if n <= STATIC_LOOP_THRESHOLD:
            chain.extend([op] * n)
        else:
            chain.append(self.lib.op_static_loop(op, n))

    # ------------------------------------------------------------ experiments --
    def vf(self):  # bench.cpp:127-163
        L, W, H = self.lib, 4096, 2160
        src = self.random_plane(W, H, U8)
        df, du = self.plane(W, H, U8), self.plane(W, H, U8)
        mul = L.op_mul(u8(3))
        recs = []
        for n in (2, 102, 202):
            chain = [L.op_read_per_thread(src)]
            self.compressed(chain, mul, n)
            fused = L.validate_chain(chain + [L.op_write_per_thread(df)])
            unfused = L.validate_chain([L.op_read_per_thread(src)] + [mul] * n + [L.op_write_per_thread(du)])
            L.execute_fused(fused, self.cfg)
            if L.execute_unfused(unfused, self.cfg).passes != n + 1:
                raise GateFailure("vf: unexpected unfused pass count")
            self.require_equal(df, du, f"vf n_ops={n}")
            recs.append(self.record("vf", n, self.series(lambda: L.execute_fused(fused, self.cfg)),
                                    self.series(lambda: L.execute_unfused(unfused, self.cfg))))
        return recs

    def hf(self):  # bench.cpp:165-219
        L, W, H = self.lib, 60, 120
        sweep = (1, 10, 50, 150, 600)
        src = [self.random_plane(W, H, U8) for _ in range(sweep[-1])]
        dfu = [self.plane(W, H, F32) for _ in range(sweep[-1])]
        dlo = [self.plane(W, H, F32) for _ in range(sweep[-1])]
        cast, mul, sub, div = L.op_cast(U8, F32), L.op_mul(f32(1.25)), L.op_sub(f32(0.5)), L.op_div(f32(2.0))
        recs = []
        for batch in sweep:
            fused = L.validate_chain([L.op_batch_read([L.op_read_per_thread(s) for s in src[:batch]]), cast, mul, sub,
                                      div, L.op_batch_write([L.op_write_per_thread(d) for d in dfu[:batch]])])
            loop = [L.validate_chain([L.op_read_per_thread(src[z]), cast, mul, sub, div,
                                      L.op_write_per_thread(dlo[z])]) for z in range(batch)]
            L.execute_fused(fused, self.cfg)
            for p in loop:
                L.execute_fused(p, self.cfg)
            for z in range(batch):
                self.require_equal(dfu[z], dlo[z], f"hf batch={batch}")

            def run_loop():
                for p in loop:
                    L.execute_fused(p, self.cfg)
            recs.append(self.record("hf", batch, self.series(lambda: L.execute_fused(fused, self.cfg)),
                                    self.series(run_loop)))
        return recs

    def vf_hf(self):  # bench.cpp:221-277
        L, W, H, B = self.lib, 60, 120, 50
        src = [self.random_plane(W, H, U8) for _ in range(B)]
        dfu = [self.plane(W, H, U8) for _ in range(B)]
        dba = [self.plane(W, H, U8) for _ in range(B)]
        mul, add = L.op_mul(u8(3)), L.op_add(u8(7))
        tmp = [self.plane(W, H, U8), self.plane(W, H, U8)]
        passes = {}

        def single(a, op, b):  # single_op_pass, bench.cpp:110-117 (built once per (in, op, out))
            key = (id(a), id(op), id(b))
            if key not in passes:
                passes[key] = L.validate_chain([L.op_read_per_thread(a), op, L.op_write_per_thread(b)])
            return passes[key]

        def baseline(pairs):
            for z in range(B):
                cur, nxt, other = src[z], tmp[0], tmp[1]
                total = 2 * pairs
                for i in range(total):
                    op = mul if i < pairs else add
                    last = i + 1 == total
                    L.execute_fused(single(cur, op, dba[z] if last else nxt), self.cfg)
                    if not last:
                        cur = nxt
                    nxt, other = other, nxt

        recs = []
        for pairs in (2, 100, 1000) if self.opt.quick else (2, 100, 1000, 10000):
            chain = [L.op_batch_read([L.op_read_per_thread(s) for s in src])]
            self.compressed(chain, mul, pairs)
            self.compressed(chain, add, pairs)
            fused = L.validate_chain(chain + [L.op_batch_write([L.op_write_per_thread(d) for d in dfu])])
            L.execute_fused(fused, self.cfg)
            t0 = time.perf_counter()
            baseline(pairs)
            slow = time.perf_counter() - t0 > 0.5
            for z in range(B):
                self.require_equal(dfu[z], dba[z], f"vf-hf pairs={pairs}")
            reps = 3 if slow else None
            recs.append(self.record("vf-hf", pairs, self.series(lambda: L.execute_fused(fused, self.cfg), reps),
                                    self.series(lambda: baseline(pairs), reps)))
        return recs

    def ipo(self):  # bench.cpp:279-316
        L, W, H, total = self.lib, 256, 256, 500
        src = self.random_plane(W, H, F32)
        df, du = self.plane(W, H, F32), self.plane(W, H, F32)
        mul = L.op_mul(f32(1.0000001))
        fused = L.validate_chain([L.op_read_per_thread(src), L.op_static_loop(mul, total), L.op_write_per_thread(df)])
        recs = []
        for per_op in range(1, 497, 55 if self.opt.quick else 5):
            counts = split_instructions(total, per_op)
            if len(counts) != (total + per_op - 1) // per_op:
                raise GateFailure("ipo: split does not match ceil(total/per_op)")
            chain = [L.op_read_per_thread(src)] + [mul if c == 1 else L.op_static_loop(mul, c) for c in counts]
            unfused = L.validate_chain(chain + [L.op_write_per_thread(du)])
            L.execute_fused(fused, self.cfg)
            if L.execute_unfused(unfused, self.cfg).passes != len(counts) + 1:
                raise GateFailure("ipo: unexpected unfused pass count")
            self.require_equal(df, du, f"ipo per_op={per_op}")
            recs.append(self.record("ipo", per_op, self.series(lambda: L.execute_fused(fused, self.cfg)),
                                    self.series(lambda: L.execute_unfused(unfused, self.cfg))))
        return recs

    def datasize(self):  # bench.cpp:318-348
        L = self.lib
        mul, add = L.op_mul(f32(1.0000001)), L.op_add(f32(0.0001))
        recs = []
        for n in (100, 10000, 1000000) if self.opt.quick else (100, 10000, 1000000, 16654030):
            src = self.random_plane(n, 1, F32)
            df, du = self.plane(n, 1, F32), self.plane(n, 1, F32)
            fused = L.validate_chain([L.op_read_per_thread(src), L.op_static_loop(mul, 100),
                                      L.op_static_loop(add, 100), L.op_write_per_thread(df)])
            unfused = L.validate_chain([L.op_read_per_thread(src)] + [mul] * 100 + [add] * 100 +
                                       [L.op_write_per_thread(du)])
            L.execute_fused(fused, self.cfg)
            L.execute_unfused(unfused, self.cfg)
            self.require_equal(df, du, f"datasize n={n}")
            recs.append(self.record("datasize", n, self.series(lambda: L.execute_fused(fused, self.cfg)),
                                    self.series(lambda: L.execute_unfused(unfused, self.cfg))))
        return recs

    def datatype(self):  # bench.cpp:350-409
        L, W, H, B = self.lib, 60, 120, 50
        pairs = [(U8, U8), (U8, F32), (U8, F64), (F32, F32), (F32, F64), (F32, U8), (F64, F32), (F64, F64)]
        recs = []
        for kin, kout in pairs:
            src = [self.random_plane(W, H, kin) for _ in range(B)]
            dfu = [self.plane(W, H, kout) for _ in range(B)]
            dba = [self.plane(W, H, kout) for _ in range(B)]
            cast = L.op_cast(kin, kout)
            mul, sub, div = (L.make_arith(op, const_of(kout, v)) for op, v in ((7, 3), (9, 1), (10, 2)))
            fused = L.validate_chain([L.op_batch_read([L.op_read_per_thread(s) for s in src]), cast, mul, sub, div,
                                      L.op_batch_write([L.op_write_per_thread(d) for d in dfu])])
            base = [L.validate_chain([L.op_read_per_thread(src[z]), cast, mul, sub, div,
                                      L.op_write_per_thread(dba[z])]) for z in range(B)]
            label = f"{KIND_NAME[kin]}->{KIND_NAME[kout]}"
            L.execute_fused(fused, self.cfg)
            for p in base:
                L.execute_unfused(p, self.cfg)
            for z in range(B):
                self.require_equal(dfu[z], dba[z], f"datatype {label}")

            def run_base():
                for p in base:
                    L.execute_unfused(p, self.cfg)
            recs.append(self.record("datatype", label, self.series(lambda: L.execute_fused(fused, self.cfg)),
                                    self.series(run_base)))
        return recs

    def memory(self, info):  # bench.cpp:411-475
        L = self.lib
        source = self.random_plane(256, 512, F32X3)
        out = [self.plane(60, 120, F32) for _ in range(3)]
        handles = [api.resize(api.crop(source, 10, 20, 120, 240, lib=L), 60, 120, BILINEAR, lib=L),
                   api.cvt_color(SWAP_RB), api.multiply(f32x3(255, 255, 255), lib=L),
                   api.subtract(f32x3(0.485, 0.456, 0.406), lib=L), api.divide(f32x3(0.229, 0.224, 0.225), lib=L),
                   api.split(out, lib=L)]
        pipeline = api.build_pipeline(handles)
        planned = L.plan_memory_savings(pipeline)
        fr = L.execute_fused(pipeline, self.cfg)
        ur = L.execute_unfused(pipeline, self.cfg)
        if ur.intermediate_bytes_allocated != planned:
            raise GateFailure("memory: planned savings disagree with measured allocation")
        img = 3840 * 2160 * 3
        info.write(f"pipeline crop->resize->cvt->mul->sub->div->split on 60x120 f32x3:\n"
                   f"  compute passes avoided: {pipeline.n_compute}\n"
                   f"  intermediate bytes saved per image: {planned}\n"
                   f"  intermediate bytes saved per batch of 50: {planned * 50}\n"
                   f"  fused intermediates: {fr.intermediate_bytes_allocated}, passes: {fr.passes}\n"
                   f"  unfused intermediates: {ur.intermediate_bytes_allocated}, passes: {ur.passes}\n"
                   f"4k RGB u8 frame (3840x2160x3): {img} bytes per intermediate\n")
        isrc = self.random_plane(60, 120, F32)
        idst = self.plane(60, 120, F32)
        identity = L.validate_chain([L.op_read_per_thread(isrc), L.op_write_per_thread(idst)])
        info.write(f"identity pipeline: {L.plan_memory_savings(identity)} bytes saved\n")
        return [self.record("memory", "image-preproc", self.series(lambda: L.execute_fused(pipeline, self.cfg)),
                            self.series(lambda: L.execute_unfused(pipeline, self.cfg))),
                self.record("memory", "identity", self.series(lambda: L.execute_fused(identity, self.cfg)),
                            self.series(lambda: L.execute_unfused(identity, self.cfg)))]

    def run(self, name, info):  # run_experiment, bench.cpp:483-494
        return {"vf": self.vf, "hf": self.hf, "vf-hf": self.vf_hf, "ipo": self.ipo, "datasize": self.datasize,
                "datatype": self.datatype, "memory": lambda: self.memory(info)}[name]()


def split_instructions(total: int, per_op: int) -> list:  # bench.cpp:119-123
    counts = [per_op] * (total // per_op)
    if total % per_op:
        counts.append(total % per_op)
    return counts


def write_csv(out, experiment: str, opt: Options, records) -> None:  # bench.cpp:497-514
    out.write(f"# opfuse bench {experiment} repeats={opt.repeats} warmup={opt.warmup} threads={opt.threads} "
              f"coarsen={opt.coarsen} chunk_rows={opt.chunk_rows} seed={opt.seed}\n")
    out.write("experiment,param,fused_ns,unfused_ns,speedup,rsd_pct\n")
    for r in records:
        out.write(f"{r.experiment},{r.param},{r.fused_ns:.0f},{r.unfused_ns:.0f},{r.speedup:.4f},{r.rsd_pct:.3f}\n")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="bench", add_help=True)
    ap.add_argument("experiment")
    ap.add_argument("--repeats", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--coarsen", type=int, default=8)
    ap.add_argument("--csv")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--backend", default="cuda", choices=["cuda", "oracle", "reference"])
    ap.add_argument("--quick", action="store_true", help="trimmed sweeps (tests)")
    try:
        a = ap.parse_args(argv)
    except SystemExit:
        return 1
    if a.experiment not in EXPERIMENTS or a.repeats < 3 or a.warmup < 0 or a.coarsen not in (1, 2, 4, 8, 16):
        print(f"usage: bench <{'|'.join(EXPERIMENTS)}> [--repeats N>=3] [--warmup N] [--threads N] "
              "[--coarsen 1|2|4|8|16] [--csv PATH] [--seed S]", file=sys.stderr)
        return 1
    opt = Options(a.repeats, a.warmup, a.threads, a.coarsen, 8, a.seed, a.backend, a.quick)
    try:
        records = Bench(opt).run(a.experiment, sys.stderr)
    except GateFailure as e:
        print(str(e), file=sys.stderr)
        return 2
    except OpfuseError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    if a.csv:
        with open(a.csv, "w") as f:
            write_csv(f, a.experiment, opt, records)
    else:
        write_csv(sys.stdout, a.experiment, opt, records)
    return 0


if __name__ == "__main__":
    sys.exit(main())
