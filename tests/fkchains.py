"""Backend-independent chain descriptions for the parity suites.

A chain is described once as plain data (ChainSpec) and instantiated on any
backend (cuda / oracle / reference) with identical inputs, so outputs can be
compared byte for byte. The random generator covers the reference's whole op
vocabulary (oplib.hpp:31-76): every kind, crop / nearest / bilinear reads,
folded unaries, casts, colour conversion, StaticLoop, batch reads with
default values, batch writes with inactive planes, split writes.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from paper_2508_07071_b200 import opfuse as of
from paper_2508_07071_b200._ffi import (BILINEAR, F32, F32X3, F64, F64X3, NEAREST, OP_ADD, OP_DIV, OP_MUL,
                                        OP_SUB, SWAP_RB, TO_GRAY_F32, U8, U8X3, LANES)

NP = {U8: np.uint8, F32: np.float32, F64: np.float64}


def lane_kind(k):
    return k - 3 if k >= U8X3 else k


def packed(k):
    return k + 3 if k < U8X3 else k


# ----------------------------------------------------------------- spec types --

@dataclass
class ReadSpec:
    src: int                    # index into ChainSpec.sources
    x0: int = 0
    y0: int = 0
    w: int = 0                  # crop rect (0 -> whole plane, op_read_per_thread)
    h: int = 0
    out_w: int = 0              # resize target (0 -> no resize)
    out_h: int = 0
    mode: int = BILINEAR
    post: list = field(default_factory=list)   # ('swap', kind) | ('cast', from, to) | ('gray', kind)


@dataclass
class ChainSpec:
    sources: list               # numpy arrays (h, w) or (h, w, 3)
    reads: list                 # ReadSpec per plane (len 1 = plain read, else BatchRead)
    compute: list               # ('arith', op_id, kind, lanes) | ('cast', f, t) | ('swap', k) | ('gray', k)
                                # | ('loop', inner_tuple, n) | ('batch_arith', op_id, kind, [lanes per z])
    write_kind: int             # kind reaching the write
    split: bool = False
    batch: bool = False         # wrap reads/writes in BatchRead/BatchWrite
    active_read: int | None = None
    active_write: int | None = None
    default: tuple | None = None
    dst_stride_pad: int = 0     # extra elements per destination row (strided writes)


def out_dims(spec: ChainSpec):
    r = spec.reads[0]
    if r.out_w:
        return r.out_w, r.out_h
    if r.w:
        return r.w, r.h
    a = spec.sources[r.src]
    return a.shape[1], a.shape[0]


# -------------------------------------------------------------- instantiation --

def _unary(lib, u):
    if u[0] == "swap":
        return lib.op_color_convert(SWAP_RB, u[1])
    if u[0] == "gray":
        return lib.op_color_convert(TO_GRAY_F32, u[1])
    return lib.op_cast(u[1], u[2])


def _compute(lib, c):
    t = c[0]
    if t == "arith":
        return lib.make_arith(c[1], of.const_of(c[2], *c[3]))
    if t == "loop":
        return lib.op_static_loop(_compute(lib, c[1]), c[2])
    if t == "batch_arith":
        return lib.op_batch_arith(c[1], [of.const_of(c[2], *v) for v in c[3]])
    return _unary(lib, c)


def make_read(lib: of.Library, spec: ChainSpec):
    """The read IOp of `spec` on `lib` (BatchRead when spec.batch) and its source planes."""
    planes = [lib.plane_from_numpy(a) for a in spec.sources]
    reads = []
    for r in spec.reads:
        src = planes[r.src]
        op = lib.op_crop(src, r.x0, r.y0, r.w, r.h) if r.w else lib.op_read_per_thread(src)
        if r.out_w:
            op = lib.op_resize(op, r.out_w, r.out_h, r.mode)
        for u in r.post:
            op = lib.fold_unary_into_read(op, _unary(lib, u))
        reads.append(op)
    if spec.batch:
        dv = of.const_of(reads[0].output_kind, *spec.default) if spec.default is not None else None
        return lib.op_batch_read(reads, spec.active_read, dv), planes
    return reads[0], planes


def make_compute(lib: of.Library, c):
    return _compute(lib, c)


def instantiate(lib: of.Library, spec: ChainSpec):
    """Build (pipeline, destination planes) for `spec` on `lib`."""
    planes = [lib.plane_from_numpy(a) for a in spec.sources]
    reads = []
    for r in spec.reads:
        src = planes[r.src]
        op = lib.op_crop(src, r.x0, r.y0, r.w, r.h) if r.w else lib.op_read_per_thread(src)
        if r.out_w:
            op = lib.op_resize(op, r.out_w, r.out_h, r.mode)
        for u in r.post:
            op = lib.fold_unary_into_read(op, _unary(lib, u))
        reads.append(op)
    W, H = out_dims(spec)
    n = len(spec.reads)
    dests, writes = [], []
    for _ in range(n):
        if spec.split:
            d = [lib.plane_alloc(W, H, lane_kind(spec.write_kind), W + spec.dst_stride_pad) for _ in range(3)]
            writes.append(lib.op_split_write(d))
        else:
            d = [lib.plane_alloc(W, H, spec.write_kind, W + spec.dst_stride_pad)]
            writes.append(lib.op_write_per_thread(d[0]))
        dests.append(d)
    if spec.batch:
        dv = of.const_of(reads[0].output_kind, *spec.default) if spec.default is not None else None
        read = lib.op_batch_read(reads, spec.active_read, dv)
        write = lib.op_batch_write(writes, spec.active_write)
    else:
        read, write = reads[0], writes[0]
    chain = [read] + [_compute(lib, c) for c in spec.compute] + [write]
    return lib.validate_chain(chain), dests, planes


def run(lib: of.Library, spec: ChainSpec, unfused=False, cfg=None):
    p, dests, _ = instantiate(lib, spec)
    rep = (lib.execute_unfused if unfused else lib.execute_fused)(p, cfg)
    return [[d.to_numpy() for d in ds] for ds in dests], rep


def same(a: np.ndarray, b: np.ndarray) -> bool:
    """Bitwise equality; any NaN equals any NaN (payloads are not specified:
    x86 and sm_100 produce different default-NaN bit patterns)."""
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.dtype.kind != "f":
        return bool(np.array_equal(a, b))
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    ia = a.view(np.uint32 if a.dtype == np.float32 else np.uint64)
    ib = b.view(np.uint32 if b.dtype == np.float32 else np.uint64)
    return bool(np.array_equal(ia[~na], ib[~nb]))


def outputs_equal(x, y) -> bool:
    return all(same(a, b) for da, db in zip(x, y) for a, b in zip(da, db))


def mismatch_report(x, y) -> str:
    out = []
    for z, (da, db) in enumerate(zip(x, y)):
        for l, (a, b) in enumerate(zip(da, db)):
            if not same(a, b):
                diff = np.argwhere((a != b) & ~(np.isnan(a) & np.isnan(b)) if a.dtype.kind == "f" else a != b)
                i = tuple(diff[0]) if len(diff) else ()
                out.append(f"plane z={z} dest={l}: {len(diff)} mismatches, first at {i}: {a[i] if i else ''} vs {b[i] if i else ''}")
    return "; ".join(out)


# ------------------------------------------------------------------ generator --

def random_source(rng, kind, w, h):
    lk, lanes = lane_kind(kind), LANES[kind]
    shape = (h, w, 3) if lanes == 3 else (h, w)
    if lk == U8:
        return rng.integers(0, 256, shape, dtype=np.uint8)
    # mix of magnitudes and signs; occasional specials
    a = (rng.random(shape) * rng.choice([1.0, 255.0, 300.0, -3.0])).astype(NP[lk])
    if rng.random() < 0.2:
        flat = a.reshape(-1)
        idx = rng.integers(0, flat.size, max(1, flat.size // 50))
        flat[idx] = rng.choice(np.array([0.5, 1.5, 2.5, 254.5, 255.5, -0.0, np.nan, np.inf, 1e-40], dtype=NP[lk]),
                               len(idx))
    return a


def _rand_const(rng, kind, op_id):
    lk, lanes = lane_kind(kind), LANES[kind]
    vals = []
    for _ in range(lanes):
        if lk == U8:
            v = int(rng.integers(1 if op_id == OP_DIV else 0, 256))
        else:
            v = float(rng.choice([rng.uniform(-4, 4), rng.uniform(0.5, 2), 255.0, 1.25, 0.1, 3.0]))
            if op_id == OP_DIV and v == 0.0:
                v = 1.0
            if lk == F32:
                v = struct.unpack("f", struct.pack("f", v))[0]
        vals.append(v)
    return tuple(vals)


def _rand_compute(rng, kind, n_planes, allow_batch_arith):
    """One compute op taking `kind`; returns (op tuple, output kind)."""
    lanes = LANES[kind]
    r = rng.random()
    if r < 0.45:
        op_id = int(rng.choice([OP_MUL, OP_ADD, OP_SUB, OP_DIV]))
        if allow_batch_arith and rng.random() < 0.3:
            return ("batch_arith", op_id, kind, [_rand_const(rng, kind, op_id) for _ in range(n_planes)]), kind
        return ("arith", op_id, kind, _rand_const(rng, kind, op_id)), kind
    if r < 0.75:
        to = int(rng.choice([U8, F32, F64])) + (3 if lanes == 3 else 0)
        return ("cast", kind, to), to
    if r < 0.85 and lanes == 3:
        return ("swap", kind), kind
    if r < 0.9 and lanes == 3:
        return ("gray", kind), F32
    op_id = int(rng.choice([OP_MUL, OP_ADD, OP_SUB, OP_DIV]))
    inner = ("arith", op_id, kind, _rand_const(rng, kind, op_id))
    if lanes == 3 and rng.random() < 0.3:
        inner = ("swap", kind)
    return ("loop", inner, int(rng.integers(1, 20))), kind


def random_chain(rng, max_ops=8, max_dim=24, max_batch=4, allow_batch_arith=False) -> ChainSpec:
    src_kind = int(rng.integers(0, 6))
    batch = int(rng.integers(1, max_batch + 1)) if rng.random() < 0.5 else 1
    use_batch = batch > 1 or rng.random() < 0.2
    out_w, out_h = int(rng.integers(1, max_dim + 1)), int(rng.integers(1, max_dim + 1))
    mode = int(rng.integers(0, 3))  # 0 plain, 1 crop, 2 crop+resize
    resize_mode = int(rng.choice([NEAREST, BILINEAR]))
    sources, reads = [], []
    post = []
    kind = src_kind
    for _ in range(int(rng.integers(0, 3))):  # folded unaries
        if LANES[kind] == 3 and rng.random() < 0.4:
            post.append(("swap", kind))
        else:
            to = int(rng.choice([U8, F32, F64])) + (3 if LANES[kind] == 3 else 0)
            post.append(("cast", kind, to))
            kind = to
    for z in range(batch):
        if mode == 0:
            a = random_source(rng, src_kind, out_w, out_h)
            reads.append(ReadSpec(len(sources), post=list(post)))
        else:
            if mode == 1:
                w, h = out_w, out_h
            else:
                w, h = int(rng.integers(1, 2 * max_dim)), int(rng.integers(1, 2 * max_dim))
            sw, sh = w + int(rng.integers(0, 6)), h + int(rng.integers(0, 6))
            a = random_source(rng, src_kind, sw, sh)
            x0, y0 = int(rng.integers(0, sw - w + 1)), int(rng.integers(0, sh - h + 1))
            reads.append(ReadSpec(len(sources), x0, y0, w, h, out_w if mode == 2 else 0,
                                  out_h if mode == 2 else 0, resize_mode, list(post)))
        sources.append(a)
    compute = []
    for _ in range(int(rng.integers(0, max_ops + 1))):
        op, kind = _rand_compute(rng, kind, batch, allow_batch_arith and use_batch)
        compute.append(op)
    split = LANES[kind] == 3 and rng.random() < 0.5
    spec = ChainSpec(sources, reads, compute, kind, split=split, batch=use_batch,
                     dst_stride_pad=int(rng.integers(0, 3)))
    if use_batch:
        spec.active_read = int(rng.integers(1, batch + 1))
        spec.active_write = int(rng.integers(1, batch + 1))
        rk = reads_out_kind(spec)
        spec.default = _rand_const(rng, rk, OP_ADD)
    return spec


def reads_out_kind(spec: ChainSpec) -> int:
    r = spec.reads[0]
    k = of.kind_of_array(spec.sources[r.src])
    for u in r.post:
        k = u[2] if u[0] == "cast" else (F32 if u[0] == "gray" else k)
    return k


# ------------------------------------------------------------ serialisation --

def spec_to_dict(spec: ChainSpec) -> dict:
    """JSON-able description (sources are stored separately, by index)."""
    return {"reads": [vars(r) | {"post": [list(u) for u in r.post]} for r in spec.reads],
            "compute": [_ser(c) for c in spec.compute], "write_kind": spec.write_kind, "split": spec.split,
            "batch": spec.batch, "active_read": spec.active_read, "active_write": spec.active_write,
            "default": list(spec.default) if spec.default is not None else None,
            "dst_stride_pad": spec.dst_stride_pad, "n_sources": len(spec.sources)}


def _ser(c):
    if c[0] == "loop":
        return ["loop", _ser(c[1]), c[2]]
    if c[0] == "batch_arith":
        return ["batch_arith", c[1], c[2], [list(v) for v in c[3]]]
    if c[0] == "arith":
        return ["arith", c[1], c[2], list(c[3])]
    return list(c)


def _deser(c):
    if c[0] == "loop":
        return ("loop", _deser(c[1]), c[2])
    if c[0] == "batch_arith":
        return ("batch_arith", c[1], c[2], [tuple(v) for v in c[3]])
    if c[0] == "arith":
        return ("arith", c[1], c[2], tuple(c[3]))
    return tuple(c)


def spec_from_dict(d: dict, sources: list) -> ChainSpec:
    reads = [ReadSpec(**(r | {"post": [tuple(u) for u in r["post"]]})) for r in d["reads"]]
    return ChainSpec(sources, reads, [_deser(c) for c in d["compute"]], d["write_kind"], d["split"], d["batch"],
                     d["active_read"], d["active_write"], tuple(d["default"]) if d["default"] is not None else None,
                     d["dst_stride_pad"])
