"""The reference's final-user facade (api.hpp / api.cpp, §4.4) over the
fused-chain library: lazy handles that move no data, one fused execution per
`execute_operations` / `execute_batch` call.

    from paper_2508_07071_b200 import api
    handles = [api.resize(api.crop(frame, 10, 20, 120, 240), 60, 120),
               api.cvt_color(SWAP_RB), api.multiply(f32x3(255, 255, 255)),
               api.subtract(f32x3(*mean)), api.divide(f32x3(*std)), api.split(planes)]
    api.execute_operations(handles)          # builds once (cached by handle uids), one launch

Semantics follow api.cpp line by line: deferred cvt_color resolves against
the kind flowing at its position (api.cpp:94-117), leading unary ops fold
into the read (:127-143), chain errors carry the offending handle's provenance
"<name> (handle #i)" (:149-159), and a process-wide cache keyed by the handle
uid sequence skips re-validation on repeat calls (:161-202).
"""
from __future__ import annotations

import itertools
import threading
from dataclasses import dataclass, field
from typing import Sequence

from ._ffi import BILINEAR, KIND_UNARY, KIND_READ, KIND_WRITE, OP_CROP_READ, OP_PER_THREAD_READ, OP_RESIZE_READ
from .opfuse import Const, ExecConfig, ExecReport, IOp, Library, OpfuseError, Pipeline, Plane, default_library

_uids = itertools.count(1)
_SAMPLE_READS = (OP_PER_THREAD_READ, OP_CROP_READ, OP_RESIZE_READ)


@dataclass(frozen=True)
class LazyHandle:
    """A deferred operation (api.hpp:13-32): constructing one executes nothing."""
    provenance: str
    uid: int
    iop: IOp | None = None          # None: deferred cvt_color / cast
    color_order: int = 0
    cast_to: int | None = None      # deferred cast: the target kind
    lib: Library | None = field(default=None, compare=False)

    @property
    def deferred(self) -> bool:
        return self.iop is None


def _guarded(provenance: str, fn):
    try:
        return fn()
    except OpfuseError as e:
        e.provenance = provenance
        raise


def _handle(name: str, fn, lib: Library | None) -> LazyHandle:
    lib = lib or default_library()
    return LazyHandle(name, next(_uids), _guarded(name, lambda: fn(lib)), lib=lib)


def read(source: Plane, lib: Library | None = None) -> LazyHandle:
    return _handle("read", lambda L: L.op_read_per_thread(source), lib)


def write(dest: Plane, lib: Library | None = None) -> LazyHandle:
    return _handle("write", lambda L: L.op_write_per_thread(dest), lib)


def crop(source: Plane, x0: int, y0: int, w: int, h: int, lib: Library | None = None) -> LazyHandle:
    return _handle("crop", lambda L: L.op_crop(source, x0, y0, w, h), lib)


def resize(upstream, width: int, height: int, mode: int = BILINEAR, lib: Library | None = None) -> LazyHandle:
    """resize(Plane | LazyHandle, ...) — collapses with an upstream read/crop into one fused read."""
    if isinstance(upstream, LazyHandle):
        if upstream.deferred:
            raise OpfuseError(1 + 9, "UnsupportedKind: resize upstream must be a read handle", -1, "resize")
        return _handle("resize", lambda L: L.op_resize(upstream.iop, width, height, mode), lib or upstream.lib)
    return _handle("resize", lambda L: L.op_resize(upstream, width, height, mode), lib)


def cvt_color(order: int) -> LazyHandle:
    """The element kind is taken from the chain when the pipeline is built (api.hpp:43)."""
    return LazyHandle("cvt_color", next(_uids), None, order)


def cast(to: int) -> LazyHandle:
    """The handle the reference facade lacks: cast the flowing
    value to kind `to`; the source kind is taken from the chain when the pipeline
    is built (like cvt_color)."""
    return LazyHandle("cast", next(_uids), None, 0, to)


def multiply(c: Const, lib: Library | None = None) -> LazyHandle:
    return _handle("multiply", lambda L: L.op_mul(c), lib)


def subtract(c: Const, lib: Library | None = None) -> LazyHandle:
    return _handle("subtract", lambda L: L.op_sub(c), lib)


def divide(c: Const, lib: Library | None = None) -> LazyHandle:
    return _handle("divide", lambda L: L.op_div(c), lib)


def split(dest: Sequence[Plane], lib: Library | None = None) -> LazyHandle:
    return _handle("split", lambda L: L.op_split_write(dest), lib)


# ------------------------------------------------------------------- building --

def _lib_of(handles: Sequence[LazyHandle]) -> Library:
    for h in handles:
        if h.lib is not None:
            return h.lib
    return default_library()


def _resolve_chain(handles: Sequence[LazyHandle], lib: Library) -> list[IOp]:
    """api.cpp:94-117: deferred cvt_color against the kind flowing at its position."""
    ops, current = [], None
    for i, h in enumerate(handles):
        if h.deferred:
            if current is None:
                raise OpfuseError(1 + 3, f"KindMismatch: {h.provenance} has no upstream value", i, h.provenance)
            if h.cast_to is not None:
                op = _guarded(h.provenance, lambda: lib.op_cast(current, h.cast_to))
            else:
                op = _guarded(h.provenance, lambda: lib.op_color_convert(h.color_order, current))
            current = op.output_kind
            ops.append(op)
        else:
            if h.iop.output_kind is not None:
                current = h.iop.output_kind
            ops.append(h.iop)
    return ops


def _fold_leading_unaries(ops: list[IOp], lib: Library) -> tuple[list[IOp], int]:
    """api.cpp:127-143: unary ops right after a sample read fold into it."""
    if not ops or ops[0].kind != KIND_READ or ops[0].id not in _SAMPLE_READS:
        return ops, 0
    read, i, folded = ops[0], 1, 0
    while i + 1 < len(ops) and ops[i].kind == KIND_UNARY:
        read = lib.fold_unary_into_read(read, ops[i])
        i += 1
        folded += 1
    return [read] + ops[i:], folded


def build_pipeline(handles: Sequence[LazyHandle]) -> Pipeline:
    """api.cpp:183-186 + validate_with_provenance (:149-159)."""
    if not handles:
        raise OpfuseError(1 + 0, "EmptyChain: no handles")
    lib = _lib_of(handles)
    ops, folded = _fold_leading_unaries(_resolve_chain(handles, lib), lib)
    try:
        return lib.validate_chain(ops)
    except OpfuseError as e:
        idx = 0 if e.position <= 0 else e.position + folded
        if idx < len(handles) and not e.provenance:
            e.provenance = f"{handles[idx].provenance} (handle #{idx + 1})"
        raise


class _Cache:
    """api.cpp:161-202: handle-uid sequence -> built pipeline, mutex-protected, never evicted."""

    def __init__(self):
        self.lock = threading.Lock()
        self.built: dict[tuple, Pipeline] = {}
        self.validations = 0


_cache = _Cache()


def validations() -> int:
    """How many pipelines execute_operations has built (one per distinct handle chain)."""
    return _cache.validations


def execute_operations(handles: Sequence[LazyHandle], config: ExecConfig | None = None) -> ExecReport:
    """api.cpp:188-203: build (or reuse) the pipeline for this exact handle chain, one fused execution."""
    key = tuple(h.uid for h in handles)
    with _cache.lock:
        pipeline = _cache.built.get(key)
    if pipeline is None:
        pipeline = build_pipeline(handles)
        with _cache.lock:
            _cache.built.setdefault(key, pipeline)
            _cache.validations += 1
    return pipeline._lib.execute_fused(pipeline, config)


def build_batch_pipeline(per_plane_reads: Sequence[LazyHandle], shared_compute: Sequence[LazyHandle],
                         per_plane_writes: Sequence[LazyHandle]) -> Pipeline:
    """api.cpp:204-260: BatchRead/BatchWrite around the shared chain; leading unaries fold into every read."""
    if not per_plane_reads:
        raise OpfuseError(1 + 12, "EmptyBatch: batch needs at least one read")
    if len(per_plane_reads) != len(per_plane_writes):
        raise OpfuseError(1 + 14, "HeterogeneousBatch: read and write handle counts differ")
    lib = _lib_of(list(per_plane_reads) + list(shared_compute))
    resolved = _resolve_chain([per_plane_reads[0]] + list(shared_compute), lib)
    n_fold = 0
    while 1 + n_fold < len(resolved) and resolved[1 + n_fold].kind == KIND_UNARY:
        n_fold += 1
    inner_reads = []
    for i, h in enumerate(per_plane_reads):
        if h.deferred or h.iop.kind != KIND_READ or h.iop.id not in _SAMPLE_READS:
            raise OpfuseError(1 + 14, f"HeterogeneousBatch: read handle #{i + 1} is not a per-plane read", i,
                              h.provenance)
        r = h.iop
        for f in range(n_fold):
            r = _guarded(h.provenance, lambda: lib.fold_unary_into_read(r, resolved[1 + f]))
        inner_reads.append(r)
    inner_writes = []
    for i, h in enumerate(per_plane_writes):
        if h.deferred or h.iop.kind != KIND_WRITE:
            raise OpfuseError(1 + 14, f"HeterogeneousBatch: write handle #{i + 1} is not a per-plane write", i,
                              h.provenance)
        inner_writes.append(h.iop)
    chain = [lib.op_batch_read(inner_reads)] + resolved[1 + n_fold:] + [lib.op_batch_write(inner_writes)]
    return lib.validate_chain(chain)


def execute_batch(per_plane_reads: Sequence[LazyHandle], shared_compute: Sequence[LazyHandle],
                  per_plane_writes: Sequence[LazyHandle], config: ExecConfig | None = None) -> ExecReport:
    """api.cpp:262-268: horizontal + vertical fusion in one call (one launch)."""
    p = build_batch_pipeline(per_plane_reads, shared_compute, per_plane_writes)
    return p._lib.execute_fused(p, config)
