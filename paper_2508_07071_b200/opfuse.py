"""Host-side mirror of the reference's opfuse API over the include/fk.h C-ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/opfuse/{plane,ops,oplib,executor}.hpp), so a
pipeline written against the reference reads the same here:

    lib = Library()                                   # the CUDA product (sm_100a)
    src = lib.plane_from_numpy(img)                   # device plane
    dst = lib.plane_alloc(w, h, U8)
    p = lib.validate_chain([lib.op_read_per_thread(src), lib.op_mul(f32(400.0)),
                            lib.op_cast(F32, U8), lib.op_write_per_thread(dst)])
    rep = lib.execute_fused(p)

Every failure raises :class:`OpfuseError` carrying the reference's ``Errc`` name
(errors.hpp:9-38) and the chain position. ``Library()`` defaults to the CUDA
backend and raises when ``libfk_cuda.so`` is missing: the product path has no
CPU fallback. ``Library("oracle")`` / ``Library("reference")`` exist for tests.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _ffi
from ._ffi import (BILINEAR, F32, F32X3, F64, F64X3, NEAREST, SWAP_RB, TO_GRAY_F32, U8,  # noqa: F401
                   U8X3, BYTES_PER_ELEMENT, KIND_NAMES, LANES)

_NP_DTYPE = {U8: np.uint8, F32: np.float32, F64: np.float64, U8X3: np.uint8, F32X3: np.float32,
             F64X3: np.float64}
_STRUCT_FMT = {U8: "B", F32: "f", F64: "d"}


def lane_kind(kind: int) -> int:
    return kind - 3 if kind >= U8X3 else kind


class OpfuseError(RuntimeError):
    """opfuse::Error (errors.hpp:45-66): Errc name, chain position, provenance."""

    def __init__(self, status: int, message: str, position: int = -1, provenance: str = ""):
        super().__init__(message)
        self.status = status
        self.code = _ffi.errc_name(status)
        self.position = position
        self.provenance = provenance

    def __str__(self) -> str:
        s = super().__str__()
        return f"{s} [{self.provenance}]" if self.provenance else s


# ------------------------------------------------------------------ constants --

@dataclass(frozen=True)
class Const:
    """Typed per-lane constant (oplib.hpp:8-21): `kind` plus raw little-endian lanes."""
    kind: int
    lanes: tuple

    def raw(self) -> bytes:
        fmt = _STRUCT_FMT[lane_kind(self.kind)]
        return struct.pack("<" + fmt * LANES[self.kind], *self.lanes)


def u8(v) -> Const: return Const(U8, (int(v) & 0xFF,))
def f32(v) -> Const: return Const(F32, (float(v),))
def f64(v) -> Const: return Const(F64, (float(v),))
def u8x3(a, b, c) -> Const: return Const(U8X3, (int(a) & 0xFF, int(b) & 0xFF, int(c) & 0xFF))
def f32x3(a, b, c) -> Const: return Const(F32X3, (float(a), float(b), float(c)))
def f64x3(a, b, c) -> Const: return Const(F64X3, (float(a), float(b), float(c)))


def const_of(kind: int, *lanes) -> Const:
    if LANES[kind] == 1:
        return {U8: u8, F32: f32, F64: f64}[kind](lanes[0])
    if len(lanes) == 1:
        lanes = lanes * 3
    return {U8X3: u8x3, F32X3: f32x3, F64X3: f64x3}[kind](*lanes)


# --------------------------------------------------------------------- planes --

class Plane:
    """Strided 2D view (plane.hpp:60-103) over a torch uint8 storage tensor.

    Device planes (CUDA backend) live in HBM; host planes (oracle/reference) in
    RAM. row_stride is in elements; packed x3 lanes are adjacent.
    """

    def __init__(self, storage, byte_offset: int, width: int, height: int, row_stride: int, kind: int):
        self.storage = storage
        self.byte_offset = int(byte_offset)
        self.width, self.height, self.row_stride, self.kind = int(width), int(height), int(row_stride), int(kind)

    @property
    def bpe(self) -> int:
        return BYTES_PER_ELEMENT[self.kind]

    @property
    def data_ptr(self) -> int:
        return self.storage.data_ptr() + self.byte_offset

    @property
    def payload_bytes(self) -> int:
        return self.width * self.height * self.bpe

    def c(self) -> _ffi.fk_plane:
        return _ffi.fk_plane(self.data_ptr, self.width, self.height, self.row_stride, self.kind)

    def view(self, x0: int, y0: int, width: int, height: int) -> "Plane":
        """Zero-copy sub-view (Plane::view, plane.cpp:91-101)."""
        if width == 0 or height == 0 or x0 + width > self.width or y0 + height > self.height:
            raise OpfuseError(1 + 16, "BoundsError: sub-view outside plane")
        off = self.byte_offset + (y0 * self.row_stride + x0) * self.bpe
        return Plane(self.storage, off, width, height, self.row_stride, self.kind)

    def to_numpy(self) -> np.ndarray:
        """Logical contents as (h, w) or (h, w, 3) array (a copy)."""
        import torch
        row_bytes = self.row_stride * self.bpe
        total = (self.height - 1) * row_bytes + self.width * self.bpe
        flat = self.storage[self.byte_offset:self.byte_offset + total]
        if flat.device.type != "cpu":
            torch.cuda.synchronize(flat.device)
            flat = flat.cpu()
        buf = flat.numpy()
        pad = self.height * row_bytes - total
        if pad:
            buf = np.concatenate([buf, np.zeros(pad, np.uint8)])
        rows = buf.reshape(self.height, row_bytes)[:, : self.width * self.bpe]
        arr = np.ascontiguousarray(rows).view(_NP_DTYPE[self.kind])
        if LANES[self.kind] == 3:
            return arr.reshape(self.height, self.width, 3)
        return arr.reshape(self.height, self.width)

    def raw_bytes(self) -> bytes:
        return self.to_numpy().tobytes()

    def __repr__(self) -> str:
        return (f"Plane({self.width}x{self.height} {KIND_NAMES[self.kind]} stride={self.row_stride} "
                f"on {self.storage.device})")


class RawPlane:
    """A bare fk_plane view (no Python-side owner)."""

    def __init__(self, raw: "_ffi.fk_plane"):
        self._raw = raw
        self.width, self.height, self.row_stride, self.kind = raw.width, raw.height, raw.row_stride, raw.kind

    def c(self) -> "_ffi.fk_plane":
        return self._raw


class SharedPlane:
    """A plane from fk_plane_alloc (Plane::alloc, plane.cpp:60-71): the buffer is
    shared with every IOp / pipeline built from it or a view of it, like the
    reference's shared_ptr<TensorBuffer> (plane.hpp:97); free() (or garbage
    collection) only drops this handle's reference."""

    def __init__(self, lib: "Library", raw: "_ffi.fk_plane"):
        self._lib, self._raw = lib, raw
        self.width, self.height, self.row_stride, self.kind = raw.width, raw.height, raw.row_stride, raw.kind

    @property
    def bpe(self) -> int:
        return BYTES_PER_ELEMENT[self.kind]

    @property
    def data_ptr(self) -> int:
        return int(self._raw.data or 0)

    def c(self) -> "_ffi.fk_plane":
        return _ffi.fk_plane(self._raw.data, self.width, self.height, self.row_stride, self.kind)

    def view(self, x0: int, y0: int, width: int, height: int) -> "RawPlane":
        """fk_plane_view: a zero-copy sub-view (it does not keep the buffer alive by
        itself; IOps built from it do)."""
        out = _ffi.fk_plane()
        self._lib._check(self._lib._c.fk_plane_view(C.byref(self._raw), x0, y0, width, height, C.byref(out)))
        return RawPlane(out)

    def free(self):
        if self._raw.data:
            self._lib._c.fk_plane_free(C.byref(self._raw))

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def kind_of_array(arr: np.ndarray) -> int:
    packed = arr.ndim == 3
    if packed and arr.shape[2] != 3:
        raise ValueError("packed planes need a trailing dimension of 3")
    base = {np.dtype(np.uint8): U8, np.dtype(np.float32): F32, np.dtype(np.float64): F64}[arr.dtype]
    return base + 3 if packed else base


# ------------------------------------------------------------------ IOps etc --

class IOp:
    """InstantiableOp handle (ops.hpp:131-153). Keeps its planes alive."""

    def __init__(self, lib: "Library", ptr: int, keep: Iterable = ()):
        self._lib = lib
        self._ptr = C.c_void_p(ptr)
        self._keep = list(keep)

    def __del__(self):
        try:
            if self._ptr and self._ptr.value:
                self._lib._c.fk_iop_free(self._ptr)
                self._ptr = C.c_void_p(None)
        except Exception:
            pass

    @property
    def id(self) -> int: return self._lib._c.fk_iop_id(self._ptr)
    @property
    def name(self) -> str: return _ffi.OP_NAMES.get(self.id, "?")
    @property
    def kind(self) -> int: return self._lib._c.fk_iop_kind(self._ptr)

    @property
    def input_kind(self):
        k = self._lib._c.fk_iop_input_kind(self._ptr)
        return None if k < 0 else k

    @property
    def output_kind(self):
        k = self._lib._c.fk_iop_output_kind(self._ptr)
        return None if k < 0 else k

    @property
    def dims_hint(self):
        e = _ffi.fk_extent3()
        return (e.width, e.height, e.batch) if self._lib._c.fk_iop_dims(self._ptr, C.byref(e)) else None

    def __repr__(self) -> str:
        return f"IOp({self.name})"


class Pipeline:
    """Validated Read -> Compute* -> Write chain (ops.hpp:156-161)."""

    def __init__(self, lib: "Library", ptr: int, keep: Iterable = ()):
        self._lib = lib
        self._ptr = C.c_void_p(ptr)
        self._keep = list(keep)

    def __del__(self):
        try:
            if self._ptr and self._ptr.value:
                self._lib._c.fk_pipeline_free(self._ptr)
                self._ptr = C.c_void_p(None)
        except Exception:
            pass

    @property
    def iter_space(self):
        e = _ffi.fk_extent3()
        self._lib._check(self._lib._c.fk_pipeline_iter_space(self._ptr, C.byref(e)))
        return (e.width, e.height, e.batch)

    @property
    def n_compute(self) -> int:
        return self._lib._c.fk_pipeline_compute_count(self._ptr)


@dataclass
class ExecConfig:
    """ExecConfig (executor.hpp:10-14) + device fields."""
    workers: int = 0
    coarsening: int = 8
    chunk_rows: int = 8
    stream: int | None = None   # cudaStream_t as int (torch: stream.cuda_stream)
    timed: bool = False
    force_generic: bool = False
    serial: bool = False
    no_lut: bool = False

    def c(self) -> _ffi.fk_exec_config:
        flags = ((_ffi.EXEC_TIMED if self.timed else 0) | (_ffi.EXEC_FORCE_GENERIC if self.force_generic else 0)
                 | (_ffi.EXEC_SERIAL if self.serial else 0) | (_ffi.EXEC_NO_LUT if self.no_lut else 0))
        return _ffi.fk_exec_config(self.workers, self.coarsening, self.chunk_rows, flags, self.stream)


@dataclass
class ExecReport:
    """ExecReport (executor.hpp:27-34) + device fields."""
    wall_time_ns: int = 0
    bytes_read: int = 0
    bytes_written: int = 0
    intermediate_bytes_allocated: int = 0
    passes: int = 0
    points_visited: int = 0
    kernels_launched: int = 0
    device_ms: float = 0.0
    path: int = 0

    @classmethod
    def from_c(cls, r: _ffi.fk_exec_report) -> "ExecReport":
        return cls(r.wall_time_ns, r.bytes_read, r.bytes_written, r.intermediate_bytes_allocated, r.passes,
                   r.points_visited, r.kernels_launched, r.device_ms, r.path)


# -------------------------------------------------------------------- library --

class Library:
    """One loaded backend. ``Library()`` is the CUDA product."""

    def __init__(self, backend: str = "cuda"):
        self.backend = backend
        self._c = _ffi.load(backend)
        self.device = "cuda" if backend == "cuda" else "cpu"

    # -- errors
    def _check(self, status: int):
        if status != 0:
            msg = self._c.fk_last_error().decode(errors="replace")
            raise OpfuseError(status, msg, self._c.fk_last_error_position())

    def _iop(self, fn, *args, keep=()) -> IOp:
        out = C.c_void_p()
        self._check(fn(*args, C.byref(out)))
        return IOp(self, out.value, keep)

    @property
    def name(self) -> str:
        return self._c.fk_backend_name().decode()

    # -- planes
    def _storage(self, nbytes: int):
        import torch
        return torch.zeros(max(nbytes, 1), dtype=torch.uint8, device=self.device)

    def plane_alloc(self, width: int, height: int, kind: int, row_stride: int | None = None) -> Plane:
        """Zero-initialised plane (Plane::alloc, plane.cpp:60-71)."""
        if width < 1 or height < 1:
            raise OpfuseError(1 + 17, "CapacityOverflow: plane extents must be >= 1")
        rs = width if row_stride is None else row_stride
        return Plane(self._storage(rs * height * BYTES_PER_ELEMENT[kind]), 0, width, height, rs, kind)

    def plane_alloc_shared(self, width: int, height: int, kind: int, row_stride: int = 0) -> SharedPlane:
        """fk_plane_alloc: a library-owned plane whose buffer IOps keep alive (plane.hpp:97)."""
        out = _ffi.fk_plane()
        self._check(self._c.fk_plane_alloc(width, height, kind, row_stride, C.byref(out)))
        return SharedPlane(self, out)

    def plane_from_numpy(self, arr: np.ndarray, kind: int | None = None, row_stride: int | None = None) -> Plane:
        import torch
        arr = np.ascontiguousarray(arr)
        kind = kind_of_array(arr) if kind is None else kind
        h, w = arr.shape[0], arr.shape[1]
        p = self.plane_alloc(w, h, kind, row_stride)
        host = torch.from_numpy(arr.view(np.uint8).reshape(h, -1).copy())
        rows = p.storage[: h * p.row_stride * p.bpe].view(h, p.row_stride * p.bpe)
        rows[:, : w * p.bpe].copy_(host.to(self.device))
        return p

    def plane_view(self, p: Plane, x0: int, y0: int, w: int, h: int) -> Plane:
        out = _ffi.fk_plane()
        self._check(self._c.fk_plane_view(C.byref(p.c()), x0, y0, w, h, C.byref(out)))
        return p.view(x0, y0, w, h)

    # -- builders (oplib.hpp:31-76)
    def make_arith(self, op_id: int, c: Const) -> IOp:
        raw = C.create_string_buffer(c.raw(), 24)
        return self._iop(self._c.fk_op_arith, op_id, c.kind, raw)

    def op_mul(self, c: Const) -> IOp: return self.make_arith(_ffi.OP_MUL, c)
    def op_add(self, c: Const) -> IOp: return self.make_arith(_ffi.OP_ADD, c)
    def op_sub(self, c: Const) -> IOp: return self.make_arith(_ffi.OP_SUB, c)
    def op_div(self, c: Const) -> IOp: return self.make_arith(_ffi.OP_DIV, c)

    def op_batch_arith(self, op_id: int, consts: Sequence[Const]) -> IOp:
        """Extension: arithmetic whose constant is selected by batch index z."""
        if not consts:
            raise OpfuseError(1 + 12, "EmptyBatch: batch arith over zero planes")
        kind = consts[0].kind
        raw = b"".join(c.raw() for c in consts)
        buf = C.create_string_buffer(raw, len(raw))
        return self._iop(self._c.fk_op_batch_arith, op_id, kind, buf, len(consts))

    def op_cast(self, frm: int, to: int) -> IOp:
        return self._iop(self._c.fk_op_cast, frm, to)

    def op_static_loop(self, inner: IOp, repeat: int) -> IOp:
        return self._iop(self._c.fk_op_static_loop, inner._ptr, repeat)

    def op_read_per_thread(self, src: Plane) -> IOp:
        return self._iop(self._c.fk_op_read_per_thread, C.byref(src.c()), keep=[src])

    def op_write_per_thread(self, dst: Plane) -> IOp:
        return self._iop(self._c.fk_op_write_per_thread, C.byref(dst.c()), keep=[dst])

    def op_crop(self, src: Plane, x0: int, y0: int, w: int, h: int) -> IOp:
        r = _ffi.fk_crop_rect(x0, y0, w, h)
        return self._iop(self._c.fk_op_crop, C.byref(src.c()), C.byref(r), keep=[src])

    def op_resize(self, upstream, w: int, h: int, mode: int = BILINEAR) -> IOp:
        """op_resize(Plane|IOp, w, h, mode) (oplib.hpp:54-57)."""
        if isinstance(upstream, Plane):
            upstream = self.op_read_per_thread(upstream)
        return self._iop(self._c.fk_op_resize, upstream._ptr, w, h, mode, keep=[upstream])

    def op_color_convert(self, order: int, input_kind: int) -> IOp:
        return self._iop(self._c.fk_op_color_convert, order, input_kind)

    def op_split_write(self, dst: Sequence[Plane]) -> IOp:
        arr = (_ffi.fk_plane * 3)(*(d.c() for d in dst))
        return self._iop(self._c.fk_op_split_write, arr, keep=list(dst))

    def op_batch_read(self, inner: Sequence[IOp], active_count: int | None = None,
                      default_value: Const | None = None) -> IOp:
        n = len(inner)
        arr = (C.c_void_p * max(n, 1))(*(i._ptr.value for i in inner))
        dv = C.create_string_buffer(default_value.raw(), 24) if default_value is not None else None
        return self._iop(self._c.fk_op_batch_read, arr, n, n if active_count is None else active_count, dv,
                         keep=list(inner))

    def op_batch_write(self, inner: Sequence[IOp], active_count: int | None = None) -> IOp:
        n = len(inner)
        arr = (C.c_void_p * max(n, 1))(*(i._ptr.value for i in inner))
        return self._iop(self._c.fk_op_batch_write, arr, n, n if active_count is None else active_count,
                         keep=list(inner))

    def fold_unary_into_read(self, read: IOp, unary: IOp) -> IOp:
        return self._iop(self._c.fk_fold_unary_into_read, read._ptr, unary._ptr, keep=[read])

    # -- validation & execution
    def validate_chain(self, iops: Sequence[IOp]) -> Pipeline:
        n = len(iops)
        arr = (C.c_void_p * max(n, 1))(*(i._ptr.value for i in iops))
        out = C.c_void_p()
        self._check(self._c.fk_validate_chain(arr, n, C.byref(out)))
        return Pipeline(self, out.value, keep=list(iops))

    def _exec(self, fn, pipeline, cfg: ExecConfig | None) -> ExecReport:
        if not isinstance(pipeline, Pipeline):
            pipeline = self.validate_chain(pipeline)
        cfg = cfg or ExecConfig()
        rep = _ffi.fk_exec_report()
        self._check(fn(pipeline._ptr, C.byref(cfg.c()), C.byref(rep)))
        return ExecReport.from_c(rep)

    def execute_fused(self, pipeline, cfg: ExecConfig | None = None) -> ExecReport:
        return self._exec(self._c.fk_execute_fused, pipeline, cfg)

    def execute_unfused(self, pipeline, cfg: ExecConfig | None = None) -> ExecReport:
        return self._exec(self._c.fk_execute_unfused, pipeline, cfg)

    # -- FKT tensor files (tensor_io.hpp:13-18)
    def tensor_write_file(self, planes, path: str):
        """tensor_write_file: planes (Plane / SharedPlane / RawPlane, one kind) -> an FKT1 file."""
        arr = (_ffi.fk_plane * max(len(planes), 1))(*(p.c() for p in planes))
        self._check(self._c.fk_tensor_write_file(arr, len(planes), str(path).encode()))

    def tensor_read_file(self, path: str) -> list:
        """tensor_read_file: the file's planes as library-owned SharedPlanes."""
        n = C.c_uint32()
        self._check(self._c.fk_tensor_read_file(str(path).encode(), None, 0, C.byref(n)))
        arr = (_ffi.fk_plane * max(n.value, 1))()
        self._check(self._c.fk_tensor_read_file(str(path).encode(), arr, n.value, C.byref(n)))
        return [SharedPlane(self, _ffi.fk_plane(arr[i].data, arr[i].width, arr[i].height, arr[i].row_stride,
                                                arr[i].kind)) for i in range(n.value)]

    def write_ppm(self, plane, path: str):
        self._check(self._c.fk_write_ppm(C.byref(plane.c()), str(path).encode()))

    def download(self, plane) -> np.ndarray:
        """A plane's elements as a packed host array (fk_plane_download)."""
        c = plane.c()
        bpe = BYTES_PER_ELEMENT[c.kind]
        buf = np.empty(c.width * c.height * bpe, np.uint8)
        self._check(self._c.fk_plane_download(C.byref(c), buf.ctypes.data, 0))
        arr = buf.view(_NP_DTYPE[c.kind])
        return arr.reshape(c.height, c.width, 3) if LANES[c.kind] == 3 else arr.reshape(c.height, c.width)

    def upload(self, plane, arr: np.ndarray):
        c = plane.c()
        a = np.ascontiguousarray(arr)
        self._check(self._c.fk_plane_upload(C.byref(c), a.ctypes.data, 0))

    def execute_sharded(self, pipelines, devices, cfgs=None):
        """fk_execute_sharded: pipelines[i] (a batch shard) on devices[i], all enqueued
        before any wait; returns one ExecReport per shard."""
        n = len(pipelines)
        arr = (C.c_void_p * max(n, 1))(*(p._ptr.value for p in pipelines))
        devs = (C.c_int32 * max(n, 1))(*devices)
        cs = None
        if cfgs is not None:
            cs = (_ffi.fk_exec_config * max(n, 1))(*(c.c() for c in cfgs))
        reps = (_ffi.fk_exec_report * max(n, 1))()
        self._check(self._c.fk_execute_sharded(arr, devs, n, cs, reps))
        return [ExecReport.from_c(reps[i]) for i in range(n)]

    def gather(self, dst_ptr: int, dst_device: int, parts, stream: int | None = None):
        """fk_gather: parts = [(dst_offset, src_ptr, src_device, nbytes), ...] peer copies."""
        n = len(parts)
        offs = (C.c_uint64 * max(n, 1))(*(p[0] for p in parts))
        srcs = (C.c_void_p * max(n, 1))(*(p[1] for p in parts))
        devs = (C.c_int32 * max(n, 1))(*(p[2] for p in parts))
        nb = (C.c_uint64 * max(n, 1))(*(p[3] for p in parts))
        self._check(self._c.fk_gather(dst_ptr, dst_device, offs, srcs, devs, nb, n, stream))

    def last_kernel(self) -> str:
        """Kernel family of this thread's last execute / reduce (CUDA backend only)."""
        return self._c.fk_cuda_last_kernel().decode()

    def multi_reduce_plane(self, read: IOp, specs, workers: int = 0):
        """multi_reduce_plane (dpp.hpp:52): specs = [(combine, transform IOp | None,
        identity Const | None), ...]; returns (list of per-spec lane tuples in the
        spec's value kind, source elements read). One traversal of the source."""
        n = len(specs)
        arr = (_ffi.fk_reduce_spec * max(n, 1))()
        kinds = []
        for i, (combine, transform, identity) in enumerate(specs):
            arr[i].transform = transform._ptr.value if transform is not None else None
            arr[i].combine = int(combine)
            if identity is not None:
                raw = identity.raw()
                arr[i].has_identity = 1
                C.memmove(arr[i].identity, raw, len(raw))
            kinds.append(transform.output_kind if transform is not None and transform.output_kind is not None
                         else (transform.input_kind if transform is not None else read.output_kind))
        out = (C.c_uint8 * (24 * max(n, 1)))()
        reads = C.c_uint64()
        self._check(self._c.fk_multi_reduce_plane(read._ptr, arr, n, int(workers), out, C.byref(reads)))
        res = []
        for i, k in enumerate(kinds):
            fmt = _STRUCT_FMT[lane_kind(k)]
            res.append(struct.unpack_from("<" + fmt * LANES[k], bytes(out), 24 * i))
        return res, reads.value

    def reduce_plane(self, read: IOp, combine: int, transform: IOp | None = None, identity: Const | None = None,
                     workers: int = 0):
        """reduce_plane (dpp.hpp:48): one spec."""
        res, _ = self.multi_reduce_plane(read, [(combine, transform, identity)], workers)
        return res[0]

    def plan_memory_savings(self, pipeline: Pipeline) -> int:
        v = C.c_uint64()
        self._check(self._c.fk_plan_memory_savings(pipeline._ptr, C.byref(v)))
        return v.value

    def schedule(self, space, cfg: ExecConfig | None = None):
        cfg = cfg or ExecConfig()
        e = _ffi.fk_extent3(*space)
        n = C.c_uint64()
        self._check(self._c.fk_schedule(C.byref(e), C.byref(cfg.c()), None, 0, C.byref(n)))
        buf = (C.c_uint32 * (3 * max(n.value, 1)))()
        self._check(self._c.fk_schedule(C.byref(e), C.byref(cfg.c()), buf, n.value, C.byref(n)))
        return [tuple(buf[3 * i: 3 * i + 3]) for i in range(n.value)]


_default: Library | None = None


def default_library() -> Library:
    """The CUDA product library (loaded once). Raises if libfk_cuda.so is missing."""
    global _default
    if _default is None:
        _default = Library("cuda")
    return _default
