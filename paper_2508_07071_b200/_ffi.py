"""ctypes binding of the include/fk.h C-ABI.

The same declarations bind three shared libraries that export the identical ABI:

* ``cuda``      -> ``paper_2508_07071_b200/lib/libfk_cuda.so`` (the product, sm_100a kernels)
* ``oracle``    -> ``oracle/build/libfk_oracle.so`` (plain-C restatement; TEST INFRASTRUCTURE)
* ``reference`` -> ``oracle/_ref/libfk_ref.so`` (the unmodified reference; TEST INFRASTRUCTURE)

Only tests, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may load the
last two. The product path (``opfuse.Library()`` with no argument) loads ``cuda`` and
raises if it is missing — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent

LIB_PATHS = {
    "cuda": PKG_DIR / "lib" / "libfk_cuda.so",
    "oracle": REPO_DIR / "oracle" / "build" / "libfk_oracle.so",
    "reference": REPO_DIR / "oracle" / "_ref" / "libfk_ref.so",
}

# enum fk_kind
U8, F32, F64, U8X3, F32X3, F64X3 = range(6)
KIND_NAMES = ["u8", "f32", "f64", "u8x3", "f32x3", "f64x3"]
BYTES_PER_ELEMENT = [1, 4, 8, 3, 12, 24]
LANES = [1, 1, 1, 3, 3, 3]

# enum fk_op_id
(OP_PER_THREAD_READ, OP_CROP_READ, OP_RESIZE_READ, OP_BATCH_READ, OP_CAST, OP_SWAP_RB, OP_TO_GRAY,
 OP_MUL, OP_ADD, OP_SUB, OP_DIV, OP_STATIC_LOOP, OP_PER_THREAD_WRITE, OP_SPLIT_WRITE,
 OP_BATCH_WRITE) = range(15)
OP_BATCH_ARITH = 32
OP_NAMES = {0: "PerThreadRead", 1: "CropRead", 2: "ResizeRead", 3: "BatchRead", 4: "Cast", 5: "SwapRB",
            6: "ToGray", 7: "Mul", 8: "Add", 9: "Sub", 10: "Div", 11: "StaticLoop", 12: "PerThreadWrite",
            13: "SplitWrite", 14: "BatchWrite", 32: "BatchArith"}

KIND_READ, KIND_UNARY, KIND_BINARY, KIND_WRITE = range(4)
NEAREST, BILINEAR = 0, 1
SWAP_RB, TO_GRAY_F32 = 0, 1

EXEC_TIMED = 0x1
EXEC_FORCE_GENERIC = 0x2
EXEC_SERIAL = 0x4
EXEC_NO_LUT = 0x8

PATH_CPU, PATH_GENERIC, PATH_COMPILED = 0, 1, 2

# Errc names, errors.hpp:9-38 (status = 1 + ordinal)
ERRC_NAMES = ["OK", "EmptyChain", "FirstNotRead", "LastNotWrite", "KindMismatch", "DimsMismatch",
              "MissingDims", "ChainTooLong", "DivByZeroParam", "UnsupportedCast", "UnsupportedKind",
              "CropOutOfBounds", "PlaneExtentMismatch", "EmptyBatch", "InnerKindMismatch",
              "HeterogeneousBatch", "BadStaticLoop", "BoundsError", "CapacityOverflow", "BadMagic",
              "UnknownKindTag", "TruncatedPayload", "IoError", "EmptyIterSpace", "InvalidConfig"]
EXTRA_ERRC = {100: "InvalidArgument", 101: "CudaError", 102: "NoDevice", 103: "Unsupported"}


def errc_name(status: int) -> str:
    if 0 <= status < len(ERRC_NAMES):
        return ERRC_NAMES[status]
    return EXTRA_ERRC.get(status, "UnknownError")


class fk_plane(C.Structure):
    _fields_ = [("data", C.c_void_p), ("width", C.c_uint32), ("height", C.c_uint32),
                ("row_stride", C.c_uint32), ("kind", C.c_uint32)]


class fk_crop_rect(C.Structure):
    _fields_ = [("x0", C.c_uint32), ("y0", C.c_uint32), ("w", C.c_uint32), ("h", C.c_uint32)]


class fk_extent3(C.Structure):
    _fields_ = [("width", C.c_uint32), ("height", C.c_uint32), ("batch", C.c_uint32)]


class fk_exec_config(C.Structure):
    _fields_ = [("workers", C.c_int32), ("coarsen_block", C.c_int32), ("chunk_rows", C.c_int32),
                ("flags", C.c_uint32), ("stream", C.c_void_p)]


class fk_reduce_spec(C.Structure):
    _fields_ = [("transform", C.c_void_p), ("combine", C.c_uint32), ("has_identity", C.c_uint32),
                ("identity", C.c_uint8 * 24)]


class fk_exec_report(C.Structure):
    _fields_ = [("wall_time_ns", C.c_uint64), ("bytes_read", C.c_uint64), ("bytes_written", C.c_uint64),
                ("intermediate_bytes_allocated", C.c_uint64), ("passes", C.c_uint64),
                ("points_visited", C.c_uint64), ("kernels_launched", C.c_uint64), ("device_ms", C.c_double),
                ("path", C.c_uint32), ("reserved", C.c_uint32)]


P = C.c_void_p
PP = C.POINTER(C.c_void_p)
U32 = C.c_uint32
I32 = C.c_int32

# name -> (restype, argtypes); every symbol include/fk.h declares
SIGNATURES = {
    "fk_backend_name": (C.c_char_p, []),
    "fk_abi_version": (I32, []),
    "fk_last_error": (C.c_char_p, []),
    "fk_last_error_position": (I32, []),
    "fk_errc_name": (I32, [I32, C.c_char_p, C.c_size_t]),
    "fk_plane_view": (I32, [C.POINTER(fk_plane), U32, U32, U32, U32, C.POINTER(fk_plane)]),
    "fk_bytes_per_element": (U32, [U32]),
    "fk_plane_alloc": (I32, [U32, U32, U32, U32, C.POINTER(fk_plane)]),
    "fk_plane_free": (None, [C.POINTER(fk_plane)]),
    "fk_plane_upload": (I32, [C.POINTER(fk_plane), P, C.c_size_t]),
    "fk_plane_download": (I32, [C.POINTER(fk_plane), P, C.c_size_t]),
    "fk_op_arith": (I32, [U32, U32, P, PP]),
    "fk_op_cast": (I32, [U32, U32, PP]),
    "fk_op_static_loop": (I32, [P, U32, PP]),
    "fk_op_read_per_thread": (I32, [C.POINTER(fk_plane), PP]),
    "fk_op_write_per_thread": (I32, [C.POINTER(fk_plane), PP]),
    "fk_op_crop": (I32, [C.POINTER(fk_plane), C.POINTER(fk_crop_rect), PP]),
    "fk_op_resize": (I32, [P, U32, U32, U32, PP]),
    "fk_op_color_convert": (I32, [U32, U32, PP]),
    "fk_op_split_write": (I32, [C.POINTER(fk_plane), PP]),
    "fk_op_batch_read": (I32, [PP, U32, U32, P, PP]),
    "fk_op_batch_write": (I32, [PP, U32, U32, PP]),
    "fk_fold_unary_into_read": (I32, [P, P, PP]),
    "fk_op_batch_arith": (I32, [U32, U32, P, U32, PP]),
    "fk_iop_free": (None, [P]),
    "fk_iop_id": (U32, [P]),
    "fk_iop_kind": (U32, [P]),
    "fk_iop_input_kind": (I32, [P]),
    "fk_iop_output_kind": (I32, [P]),
    "fk_iop_dims": (I32, [P, C.POINTER(fk_extent3)]),
    "fk_validate_chain": (I32, [PP, U32, PP]),
    "fk_pipeline_free": (None, [P]),
    "fk_pipeline_iter_space": (I32, [P, C.POINTER(fk_extent3)]),
    "fk_pipeline_compute_count": (U32, [P]),
    "fk_execute_fused": (I32, [P, C.POINTER(fk_exec_config), C.POINTER(fk_exec_report)]),
    "fk_execute_unfused": (I32, [P, C.POINTER(fk_exec_config), C.POINTER(fk_exec_report)]),
    "fk_plan_memory_savings": (I32, [P, C.POINTER(C.c_uint64)]),
    "fk_schedule": (I32, [C.POINTER(fk_extent3), C.POINTER(fk_exec_config), C.POINTER(C.c_uint32),
                          C.c_uint64, C.POINTER(C.c_uint64)]),
    "fk_multi_reduce_plane": (I32, [P, C.POINTER(fk_reduce_spec), U32, I32, P, C.POINTER(C.c_uint64)]),
    "fk_tensor_write_file": (I32, [C.POINTER(fk_plane), U32, C.c_char_p]),
    "fk_tensor_read_file": (I32, [C.c_char_p, C.POINTER(fk_plane), U32, C.POINTER(U32)]),
    "fk_write_ppm": (I32, [C.POINTER(fk_plane), C.c_char_p]),
    "fk_execute_sharded": (I32, [PP, C.POINTER(I32), U32, C.POINTER(fk_exec_config), C.POINTER(fk_exec_report)]),
    "fk_gather": (I32, [P, I32, C.POINTER(C.c_uint64), PP, C.POINTER(I32), C.POINTER(C.c_uint64), U32, P]),
}

REDUCE_SUM, REDUCE_MAX, REDUCE_MIN = 0, 1, 2  # fk_reducer (dpp.hpp:32)

# symbols only the CUDA product exports (declared in include/fk_cuda.h)
CUDA_SIGNATURES = {
    "fk_cuda_device_info": (I32, [C.c_char_p, C.c_size_t]),
    "fk_cuda_kernel_launch_count": (C.c_uint64, []),
    "fk_cuda_last_kernel": (C.c_char_p, []),
}

_loaded: dict[str, C.CDLL] = {}


def library_path(backend: str) -> Path:
    if backend not in LIB_PATHS:
        raise ValueError(f"unknown backend {backend!r}; expected one of {sorted(LIB_PATHS)}")
    return LIB_PATHS[backend]


def load(backend: str) -> C.CDLL:
    """Load and declare one backend's shared library. Raises FileNotFoundError if absent."""
    if backend in _loaded:
        return _loaded[backend]
    path = library_path(backend)
    if not path.exists():
        hint = "python -c 'import __graft_entry__ as g; g.build()'"
        raise FileNotFoundError(f"fk backend {backend!r} not built: {path} is missing (run {hint})")
    lib = C.CDLL(os.fspath(path), mode=C.RTLD_LOCAL)
    sigs = dict(SIGNATURES)
    if backend == "cuda":
        sigs.update(CUDA_SIGNATURES)
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _loaded[backend] = lib
    return lib
