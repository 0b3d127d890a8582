"""B200-native Fused Kernel Library (arXiv 2508.07071 capabilities, sm_100a).

The product is ``lib/libfk_cuda.so`` behind the C-ABI in ``include/fk.h``;
:mod:`.opfuse` mirrors the reference's opfuse API on top of it and
:mod:`.api` mirrors its lazy facade (execute_operations / execute_batch).
"""
from .opfuse import (Const, ExecConfig, ExecReport, IOp, Library, OpfuseError, Pipeline, Plane,  # noqa: F401
                     const_of, default_library, f32, f32x3, f64, f64x3, u8, u8x3)
from ._ffi import (BILINEAR, F32, F32X3, F64, F64X3, NEAREST, SWAP_RB, TO_GRAY_F32, U8, U8X3)  # noqa: F401
