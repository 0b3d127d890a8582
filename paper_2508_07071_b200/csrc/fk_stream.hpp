// fk_stream.hpp — the roofline-grade unfused comparator's pass kernels
// (fk_stream.cu): execute_unfused (executor.cpp:134-217) as one compiled,
// 128-bit vectorised streaming kernel per compute op plus the write pass.
//
// Intermediates of 3-lane kinds are kept PLANAR ([z][lane][H x W]) so every
// pass is a plain stream of 4-value chunks whose lane and plane are uniform
// (the bytes per pass equal the reference's packed intermediates': P B bpe).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "fk_devprog.hpp"

namespace fk {

enum : uint32_t { SP_ARITH = 0, SP_TO_U8 = 1, SP_COPY = 2 };

struct StreamPass {
  const uint8_t* src;        // pass input: contiguous values (f32; u8 for SP_COPY of u8)
  uint8_t* dst;              // pass output (contiguous) — null when writing through `writes`
  uint64_t chunks;           // 4-value chunks in total (n / 4)
  FastDiv plane_chunks;      // chunks per (z, lane) plane: H W / 4
  uint32_t nl;               // lanes of the kind (1 or 3)
  uint32_t op;               // SP_*
  uint32_t fn;               // AF_* (SP_ARITH)
  uint32_t repeat;           // StaticLoop count (>= 1)
  float c[3];                // per-lane constants (uniform over planes)
  const uint64_t* per_z;     // BatchArith: 3 raw Element lanes per plane (f32 bits), or null
  uint32_t per_z_n;
  uint32_t vbytes;           // bytes per value of src/dst (4 = f32, 1 = u8)
  // final write pass (dst == null): plane q = (z, lane) row-major W wide into
  // writes[z].dst[lane] with writes[z].pitch[lane] (BatchWrite split / per-thread)
  const DWrite* writes;
  DWrite wr;                 // non-batch write
  FastDiv row_chunks;        // W / 4
  uint32_t width;
  uint64_t negz;             // kNegZero2 (fk_pack2.cuh)
};

// one launch over P.chunks chunks; false when the pass is not streamable
cudaError_t launch_stream(const StreamPass& P, cudaStream_t st);

}  // namespace fk
