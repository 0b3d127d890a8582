// fk_stream.cu — pass kernels of the roofline-grade unfused comparator
// (execute_unfused, executor.cpp:134-217): one launch per compute op, each a
// grid-stride stream of 4-value chunks (one 16-byte load and store per chunk,
// streaming cache hints), plus the final write pass through the pipeline's
// write op. Same IEEE ops as the fused kernels and the reference (arith
// ops.cpp:88-159, round_clamp_u8 scalar.hpp:161-167), so the unfused output is
// bit-identical to the fused one.
#include <cuda_runtime.h>

#include "fk_device.cuh"
#include "fk_pack2.cuh"
#include "fk_stream.hpp"

namespace fk {
namespace {

__device__ __forceinline__ float4 ld_cs4(const uint8_t* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ uint32_t ld_cs1(const uint8_t* p) { return __ldcs(reinterpret_cast<const uint32_t*>(p)); }

// v = v (op) k on a chunk, as two packed pairs (products as fma(a, k, -0), fk_pack2.cuh)
template <uint32_t FN>
__device__ __forceinline__ void apply(float4& v, float k, uint64_t z) {
  if constexpr (FN == AF_DIV) {
    v.x = __fdiv_rn(v.x, k);
    v.y = __fdiv_rn(v.y, k);
    v.z = __fdiv_rn(v.z, k);
    v.w = __fdiv_rn(v.w, k);
  } else {
    const uint64_t kk = p2::pack(k, k);
    uint64_t a = p2::pack(v.x, v.y), b = p2::pack(v.z, v.w);
    if constexpr (FN == AF_MUL) {
      a = p2::mul_z(a, kk, z);
      b = p2::mul_z(b, kk, z);
    } else if constexpr (FN == AF_ADD) {
      a = p2::add(a, kk);
      b = p2::add(b, kk);
    } else {
      a = p2::sub(a, kk);
      b = p2::sub(b, kk);
    }
    v = make_float4(p2::lo(a), p2::hi(a), p2::lo(b), p2::hi(b));
  }
}

template <uint32_t OP, uint32_t FN, bool PERZ, bool WRITE, uint32_t VB>
__global__ void __launch_bounds__(256) fk_stream(const __grid_constant__ StreamPass P) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < P.chunks; c += stride) {
    const uint32_t q = dev::fastdiv(uint32_t(c), P.plane_chunks);  // plane (z, lane)
    const uint32_t z = P.nl == 3 ? q / 3u : q, m = q - z * P.nl;
    if constexpr (OP == SP_ARITH) {
      float4 v = ld_cs4(P.src + 16 * c);
      const float k = PERZ ? __uint_as_float(uint32_t(P.per_z[3 * size_t(z < P.per_z_n ? z : P.per_z_n - 1) + m]))
                           : P.c[m];
      for (uint32_t r = 0; r < P.repeat; ++r) apply<FN>(v, k, P.negz);
      __stcs(reinterpret_cast<float4*>(P.dst + 16 * c), v);
    } else if constexpr (OP == SP_TO_U8) {
      const float4 v = ld_cs4(P.src + 16 * c);
      const uint32_t w = dev::round_clamp_u8(v.x) | (dev::round_clamp_u8(v.y) << 8) | (dev::round_clamp_u8(v.z) << 16) |
                         (dev::round_clamp_u8(v.w) << 24);
      __stcs(reinterpret_cast<uint32_t*>(P.dst + 4 * c), w);
    } else {  // SP_COPY through the write op (store_block / split_block, ops.cpp:396-424)
      const DWrite& wr = P.writes ? P.writes[z] : P.wr;
      if (!(wr.flags & WF_ACTIVE)) continue;  // BatchWrite: z >= active skips (ops.cpp:437-445)
      const uint32_t r = uint32_t(c) - q * P.plane_chunks.d;
      const uint32_t y = dev::fastdiv(r, P.row_chunks), x4 = r - y * P.row_chunks.d;
      uint8_t* d = reinterpret_cast<uint8_t*>(wr.dst[m]) + uint64_t(y) * wr.pitch[m] + uint64_t(x4) * 4 * VB;
      if constexpr (VB == 4) __stcs(reinterpret_cast<float4*>(d), ld_cs4(P.src + 16 * c));
      else __stcs(reinterpret_cast<uint32_t*>(d), ld_cs1(P.src + 4 * c));
    }
  }
}

template <uint32_t OP, uint32_t FN, bool PERZ, bool WRITE, uint32_t VB>
cudaError_t run(const StreamPass& P, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t want = (P.chunks + 255) / 256;
  const uint32_t blocks = uint32_t(want < uint64_t(sms) * 8 ? want : uint64_t(sms) * 8);  // 8 x 256 threads per SM
  fk_stream<OP, FN, PERZ, WRITE, VB><<<blocks ? blocks : 1, 256, 0, st>>>(P);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_stream(const StreamPass& P, cudaStream_t st) {
  if (P.chunks == 0) return cudaSuccess;
  if (P.op == SP_COPY) return P.vbytes == 4 ? run<SP_COPY, 0, false, true, 4>(P, st) : run<SP_COPY, 0, false, true, 1>(P, st);
  if (P.op == SP_TO_U8) return run<SP_TO_U8, 0, false, false, 4>(P, st);
  const bool pz = P.per_z != nullptr;
  switch (P.fn) {
    case AF_MUL: return pz ? run<SP_ARITH, AF_MUL, true, false, 4>(P, st) : run<SP_ARITH, AF_MUL, false, false, 4>(P, st);
    case AF_ADD: return pz ? run<SP_ARITH, AF_ADD, true, false, 4>(P, st) : run<SP_ARITH, AF_ADD, false, false, 4>(P, st);
    case AF_SUB: return pz ? run<SP_ARITH, AF_SUB, true, false, 4>(P, st) : run<SP_ARITH, AF_SUB, false, false, 4>(P, st);
    default: return pz ? run<SP_ARITH, AF_DIV, true, false, 4>(P, st) : run<SP_ARITH, AF_DIV, false, false, 4>(P, st);
  }
}

}  // namespace fk
