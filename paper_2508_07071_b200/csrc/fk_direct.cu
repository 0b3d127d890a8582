// fk_direct.cu — compiled kernel for element-wise f32 chains (vertical fusion,
// PAPER.md:530-541; configs[0] and configs[2]).
//
//   Read f32 (PerThreadRead / Crop, any batch) -> registered chain of f32
//   Mul/Add/Sub/Div, each with a runtime StaticLoop repeat count
//   -> [Cast f32 -> u8] -> Write (f32 or u8)
//
// The op sequence is a template signature (fk_sig.cuh) — the kernel is the
// paper's variadic fused kernel for that chain, constants and repeat counts in
// kernel parameters. Each thread owns 16 consecutive elements: four 128-bit
// loads, the chain in registers, one 128-bit (u8) or four (f32) streaming stores.
//
// Division by a constant d uses r = RN(1/d) and one FMA correction
// (div_guarded) once fk_verify_recip_div has proven, on all 2^32 f32 inputs,
// that it returns exactly __fdiv_rn(x, d) for this d; otherwise IEEE division.
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <mutex>

#include "fk_launch.hpp"
#include "fk_sig.cuh"
#include "fk_stages.cuh"

namespace fk {

namespace {

constexpr int kD = 16;  // elements per thread

// registered chains; bit 12+k marks op k as a verified reciprocal division
#define FK_DIRECT_SIGS(X)                                                                         \
  X(sig_make(0)) X(sig_make(1, AF_MUL)) X(sig_make(1, AF_ADD)) X(sig_make(1, AF_SUB))               \
  X(sig_make(1, AF_DIV)) X(sig_make(1, AF_DIV, 0, 0, 0, 1)) X(sig_make(2, AF_MUL, AF_ADD))          \
  X(sig_make(2, AF_SUB, AF_DIV)) X(sig_make(2, AF_SUB, AF_DIV, 0, 0, 2))                            \
  X(sig_make(3, AF_MUL, AF_SUB, AF_DIV)) X(sig_make(3, AF_MUL, AF_SUB, AF_DIV, 0, 4))               \
  X(sig_make(4, AF_MUL, AF_ADD, AF_SUB, AF_DIV)) X(sig_make(4, AF_MUL, AF_ADD, AF_SUB, AF_DIV, 8))

template <uint32_t SIG, int K>
__device__ __forceinline__ float direct_elem(float v, float c, float r) {
  if constexpr (sig_fn(SIG, K) == AF_DIV && sig_fast(SIG, K)) return div_guarded(v, c, r);
  else return sig_op<SIG, K>(v, c, r);
}

template <uint32_t SIG, int K>
__device__ __forceinline__ void direct_op(float (&v)[kD], float c, float r, uint32_t reps) {
  if constexpr (K < sig_n(SIG)) {
#pragma unroll 1
    for (uint32_t i = 0; i < reps; ++i)
#pragma unroll
      for (int e = 0; e < kD; ++e) v[e] = direct_elem<SIG, K>(v[e], c, r);
  }
}

// round_clamp_u8 (scalar.hpp:161-167) in one instruction: cvt.rni.sat rounds to
// nearest-even, saturates to [0, 255] and maps NaN to 0.
__device__ __forceinline__ uint32_t f32_to_u8(float x) {
  uint32_t r;
  asm("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r & 0xffu;
}

}  // namespace

template <bool TO_U8>
__device__ __forceinline__ void load_tile(const DPlan& P, const DSample& s, uint32_t t, float (&v)[kD]) {
  const uint32_t y = dev::fastdiv(t, P.tpr);
  const uint32_t x = (t - y * P.tiles_per_row) * kD;
  const int n = (P.width - x) < uint32_t(kD) ? int(P.width - x) : kD;
  const uint8_t* p = reinterpret_cast<const uint8_t*>(s.src) + uint64_t(s.y0 + y) * s.pitch + uint64_t(s.x0 + x) * 4;
  if (n == kD && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
    for (int i = 0; i < kD / 4; ++i) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(p) + i);
      v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < kD; ++e) v[e] = e < n ? __ldg(reinterpret_cast<const float*>(p) + e) : 0.f;
  }
}

template <uint32_t SIG, bool TO_U8>
__device__ __forceinline__ void finish_tile(const DPlan& P, const DWrite& w, uint32_t t, float (&v)[kD],
                                            const float (&c)[4], const float (&r)[4], const uint32_t (&rep)[4]) {
  const uint32_t y = dev::fastdiv(t, P.tpr);
  const uint32_t x = (t - y * P.tiles_per_row) * kD;
  const int n = (P.width - x) < uint32_t(kD) ? int(P.width - x) : kD;
  const bool st = (w.flags & WF_STREAM) != 0;
  direct_op<SIG, 0>(v, c[0], r[0], rep[0]);
  direct_op<SIG, 1>(v, c[1], r[1], rep[1]);
  direct_op<SIG, 2>(v, c[2], r[2], rep[2]);
  direct_op<SIG, 3>(v, c[3], r[3], rep[3]);
  uint8_t* q = reinterpret_cast<uint8_t*>(w.dst[0]) + uint64_t(y) * w.pitch[0];
  if constexpr (TO_U8) {
    uint32_t b[kD];
#pragma unroll
    for (int e = 0; e < kD; ++e) b[e] = f32_to_u8(v[e]);
    q += x;
    if (n == kD && (reinterpret_cast<uintptr_t>(q) & 15) == 0) {
      uint32_t wd[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        wd[i] = b[4 * i] | (b[4 * i + 1] << 8) | (b[4 * i + 2] << 16) | (b[4 * i + 3] << 24);
      dev::store_words<4>(q, wd, st);
    } else {
      for (int e = 0; e < n; ++e) q[e] = uint8_t(b[e]);
    }
  } else {
    q += uint64_t(x) * 4;
    if (n == kD && (reinterpret_cast<uintptr_t>(q) & 15) == 0) {
      uint32_t wd[kD];
#pragma unroll
      for (int e = 0; e < kD; ++e) wd[e] = __float_as_uint(v[e]);
      dev::store_words<kD>(q, wd, st);
    } else {
      for (int e = 0; e < n; ++e) reinterpret_cast<float*>(q)[e] = v[e];
    }
  }
}

// Grid-stride over the tiles of plane z with a machine-sized grid (no tail
// wave), two tiles in flight per thread: both tiles' loads are issued before
// either is computed, doubling the bytes in flight per SM.
template <uint32_t SIG, bool TO_U8>
__global__ void __launch_bounds__(kBlock) fk_direct(const __grid_constant__ DPlan P) {
  float c[4] = {0.f, 0.f, 0.f, 0.f}, r[4] = {0.f, 0.f, 0.f, 0.f};
  uint32_t rep[4] = {0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < sig_n(SIG)) {
      const DOp op = dev::prog_op(P, P.op_base + k);
      c[k] = __uint_as_float(uint32_t(op.c[0]));
      r[k] = __frcp_rn(c[k]);
      rep[k] = op.repeat;
    }
  }
  const uint32_t stride = gridDim.x * kBlock;
  for (uint32_t z = blockIdx.z; z < P.batch; z += gridDim.z) {
    const DSample s = P.reads[z];
    const DWrite w = P.writes[z];
    if (!(w.flags & WF_ACTIVE)) continue;
    for (uint32_t t = blockIdx.x * kBlock + threadIdx.x; t < P.tiles; t += 2 * stride) {
      const uint32_t t2 = t + stride;
      float va[kD], vb[kD];
      load_tile<TO_U8>(P, s, t, va);
      if (t2 < P.tiles) load_tile<TO_U8>(P, s, t2, vb);
      finish_tile<SIG, TO_U8>(P, w, t, va, c, r, rep);
      if (t2 < P.tiles) finish_tile<SIG, TO_U8>(P, w, t2, vb, c, r, rep);
    }
  }
}

// Exhaustive proof for one divisor: div_guarded(x, d, RN(1/d)) == __fdiv_rn(x, d)
// for every one of the 2^32 f32 bit patterns x (NaN results compare equal).
__global__ void fk_verify_recip_div(float d, unsigned int* bad) {
  const float r = __frcp_rn(d);
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  unsigned int found = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < (uint64_t(1) << 32); i += stride) {
    const float x = __uint_as_float(uint32_t(i));
    const float a = div_guarded(x, d, r), b = __fdiv_rn(x, d);
    if (__float_as_uint(a) != __float_as_uint(b) && !(isnan(a) && isnan(b))) found = 1;
  }
  if (found) atomicOr(bad, 1u);
}

bool recip_div_verified(float d) {
  static std::mutex mu;
  static std::map<uint32_t, bool> cache;
  uint32_t key;
  std::memcpy(&key, &d, 4);
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  unsigned int* flag = nullptr;
  bool ok = false;
  if (cudaMalloc(&flag, sizeof(unsigned int)) == cudaSuccess) {
    cudaMemset(flag, 0, sizeof(unsigned int));
    fk_verify_recip_div<<<148 * 16, 256>>>(d, flag);
    unsigned int h = 1;
    if (cudaMemcpy(&h, flag, sizeof h, cudaMemcpyDeviceToHost) == cudaSuccess) ok = h == 0;
    cudaFree(flag);
  }
  cudaGetLastError();
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = ok;
  return ok;
}

int direct_elems() { return kD; }

bool direct_registered(uint32_t sig) {
#define FK_CASE(S) if (sig == (S)) return true;
  FK_DIRECT_SIGS(FK_CASE)
#undef FK_CASE
  return false;
}

// CTAs per plane: enough to fill every SM at full occupancy (two tiles per thread), no more.
template <class K>
uint32_t direct_grid_x(K kernel, uint32_t tiles, uint32_t planes) {
  static int resident = 0;  // CTAs per SM, queried once per instantiation
  if (!resident) {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kBlock, 0);
    resident = (sms > 0 ? sms : 148) * (occ > 0 ? occ : 1);
  }
  const uint64_t want = (uint64_t(tiles) + 2 * kBlock - 1) / (2 * kBlock);
  const uint64_t per_plane = (uint64_t(resident) + planes - 1) / planes;
  return uint32_t(want < per_plane ? (want > 0 ? want : 1) : (per_plane > 0 ? per_plane : 1));
}

cudaError_t launch_direct(uint32_t sig, bool to_u8, const DPlan& P, cudaStream_t st) {
  if (P.tiles == 0 || P.batch == 0) return cudaSuccess;
  const uint32_t gz = P.batch < 65535u ? P.batch : 65535u;
#define FK_CASE(S)                                                                            \
  if (sig == (S)) {                                                                           \
    if (to_u8) {                                                                              \
      const dim3 grid(direct_grid_x(fk_direct<S, true>, P.tiles, gz), 1, gz);                 \
      fk_direct<S, true><<<grid, kBlock, 0, st>>>(P);                                         \
    } else {                                                                                  \
      const dim3 grid(direct_grid_x(fk_direct<S, false>, P.tiles, gz), 1, gz);                \
      fk_direct<S, false><<<grid, kBlock, 0, st>>>(P);                                        \
    }                                                                                         \
    return cudaGetLastError();                                                                \
  }
  FK_DIRECT_SIGS(FK_CASE)
#undef FK_CASE
  return cudaErrorInvalidValue;
}

}  // namespace fk
