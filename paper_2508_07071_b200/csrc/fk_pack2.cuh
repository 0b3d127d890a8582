// fk_pack2.cuh — packed FP32 pairs (FADD2 / FFMA2 on sm_100): two f32 lanes in
// one 64-bit register pair, each lane rounded exactly like the scalar IEEE op.
//
// A chain's product is issued as fma(a, b, z) with z a RUNTIME -0.0 pair (a
// kernel parameter), never as mul.rn.f32x2: ptxas contracts a packed mul
// followed by a packed add/sub into one FFMA2 even with .rn and -fmad=false
// (found by fk_walk's Mul -> Sub -> Div chain test: 1-ulp differences), and it
// folds a literal -0 addend the same way; an FMA with an unknown addend cannot
// be fused with its consumer. fma(a, b, -0) == RN(a b) for every input, zero
// signs included (+0 + -0 = +0, -0 + -0 = -0). kNegZero2 is the value to pass.
#pragma once

#include <cstdint>

namespace fk {
constexpr uint64_t kNegZero2 = 0x8000000080000000ull;  // (-0.0f, -0.0f)
namespace p2 {
__device__ __forceinline__ uint64_t pack(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ uint64_t of(float2 v) { return pack(v.x, v.y); }
__device__ __forceinline__ float lo(uint64_t v) { return __uint_as_float(uint32_t(v)); }
__device__ __forceinline__ float hi(uint64_t v) { return __uint_as_float(uint32_t(v >> 32)); }
__device__ __forceinline__ uint64_t add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t sub(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
// products whose consumer is not an add/sub (an FMA operand, a store) may use FMUL2
__device__ __forceinline__ uint64_t mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// a product that may feed an add/sub: z must be kNegZero2 loaded at run time
__device__ __forceinline__ uint64_t mul_z(uint64_t a, uint64_t b, uint64_t z) { return fma(a, b, z); }
}  // namespace p2
}  // namespace fk
