// fk_sig.cuh — compile-time chain signatures for the compiled kernels.
//
// A signature names a straight-line chain of up to four f32 Mul/Add/Sub/Div ops
// (the paper's variadic op chain, as one integer so a registry
// can list its instantiations): bits 0-3 = op count, bits 4+2k = op k's function
// (AF_*), bit 12+k = op k is a division whose verified reciprocal form may be
// used. Constants stay runtime values (kernel parameters), so one instantiation
// serves every constant set with that op sequence.
#pragma once

#include <cstdint>

#include "fk_devprog.hpp"

namespace fk {

constexpr uint32_t kSigLut = 0xffffffffu;  // not a straight-line chain: tabulate (LUT mode)

__host__ __device__ constexpr uint32_t sig_make(int n, uint32_t f0 = 0, uint32_t f1 = 0, uint32_t f2 = 0, uint32_t f3 = 0,
                            uint32_t fast = 0, uint32_t total = 0) {
  return uint32_t(n) | (f0 << 4) | (f1 << 6) | (f2 << 8) | (f3 << 10) | (fast << 12) | (total << 16);
}
__host__ __device__ constexpr int sig_n(uint32_t s) { return int(s & 0xfu); }
__host__ __device__ constexpr uint32_t sig_fn(uint32_t s, int k) { return (s >> (4 + 2 * k)) & 3u; }
__host__ __device__ constexpr bool sig_fast(uint32_t s, int k) { return (s >> (12 + k)) & 1u; }
// bit 16+k: the reciprocal form is exact for EVERY f32 input of op k (no range guard)
__host__ __device__ constexpr bool sig_total(uint32_t s, int k) { return (s >> (16 + k)) & 1u; }

// Correctly rounded x / d from r = RN(1/d): q = RN(x r), e = x - q d (exact via
// FMA), q' = RN(q + e r). Used only where the host has verified it equals
// __fdiv_rn on every input the op can see (all 256 u8-derived values).
__device__ __forceinline__ float div_by_recip(float x, float d, float r) {
  const float q = __fmul_rn(x, r);
  const float e = __fmaf_rn(-q, d, x);
  return __fmaf_rn(e, r, q);
}

// The same for any f32 input: normal-range magnitudes take the reciprocal form,
// zeros / denormals / huge values / inf / NaN take IEEE division. Used for a
// divisor only after fk_verify_recip_div has checked it against __fdiv_rn on all
// 2^32 inputs (fk_direct.cu).
// |x| in [2^-100, 2^100) as one integer compare on the bit pattern (NaN/inf/0/denormal fail).
__device__ __forceinline__ bool recip_range(float x) {
  return ((__float_as_uint(x) & 0x7fffffffu) - 0x0d800000u) < 0x64000000u;
}
__device__ __forceinline__ float div_guarded(float x, float d, float r) {
  return recip_range(x) ? div_by_recip(x, d, r) : __fdiv_rn(x, d);
}

template <uint32_t SIG, int K>
__device__ __forceinline__ float sig_op(float v, float c, float r) {
  constexpr uint32_t fn = sig_fn(SIG, K);
  if constexpr (fn == AF_MUL) return __fmul_rn(v, c);
  else if constexpr (fn == AF_ADD) return __fadd_rn(v, c);
  else if constexpr (fn == AF_SUB) return __fsub_rn(v, c);
  else if constexpr (sig_fast(SIG, K)) return div_by_recip(v, c, r);
  else return __fdiv_rn(v, c);
}

// Apply the whole signature to one f32 lane value: c[k] constants, r[k] reciprocals.
template <uint32_t SIG>
__device__ __forceinline__ float sig_apply(float v, const float (&c)[4], const float (&r)[4]) {
  if constexpr (sig_n(SIG) > 0) v = sig_op<SIG, 0>(v, c[0], r[0]);
  if constexpr (sig_n(SIG) > 1) v = sig_op<SIG, 1>(v, c[1], r[1]);
  if constexpr (sig_n(SIG) > 2) v = sig_op<SIG, 2>(v, c[2], r[2]);
  if constexpr (sig_n(SIG) > 3) v = sig_op<SIG, 3>(v, c[3], r[3]);
  return v;
}

// The resample kernel's registered AFFINE chains (after Cast u8 -> f32).
// X-macro: FK_AFFINE_SIG(sig) for every instantiated signature.
#define FK_AFFINE_SIGS(X)                                                      \
  X(sig_make(0))                                                               \
  X(sig_make(1, AF_MUL)) X(sig_make(1, AF_ADD)) X(sig_make(1, AF_SUB))        \
  X(sig_make(1, AF_DIV)) X(sig_make(1, AF_DIV, 0, 0, 0, 1))                  \
  X(sig_make(2, AF_SUB, AF_DIV)) X(sig_make(2, AF_SUB, AF_DIV, 0, 0, 2))      \
  X(sig_make(2, AF_MUL, AF_ADD)) X(sig_make(2, AF_SUB, AF_MUL))               \
  X(sig_make(3, AF_MUL, AF_SUB, AF_DIV)) X(sig_make(3, AF_MUL, AF_SUB, AF_DIV, 0, 4))

}  // namespace fk
