// fk_device.cuh — device numerics and tile I/O shared by every fused kernel.
//
// Numerics reproduce the reference bit-for-bit (scalar.hpp:146-167, scalar.cpp:15-42,
// ops.cpp:88-310): every float/double op is an explicitly rounded intrinsic
// (__fmul_rn, __dadd_rn, ...) so nvcc can never contract a mul+add into an FMA,
// and the library is additionally compiled with -fmad=false.
//
// Values flow between ops in a register "state" Lane v[E][L]: E consecutive x
// positions of one row (thread coarsening), L lanes. A u8 lane holds 0..255 in
// the low bits, an f32 lane its IEEE bits, an f64 lane (64-bit states only) its
// IEEE bits.
#pragma once

#include <cstdint>

#include "fk.h"
#include "fk_devprog.hpp"

namespace fk {
namespace dev {

template <uint32_t K> struct KindT {
  static constexpr uint32_t lk = K >= FK_U8X3 ? K - 3 : K;
  static constexpr int nl = K >= FK_U8X3 ? 3 : 1;
  static constexpr int lb = lk == FK_U8 ? 1 : (lk == FK_F32 ? 4 : 8);
  static constexpr int bpe = nl * lb;
};

// Can a state of (Lane, L) hold values of kind K?
template <uint32_t K, class Lane, int L>
__host__ __device__ constexpr bool fits() {
  return KindT<K>::nl <= L && (KindT<K>::lk != FK_F64 || sizeof(Lane) == 8);
}
template <uint32_t LK, int NL, class Lane, int L>
__host__ __device__ constexpr bool fits_lanes() {
  return NL <= L && (LK != FK_F64 || sizeof(Lane) == 8);
}

// ------------------------------------------------------------- numerics --
__device__ __forceinline__ float as_f32(uint64_t v) { return __uint_as_float(uint32_t(v)); }
__device__ __forceinline__ float as_f32(uint32_t v) { return __uint_as_float(v); }
__device__ __forceinline__ double as_f64(uint64_t v) { return __longlong_as_double((long long)v); }
__device__ __forceinline__ uint32_t bits(float f) { return __float_as_uint(f); }
__device__ __forceinline__ uint64_t bits(double d) { return (uint64_t)__double_as_longlong(d); }

// round_clamp_u8, scalar.hpp:161-167: NaN -> 0, nearbyint (ties-to-even), clamp.
__device__ __forceinline__ uint32_t round_clamp_u8(double x) {
  if (isnan(x)) return 0u;
  const double r = rint(x);
  if (r < 0.0) return 0u;
  if (r > 255.0) return 255u;
  return (uint32_t)r;
}
// Same result for a float input: (double)f is exact and rint commutes with it.
__device__ __forceinline__ uint32_t round_clamp_u8(float x) {
  if (isnan(x)) return 0u;
  const float r = rintf(x);
  if (r < 0.0f) return 0u;
  if (r > 255.0f) return 255u;
  return (uint32_t)r;
}

template <class Lane>
__device__ __forceinline__ double lane_to_double(uint32_t lk, Lane v) {
  if (lk == FK_U8) return (double)(uint32_t)(v & 0xffu);
  if (lk == FK_F32) return (double)as_f32(v);
  if constexpr (sizeof(Lane) == 8) return as_f64(v);
  return 0.0;
}
template <uint32_t LK, class Lane>
__device__ __forceinline__ double lane_to_double(Lane v) {
  if constexpr (LK == FK_U8) return (double)(uint32_t)(v & 0xffu);
  else if constexpr (LK == FK_F32) return (double)as_f32(v);
  else return as_f64((uint64_t)v);
}
// set_lane, scalar.cpp:21-31 (narrowing policies applied once at the destination)
template <uint32_t LK, class Lane>
__device__ __forceinline__ Lane lane_from_double(double x) {
  if constexpr (LK == FK_U8) return (Lane)round_clamp_u8(x);
  else if constexpr (LK == FK_F32) return (Lane)bits(__double2float_rn(x));
  else return (Lane)bits(x);
}

// u8 ops wrap mod 256 (scalar.hpp:146-157), IEEE float/double ops (ops.cpp:88-107)
template <uint32_t FN> __device__ __forceinline__ uint32_t u8_op(uint32_t a, uint32_t b) {
  if constexpr (FN == AF_MUL) return a * b;       // wrap deferred: mod 2^32 preserves mod 256
  else if constexpr (FN == AF_ADD) return a + b;
  else if constexpr (FN == AF_SUB) return a - b;
  else return (a & 0xffu) / b;
}
template <uint32_t FN> __device__ __forceinline__ float f32_op(float a, float b) {
  if constexpr (FN == AF_MUL) return __fmul_rn(a, b);
  else if constexpr (FN == AF_ADD) return __fadd_rn(a, b);
  else if constexpr (FN == AF_SUB) return __fsub_rn(a, b);
  else return __fdiv_rn(a, b);
}
template <uint32_t FN> __device__ __forceinline__ double f64_op(double a, double b) {
  if constexpr (FN == AF_MUL) return __dmul_rn(a, b);
  else if constexpr (FN == AF_ADD) return __dadd_rn(a, b);
  else if constexpr (FN == AF_SUB) return __dsub_rn(a, b);
  else return __ddiv_rn(a, b);
}

__device__ __forceinline__ double lerp(double a, double b, double t) {  // ops.cpp:250
  return __dadd_rn(a, __dmul_rn(__dsub_rn(b, a), t));
}
// center_coord, ops.cpp:253-257: ((i + 0.5) * rect) / out - 0.5
__device__ __forceinline__ double center_coord(uint32_t i, uint32_t rect, uint32_t out) {
  return __dsub_rn(__ddiv_rn(__dmul_rn(__dadd_rn((double)i, 0.5), (double)rect), (double)out), 0.5);
}
__device__ __forceinline__ long long clamp_ll(long long v, long long lo, long long hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

__device__ __forceinline__ uint32_t fastdiv(uint32_t n, const FastDiv& f) {
  return (uint32_t)(((uint64_t)__umulhi(n, f.m) + n) >> f.s);
}

// ------------------------------------------------------------ memory I/O --
// Word-granular tile moves with the widest alignment the address allows.
template <int NW>
__device__ __forceinline__ void load_words(const uint8_t* p, uint32_t (&w)[NW]) {
  const uintptr_t a = (uintptr_t)p;
  if constexpr (NW % 4 == 0) {
    if ((a & 15) == 0) {
#pragma unroll
      for (int i = 0; i < NW / 4; ++i) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(p) + i);
        w[4 * i] = q.x; w[4 * i + 1] = q.y; w[4 * i + 2] = q.z; w[4 * i + 3] = q.w;
      }
      return;
    }
  }
  if constexpr (NW % 2 == 0) {
    if ((a & 7) == 0) {
#pragma unroll
      for (int i = 0; i < NW / 2; ++i) {
        const uint2 q = __ldg(reinterpret_cast<const uint2*>(p) + i);
        w[2 * i] = q.x; w[2 * i + 1] = q.y;
      }
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < NW; ++i) w[i] = __ldg(reinterpret_cast<const uint32_t*>(p) + i);
}

template <int NW>
__device__ __forceinline__ void store_words(uint8_t* p, const uint32_t (&w)[NW], bool stream) {
  const uintptr_t a = (uintptr_t)p;
  if constexpr (NW % 4 == 0) {
    if ((a & 15) == 0) {
#pragma unroll
      for (int i = 0; i < NW / 4; ++i) {
        const uint4 q = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        if (stream) __stcs(reinterpret_cast<uint4*>(p) + i, q);
        else reinterpret_cast<uint4*>(p)[i] = q;
      }
      return;
    }
  }
  if constexpr (NW % 2 == 0) {
    if ((a & 7) == 0) {
#pragma unroll
      for (int i = 0; i < NW / 2; ++i) {
        const uint2 q = make_uint2(w[2 * i], w[2 * i + 1]);
        if (stream) __stcs(reinterpret_cast<uint2*>(p) + i, q);
        else reinterpret_cast<uint2*>(p)[i] = q;
      }
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    if (stream) __stcs(reinterpret_cast<uint32_t*>(p) + i, w[i]);
    else reinterpret_cast<uint32_t*>(p)[i] = w[i];
  }
}

// One lane of lane-kind LK at p (aligned -> typed load, else byte assembly).
template <uint32_t LK, class Lane>
__device__ __forceinline__ Lane load_lane(const uint8_t* p, bool aligned) {
  if constexpr (LK == FK_U8) {
    return (Lane)__ldg(p);
  } else if constexpr (LK == FK_F32) {
    if (aligned) return (Lane)__ldg(reinterpret_cast<const uint32_t*>(p));
    uint32_t r = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) r |= (uint32_t)__ldg(p + b) << (8 * b);
    return (Lane)r;
  } else {
    if (aligned) return (Lane)__ldg(reinterpret_cast<const unsigned long long*>(p));
    uint64_t r = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) r |= (uint64_t)__ldg(p + b) << (8 * b);
    return (Lane)r;
  }
}

template <uint32_t LK, class Lane>
__device__ __forceinline__ void store_lane(uint8_t* p, Lane v, bool aligned) {
  if constexpr (LK == FK_U8) {
    *p = (uint8_t)(v & 0xffu);
  } else if constexpr (LK == FK_F32) {
    if (aligned) { *reinterpret_cast<uint32_t*>(p) = (uint32_t)v; return; }
#pragma unroll
    for (int b = 0; b < 4; ++b) p[b] = (uint8_t)((uint32_t)v >> (8 * b));
  } else {
    if (aligned) { *reinterpret_cast<unsigned long long*>(p) = (unsigned long long)v; return; }
#pragma unroll
    for (int b = 0; b < 8; ++b) p[b] = (uint8_t)((uint64_t)v >> (8 * b));
  }
}

// Decode the words of E consecutive elements of kind K into the state.
template <uint32_t K, class Lane, int L, int E, int NW>
__device__ __forceinline__ void decode(const uint32_t (&w)[NW], Lane (&v)[E][L]) {
  using T = KindT<K>;
#pragma unroll
  for (int e = 0; e < E; ++e)
#pragma unroll
    for (int l = 0; l < T::nl; ++l) {
      const int o = e * T::bpe + l * T::lb;
      if constexpr (T::lk == FK_U8) v[e][l] = (Lane)((w[o >> 2] >> ((o & 3) * 8)) & 0xffu);
      else if constexpr (T::lk == FK_F32) v[e][l] = (Lane)w[o >> 2];
      else v[e][l] = (Lane)((uint64_t)w[o >> 2] | ((uint64_t)w[(o >> 2) + 1] << 32));
    }
}

template <uint32_t K, class Lane, int L, int E, int NW>
__device__ __forceinline__ void encode(const Lane (&v)[E][L], uint32_t (&w)[NW]) {
  using T = KindT<K>;
#pragma unroll
  for (int i = 0; i < NW; ++i) w[i] = 0;
#pragma unroll
  for (int e = 0; e < E; ++e)
#pragma unroll
    for (int l = 0; l < T::nl; ++l) {
      const int o = e * T::bpe + l * T::lb;
      if constexpr (T::lk == FK_U8) w[o >> 2] |= ((uint32_t)v[e][l] & 0xffu) << ((o & 3) * 8);
      else if constexpr (T::lk == FK_F32) w[o >> 2] = (uint32_t)v[e][l];
      else {
        w[o >> 2] = (uint32_t)(uint64_t)v[e][l];
        w[(o >> 2) + 1] = (uint32_t)((uint64_t)v[e][l] >> 32);
      }
    }
}

}  // namespace dev
}  // namespace fk
