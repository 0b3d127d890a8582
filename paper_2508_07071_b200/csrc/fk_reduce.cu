// fk_reduce.cu — ReduceDPP on B200 (dpp.hpp:32-53, dpp.cpp:46-246): several
// Sum / Max / Min folds over one read, in ONE traversal of the source.
//
// Every thread folds tiles of E consecutive x (grid-stride, coalesced), reading
// each element once through the same read stage as the fused kernels (crop,
// resize, batch, default values, folded unaries) and running each spec's
// transform in registers. Partials combine through warp shuffles, shared
// memory and a final pass of one CTA per spec. The parallel fold reproduces the
// reference's sequential one:
//   * u8 Sum wraps mod 256: accumulated in 32 bits, reduced mod 256 at the end;
//   * float Sum accumulates in double (as the reference); the order of the
//     double additions differs, agreement is within 2^-20 relative
//     (SPEC.md:388), ~2^-40 in practice;
//   * Max / Min keep "a < b ? b : a" (NaN is never adopted). The result is the
//     FIRST element numerically equal to the extremum; only a zero extremum can
//     differ in bits (+0 / -0), so when one comes out zero the host runs a
//     second pass (fk_reduce_zero_sign) that finds the earliest +0 and -0.
#include <cuda_runtime.h>

#include <algorithm>

#include "fk_launch.hpp"
#include "fk_reduce.hpp"
#include "fk_stages.cuh"

namespace fk {

namespace {

constexpr int kRE = 4;            // elements per tile
constexpr uint32_t kRBlock = 256;  // threads per CTA
#ifndef FK_PLAIN_U
#define FK_PLAIN_U 2
#endif
#ifndef FK_PLAIN_MINB
#define FK_PLAIN_MINB 4
#endif
constexpr int kPlainU = FK_PLAIN_U;  // vectors in flight per thread (plain rows)

struct Acc {
  uint64_t v[3];  // double bits (float Sum), 32-bit running u8 sum, or the extremum's lane bits
};

__device__ __forceinline__ double as_d(uint64_t b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ uint64_t d_bits(double d) { return (uint64_t)__double_as_longlong(d); }

// a < b in the lane kind (u8 / f32 / f64 bits)
__device__ __forceinline__ bool lane_less(uint32_t lk, uint64_t a, uint64_t b) {
  if (lk == FK_U8) return (a & 0xffu) < (b & 0xffu);
  if (lk == FK_F32) return __uint_as_float(uint32_t(a)) < __uint_as_float(uint32_t(b));
  return as_d(a) < as_d(b);
}

// a = a (+) x for one spec
__device__ __forceinline__ void combine(const RSpecDev& s, Acc& a, const Acc& x) {
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    if (l >= int(s.lanes)) break;
    if (s.combine == FK_REDUCE_SUM) {
      if (s.dsum) a.v[l] = d_bits(as_d(a.v[l]) + as_d(x.v[l]));
      else a.v[l] = uint32_t(a.v[l]) + uint32_t(x.v[l]);  // u8_add, mod 256 at the end
    } else {
      const bool take = s.combine == FK_REDUCE_MAX ? lane_less(s.lane_kind, a.v[l], x.v[l])
                                                   : lane_less(s.lane_kind, x.v[l], a.v[l]);
      if (take) a.v[l] = x.v[l];
    }
  }
}

__device__ __forceinline__ void identity_acc(const RSpecDev& s, Acc& a) {
#pragma unroll
  for (int l = 0; l < 3; ++l) a.v[l] = s.dsum ? d_bits(0.0) : (s.combine == FK_REDUCE_SUM ? 0 : s.ident[l]);
}

// one element's lanes in the accumulator's encoding
template <class Lane, int L>
__device__ __forceinline__ Acc as_acc(const RSpecDev& s, const Lane (&v)[L]) {
  Acc x;
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const uint64_t b = l < L ? uint64_t(v[l]) : 0;
    if (s.dsum) x.v[l] = d_bits(s.lane_kind == FK_F32 ? double(__uint_as_float(uint32_t(b))) : as_d(b));
    else x.v[l] = s.lane_kind == FK_F32 ? (b & 0xffffffffu) : (s.lane_kind == FK_U8 ? (b & 0xffu) : b);
  }
  return x;
}

__device__ __forceinline__ Acc shfl_down(const Acc& a, int d) {
  Acc r;
#pragma unroll
  for (int l = 0; l < 3; ++l) r.v[l] = __shfl_down_sync(0xffffffffu, a.v[l], d);
  return r;
}

// the tile at linear tile index t: plane z, row y, first column x, element count n
struct TileAt {
  uint32_t z, y, x;
  int n;
};
__device__ __forceinline__ TileAt tile_at(const DPlan& P, uint64_t t) {
  const uint64_t tiles_plane = uint64_t(P.tiles);
  TileAt a;
  // plane index: none for one plane, a 32-bit reciprocal division when the
  // whole space has < 2^32 tiles (P.zdiv), a 64-bit division otherwise
  a.z = P.batch == 1 ? 0u : (t < (uint64_t(1) << 32) ? dev::fastdiv(uint32_t(t), P.zdiv) : uint32_t(t / tiles_plane));
  const uint32_t tt = uint32_t(t - uint64_t(a.z) * tiles_plane);
  a.y = dev::fastdiv(tt, P.tpr);
  a.x = (tt - a.y * P.tiles_per_row) * kRE;
  a.n = (P.width - a.x) < uint32_t(kRE) ? int(P.width - a.x) : kRE;
  return a;
}

template <class Lane, int L>
__device__ __forceinline__ void read_tile(const DPlan& P, const TileAt& at, Lane (&v)[kRE][L]) {
  const DSample s = P.reads[at.z];
  if constexpr (L == 1) {  // plain u8 / f32 rows, whole aligned tile: one vector load
    if (s.mode == RD_DIRECT && !(s.flags & SF_DEFAULT) && s.post_len == 0 && at.n == kRE &&
        (s.kind == FK_F32 || s.kind == FK_U8)) {
      const uint32_t b = s.kind == FK_F32 ? 4u : 1u;
      const uint64_t a = s.src + uint64_t(s.y0 + at.y) * s.pitch + uint64_t(s.x0 + at.x) * b;
      if ((a & (kRE * b - 1)) == 0) {
        if (s.kind == FK_F32) {
          const uint4 q = __ldg(reinterpret_cast<const uint4*>(a));
          v[0][0] = Lane(q.x); v[1][0] = Lane(q.y); v[2][0] = Lane(q.z); v[3][0] = Lane(q.w);
        } else {
          const uint32_t q = __ldg(reinterpret_cast<const uint32_t*>(a));
#pragma unroll
          for (int e = 0; e < kRE; ++e) v[e][0] = Lane((q >> (8 * e)) & 0xffu);
        }
        return;
      }
    }
  }
  dev::read_raw(P, s, at.x, at.y, at.n, v, nullptr, nullptr);
  if (!(s.flags & SF_DEFAULT)) dev::run_ops(P, s.post_off, s.post_len, at.z, v);
}

template <class Lane, int L>
__device__ __forceinline__ void spec_values(const DPlan& P, const RSpecDev& s, uint32_t z, const Lane (&v)[kRE][L],
                                            Lane (&w)[kRE][L]) {
#pragma unroll
  for (int e = 0; e < kRE; ++e)
#pragma unroll
    for (int l = 0; l < L; ++l) w[e][l] = v[e][l];
  if (s.op != kNoOp) dev::run_ops(P, s.op, 1, z, w);
}

// Fold a tile's n values into one spec's accumulator, specialised on the
// combine and the lane kind (the dispatch is per tile and warp-uniform). Every
// one of the L lanes is folded; lanes beyond the spec's value are never output.
template <uint32_t CB, uint32_t LK, class Lane, int E, int L>
__device__ __forceinline__ void fold_tile(Acc& a, const Lane (&w)[E][L], int n) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (e >= n) break;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      const uint64_t b = uint64_t(w[e][l]);
      if constexpr (CB == FK_REDUCE_SUM && LK == FK_U8) {
        a.v[l] = uint32_t(a.v[l]) + uint32_t(b & 0xffu);
      } else if constexpr (CB == FK_REDUCE_SUM) {
        const double x = LK == FK_F32 ? double(__uint_as_float(uint32_t(b))) : as_d(b);
        a.v[l] = d_bits(as_d(a.v[l]) + x);
      } else {
        const uint64_t x = LK == FK_U8 ? (b & 0xffu) : (LK == FK_F32 ? (b & 0xffffffffu) : b);
        const bool take = CB == FK_REDUCE_MAX ? lane_less(LK, a.v[l], x) : lane_less(LK, x, a.v[l]);
        if (take) a.v[l] = x;
      }
    }
  }
}

template <class Lane, int E, int L>
__device__ __forceinline__ void fold_spec(const RSpecDev& s, Acc& a, const Lane (&w)[E][L], int n) {
  switch (s.combine * 3 + s.lane_kind) {
    case FK_REDUCE_SUM * 3 + FK_U8: fold_tile<FK_REDUCE_SUM, FK_U8>(a, w, n); break;
    case FK_REDUCE_SUM * 3 + FK_F32: fold_tile<FK_REDUCE_SUM, FK_F32>(a, w, n); break;
    case FK_REDUCE_SUM * 3 + FK_F64: fold_tile<FK_REDUCE_SUM, FK_F64>(a, w, n); break;
    case FK_REDUCE_MAX * 3 + FK_U8: fold_tile<FK_REDUCE_MAX, FK_U8>(a, w, n); break;
    case FK_REDUCE_MAX * 3 + FK_F32: fold_tile<FK_REDUCE_MAX, FK_F32>(a, w, n); break;
    case FK_REDUCE_MAX * 3 + FK_F64: fold_tile<FK_REDUCE_MAX, FK_F64>(a, w, n); break;
    case FK_REDUCE_MIN * 3 + FK_U8: fold_tile<FK_REDUCE_MIN, FK_U8>(a, w, n); break;
    case FK_REDUCE_MIN * 3 + FK_F32: fold_tile<FK_REDUCE_MIN, FK_F32>(a, w, n); break;
    default: fold_tile<FK_REDUCE_MIN, FK_F64>(a, w, n); break;
  }
}

// CTA partials of every spec: per-thread folds, then warp / CTA combines
template <class Lane, int L>
__global__ void __launch_bounds__(kRBlock) fk_reduce_partial(const __grid_constant__ DPlan P,
                                                           const __grid_constant__ RSpecsDev S, Acc* partials) {
  __shared__ Acc warp_acc[kRBlock / 32][kMaxReduceSpecs];
  Acc acc[kMaxReduceSpecs];
#pragma unroll
  for (int k = 0; k < kMaxReduceSpecs; ++k)
    if (k < int(S.n)) identity_acc(S.s[k], acc[k]);
  const uint64_t total = uint64_t(P.tiles) * P.batch;
  const uint64_t stride = uint64_t(gridDim.x) * kRBlock;
  for (uint64_t t = uint64_t(blockIdx.x) * kRBlock + threadIdx.x; t < total; t += stride) {
    const TileAt at = tile_at(P, t);
    Lane v[kRE][L];
    read_tile<Lane, L>(P, at, v);
#pragma unroll
    for (int k = 0; k < kMaxReduceSpecs; ++k) {
      if (k >= int(S.n)) break;
      if (S.s[k].op == kNoOp) {
        fold_spec<Lane, kRE, L>(S.s[k], acc[k], v, at.n);
      } else {
        Lane w[kRE][L];
        spec_values<Lane, L>(P, S.s[k], at.z, v, w);
        fold_spec<Lane, kRE, L>(S.s[k], acc[k], w, at.n);
      }
    }
  }
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kMaxReduceSpecs; ++k) {
    if (k >= int(S.n)) break;
    for (int d = 16; d > 0; d >>= 1) {
      const Acc o = shfl_down(acc[k], d);
      if (lane < uint32_t(d)) combine(S.s[k], acc[k], o);
    }
    if (lane == 0) warp_acc[warp][k] = acc[k];
  }
  __syncthreads();
  if (threadIdx.x < uint32_t(S.n)) {
    const int k = int(threadIdx.x);
    Acc a = warp_acc[0][k];
    for (uint32_t w = 1; w < kRBlock / 32; ++w) combine(S.s[k], a, warp_acc[w][k]);
    partials[uint64_t(blockIdx.x) * kMaxReduceSpecs + k] = a;
  }
}

// Plain single-lane rows (one plane, direct read, no default values or folded
// unaries, 16-byte aligned rows): each thread folds 16-byte vectors (16 u8 or
// 4 f32), two in flight per iteration, with the read stage's bookkeeping
// reduced to one reciprocal division per vector.
// A thread's walk over the vectors v, v + stride, ...: a 32-bit byte offset
// from the plane's first element (the host keeps the plane under 4 GiB) that
// advances by the stride's (rows, vectors) with one carry, no division.
struct PlainCursor {
  uint32_t off;  // byte offset of the vector
  uint32_t xv;   // vector index in its row
};

__device__ __forceinline__ PlainCursor plain_start(const PlainRows& R, uint32_t v) {
  const uint32_t y = dev::fastdiv(v, R.vdiv);
  const uint32_t xv = v - y * R.vpr;
  return PlainCursor{y * uint32_t(R.pitch) + xv * R.vb, xv};
}

__device__ __forceinline__ void plain_advance(const PlainRows& R, PlainCursor& c, uint32_t sx, uint32_t dstep,
                                              uint32_t wrap) {
  c.off += dstep;
  c.xv += sx;
  if (c.xv >= R.vpr) {
    c.xv -= R.vpr;
    c.off += wrap;
  }
}

// the row's last, partial vector (its bytes past the row are never touched)
template <uint32_t KIND>
__device__ __noinline__ uint4 plain_partial(uint64_t a, uint32_t n) {
  uint32_t w[4] = {0, 0, 0, 0};
  for (uint32_t e = 0; e < n; ++e) {
    const uint32_t b = KIND == FK_U8 ? uint32_t(*reinterpret_cast<const uint8_t*>(a + e))
                                     : *reinterpret_cast<const uint32_t*>(a + 4 * e);
    if (KIND == FK_U8) w[e >> 2] |= b << (8 * (e & 3)); else w[e] = b;
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <uint32_t KIND>
__device__ __forceinline__ int plain_load(const PlainRows& R, const PlainCursor& c, uint4& q) {
  constexpr uint32_t VE = KIND == FK_U8 ? 16u : 4u;
  const uint32_t left = R.width - c.xv * VE;
  const uint64_t a = R.base + c.off;
  if (left >= VE) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "l"(a));
    return int(VE);
  }
  q = plain_partial<KIND>(a, left);
  return int(left);
}

// The general fold of one spec over one vector (a transform, or a partial
// vector at a row's end): out of line, accumulator in and out by value, so the
// hot loop's code stays small and its accumulators stay in registers.
template <uint32_t KIND>
__device__ __noinline__ uint64_t fold_vector_general(const DPlan& P, const RSpecDev& s, uint64_t a0, uint4 q, int n) {
  constexpr int VE = KIND == FK_U8 ? 16 : 4;
  Acc a;
  a.v[0] = a0;
  a.v[1] = a.v[2] = 0;
  uint32_t w[VE][1];
  const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int e = 0; e < VE; ++e) w[e][0] = KIND == FK_U8 ? (qw[e >> 2] >> (8 * (e & 3))) & 0xffu : qw[e];
  if (s.op != kNoOp) dev::run_ops(P, s.op, 1, 0, w);
  fold_spec<uint32_t, VE, 1>(s, a, w, n);
  return a.v[0];
}

// A whole vector, no transform.
//   f32 Sum: a pairwise tree in double (the order of the double additions is
//     free within the 2^-20 agreement);
//   f32 Max / Min: fmaxf / fminf trees, which keep "a < b ? b : a"'s value (NaN
//     never adopted; only the sign of a zero result can differ, and the
//     zero-sign pass settles that);
//   u8 Sum: dp4a into the running 32-bit sum (only ever read mod 256);
//   u8 Max / Min: the bytes as two 16-bit lanes per word (even / odd bytes),
//     folded with VIMNMX.U16x2 into a packed accumulator pk that is reduced
//     horizontally once, after the walk.
struct U8Split {
  uint32_t e[4], o[4];
};
__device__ __forceinline__ U8Split u8_split(const uint4& q) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
  U8Split r;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    r.e[i] = w[i] & 0x00ff00ffu;
    r.o[i] = (w[i] >> 8) & 0x00ff00ffu;
  }
  return r;
}
__device__ __forceinline__ uint32_t mm2(uint32_t a, uint32_t b, bool mx) { return mx ? __vmaxu2(a, b) : __vminu2(a, b); }

template <uint32_t KIND>
__device__ __forceinline__ void fold_vector_fast(const RSpecDev& s, uint64_t& a0, uint32_t& pk, const uint4& q,
                                                 const U8Split& sp) {
  if constexpr (KIND == FK_U8) {
    if (s.combine == FK_REDUCE_SUM) {
      uint32_t t = uint32_t(a0);
      t = __dp4a(q.x, 0x01010101u, t);
      t = __dp4a(q.y, 0x01010101u, t);
      t = __dp4a(q.z, 0x01010101u, t);
      t = __dp4a(q.w, 0x01010101u, t);
      a0 = t;
    } else {
      const bool mx = s.combine == FK_REDUCE_MAX;
      const uint32_t m = mm2(mm2(mm2(sp.e[0], sp.o[0], mx), mm2(sp.e[1], sp.o[1], mx), mx),
                             mm2(mm2(sp.e[2], sp.o[2], mx), mm2(sp.e[3], sp.o[3], mx), mx), mx);
      pk = mm2(pk, m, mx);
    }
  } else {
    const float x0 = __uint_as_float(q.x), x1 = __uint_as_float(q.y), x2 = __uint_as_float(q.z),
                x3 = __uint_as_float(q.w);
    if (s.combine == FK_REDUCE_SUM) {
      const double t = (double(x0) + double(x1)) + (double(x2) + double(x3));
      a0 = d_bits(as_d(a0) + t);
    } else if (s.combine == FK_REDUCE_MAX) {
      a0 = __float_as_uint(fmaxf(__uint_as_float(uint32_t(a0)), fmaxf(fmaxf(x0, x1), fmaxf(x2, x3))));
    } else {
      a0 = __float_as_uint(fminf(__uint_as_float(uint32_t(a0)), fminf(fminf(x0, x1), fminf(x2, x3))));
    }
  }
}

template <uint32_t KIND>
__device__ __forceinline__ void plain_fold(const DPlan& P, const RSpecsDev& S, uint64_t (&acc)[kMaxReduceSpecs],
                                           uint32_t (&pk)[kMaxReduceSpecs], const uint4& q, int n) {
  constexpr int VE = KIND == FK_U8 ? 16 : 4;
  const U8Split sp = KIND == FK_U8 ? u8_split(q) : U8Split{};
#pragma unroll
  for (int k = 0; k < kMaxReduceSpecs; ++k) {
    if (k >= int(S.n)) break;
    const RSpecDev& s = S.s[k];
    if (s.op == kNoOp && n == VE) fold_vector_fast<KIND>(s, acc[k], pk[k], q, sp);
    else acc[k] = fold_vector_general<KIND>(P, s, acc[k], q, n);
  }
}

template <uint32_t KIND>
__global__ void __launch_bounds__(kRBlock, FK_PLAIN_MINB) fk_reduce_plain(const __grid_constant__ DPlan P,
                                                                         const __grid_constant__ RSpecsDev S,
                                                                         const __grid_constant__ PlainRows R,
                                                                         Acc* partials) {
  __shared__ Acc warp_acc[kRBlock / 32][kMaxReduceSpecs];
  uint64_t a1[kMaxReduceSpecs];  // single-lane accumulators
  uint32_t pk[kMaxReduceSpecs];  // u8 Max / Min: packed 16x2 accumulators
#pragma unroll
  for (int k = 0; k < kMaxReduceSpecs; ++k) {
    Acc i;
    identity_acc(S.s[k], i);
    a1[k] = i.v[0];
    pk[k] = uint32_t(i.v[0] & 0xffu) * 0x00010001u;
  }
  const uint32_t total = R.vecs;
  const uint32_t stride = gridDim.x * kRBlock;
  uint32_t v = blockIdx.x * kRBlock + threadIdx.x;
  if (v < total) {
    const uint32_t sy = dev::fastdiv(stride, R.vdiv), sx = stride - sy * R.vpr;
    const uint32_t dstep = sy * uint32_t(R.pitch) + sx * R.vb;
    const uint32_t wrap = uint32_t(R.pitch) - R.vpr * R.vb;
    PlainCursor c = plain_start(R, v);
    for (; v + (kPlainU - 1) * stride < total; v += kPlainU * stride) {  // kPlainU loads in flight
      uint4 q[kPlainU];
      int n[kPlainU];
#pragma unroll
      for (int u = 0; u < kPlainU; ++u) {
        n[u] = plain_load<KIND>(R, c, q[u]);
        plain_advance(R, c, sx, dstep, wrap);
      }
#ifdef FK_PLAIN_PROBE  // memory-only probe: no fold
#pragma unroll
      for (int u = 0; u < kPlainU; ++u) a1[0] ^= q[u].x ^ q[u].y ^ q[u].z ^ q[u].w ^ n[u];
#else
#pragma unroll
      for (int u = 0; u < kPlainU; ++u) plain_fold<KIND>(P, S, a1, pk, q[u], n[u]);
#endif
    }
    for (; v < total; v += stride) {
      uint4 q;
      const int n = plain_load<KIND>(R, c, q);
      plain_advance(R, c, sx, dstep, wrap);
      plain_fold<KIND>(P, S, a1, pk, q, n);
    }
  }
  Acc acc[kMaxReduceSpecs];
#pragma unroll
  for (int k = 0; k < kMaxReduceSpecs; ++k) {
    acc[k].v[0] = a1[k];
    acc[k].v[1] = acc[k].v[2] = 0;
    // the packed lanes' extremum joins the scalar one — only for specs that fed
    // them (u8 values, no transform: fold_vector_fast); any other spec's pk is
    // an untouched seed (e.g. 0 for an f32 Min's +inf identity)
    if (KIND == FK_U8 && k < int(S.n) && S.s[k].combine != FK_REDUCE_SUM && S.s[k].op == kNoOp &&
        S.s[k].lane_kind == FK_U8) {
      const bool mx = S.s[k].combine == FK_REDUCE_MAX;
      const uint32_t m = mm2(pk[k], pk[k] >> 16, mx) & 0xffu;
      if (mx ? uint32_t(a1[k]) < m : m < uint32_t(a1[k])) acc[k].v[0] = m;
    }
  }
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kMaxReduceSpecs; ++k) {
    if (k >= int(S.n)) break;
    for (int d = 16; d > 0; d >>= 1) {
      const Acc o = shfl_down(acc[k], d);
      if (lane < uint32_t(d)) combine(S.s[k], acc[k], o);
    }
    if (lane == 0) warp_acc[warp][k] = acc[k];
  }
  __syncthreads();
  if (threadIdx.x < uint32_t(S.n)) {
    const int k = int(threadIdx.x);
    Acc a = warp_acc[0][k];
    for (uint32_t w = 1; w < kRBlock / 32; ++w) combine(S.s[k], a, warp_acc[w][k]);
    partials[uint64_t(blockIdx.x) * kMaxReduceSpecs + k] = a;
  }
}

// Plain u8x3 rows (interleaved 3-channel bytes): vectors of 16 pixels = 48
// bytes (three 16-byte loads), the same cursor walk; per channel, Sum through
// dp4a with the channel's byte mask (the channel pattern repeats every three
// words), Max / Min on the extracted bytes.
struct Px16 {
  uint32_t w[12];
};

__device__ __forceinline__ Px16 plain3_load(const PlainRows& R, const PlainCursor& c, int& n) {
  Px16 p;
  const uint32_t left = R.width - c.xv * 16u;
  const uint64_t a = R.base + c.off;
  if (left >= 16u) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(p.w[4 * i]), "=r"(p.w[4 * i + 1]), "=r"(p.w[4 * i + 2]), "=r"(p.w[4 * i + 3])
                   : "l"(a + 16u * i));
    n = 16;
  } else {
#pragma unroll
    for (int i = 0; i < 12; ++i) p.w[i] = 0;
    for (uint32_t b = 0; b < 3 * left; ++b)
      p.w[b >> 2] |= uint32_t(*reinterpret_cast<const uint8_t*>(a + b)) << (8 * (b & 3));
    n = int(left);
  }
  return p;
}

__device__ __noinline__ Acc fold3_general(const DPlan& P, const RSpecDev& s, Acc a, Px16 p, int n) {
  uint32_t w[16][3];
#pragma unroll
  for (int e = 0; e < 16; ++e)
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const int b = 3 * e + l;
      w[e][l] = (p.w[b >> 2] >> (8 * (b & 3))) & 0xffu;
    }
  if (s.op != kNoOp) dev::run_ops(P, s.op, 1, 0, w);
  fold_spec<uint32_t, 16, 3>(s, a, w, n);
  return a;
}

__device__ __forceinline__ void fold3_fast(const RSpecDev& s, Acc& a, const Px16& p) {
  if (s.combine == FK_REDUCE_SUM) {
    // byte p = 4 i + b of the vector is channel p % 3; masks per (channel, i % 3)
    constexpr uint32_t M[3][3] = {{0x01000001u, 0x00010000u, 0x00000100u},
                                  {0x00000100u, 0x01000001u, 0x00010000u},
                                  {0x00010000u, 0x00000100u, 0x01000001u}};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      uint32_t t = uint32_t(a.v[c]);
#pragma unroll
      for (int i = 0; i < 12; ++i) t = __dp4a(p.w[i], M[c][i % 3], t);
      a.v[c] = t;
    }
  } else {
    const bool mx = s.combine == FK_REDUCE_MAX;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      uint32_t m = uint32_t(a.v[c]);
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int b = 3 * e + c;
        const uint32_t x = (p.w[b >> 2] >> (8 * (b & 3))) & 0xffu;
        m = mx ? max(m, x) : min(m, x);
      }
      a.v[c] = m;
    }
  }
}

__global__ void __launch_bounds__(kRBlock, 2) fk_reduce_plain3(const __grid_constant__ DPlan P,
                                                                          const __grid_constant__ RSpecsDev S,
                                                                          const __grid_constant__ PlainRows R,
                                                                          Acc* partials) {
  __shared__ Acc warp_acc[kRBlock / 32][kMaxReduceSpecs];
  Acc acc[kMaxReduceSpecs];
#pragma unroll
  for (int k = 0; k < kMaxReduceSpecs; ++k) identity_acc(S.s[k], acc[k]);
  const uint32_t total = R.vecs;
  const uint32_t stride = gridDim.x * kRBlock;
  uint32_t v = blockIdx.x * kRBlock + threadIdx.x;
  if (v < total) {
    const uint32_t sy = dev::fastdiv(stride, R.vdiv), sx = stride - sy * R.vpr;
    const uint32_t dstep = sy * uint32_t(R.pitch) + sx * R.vb;
    const uint32_t wrap = uint32_t(R.pitch) - R.vpr * R.vb;
    PlainCursor c = plain_start(R, v);
    for (; v < total; v += stride) {
      int n;
      const Px16 p = plain3_load(R, c, n);
      plain_advance(R, c, sx, dstep, wrap);
#pragma unroll
      for (int k = 0; k < kMaxReduceSpecs; ++k) {
        if (k >= int(S.n)) break;
        const RSpecDev& s = S.s[k];
        if (s.op == kNoOp && n == 16) fold3_fast(s, acc[k], p);
        else acc[k] = fold3_general(P, s, acc[k], p, n);
      }
    }
  }
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kMaxReduceSpecs; ++k) {
    if (k >= int(S.n)) break;
    for (int d = 16; d > 0; d >>= 1) {
      const Acc o = shfl_down(acc[k], d);
      if (lane < uint32_t(d)) combine(S.s[k], acc[k], o);
    }
    if (lane == 0) warp_acc[warp][k] = acc[k];
  }
  __syncthreads();
  if (threadIdx.x < uint32_t(S.n)) {
    const int k = int(threadIdx.x);
    Acc a = warp_acc[0][k];
    for (uint32_t w = 1; w < kRBlock / 32; ++w) combine(S.s[k], a, warp_acc[w][k]);
    partials[uint64_t(blockIdx.x) * kMaxReduceSpecs + k] = a;
  }
}

// Zero-sign pass over plain rows (u8 / f32 reads whose spec values are f32):
// each thread keeps the first +0 / -0 it meets per flagged spec (its walk is
// in increasing (y, x) order, and v * VE + e is monotone in it), then one
// atomicMin per warp — no per-element atomics on zero-heavy planes.
template <uint32_t KIND>
__global__ void __launch_bounds__(kRBlock) fk_reduce_plain_zero_sign(const __grid_constant__ DPlan P,
                                                                   const __grid_constant__ RSpecsDev S,
                                                                   const __grid_constant__ PlainRows R,
                                                                   uint32_t zmask, unsigned long long* first) {
  constexpr int VE = KIND == FK_U8 ? 16 : 4;
  unsigned long long f[kMaxReduceSpecs][2];
#pragma unroll
  for (int k = 0; k < kMaxReduceSpecs; ++k) f[k][0] = f[k][1] = ~0ull;
  const uint32_t total = R.vecs;
  const uint32_t stride = gridDim.x * kRBlock;
  uint32_t v = blockIdx.x * kRBlock + threadIdx.x;
  if (v < total) {
    const uint32_t sy = dev::fastdiv(stride, R.vdiv), sx = stride - sy * R.vpr;
    const uint32_t dstep = sy * uint32_t(R.pitch) + sx * R.vb;
    const uint32_t wrap = uint32_t(R.pitch) - R.vpr * R.vb;
    PlainCursor c = plain_start(R, v);
    for (; v < total; v += stride) {
      uint4 q;
      const int n = plain_load<KIND>(R, c, q);
      plain_advance(R, c, sx, dstep, wrap);
      uint32_t x[VE][1];
      const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < VE; ++e) x[e][0] = KIND == FK_U8 ? (qw[e >> 2] >> (8 * (e & 3))) & 0xffu : qw[e];
#pragma unroll
      for (int k = 0; k < kMaxReduceSpecs; ++k) {
        if (k >= int(S.n) || !((zmask >> (3 * k)) & 1u)) continue;
        uint32_t w[VE][1];
#pragma unroll
        for (int e = 0; e < VE; ++e) w[e][0] = x[e][0];
        if (S.s[k].op != kNoOp) dev::run_ops(P, S.s[k].op, 1, 0, w);
#pragma unroll
        for (int e = 0; e < VE; ++e) {
          if (e < n && (w[e][0] & 0x7fffffffu) == 0) {
            const unsigned long long i = uint64_t(v) * VE + e;
            if (w[e][0] >> 31) f[k][1] = i < f[k][1] ? i : f[k][1];
            else f[k][0] = i < f[k][0] ? i : f[k][0];
          }
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kMaxReduceSpecs; ++k) {
    if (k >= int(S.n) || !((zmask >> (3 * k)) & 1u)) continue;
#pragma unroll
    for (int sgn = 0; sgn < 2; ++sgn) {
      unsigned long long m = f[k][sgn];
      for (int d = 16; d > 0; d >>= 1) {
        const unsigned long long o = __shfl_down_sync(0xffffffffu, m, d);
        m = o < m ? o : m;
      }
      if ((threadIdx.x & 31u) == 0 && m != ~0ull) atomicMin(first + 6 * k + sgn, m);
    }
  }
}

// one CTA per spec: the CTA partials, then the spec's identity (the left-most
// operand of the reference's merge, dpp.cpp:232-237) and finish_accum
// (dpp.cpp:138-152). out: 3 lane words per spec (value kind bits).
__global__ void __launch_bounds__(kRBlock) fk_reduce_final(const __grid_constant__ RSpecsDev S, const Acc* partials,
                                                          uint32_t nparts, uint64_t* out) {
  __shared__ Acc warp_acc[kRBlock / 32];
  const int k = int(blockIdx.x);
  const RSpecDev& s = S.s[k];
  Acc a;
  identity_acc(s, a);
  uint32_t p = threadIdx.x;
  for (; p + 3 * kRBlock < nparts; p += 4 * kRBlock) {  // four partials in flight
    Acc x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = partials[uint64_t(p + u * kRBlock) * kMaxReduceSpecs + k];
#pragma unroll
    for (int u = 0; u < 4; ++u) combine(s, a, x[u]);
  }
  for (; p < nparts; p += kRBlock) combine(s, a, partials[uint64_t(p) * kMaxReduceSpecs + k]);
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (int d = 16; d > 0; d >>= 1) {
    const Acc o = shfl_down(a, d);
    if (lane < uint32_t(d)) combine(s, a, o);
  }
  if (lane == 0) warp_acc[warp] = a;
  __syncthreads();
  if (threadIdx.x != 0) return;
  a = warp_acc[0];
  for (uint32_t w = 1; w < kRBlock / 32; ++w) combine(s, a, warp_acc[w]);
  for (int l = 0; l < 3; ++l) {
    if (s.dsum) {
      const double total = as_d(s.user_ident[l]) + as_d(a.v[l]);  // identity as double + the sum
      out[3 * k + l] = s.lane_kind == FK_F32 ? uint64_t(__float_as_uint(float(total))) : d_bits(total);
    } else if (s.combine == FK_REDUCE_SUM) {
      out[3 * k + l] = (s.user_ident[l] + a.v[l]) & 0xffu;
    } else {
      Acc r, m;
      r.v[0] = r.v[1] = r.v[2] = s.user_ident[l];
      m.v[0] = m.v[1] = m.v[2] = a.v[l];
      combine(s, r, m);  // keeps the identity on equality: it comes first
      out[3 * k + l] = r.v[0];
    }
  }
}

// Second pass for a zero Max / Min: the linear index of the first +0 and of the
// first -0 of each (spec, lane) flagged in zmask (bit 3 * spec + lane).
template <class Lane, int L>
__global__ void __launch_bounds__(kRBlock) fk_reduce_zero_sign(const __grid_constant__ DPlan P,
                                                             const __grid_constant__ RSpecsDev S, uint32_t zmask,
                                                             unsigned long long* first) {
  uint32_t done = 0;  // (spec, lane, sign) keys this thread has already recorded
  const uint64_t total = uint64_t(P.tiles) * P.batch;
  const uint64_t stride = uint64_t(gridDim.x) * kRBlock;
  for (uint64_t t = uint64_t(blockIdx.x) * kRBlock + threadIdx.x; t < total; t += stride) {
    const TileAt at = tile_at(P, t);
    Lane v[kRE][L];
    read_tile<Lane, L>(P, at, v);
    const uint64_t i0 = (uint64_t(at.z) * P.height + at.y) * P.width + at.x;
    for (int k = 0; k < int(S.n); ++k) {
      if (!((zmask >> (3 * k)) & 7u)) continue;
      Lane w[kRE][L];
      spec_values<Lane, L>(P, S.s[k], at.z, v, w);
      for (int e = 0; e < at.n; ++e) {
        const Acc x = as_acc<Lane, L>(S.s[k], w[e]);
        for (int l = 0; l < int(S.s[k].lanes); ++l) {
          if (!((zmask >> (3 * k + l)) & 1u)) continue;
          const bool f32 = S.s[k].lane_kind == FK_F32;
          const uint64_t mag = f32 ? (x.v[l] & 0x7fffffffu) : (x.v[l] & 0x7fffffffffffffffull);
          if (mag == 0) {
            const bool neg = f32 ? ((x.v[l] >> 31) & 1u) : ((x.v[l] >> 63) & 1u);
            const uint32_t bit = 1u << (6 * k + 2 * l + (neg ? 1 : 0));
            if (!(done & bit)) {  // the thread walks in increasing (z, y, x): its first is its minimum
              atomicMin(first + 6 * k + 2 * l + (neg ? 1 : 0), (unsigned long long)(i0 + e));
              done |= bit;
            }
          }
        }
      }
    }
  }
}

}  // namespace

cudaError_t launch_reduce(int cls, const DPlan& P, const RSpecsDev& S, void* scratch, uint32_t nblocks, uint64_t* out,
                          cudaStream_t st) {
  Acc* parts = static_cast<Acc*>(scratch);
  switch (cls) {
    case 0: fk_reduce_partial<uint32_t, 1><<<nblocks, kRBlock, 0, st>>>(P, S, parts); break;
    case 1: fk_reduce_partial<uint32_t, 3><<<nblocks, kRBlock, 0, st>>>(P, S, parts); break;
    case 2: fk_reduce_partial<uint64_t, 1><<<nblocks, kRBlock, 0, st>>>(P, S, parts); break;
    default: fk_reduce_partial<uint64_t, 3><<<nblocks, kRBlock, 0, st>>>(P, S, parts); break;
  }
  fk_reduce_final<<<S.n, kRBlock, 0, st>>>(S, parts, nblocks, out);
  return cudaGetLastError();
}

cudaError_t launch_reduce_zero_sign(int cls, const DPlan& P, const RSpecsDev& S, uint32_t zmask, uint32_t nblocks,
                                    unsigned long long* first, cudaStream_t st) {
  switch (cls) {
    case 0: fk_reduce_zero_sign<uint32_t, 1><<<nblocks, kRBlock, 0, st>>>(P, S, zmask, first); break;
    case 1: fk_reduce_zero_sign<uint32_t, 3><<<nblocks, kRBlock, 0, st>>>(P, S, zmask, first); break;
    case 2: fk_reduce_zero_sign<uint64_t, 1><<<nblocks, kRBlock, 0, st>>>(P, S, zmask, first); break;
    default: fk_reduce_zero_sign<uint64_t, 3><<<nblocks, kRBlock, 0, st>>>(P, S, zmask, first); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_reduce_plain(const DPlan& P, const RSpecsDev& S, const PlainRows& R, void* scratch,
                                uint32_t nblocks, uint64_t* out, cudaStream_t st) {
  Acc* parts = static_cast<Acc*>(scratch);
  if (R.kind == FK_U8) fk_reduce_plain<FK_U8><<<nblocks, kRBlock, 0, st>>>(P, S, R, parts);
  else if (R.kind == FK_U8X3) fk_reduce_plain3<<<nblocks, kRBlock, 0, st>>>(P, S, R, parts);
  else fk_reduce_plain<FK_F32><<<nblocks, kRBlock, 0, st>>>(P, S, R, parts);
  fk_reduce_final<<<S.n, kRBlock, 0, st>>>(S, parts, nblocks, out);
  return cudaGetLastError();
}

cudaError_t launch_reduce_plain_zero_sign(const DPlan& P, const RSpecsDev& S, const PlainRows& R, uint32_t zmask,
                                          uint32_t nblocks, unsigned long long* first, cudaStream_t st) {
  if (R.kind == FK_U8) fk_reduce_plain_zero_sign<FK_U8><<<nblocks, kRBlock, 0, st>>>(P, S, R, zmask, first);
  else fk_reduce_plain_zero_sign<FK_F32><<<nblocks, kRBlock, 0, st>>>(P, S, R, zmask, first);
  return cudaGetLastError();
}

uint32_t reduce_plain_blocks(uint32_t kind, int sms) {
  int per_sm = 0;
  if (kind == FK_U8) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fk_reduce_plain<FK_U8>, kRBlock, 0);
  else if (kind == FK_U8X3) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fk_reduce_plain3, kRBlock, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fk_reduce_plain<FK_F32>, kRBlock, 0);
  return uint32_t(std::max(1, per_sm)) * uint32_t(sms);
}

size_t reduce_scratch_bytes(uint32_t nblocks) { return size_t(nblocks) * kMaxReduceSpecs * sizeof(Acc); }
int reduce_tile_elems() { return kRE; }

}  // namespace fk
