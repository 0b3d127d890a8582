// fk_reduce.cu — ReduceDPP on B200 (dpp.hpp:32-53, dpp.cpp:46-246): several
// Sum / Max / Min folds over one read, in ONE traversal of the source.
//
// Every thread folds tiles of E consecutive x (grid-stride, coalesced), reading
// each element once through the same read stage as the fused kernels (crop,
// resize, batch, default values, folded unaries) and running each spec's
// transform in registers. Partials then combine through warp shuffles, shared
// memory and a last single-CTA pass. The fold is made order-independent so the
// parallel order reproduces the reference's sequential one:
//   * u8 Sum wraps mod 256 (associative, exact);
//   * float Sum accumulates in double (the reference does too); the order of
//     the double additions differs, agreement is within 2^-20 relative
//     (SPEC.md:388), ~2^-40 in practice;
//   * Max / Min keep "a < b ? b : a": values that compare equal but differ in
//     bits (+0 / -0) are resolved to the earliest element in (z, y, x) order, so
//     each partial carries the linear index of its value; NaN is never adopted
//     (it only survives as a user identity), exactly as in the reference.
#include <cuda_runtime.h>

#include "fk_launch.hpp"
#include "fk_reduce.hpp"
#include "fk_stages.cuh"

namespace fk {

namespace {

constexpr int kRE = 4;            // elements per tile
constexpr uint32_t kRBlock = 256;  // threads per CTA

struct Acc {          // one spec's partial
  uint64_t v[3];      // double bits (float Sum) or the value's lane bits
  uint64_t idx[3];    // Max / Min: 1 + linear index of v[l] (earliest wins ties); 0 = user identity,
                      // ~0 = default identity (ties with it have identical bits)
};

__device__ __forceinline__ double as_d(uint64_t b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ uint64_t d_bits(double d) { return (uint64_t)__double_as_longlong(d); }

// a < b in the lane kind (u8 / f32 / f64 bits)
__device__ __forceinline__ bool lane_less(uint32_t lk, uint64_t a, uint64_t b) {
  if (lk == FK_U8) return (a & 0xffu) < (b & 0xffu);
  if (lk == FK_F32) return __uint_as_float(uint32_t(a)) < __uint_as_float(uint32_t(b));
  return as_d(a) < as_d(b);
}

__device__ __forceinline__ bool lane_eq(uint32_t lk, uint64_t a, uint64_t b) {  // as numbers: +0 == -0, NaN != NaN
  if (lk == FK_U8) return (a & 0xffu) == (b & 0xffu);
  if (lk == FK_F32) return __uint_as_float(uint32_t(a)) == __uint_as_float(uint32_t(b));
  return as_d(a) == as_d(b);
}

// fold x (at linear index i) into a, or combine partial x into a
__device__ __forceinline__ void combine(const RSpecDev& s, Acc& a, const Acc& x) {
  const uint32_t lk = s.lane_kind;
  if (s.combine == FK_REDUCE_SUM) {
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      if (l >= int(s.lanes)) break;
      if (s.dsum) a.v[l] = d_bits(as_d(a.v[l]) + as_d(x.v[l]));
      else a.v[l] = (a.v[l] + x.v[l]) & 0xffu;  // u8_add, scalar.hpp:146-157
    }
    return;
  }
  // Max: take x where a < x; Min: where x < a; equal values (+0 / -0) -> the
  // earlier index; unordered (NaN) -> keep a, as the reference's `a < b ? b : a`
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    if (l >= int(s.lanes)) break;
    const bool gt = s.combine == FK_REDUCE_MAX ? lane_less(lk, a.v[l], x.v[l]) : lane_less(lk, x.v[l], a.v[l]);
    if (gt || (lane_eq(lk, a.v[l], x.v[l]) && x.idx[l] < a.idx[l])) {
      a.v[l] = x.v[l];
      a.idx[l] = x.idx[l];
    }
  }
}

__device__ __forceinline__ void identity_acc(const RSpecDev& s, Acc& a) {
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    a.v[l] = s.dsum ? d_bits(0.0) : s.ident[l];
    a.idx[l] = ~uint64_t(0);
  }
}

template <class Lane, int L>
__device__ __forceinline__ void fold_value(const RSpecDev& s, Acc& a, const Lane (&v)[L], uint64_t i) {
  Acc x;
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const uint64_t b = l < L ? uint64_t(v[l]) : 0;
    if (s.dsum)
      x.v[l] = d_bits(s.lane_kind == FK_F32 ? double(__uint_as_float(uint32_t(b))) : as_d(b));
    else
      x.v[l] = s.lane_kind == FK_F32 ? (b & 0xffffffffu) : (s.lane_kind == FK_U8 ? (b & 0xffu) : b);
  }
#pragma unroll
  for (int l = 0; l < 3; ++l) x.idx[l] = i + 1;
  combine(s, a, x);
}

__device__ __forceinline__ Acc shfl_down(const Acc& a, int d) {
  Acc r;
#pragma unroll
  for (int l = 0; l < 3; ++l) r.v[l] = __shfl_down_sync(0xffffffffu, a.v[l], d);
#pragma unroll
  for (int l = 0; l < 3; ++l) r.idx[l] = __shfl_down_sync(0xffffffffu, a.idx[l], d);
  return r;
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
  const uint64_t tiles_plane = uint64_t(P.tiles), total = tiles_plane * P.batch;
  const uint64_t stride = uint64_t(gridDim.x) * kRBlock;
  for (uint64_t t = uint64_t(blockIdx.x) * kRBlock + threadIdx.x; t < total; t += stride) {
    const uint32_t z = uint32_t(t / tiles_plane);
    const uint32_t tt = uint32_t(t - uint64_t(z) * tiles_plane);
    const uint32_t y = dev::fastdiv(tt, P.tpr);
    const uint32_t x = (tt - y * P.tiles_per_row) * kRE;
    const int n = (P.width - x) < uint32_t(kRE) ? int(P.width - x) : kRE;
    const DSample s = P.reads[z];
    Lane v[kRE][L];
    dev::read_raw(P, s, x, y, n, v, nullptr, nullptr);
    if (!(s.flags & SF_DEFAULT)) dev::run_ops(P, s.post_off, s.post_len, z, v);
    const uint64_t i0 = (uint64_t(z) * P.height + y) * P.width + x;
#pragma unroll
    for (int k = 0; k < kMaxReduceSpecs; ++k) {
      if (k >= int(S.n)) break;
      Lane w[kRE][L];
#pragma unroll
      for (int e = 0; e < kRE; ++e)
#pragma unroll
        for (int l = 0; l < L; ++l) w[e][l] = v[e][l];
      if (S.s[k].op != kNoOp) dev::run_ops(P, S.s[k].op, 1, z, w);
#pragma unroll
      for (int e = 0; e < kRE; ++e)
        if (e < n) fold_value<Lane, L>(S.s[k], acc[k], w[e], i0 + e);
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

// one thread per spec: CTA partials in order, then identity and finish_accum (dpp.cpp:138-152)
__global__ void fk_reduce_final(const __grid_constant__ RSpecsDev S, const Acc* partials, uint32_t nparts,
                                uint64_t* out /* 3 lanes per spec, lane bits in the value kind */) {
  const int k = int(threadIdx.x);
  if (k >= int(S.n)) return;
  const RSpecDev& s = S.s[k];
  Acc a;
  identity_acc(s, a);
  for (uint32_t p = 0; p < nparts; ++p) combine(s, a, partials[uint64_t(p) * kMaxReduceSpecs + k]);
  if (!s.dsum) {  // the merge starts from the spec's identity (dpp.cpp:232-237): it is the left-most operand
    Acc r;
    for (int l = 0; l < 3; ++l) {
      r.v[l] = s.user_ident[l];
      r.idx[l] = 0;
    }
    combine(s, r, a);
    for (int l = 0; l < 3; ++l) out[3 * k + l] = r.v[l];
  } else {
    for (int l = 0; l < 3; ++l) {
      const double total = as_d(s.user_ident[l]) + as_d(a.v[l]);  // identity as double + the sum
      out[3 * k + l] = s.lane_kind == FK_F32 ? uint64_t(__float_as_uint(float(total))) : d_bits(total);
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
  fk_reduce_final<<<1, 32, 0, st>>>(S, parts, nblocks, out);
  return cudaGetLastError();
}

size_t reduce_scratch_bytes(uint32_t nblocks) { return size_t(nblocks) * kMaxReduceSpecs * sizeof(Acc); }
int reduce_tile_elems() { return kRE; }

}  // namespace fk
