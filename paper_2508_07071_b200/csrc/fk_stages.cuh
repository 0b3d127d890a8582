// fk_stages.cuh — the three stages of the TransformDPP body (PAPER.md:393-402,
// dpp.cpp:14-32) over a register tile: read (sample_block, ops.cpp:327-381),
// compute (compute_exec_block, ops.cpp:214-235), write (write_exec_block,
// ops.cpp:396-448). Used by the interpreted-chain kernel (fk_generic.cu).
#pragma once

#include "fk_device.cuh"

namespace fk {
namespace dev {

// ------------------------------------------------------------------ compute --

template <uint32_t LK, int NL, uint32_t FN, class Lane, int L, int E>
__device__ __forceinline__ void arith(Lane (&v)[E][L], const uint64_t (&c)[3], uint32_t reps) {
  if constexpr (fits_lanes<LK, NL, Lane, L>()) {
    if constexpr (LK == FK_U8) {  // arith_block_repeat, ops.cpp:114-120 (u8 wraps)
      uint32_t a[E][NL], cc[NL];
#pragma unroll
      for (int l = 0; l < NL; ++l) cc[l] = uint32_t(c[l]) & 0xffu;
#pragma unroll
      for (int e = 0; e < E; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l) a[e][l] = uint32_t(v[e][l]);
#pragma unroll 1
      for (uint32_t r = 0; r < reps; ++r)
#pragma unroll
        for (int e = 0; e < E; ++e)
#pragma unroll
          for (int l = 0; l < NL; ++l) a[e][l] = u8_op<FN>(a[e][l], cc[l]);
#pragma unroll
      for (int e = 0; e < E; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l) v[e][l] = Lane(a[e][l] & 0xffu);
    } else if constexpr (LK == FK_F32) {  // ops.cpp:121-126
      float a[E][NL], cc[NL];
#pragma unroll
      for (int l = 0; l < NL; ++l) cc[l] = as_f32(c[l]);
#pragma unroll
      for (int e = 0; e < E; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l) a[e][l] = as_f32(v[e][l]);
#pragma unroll 1
      for (uint32_t r = 0; r < reps; ++r)
#pragma unroll
        for (int e = 0; e < E; ++e)
#pragma unroll
          for (int l = 0; l < NL; ++l) a[e][l] = f32_op<FN>(a[e][l], cc[l]);
#pragma unroll
      for (int e = 0; e < E; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l) v[e][l] = Lane(bits(a[e][l]));
    } else {  // ops.cpp:127-132
      double a[E][NL], cc[NL];
#pragma unroll
      for (int l = 0; l < NL; ++l) cc[l] = as_f64(c[l]);
#pragma unroll
      for (int e = 0; e < E; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l) a[e][l] = as_f64(uint64_t(v[e][l]));
#pragma unroll 1
      for (uint32_t r = 0; r < reps; ++r)
#pragma unroll
        for (int e = 0; e < E; ++e)
#pragma unroll
          for (int l = 0; l < NL; ++l) a[e][l] = f64_op<FN>(a[e][l], cc[l]);
#pragma unroll
      for (int e = 0; e < E; ++e)
#pragma unroll
        for (int l = 0; l < NL; ++l) v[e][l] = Lane(bits(a[e][l]));
    }
  }
}

template <uint32_t LK, int NL, class Lane, int L, int E>
__device__ __forceinline__ void arith_fn(uint32_t fn, Lane (&v)[E][L], const uint64_t (&c)[3], uint32_t reps) {
  switch (fn) {
    case AF_MUL: arith<LK, NL, AF_MUL>(v, c, reps); break;
    case AF_ADD: arith<LK, NL, AF_ADD>(v, c, reps); break;
    case AF_SUB: arith<LK, NL, AF_SUB>(v, c, reps); break;
    default: arith<LK, NL, AF_DIV>(v, c, reps); break;
  }
}

// cast_element, scalar.cpp:35-42: lane-wise through double, narrowing at the destination.
template <uint32_t LI, uint32_t LO, int NL, class Lane, int L, int E>
__device__ __forceinline__ void cast(Lane (&v)[E][L]) {
  if constexpr (fits_lanes<LI, NL, Lane, L>() && fits_lanes<LO, NL, Lane, L>()) {
#pragma unroll
    for (int e = 0; e < E; ++e)
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        if constexpr (LI == FK_F32 && LO == FK_U8) {
          v[e][l] = Lane(round_clamp_u8(as_f32(v[e][l])));           // exact: rint((double)f) == rintf(f)
        } else if constexpr (LI == FK_U8 && LO == FK_F32) {
          v[e][l] = Lane(bits((float)(uint32_t(v[e][l]) & 0xffu)));   // exact widening
        } else {
          v[e][l] = lane_from_double<LO, Lane>(lane_to_double<LI>(v[e][l]));
        }
      }
  }
}

template <uint32_t LI, class Lane, int L, int E>
__device__ __forceinline__ void cast_from(uint32_t lo, int nl, Lane (&v)[E][L]) {
  if (nl == 3) {
    if (lo == FK_U8) cast<LI, FK_U8, 3>(v);
    else if (lo == FK_F32) cast<LI, FK_F32, 3>(v);
    else cast<LI, FK_F64, 3>(v);
  } else {
    if (lo == FK_U8) cast<LI, FK_U8, 1>(v);
    else if (lo == FK_F32) cast<LI, FK_F32, 1>(v);
    else cast<LI, FK_F64, 1>(v);
  }
}

// to_gray_block, ops.cpp:178-185: ((0.299 r + 0.587 g) + 0.114 b) in double, one f32 rounding.
template <uint32_t LI, class Lane, int L, int E>
__device__ __forceinline__ void gray(Lane (&v)[E][L]) {
  if constexpr (L == 3 && fits_lanes<LI, 3, Lane, L>()) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double g = __dadd_rn(__dadd_rn(__dmul_rn(0.299, lane_to_double<LI>(v[e][0])),
                                           __dmul_rn(0.587, lane_to_double<LI>(v[e][1]))),
                                 __dmul_rn(0.114, lane_to_double<LI>(v[e][2])));
      v[e][0] = Lane(bits(__double2float_rn(g)));
    }
  }
}

template <class Lane, int L, int E>
__device__ __forceinline__ void apply_op(const DOp& op, uint32_t z, Lane (&v)[E][L]) {
  switch (op.cls) {
    case OC_ARITH: {
      uint64_t c[3] = {op.c[0], op.c[1], op.c[2]};
      if (op.per_z) {  // BatchArith: the constant row of plane z
        const uint64_t* row = reinterpret_cast<const uint64_t*>(op.per_z) + 3ull * (z < op.per_z_n ? z : op.per_z_n - 1);
        c[0] = __ldg(row); c[1] = __ldg(row + 1); c[2] = __ldg(row + 2);
      }
      const uint32_t sel = op.lk_in * 2 + (op.nl == 3 ? 1 : 0);
      switch (sel) {
        case 0: arith_fn<FK_U8, 1>(op.fn, v, c, op.repeat); break;
        case 1: arith_fn<FK_U8, 3>(op.fn, v, c, op.repeat); break;
        case 2: arith_fn<FK_F32, 1>(op.fn, v, c, op.repeat); break;
        case 3: arith_fn<FK_F32, 3>(op.fn, v, c, op.repeat); break;
        case 4: arith_fn<FK_F64, 1>(op.fn, v, c, op.repeat); break;
        default: arith_fn<FK_F64, 3>(op.fn, v, c, op.repeat); break;
      }
      break;
    }
    case OC_SWAP:  // swap_rb_block, ops.cpp:161-176 (parity of the repeat count)
      if constexpr (L == 3) {
        if (op.repeat & 1u) {
#pragma unroll
          for (int e = 0; e < E; ++e) { const Lane t = v[e][0]; v[e][0] = v[e][2]; v[e][2] = t; }
        }
      }
      break;
    case OC_CAST:
      if (op.lk_in == FK_U8) cast_from<FK_U8>(op.lk_out, op.nl, v);
      else if (op.lk_in == FK_F32) cast_from<FK_F32>(op.lk_out, op.nl, v);
      else cast_from<FK_F64>(op.lk_out, op.nl, v);
      break;
    case OC_GRAY:
      if (op.lk_in == FK_U8) gray<FK_U8>(v);
      else if (op.lk_in == FK_F32) gray<FK_F32>(v);
      else gray<FK_F64>(v);
      break;
    default: break;
  }
}

// --------------------------------------------------------------------- read --

// One element of kind K at p into state slot e.
template <uint32_t K, class Lane, int L, int E>
__device__ __forceinline__ void load_elem(const uint8_t* p, bool al, Lane (&v)[E][L], int e) {
  using T = KindT<K>;
#pragma unroll
  for (int l = 0; l < T::nl; ++l) v[e][l] = load_lane<T::lk, Lane>(p + l * T::lb, al);
}

template <uint32_t K, class Lane, int L, int E>
__device__ __forceinline__ void read_kind(const DSample& s, uint32_t x, uint32_t y, int n, Lane (&v)[E][L]) {
  if constexpr (fits<K, Lane, L>()) {
    using T = KindT<K>;
    const bool al = (s.flags & SF_LANE_ALIGNED) != 0;
    const uint8_t* base = reinterpret_cast<const uint8_t*>(s.src);
    if (s.mode == RD_DIRECT) {  // identity / crop: source(x0 + x, y0 + y)
      const uint8_t* p = base + uint64_t(s.y0 + y) * s.pitch + uint64_t(s.x0 + x) * T::bpe;
      constexpr int NB = E * T::bpe;
      if constexpr (NB % 4 == 0) {
        if (n == E && (reinterpret_cast<uintptr_t>(p) & 3) == 0) {
          uint32_t w[NB / 4];
          load_words<NB / 4>(p, w);
          decode<K, Lane, L, E>(w, v);
          return;
        }
      }
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (e < n) load_elem<K>(p + e * T::bpe, al, v, e);
    } else if (s.mode == RD_NEAREST) {  // nearest_sample, ops.cpp:301-310
      const double cy = __ddiv_rn(__dmul_rn(__dadd_rn((double)y, 0.5), (double)s.rect_h), (double)s.out_h);
      const long long sy = s.y0 + clamp_ll((long long)floor(cy), 0, (long long)s.rect_h - 1);
      const uint8_t* row = base + uint64_t(sy) * s.pitch;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (e < n) {
          const double cx = __ddiv_rn(__dmul_rn(__dadd_rn((double)(x + e), 0.5), (double)s.rect_w), (double)s.out_w);
          const long long sx = s.x0 + clamp_ll((long long)floor(cx), 0, (long long)s.rect_w - 1);
          load_elem<K>(row + uint64_t(sx) * T::bpe, al, v, e);
        }
      }
    } else {  // bilinear_sample, ops.cpp:259-299
      const double cy = center_coord(y, s.rect_h, s.out_h);
      const double fiy = floor(cy);
      const long long iy = (long long)fiy;
      const double fy = __dsub_rn(cy, fiy);
      const long long maxy = (long long)s.rect_h - 1, maxx = (long long)s.rect_w - 1;
      const uint8_t* r0 = base + uint64_t(s.y0 + clamp_ll(iy, 0, maxy)) * s.pitch;
      const uint8_t* r1 = base + uint64_t(s.y0 + clamp_ll(iy + 1, 0, maxy)) * s.pitch;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (e < n) {
          const double cx = center_coord(x + e, s.rect_w, s.out_w);
          const double fix = floor(cx);
          const long long ix = (long long)fix;
          const double fx = __dsub_rn(cx, fix);
          const uint64_t o0 = uint64_t(s.x0 + clamp_ll(ix, 0, maxx)) * T::bpe;
          const uint64_t o1 = uint64_t(s.x0 + clamp_ll(ix + 1, 0, maxx)) * T::bpe;
#pragma unroll
          for (int l = 0; l < T::nl; ++l) {
            const int lo = l * T::lb;
            const double a = lane_to_double<T::lk>(load_lane<T::lk, Lane>(r0 + o0 + lo, al));
            const double b = lane_to_double<T::lk>(load_lane<T::lk, Lane>(r0 + o1 + lo, al));
            const double c = lane_to_double<T::lk>(load_lane<T::lk, Lane>(r1 + o0 + lo, al));
            const double d = lane_to_double<T::lk>(load_lane<T::lk, Lane>(r1 + o1 + lo, al));
            const double top = lerp(a, b, fx);
            const double bot = lerp(c, d, fx);
            v[e][l] = lane_from_double<T::lk, Lane>(lerp(top, bot, fy));
          }
        }
      }
    }
  }
}

// read_exec_block, ops.cpp:361-381, plus the folded unaries (sample_block :343)
template <class Lane, int L, int E>
__device__ __forceinline__ void read_tile(const DPlan& P, const DSample& s, uint32_t z, uint32_t x, uint32_t y,
                                          int n, Lane (&v)[E][L]) {
  if (s.flags & SF_DEFAULT) {  // z >= active_count: default value, no post ops
#pragma unroll
    for (int e = 0; e < E; ++e)
#pragma unroll
      for (int l = 0; l < L; ++l) v[e][l] = Lane(P.def[l]);
    return;
  }
  switch (s.kind) {
    case FK_U8: read_kind<FK_U8>(s, x, y, n, v); break;
    case FK_F32: read_kind<FK_F32>(s, x, y, n, v); break;
    case FK_F64: read_kind<FK_F64>(s, x, y, n, v); break;
    case FK_U8X3: read_kind<FK_U8X3>(s, x, y, n, v); break;
    case FK_F32X3: read_kind<FK_F32X3>(s, x, y, n, v); break;
    default: read_kind<FK_F64X3>(s, x, y, n, v); break;
  }
  for (uint32_t i = 0; i < s.post_len; ++i) {
    const DOp op = P.post[s.post_off + i];
    apply_op(op, z, v);
  }
}

// -------------------------------------------------------------------- write --

template <uint32_t K, class Lane, int L, int E>
__device__ __forceinline__ void write_kind(const DWrite& w, uint32_t x, uint32_t y, int n, const Lane (&v)[E][L]) {
  if constexpr (fits<K, Lane, L>()) {
    using T = KindT<K>;
    const bool al = (w.flags & WF_LANE_ALIGNED) != 0;
    const bool st = (w.flags & WF_STREAM) != 0;
    uint8_t* p = reinterpret_cast<uint8_t*>(w.dst[0]) + uint64_t(y) * w.pitch[0] + uint64_t(x) * T::bpe;
    constexpr int NB = E * T::bpe;
    if constexpr (NB % 4 == 0) {
      if (n == E && (reinterpret_cast<uintptr_t>(p) & 3) == 0) {
        uint32_t wd[NB / 4];
        encode<K, Lane, L, E>(v, wd);
        store_words<NB / 4>(p, wd, st);
        return;
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (e < n)
#pragma unroll
        for (int l = 0; l < T::nl; ++l) store_lane<T::lk, Lane>(p + e * T::bpe + l * T::lb, v[e][l], al);
  }
}

// split_block, ops.cpp:402-424: lane l of the packed value lands in dest[l]
template <uint32_t LK, class Lane, int L, int E>
__device__ __forceinline__ void write_split(const DWrite& w, uint32_t x, uint32_t y, int n, const Lane (&v)[E][L]) {
  if constexpr (fits_lanes<LK, 3, Lane, L>()) {
    constexpr int LB = LK == FK_U8 ? 1 : (LK == FK_F32 ? 4 : 8);
    constexpr uint32_t K = LK;  // scalar kind of each destination plane
    const bool al = (w.flags & WF_LANE_ALIGNED) != 0;
    const bool st = (w.flags & WF_STREAM) != 0;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      uint8_t* p = reinterpret_cast<uint8_t*>(w.dst[l]) + uint64_t(y) * w.pitch[l] + uint64_t(x) * LB;
      constexpr int NB = E * LB;
      if constexpr (NB % 4 == 0) {
        if (n == E && (reinterpret_cast<uintptr_t>(p) & 3) == 0) {
          Lane s[E][L];
#pragma unroll
          for (int e = 0; e < E; ++e) s[e][0] = v[e][l];
          uint32_t wd[NB / 4];
          encode<K, Lane, L, E>(s, wd);
          store_words<NB / 4>(p, wd, st);
          continue;
        }
      }
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (e < n) store_lane<LK, Lane>(p + e * LB, v[e][l], al);
    }
  }
}

template <class Lane, int L, int E>
__device__ __forceinline__ void write_tile(const DPlan& P, const DWrite& w, uint32_t x, uint32_t y, int n,
                                           const Lane (&v)[E][L]) {
  if (!(w.flags & WF_ACTIVE)) return;  // BatchWrite z >= active_count: skip (ops.cpp:437-445)
  if (P.write_mode == WR_DIRECT) {
    switch (P.write_kind) {
      case FK_U8: write_kind<FK_U8>(w, x, y, n, v); break;
      case FK_F32: write_kind<FK_F32>(w, x, y, n, v); break;
      case FK_F64: write_kind<FK_F64>(w, x, y, n, v); break;
      case FK_U8X3: write_kind<FK_U8X3>(w, x, y, n, v); break;
      case FK_F32X3: write_kind<FK_F32X3>(w, x, y, n, v); break;
      default: write_kind<FK_F64X3>(w, x, y, n, v); break;
    }
  } else {
    switch (P.write_kind) {
      case FK_U8X3: write_split<FK_U8>(w, x, y, n, v); break;
      case FK_F32X3: write_split<FK_F32>(w, x, y, n, v); break;
      default: write_split<FK_F64>(w, x, y, n, v); break;
    }
  }
}

}  // namespace dev
}  // namespace fk
