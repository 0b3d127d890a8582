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

// The two u8x3 taps of one source row (3 bytes at o0, 3 bytes at o1, o1 - o0 in
// {0, 3}) from aligned 32-bit words: the bytes [o0, o1 + 3) lie in at most three
// words from (row + o0) & ~3. A word that holds none of those bytes is not read
// (its load is redirected to the first word), so the gather never touches memory
// past the plane, and it has no branches.
__device__ __forceinline__ void load_u8x3_taps(const uint8_t* row, uint32_t o0, uint32_t o1, uint32_t& a,
                                               uint32_t& b) {
  const uintptr_t p = reinterpret_cast<uintptr_t>(row + o0);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(p & ~uintptr_t(3));
  const uint32_t r = uint32_t(p & 3);
  const uint32_t d = o1 - o0;
  const uint32_t last = r + d + 2;  // relative index of the last byte needed
  const uint32_t w0 = __ldg(w);
  const uint32_t w1 = __ldg(w + (last >= 4 ? 1 : 0));
  const uint32_t w2 = __ldg(w + (last >= 8 ? 2 : 0));
  const uint32_t sa = 8 * r, sb = 8 * (r + d);
  a = __funnelshift_r(w0, w1, sa) & 0xffffffu;
  b = (sb < 32 ? __funnelshift_r(w0, w1, sb) : __funnelshift_r(w1, w2, sb - 32)) & 0xffffffu;
}

// bilinear_sample, ops.cpp:259-299, for one output pixel whose taps are at byte
// offsets o0/o1 of rows r0/r1. u8 lanes take an exact shortcut for int->double
// (2^52 + v is a double whose low word is v) and for nearbyint (adding 1.5*2^52
// rounds to an integer ties-to-even in the low word); the lerp arithmetic is the
// reference's, op for op, in double.
template <uint32_t K, class Lane, int L, int E>
__device__ __forceinline__ void bilinear_px(const uint8_t* r0, const uint8_t* r1, uint32_t o0, uint32_t o1,
                                            double fx, double fy, bool al, Lane (&v)[E][L], int e) {
  using T = KindT<K>;
  if constexpr (T::lk == FK_U8) {
    uint32_t ta[T::nl], tb[T::nl], tc[T::nl], td[T::nl];
    if constexpr (T::nl == 3) {
      uint32_t a, b, c, d;
      load_u8x3_taps(r0, o0, o1, a, b);
      load_u8x3_taps(r1, o0, o1, c, d);
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        ta[l] = (a >> (8 * l)) & 0xffu;
        tb[l] = (b >> (8 * l)) & 0xffu;
        tc[l] = (c >> (8 * l)) & 0xffu;
        td[l] = (d >> (8 * l)) & 0xffu;
      }
    } else {
      ta[0] = __ldg(r0 + o0);
      tb[0] = __ldg(r0 + o1);
      tc[0] = __ldg(r1 + o0);
      td[0] = __ldg(r1 + o1);
    }
    constexpr double kTwo52 = 4503599627370496.0;        // 2^52
    constexpr double kRound = 6755399441055744.0;        // 1.5 * 2^52
#pragma unroll
    for (int l = 0; l < T::nl; ++l) {
      const double A = __hiloint2double(0x43300000, int(ta[l]));   // 2^52 + a, exact
      const double B = __hiloint2double(0x43300000, int(tb[l]));
      const double C = __hiloint2double(0x43300000, int(tc[l]));
      const double D = __hiloint2double(0x43300000, int(td[l]));
      const double a = __dsub_rn(A, kTwo52), c = __dsub_rn(C, kTwo52);         // exact
      const double top = __dadd_rn(a, __dmul_rn(__dsub_rn(B, A), fx));          // a + (b - a) * fx
      const double bot = __dadd_rn(c, __dmul_rn(__dsub_rn(D, C), fx));          // c + (d - c) * fx
      const double res = __dadd_rn(top, __dmul_rn(__dsub_rn(bot, top), fy));   // top + (bot - top) * fy
      // res is in [0, 255] (a lerp of values in [0, 255] with t in [0, 1) under RN), so
      // round_clamp_u8 reduces to nearbyint, i.e. the low word of res + 1.5 * 2^52.
      v[e][l] = Lane(uint32_t(__double2loint(__dadd_rn(res, kRound))));
    }
  } else {
#pragma unroll
    for (int l = 0; l < T::nl; ++l) {
      const int lo = l * T::lb;
      const double a = lane_to_double<T::lk>(load_lane<T::lk, Lane>(r0 + o0 + lo, al));
      const double b = lane_to_double<T::lk>(load_lane<T::lk, Lane>(r0 + o1 + lo, al));
      const double c = lane_to_double<T::lk>(load_lane<T::lk, Lane>(r1 + o0 + lo, al));
      const double d = lane_to_double<T::lk>(load_lane<T::lk, Lane>(r1 + o1 + lo, al));
      v[e][l] = lane_from_double<T::lk, Lane>(lerp(lerp(a, b, fx), lerp(c, d, fx), fy));
    }
  }
}

// Sampling coordinates of output column i (ops.cpp:259-270 / 301-306) for a table entry.
__device__ __forceinline__ XEnt x_entry(const DSample& s, uint32_t i, uint32_t bpe) {
  XEnt x;
  const long long maxx = (long long)s.rect_w - 1;
  if (s.mode == RD_BILINEAR) {
    const double cx = center_coord(i, s.rect_w, s.out_w);
    const double fl = floor(cx);
    const long long ix = (long long)fl;
    x.o0 = uint32_t((s.x0 + clamp_ll(ix, 0, maxx)) * bpe);
    x.o1 = uint32_t((s.x0 + clamp_ll(ix + 1, 0, maxx)) * bpe);
    x.f = __dsub_rn(cx, fl);
  } else {
    const double cx = __ddiv_rn(__dmul_rn(__dadd_rn((double)i, 0.5), (double)s.rect_w), (double)s.out_w);
    x.o0 = x.o1 = uint32_t((s.x0 + clamp_ll((long long)floor(cx), 0, maxx)) * bpe);
    x.f = 0.0;
  }
  return x;
}
__device__ __forceinline__ YEnt y_entry(const DSample& s, uint32_t j) {
  YEnt y;
  const long long maxy = (long long)s.rect_h - 1;
  if (s.mode == RD_BILINEAR) {
    const double cy = center_coord(j, s.rect_h, s.out_h);
    const double fl = floor(cy);
    const long long iy = (long long)fl;
    y.r0 = uint64_t(s.y0 + clamp_ll(iy, 0, maxy)) * s.pitch;
    y.r1 = uint64_t(s.y0 + clamp_ll(iy + 1, 0, maxy)) * s.pitch;
    y.f = __dsub_rn(cy, fl);
  } else {
    const double cy = __ddiv_rn(__dmul_rn(__dadd_rn((double)j, 0.5), (double)s.rect_h), (double)s.out_h);
    y.r0 = y.r1 = uint64_t(s.y0 + clamp_ll((long long)floor(cy), 0, maxy)) * s.pitch;
    y.f = 0.0;
  }
  return y;
}

__device__ __forceinline__ uint32_t kind_bpe(uint32_t k) {
  return k == FK_U8 ? 1u : k == FK_F32 ? 4u : k == FK_F64 ? 8u : k == FK_U8X3 ? 3u : k == FK_F32X3 ? 12u : 24u;
}

// Resample tables for this CTA's rows [y_first, y_first + rows) (block-cooperative).
// The column table is struct-of-arrays so a thread reads its E consecutive
// entries with 128-bit shared loads: conflict-free across the warp.
__device__ __forceinline__ void build_tables(const DSample& s, uint32_t width, uint32_t y_first, uint32_t rows,
                                             XTab& xt, YEnt* yt) {
  const uint32_t b = kind_bpe(s.kind);
  const uint32_t padded = (width + 7u) & ~7u;
  for (uint32_t i = threadIdx.x; i < padded; i += blockDim.x) {
    const XEnt e = x_entry(s, i < width ? i : width - 1, b);
    xt.o[i] = e.o0 | (e.o1 == e.o0 ? kEdge : 0u);
    xt.f[i] = e.f;
  }
  for (uint32_t j = threadIdx.x; j < rows; j += blockDim.x) yt[j] = y_entry(s, y_first + j);
}

template <int E>
__device__ __forceinline__ void load_xtab(const XTab& xt, uint32_t x, uint32_t (&o)[E], double (&f)[E]) {
  static_assert(E % 4 == 0, "tile width must be a multiple of 4");
#pragma unroll
  for (int i = 0; i < E / 4; ++i) {
    const uint4 q = *reinterpret_cast<const uint4*>(&xt.o[x + 4 * i]);
    o[4 * i] = q.x; o[4 * i + 1] = q.y; o[4 * i + 2] = q.z; o[4 * i + 3] = q.w;
  }
#pragma unroll
  for (int i = 0; i < E / 2; ++i) {
    const double2 d = *reinterpret_cast<const double2*>(&xt.f[x + 2 * i]);
    f[2 * i] = d.x; f[2 * i + 1] = d.y;
  }
}

template <uint32_t K, class Lane, int L, int E>
__device__ __forceinline__ void read_kind(const DSample& s, uint32_t x, uint32_t y, int n, Lane (&v)[E][L],
                                          const XTab* xt, const YEnt* yt) {
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
      return;
    }
    // resampling read: coordinates from the CTA tables when present, else computed here
    const YEnt ye = yt ? *yt : y_entry(s, y);
    const uint8_t* r0 = base + ye.r0;
    const uint8_t* r1 = base + ye.r1;
    uint32_t o[E];
    double f[E];
    if (xt) {
      load_xtab<E>(*xt, x, o, f);
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const XEnt xe = x_entry(s, x + (e < n ? e : 0), T::bpe);
        o[e] = xe.o0 | (xe.o1 == xe.o0 ? kEdge : 0u);
        f[e] = xe.f;
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e < n) {
        const uint32_t o0 = o[e] & ~kEdge, o1 = (o[e] & kEdge) ? o0 : o0 + T::bpe;
        if (s.mode == RD_NEAREST) load_elem<K>(r0 + o0, al, v, e);  // nearest_sample, ops.cpp:301-310
        else bilinear_px<K>(r0, r1, o0, o1, f[e], ye.f, al, v, e);
      }
    }
  }
}

// Program table access: inline in kernel-parameter space (constant bank) when the
// whole table fits, else HBM.
__device__ __forceinline__ DOp prog_op(const DPlan& P, uint32_t i) {
  return P.prog_inline ? P.prog[i] : P.table[i];
}

template <class Lane, int L, int E>
__device__ __forceinline__ void run_ops(const DPlan& P, uint32_t first, uint32_t count, uint32_t z, Lane (&v)[E][L]) {
  for (uint32_t i = 0; i < count; ++i) {
    const DOp op = prog_op(P, first + i);
    apply_op(op, z, v);
  }
}

// read_exec_block, ops.cpp:361-381, without the folded unaries (sample_block :343
// applies them; the caller runs them or their LUT).
template <class Lane, int L, int E>
__device__ __forceinline__ void read_raw(const DPlan& P, const DSample& s, uint32_t x, uint32_t y, int n,
                                         Lane (&v)[E][L], const XTab* xt, const YEnt* yt) {
  if (s.flags & SF_DEFAULT) {  // z >= active_count: default value, no post ops
#pragma unroll
    for (int e = 0; e < E; ++e)
#pragma unroll
      for (int l = 0; l < L; ++l) v[e][l] = Lane(P.def[l]);
    return;
  }
  switch (s.kind) {
    case FK_U8: read_kind<FK_U8>(s, x, y, n, v, xt, yt); break;
    case FK_F32: read_kind<FK_F32>(s, x, y, n, v, xt, yt); break;
    case FK_F64: read_kind<FK_F64>(s, x, y, n, v, xt, yt); break;
    case FK_U8X3: read_kind<FK_U8X3>(s, x, y, n, v, xt, yt); break;
    case FK_F32X3: read_kind<FK_F32X3>(s, x, y, n, v, xt, yt); break;
    default: read_kind<FK_F64X3>(s, x, y, n, v, xt, yt); break;
  }
}

// The folded unaries followed by the compute program, tabulated over the 256
// values a u8 lane can take (every op involved is lane-wise, so output lane l is
// g_l(input lane perm(l)) and g_l(t) is the program run on the lane vector (t,t,t)).
// Each entry is computed by the same device ops as the direct path: bit-exact by
// construction.
template <class Lane, int L, int E>
__device__ __forceinline__ void build_lut(const DPlan& P, const DSample& s, uint32_t z, Lane (*lut)[256]) {
  for (uint32_t t = threadIdx.x; t < 256; t += blockDim.x) {
    Lane v[E][L];
#pragma unroll
    for (int e = 0; e < E; ++e)
#pragma unroll
      for (int l = 0; l < L; ++l) v[e][l] = Lane(t);
    run_ops(P, s.post_off, s.post_len, z, v);
    run_ops(P, P.op_base, P.n_ops, z, v);
#pragma unroll
    for (int l = 0; l < L; ++l) lut[l][t] = v[0][l];
  }
}

template <class Lane, int L, int E>
__device__ __forceinline__ void apply_lut(const Lane (*lut)[256], bool swap, Lane (&v)[E][L]) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if constexpr (L == 3) {
      const uint32_t i0 = uint32_t(v[e][0]) & 0xffu, i1 = uint32_t(v[e][1]) & 0xffu, i2 = uint32_t(v[e][2]) & 0xffu;
      v[e][0] = lut[0][swap ? i2 : i0];
      v[e][1] = lut[1][i1];
      v[e][2] = lut[2][swap ? i0 : i2];
    } else {
      v[e][0] = lut[0][uint32_t(v[e][0]) & 0xffu];
    }
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
