// fk_resample_sep.cuh — column-streaming kernel for batched u8 crop/resize
// pipelines (configs[1], [3], [4]; the cvGS / FastNPP preprocessing family,
// PAPER.md:695-703).
//
// The reference's bilinear sample (ops.cpp:259-299) is, per lane,
//     top = lerp(a, b, fx)   taps of source row sy0
//     bot = lerp(c, d, fx)   taps of source row sy1
//     res = lerp(top, bot, fy)
//     u8  = round_clamp_u8(res)            (nearbyint, ties to even)
// in double. `top`/`bot` depend only on (source row, output column), so each
// thread owns a PAIR of adjacent output columns and walks down a band of output
// rows, holding the horizontal lerps of the two current source rows in
// registers: a source row's H-lerp is computed once however many output rows use
// it, and the V-lerp is the only per-pixel work.
//
// Exact-result filter. The lerps run in FP32, two columns per instruction
// (FFMA2/FADD2 on sm_100), and the double computation is only redone where FP32
// could round differently:
//   |v_f32 - res_f64| <= 6.9e-5 < E = 2^-13 for every tap/coordinate
// (fx, fy rounded to f32: 255*2^-25 each; three f32 roundings at magnitude < 256:
// 2^-17 each, the difference bot - top carries both H-lerp errors), so when
// |v_f32 - rint(v_f32)| <= 0.5 - E no value within E of v_f32 rounds differently
// and rint(v_f32) == nearbyint(res_f64). Otherwise (a lane within E of a
// half-integer, ~2.4e-4 of lanes on random data) the pixel pair is recomputed
// with the reference's double arithmetic op for op (exact_pair). When fx and fy
// are multiples of 2^-8 every FP32 and FP64 operation above is exact, so both
// produce the same value — including exact ties — and the check is skipped
// (RowEnt::thr[1] / the column pair's `exact` flag): integer scale factors such
// as 448 -> 224 (fx = fy = 0.5) never take the slow path.
//
//   CTA = a strip of up to 2 * 256 consecutive output columns x a band of rows
//   of one plane z (blockIdx.z, horizontal fusion). Per CTA and plane: the rows'
//   coordinates and visit list in shared memory; the chain's constants in
//   registers (AFFINE: Cast u8->f32 + a registered f32 chain, evaluated with
//   packed FP32 ops) or its 256-entry table (LUT: any lane-wise chain).
#pragma once
#include <cuda_runtime.h>

#include <cstdio>
#include <type_traits>

#include "fk_launch.hpp"
#include "fk_sig.cuh"
#include "fk_stages.cuh"

namespace fk {

namespace {

#ifndef FK_SEP_MINB
#define FK_SEP_MINB 20  // resident one-warp CTAs per SM (96 registers; ~11 KB shared each)
#endif
constexpr uint32_t kBandMax = 256;     // output rows per CTA (host picks <= this)
constexpr float kNearTol = 1.0f / 8192.0f;  // E = 2^-13 (bound 6.9e-5, see header)

// ---------------------------------------------------------- packed FP32 --
// Two f32 values in one 64-bit register pair (lo = column x, hi = column x + 1).
namespace f2 {
__device__ __forceinline__ uint64_t pack(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ uint64_t bc(float v) { return pack(v, v); }
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
__device__ __forceinline__ uint64_t mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
}  // namespace f2

// The registered AFFINE chain (fk_sig.cuh) on a column pair: same IEEE ops in
// the same order as sig_apply, two values per instruction.
template <uint32_t SIG, int K>
__device__ __forceinline__ uint64_t sig_op2(uint64_t v, float c, float r) {
  constexpr uint32_t fn = sig_fn(SIG, K);
  // a chain product as two scalar mul.rn: ptxas contracts a packed mul + add into FFMA2 (fk_pack2.cuh)
  if constexpr (fn == AF_MUL) return f2::pack(__fmul_rn(f2::lo(v), c), __fmul_rn(f2::hi(v), c));
  else if constexpr (fn == AF_ADD) return f2::add(v, f2::bc(c));
  else if constexpr (fn == AF_SUB) return f2::sub(v, f2::bc(c));
  else if constexpr (sig_fast(SIG, K)) {  // div_by_recip: q = x r; e = fma(-q, d, x); q + e r
    const uint64_t q = f2::mul(v, f2::bc(r));
    const uint64_t e = f2::fma(q, f2::bc(-c), v);
    return f2::fma(e, f2::bc(r), q);
  } else {
    return f2::pack(__fdiv_rn(f2::lo(v), c), __fdiv_rn(f2::hi(v), c));
  }
}
template <uint32_t SIG, class KS>
__device__ __forceinline__ uint64_t sig_apply2(uint64_t v, const KS& ks, int l) {
  if constexpr (sig_n(SIG) > 0) v = sig_op2<SIG, 0>(v, ks.c(l, 0), ks.r(l, 0));
  if constexpr (sig_n(SIG) > 1) v = sig_op2<SIG, 1>(v, ks.c(l, 1), ks.r(l, 1));
  if constexpr (sig_n(SIG) > 2) v = sig_op2<SIG, 2>(v, ks.c(l, 2), ks.r(l, 2));
  if constexpr (sig_n(SIG) > 3) v = sig_op2<SIG, 3>(v, ks.c(l, 3), ks.r(l, 3));
  return v;
}

// ------------------------------------------------------------ row tables --
// The band's output rows: per row {fy_f32, the row's filter threshold} (0.5,
// i.e. never flagged, when fy is a multiple of 2^-8; a pair's threshold is the
// min of its row's and its columns') and the source rows of the top / bottom
// taps relative to the plane's y0 (s0 | s1 << 16; rect_h < 2^16, host-checked).
struct BandRows {
  float2 q[kBandMax];
  uint32_t s[kBandMax];
};

// fx (or fy) is a multiple of 2^-8: the FP32 lerps are exact (see header)
__device__ __forceinline__ bool coord_exact8(double f) {
  const double s = __dmul_rn(f, 256.0);
  return s == floor(s);
}

// 64-bit address base + row * pitch: one IMAD.WIDE.U32
__device__ __forceinline__ uint64_t at_row(uint64_t base, uint32_t row, uint32_t pitch) {
  uint64_t a;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a) : "r"(row), "r"(pitch), "l"(base));
  return a;
}

// One column's two taps in a source row. Word path (u8x3 rows 4-byte aligned):
// tap t's 3 bytes start at byte (o_t & 3) of the word at (o_t & ~3); the next
// word is loaded only if the tap reaches into it (so nothing past the plane is
// touched) and a funnel shift aligns the tap. Byte path: the bytes themselves.
// `issue` starts the loads of source row `row`, `taps` extracts them, so the next row's loads are in flight while
// this row is lerped.
template <int NL, bool ALIGNED>
struct ColTap {
  uint64_t pa, pb;       // source origin + word (or byte) offset of tap a / tap b
  uint32_t sa, sb;       // funnel-shift amounts (bits)
  bool na, nb;           // tap a / b spans two words
  uint32_t wa0, wa1, wb0, wb1;
  uint64_t pa_row, pb_row;  // byte path only
  __device__ __forceinline__ void init(uint64_t src, uint32_t o0, uint32_t o1) {
    if constexpr (NL == 3 && ALIGNED) {
      pa = src + (o0 & ~3u);
      pb = src + (o1 & ~3u);
      sa = 8 * (o0 & 3u);
      sb = 8 * (o1 & 3u);
      na = (o0 & 3u) >= 2;
      nb = (o1 & 3u) >= 2;
    } else {
      pa = src + o0;
      pb = src + o1;
    }
  }
  __device__ __forceinline__ void issue(uint32_t row, uint32_t pitch) {
    if constexpr (NL == 3 && ALIGNED) {
      const uint32_t* a = reinterpret_cast<const uint32_t*>(at_row(pa, row, pitch));
      const uint32_t* b = reinterpret_cast<const uint32_t*>(at_row(pb, row, pitch));
      wa0 = __ldg(a);
      wb0 = __ldg(b);
      wa1 = na ? __ldg(a + 1) : 0u;
      wb1 = nb ? __ldg(b + 1) : 0u;
    } else if constexpr (NL == 3) {
      pa_row = at_row(pa, row, pitch);  // the byte path loads at use
      pb_row = at_row(pb, row, pitch);
    } else {
      wa0 = __ldg(reinterpret_cast<const uint8_t*>(at_row(pa, row, pitch)));
      wb0 = __ldg(reinterpret_cast<const uint8_t*>(at_row(pb, row, pitch)));
    }
  }
  __device__ __forceinline__ void taps(uint32_t& a, uint32_t& b) const {
    if constexpr (NL == 3 && ALIGNED) {
      a = __funnelshift_r(wa0, wa1, sa);
      b = __funnelshift_r(wb0, wb1, sb);
    } else if constexpr (NL == 3) {
      const uint8_t* p = reinterpret_cast<const uint8_t*>(pa_row);
      const uint8_t* q = reinterpret_cast<const uint8_t*>(pb_row);
      a = uint32_t(__ldg(p)) | uint32_t(__ldg(p + 1)) << 8 | uint32_t(__ldg(p + 2)) << 16;
      b = uint32_t(__ldg(q)) | uint32_t(__ldg(q + 1)) << 8 | uint32_t(__ldg(q + 2)) << 16;
    } else {
      a = wa0;
      b = wb0;
    }
  }
};

// byte l of v as the float 2^23 + v (bit pattern 0x4B0000vv): one PRMT with an
// immediate selector; `bias` holds 0x4B000000 in a register (opaque to the
// compiler, which would otherwise materialise a selector register per PRMT,
// so it is read from the constant bank)
__constant__ uint32_t kBiasWord = 0x4B000000u;
__device__ __forceinline__ uint32_t bias_reg() { return kBiasWord; }
__device__ __forceinline__ float byte_biased(uint32_t v, uint32_t bias, int l) {
  return __uint_as_float(__byte_perm(v, bias, 0x7540u | uint32_t(l)));
}
constexpr float kTwo23 = 8388608.0f;
constexpr float kRound = 12582912.0f;  // 1.5 * 2^23: x + kRound rounds x to an integer (ties to even)

// Horizontal lerp of one source row for the column pair, per lane, in FP32:
// h = a + (b - a) * fx with a, b exact (PRMT-built biased floats).
template <int NL>
__device__ __forceinline__ void hlerp2(uint32_t a0, uint32_t b0, uint32_t a1, uint32_t b1, uint64_t fx,
                                       uint32_t bias, uint64_t (&h)[3]) {
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const uint64_t A = f2::pack(byte_biased(a0, bias, l), byte_biased(a1, bias, l));
    const uint64_t B = f2::pack(byte_biased(b0, bias, l), byte_biased(b1, bias, l));
    h[l] = f2::fma(f2::sub(B, A), fx, f2::sub(A, f2::bc(kTwo23)));
  }
}

// The reference's bilinear value of one lane in double, op for op
// (ops.cpp:250,283-296; u8 -> double as the low word of 2^52 + v, nearbyint as
// the low word of res + 1.5 * 2^52), returned as the float of the u8 result.
__device__ __forceinline__ float exact_lane(uint32_t a, uint32_t b, uint32_t c, uint32_t d, double fx, double fy) {
  constexpr double kTwo52 = 4503599627370496.0;
  const double A = __hiloint2double(0x43300000, int(a)) - kTwo52, B = __hiloint2double(0x43300000, int(b)) - kTwo52;
  const double C = __hiloint2double(0x43300000, int(c)) - kTwo52, D = __hiloint2double(0x43300000, int(d)) - kTwo52;
  const double top = __dadd_rn(A, __dmul_rn(__dsub_rn(B, A), fx));
  const double bot = __dadd_rn(C, __dmul_rn(__dsub_rn(D, C), fx));
  const double res = __dadd_rn(top, __dmul_rn(__dsub_rn(bot, top), fy));
  return float(uint32_t(__double2loint(__dadd_rn(res, 6755399441055744.0))) & 0xffu);
}

// Per-plane chain constants for the AFFINE mode, indexed by INPUT lane m (the
// constants of the output lane sigma(m) it lands in).
struct AffConsts {
  float c[3][4], r[3][4];
};

// Where the AFFINE chain's constants come from inside the walk: registers
// (per-plane constants, or a plane-dependent lane swap), or — when every plane
// shares them (DPlan::aff_inline) and the warp's lane swap is known at compile
// time — straight from kernel-parameter space, so they cost no registers.
struct KReg {
  const AffConsts& K;
  __device__ __forceinline__ float c(int l, int k) const { return K.c[l][k]; }
  __device__ __forceinline__ float r(int l, int k) const { return K.r[l][k]; }
};
template <int NL, bool SW>
struct KPar {
  const DPlan& P;
  __device__ __forceinline__ float c(int l, int k) const { return P.aff_c[k][NL == 3 && SW ? 2 - l : l]; }
  __device__ __forceinline__ float r(int l, int k) const { return P.aff_r[k][NL == 3 && SW ? 2 - l : l]; }
};
// The same constants loaded once into registers the compiler must keep (it
// otherwise reloads them from the constant bank on every output row).
__device__ __forceinline__ float pinf(float v) {
  asm volatile("" : "+f"(v));
  return v;
}
template <int NL, uint32_t SIG, bool SW>
struct KPin {
  float cc[3][4], rr[3][4];
  // staged through shared memory with volatile loads: ptxas may re-read a
  // kernel parameter inside the loop (LDCU per output row), not a volatile load
  __device__ __forceinline__ KPin(const DPlan& P, float* scratch) {
    const uint32_t lane = threadIdx.x & 31u;
    if (lane == 0) {
#pragma unroll
      for (int l = 0; l < 3; ++l)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int m = NL == 3 && SW ? 2 - l : l;
          scratch[l * 4 + k] = P.aff_c[k][m];
          scratch[12 + l * 4 + k] = P.aff_r[k][m];
        }
    }
    __syncwarp();
    const uint32_t sb = uint32_t(__cvta_generic_to_shared(scratch));
#pragma unroll
    for (int l = 0; l < 3; ++l)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool used = l < NL && k < sig_n(SIG);
        float c = 0.f, r = 0.f;
        if (used) asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(c) : "r"(sb + 4 * (l * 4 + k)));
        if (used && sig_fn(SIG, k) == AF_DIV)
          asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(r) : "r"(sb + 4 * (12 + l * 4 + k)));
        cc[l][k] = c;
        rr[l][k] = r;
      }
    __syncwarp();
  }
  __device__ __forceinline__ float c(int l, int k) const { return cc[l][k]; }
  __device__ __forceinline__ float r(int l, int k) const { return rr[l][k]; }
};

template <int NL, uint32_t SIG>
__device__ __forceinline__ void load_affine(const DPlan& P, uint32_t z, bool swap, AffConsts& K) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k >= sig_n(SIG)) {
#pragma unroll
      for (int m = 0; m < 3; ++m) K.c[m][k] = K.r[m][k] = 0.f;
      continue;
    }
    float c[3], r[3];
    if (P.aff_inline) {
#pragma unroll
      for (int l = 0; l < 3; ++l) { c[l] = P.aff_c[k][l]; r[l] = P.aff_r[k][l]; }
    } else {
      const DOp op = dev::prog_op(P, P.op_base + k);
      uint64_t v[3] = {op.c[0], op.c[1], op.c[2]};
      if (op.per_z) {
        const uint64_t* row = reinterpret_cast<const uint64_t*>(op.per_z) + 3ull * (z < op.per_z_n ? z : op.per_z_n - 1);
        v[0] = __ldg(row); v[1] = __ldg(row + 1); v[2] = __ldg(row + 2);
      }
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        c[l] = __uint_as_float(uint32_t(v[op.nl == 3 ? l : 0]));
        r[l] = __frcp_rn(c[l]);
      }
    }
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int l = (NL == 3 && swap) ? 2 - m : m;
      K.c[m][k] = l == 0 ? c[0] : (l == 1 ? c[1] : c[2]);
      K.r[m][k] = l == 0 ? r[0] : (l == 1 ? r[1] : r[2]);
    }
  }
}

// Pixel pairs the filter flagged, recomputed after the band walk: (row k << 5 |
// lane) entries in the warp's shared memory. A 224-row plane of random data
// flags ~60 pairs; scale factors with small denominators (e.g. 176 -> 224) make
// exact rational ties common (up to ~1700 pairs, ~500 per warp). A lane whose
// push finds the list full marks itself and recomputes its whole column pair
// afterwards.
constexpr uint32_t kFixCap = 512;
struct FixShared {
  uint32_t n;
  uint16_t e[kFixCap];
};
struct FixList {
  FixShared* sh;
  bool ovf;
  __device__ __forceinline__ void push(uint32_t k) {
    const uint32_t i = atomicAdd(&sh->n, 1u);
    if (i < kFixCap) sh->e[i] = uint16_t((k << 5) | (threadIdx.x & 31u));
    else ovf = true;
  }
};

// One output pixel (xc, y) exactly as the reference computes it: bilinear_sample
// in double (ops.cpp:259-299), round_clamp_u8, then the chain and the store.
template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG, class Out>
__device__ __forceinline__ void fix_pixel(const DSample& s, const DWrite& w, uint32_t xc, uint32_t y, bool swap, bool al,
                                       const AffConsts& K, const Out* lut) {
  constexpr int OB = OLK == FK_U8 ? 1 : (OLK == FK_F32 ? 4 : 8);
  const XEnt xe = dev::x_entry(s, xc, NL);
  const YEnt ye = dev::y_entry(s, y);
  const uint8_t* r0 = reinterpret_cast<const uint8_t*>(s.src) + ye.r0;
  const uint8_t* r1 = reinterpret_cast<const uint8_t*>(s.src) + ye.r1;
  Out o[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const float u = exact_lane(__ldg(r0 + xe.o0 + l), __ldg(r0 + xe.o1 + l), __ldg(r1 + xe.o0 + l),
                               __ldg(r1 + xe.o1 + l), xe.f, ye.f);
    if constexpr (SIG != kSigLut) o[l] = Out(__float_as_uint(sig_apply<SIG>(u, K.c[l], K.r[l])));
    else o[l] = lut[l * 256 + uint32_t(u)];
  }
  if constexpr (SPLIT) {
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const int e = swap ? 2 - l : l;
      dev::store_lane<OLK, Out>(reinterpret_cast<uint8_t*>(w.dst[e]) + uint64_t(y) * w.pitch[e] + uint64_t(xc) * OB,
                                o[l], al);
    }
  } else {
    if constexpr (NL == 3) {
      if (swap) { const Out t = o[0]; o[0] = o[2]; o[2] = t; }
    }
#pragma unroll
    for (int l = 0; l < NL; ++l)
      dev::store_lane<OLK, Out>(
          reinterpret_cast<uint8_t*>(w.dst[0]) + uint64_t(y) * w.pitch[0] + (uint64_t(xc) * NL + l) * OB, o[l], al);
  }
}

// Both columns (x, x + 1 if in the plane) of output row y of plane z, exactly.
template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG, class Out>
__device__ __noinline__ void fix_pair(const DPlan& P, uint32_t z, uint32_t x, uint32_t y, const Out* lut) {
  const DSample s = P.reads[z];
  const DWrite w = P.writes[z];
  const bool swap = ((s.flags & SF_POST_SWAP) != 0) != (P.prog_swap != 0);
  const bool al = (w.flags & WF_LANE_ALIGNED) != 0;
  AffConsts K;
  if constexpr (SIG != kSigLut) load_affine<NL, SIG>(P, z, swap, K);
  fix_pixel<NL, OLK, SPLIT, SIG, Out>(s, w, x, y, swap, al, K, lut);
  if (x + 1 < P.width) fix_pixel<NL, OLK, SPLIT, SIG, Out>(s, w, x + 1, y, swap, al, K, lut);
}

// Destination cursor of one column pair: the byte address of (x, y) in each
// destination plane, advanced by the pitch per output row.
template <int NL, uint32_t OLK, bool SPLIT>
struct PairOut {
  static constexpr int OB = OLK == FK_U8 ? 1 : (OLK == FK_F32 ? 4 : 8);
  static constexpr int ND = SPLIT ? 3 : 1;
  uint8_t* p[ND];
  uint32_t pitch[ND];  // < 2^32 (checked by the host)
  __device__ __forceinline__ PairOut(const DWrite& w, uint32_t x, uint32_t y, bool swap) {
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      const int e = (SPLIT && swap) ? 2 - d : d;  // split + lane swap: lane m goes to plane sigma(m)
      pitch[d] = uint32_t(w.pitch[e]);
      // one row above (x, y): next() advances first, then stores
      p[d] = reinterpret_cast<uint8_t*>(w.dst[e]) + (uint64_t(y) - 1) * w.pitch[e] + uint64_t(x) * OB * (SPLIT ? 1 : NL);
    }
  }
  __device__ __forceinline__ void next() {
#pragma unroll
    for (int d = 0; d < ND; ++d) p[d] += pitch[d];
  }
  // store_block (:396-400) / split of column c's lanes (generic)
  template <class Out>
  __device__ __forceinline__ void put_col(int c, const Out (&o)[NL], bool al) {
    if constexpr (SPLIT) {
#pragma unroll
      for (int l = 0; l < 3; ++l) dev::store_lane<OLK, Out>(p[l] + c * OB, o[l], al);
    } else {
#pragma unroll
      for (int l = 0; l < NL; ++l) dev::store_lane<OLK, Out>(p[0] + (c * NL + l) * OB, o[l], al);
    }
  }
};


// Destination cursor of the split-f32 fast path: three planes with one pitch,
// the row address as base + y * pitch (one IMAD.WIDE), and lane l of both
// columns written as one 8-byte streaming store.
struct VecOut {
  uint64_t base[3];
  uint32_t y, pitch;
  __device__ __forceinline__ VecOut(const DWrite& w, uint32_t x, uint32_t y0, bool swap) {
#pragma unroll
    for (int d = 0; d < 3; ++d) base[d] = w.dst[swap ? 2 - d : d] + uint64_t(x) * 4;
    pitch = uint32_t(w.pitch[0]);
    y = y0 - 1;  // next() advances first
  }
  __device__ __forceinline__ void next() { ++y; }
  __device__ __forceinline__ void put(int l, uint64_t v) {
    asm volatile("st.global.cs.v2.b32 [%0], {%1, %2};" ::"l"(at_row(base[l], y, pitch)), "r"(uint32_t(v)),
                 "r"(uint32_t(v >> 32))
                 : "memory");
  }
};

// Output row k of the column pair: V-lerp, exact-result filter, chain, store.
// top / bot = H-lerps of source rows s0 / s1 (lane-packed pairs).
template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG, bool VEC, class Out, class Cur, class KS>
__device__ __forceinline__ void emit2(const uint64_t (&top)[3], const uint64_t (&bot)[3], float2 q,
                                      uint32_t row_k, float col_thr, const KS& ks, const Out* lut, bool swap,
                                      bool col1, bool al, Cur& out, FixList& fix) {
  constexpr bool AFFINE = SIG != kSigLut;
  const float thr = fminf(q.y, col_thr);  // 0.5 (never flagged) only if fx and fy are multiples of 2^-8
  uint64_t t[3], k[3];
  bool near = false;
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const uint64_t v = f2::fma(f2::sub(bot[l], top[l]), f2::bc(q.x), top[l]);
    t[l] = f2::add(v, f2::bc(kRound));
    k[l] = f2::sub(t[l], f2::bc(kRound));
    const uint64_t e = f2::sub(v, k[l]);
    near |= fabsf(f2::lo(e)) > thr;
    near |= fabsf(f2::hi(e)) > thr;
  }
  out.next();
  if (near) fix.push(row_k);  // rare: fixed after the walk in the reference's double arithmetic
  if constexpr (VEC) {  // split f32, both columns in the plane: 8-byte stores
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      if constexpr (AFFINE) {
        out.put(l, sig_apply2<SIG>(k[l], ks, l));
      } else {
        out.put(l, uint64_t(lut[l * 256 + (uint32_t(t[l]) & 0xffu)]) |
                       uint64_t(lut[l * 256 + (uint32_t(t[l] >> 32) & 0xffu)]) << 32);
      }
    }
  } else if constexpr (AFFINE) {  // generic stores; packed output: lane m lands in lane sigma(m)
    uint64_t o[3];
#pragma unroll
    for (int l = 0; l < NL; ++l) o[l] = sig_apply2<SIG>(k[l], ks, l);
    if constexpr (NL == 3 && !SPLIT) {
      if (swap) { const uint64_t tt = o[0]; o[0] = o[2]; o[2] = tt; }
    }
    Out a[NL], b[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) { a[l] = Out(uint32_t(o[l])); b[l] = Out(uint32_t(o[l] >> 32)); }
    out.put_col(0, a, al);
    if (col1) out.put_col(1, b, al);
  } else {  // LUT: index = the low bits of t (t = 1.5 * 2^23 + u8)
    Out a[NL], b[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      a[l] = lut[l * 256 + (uint32_t(t[l]) & 0xffu)];
      b[l] = lut[l * 256 + (uint32_t(t[l] >> 32) & 0xffu)];
    }
    if constexpr (NL == 3 && !SPLIT) {
      if (swap) {
        Out tt = a[0]; a[0] = a[2]; a[2] = tt;
        tt = b[0]; b[0] = b[2]; b[2] = tt;
      }
    }
    out.put_col(0, a, al);
    if (col1) out.put_col(1, b, al);
  }
}

// The source rows a band visits, in order, and the output rows each visit
// completes: output row k (source rows s0, s1) is emitted right after the visits
// s0, s1 — the last two visits are always exactly (s0, s1), so an edge row whose
// s0 == s1 (clamped) visits that row twice. Output rows [v[i - 1].end, v[i].end)
// are emitted at visit i; v[n] repeats v[n - 1]'s row (the walk prefetches one
// visit ahead).
struct Visits {
  uint32_t v[2 * kBandMax + 1];  // source row relative to y0 | (output rows emitted up to here) << 16
  uint32_t n;
};
__device__ __forceinline__ uint32_t visit_row(uint32_t e) { return e & 0xffffu; }
__device__ __forceinline__ uint32_t visit_end(uint32_t e) { return e >> 16; }

// Built by warp 0 for the band's n output rows. Output row k adds no visit when
// (s0, s1) equals row k - 1's, one visit (s1) when its s0 is row k - 1's s1,
// two (s0, s1) otherwise; a warp scan places them.
__device__ __forceinline__ void build_visits_warp(const BandRows& R, uint32_t n, Visits& V) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t base = 0;
  for (uint32_t c = 0; c < n; c += 32) {
    const uint32_t k = c + lane;
    const bool in = k < n;
    const uint32_t s0 = in ? (R.s[k] & 0xffffu) : 0, s1 = in ? (R.s[k] >> 16) : 0;
    const bool first = k == 0;
    const uint32_t p0 = (in && !first) ? (R.s[k - 1] & 0xffffu) : 0, p1 = (in && !first) ? (R.s[k - 1] >> 16) : 0;
    const uint32_t cnt = !in ? 0u : (!first && s0 == p0 && s1 == p1) ? 0u : (!first && s0 == p1) ? 1u : 2u;
    uint32_t incl = cnt;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    const uint32_t pos = base + incl - cnt;
    if (cnt == 2) V.v[pos] = s0 | (k << 16);
    // the last output row attached to a visit closes it
    const bool closes = in && (k + 1 == n || R.s[k + 1] != R.s[k]);
    if (cnt != 0) V.v[pos + cnt - 1] = s1 | ((closes ? k + 1 : k) << 16);
    __syncwarp();
    if (closes && cnt == 0) V.v[pos - 1] = (V.v[pos - 1] & 0xffffu) | ((k + 1) << 16);
    base += __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();
  }
  if (lane == 0) {
    V.v[base] = V.v[base - 1];
    V.n = base;
  }
}

// Walk the band's visits for the column pair (x, x + 1) (bilinear). Each visit
// H-lerps ONE source row and emits the output rows it completes. hA / hB
// alternate as the current row by unrolling the walk by two, so no H-lerp is
// ever copied between registers.
template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG, bool ALIGNED, bool VEC, class Out>
__device__ __forceinline__ void pair_bilinear(const DSample& s, const DWrite& w, const BandRows& R, const Visits& V,
                                              uint32_t x, bool col1, uint32_t y0, bool swap, bool al,
                                              const AffConsts& K, const Out* lut, FixList& fix) {
  const XEnt e0 = dev::x_entry(s, x, NL);
  const XEnt e1 = dev::x_entry(s, col1 ? x + 1 : x, NL);
  const uint64_t fx = f2::pack(float(e0.f), float(e1.f));
  const float col_thr = (coord_exact8(e0.f) && coord_exact8(e1.f)) ? 0.5f : 0.5f - kNearTol;
  const uint32_t bias = bias_reg();
  ColTap<NL, ALIGNED> T0, T1;
  const uint64_t origin = s.src + uint64_t(s.y0) * s.pitch;  // visit rows are relative to y0
  T0.init(origin, e0.o0, e0.o1);
  T1.init(origin, e1.o0, e1.o1);
  using Cur = typename std::conditional<VEC, VecOut, PairOut<NL, OLK, SPLIT>>::type;
  Cur out(w, x, y0, swap);
  const uint32_t pitch = uint32_t(s.pitch);
  T0.issue(visit_row(V.v[0]), pitch);
  T1.issue(visit_row(V.v[0]), pitch);
  uint64_t hA[3] = {0, 0, 0}, hB[3] = {0, 0, 0};
  uint32_t k = 0;
  const uint32_t nv = V.n;
  // visit i: H-lerp its row into `cur`, prefetch visit i + 1, emit its outputs
  auto visit = [&](uint32_t i, uint64_t (&cur)[3], const uint64_t (&prev)[3]) {
    uint32_t a0, b0, a1, b1;
    T0.taps(a0, b0);
    T1.taps(a1, b1);
    const uint32_t nx = visit_row(V.v[i + 1]);
    const uint32_t end = visit_end(V.v[i]);
    T0.issue(nx, pitch);
    T1.issue(nx, pitch);
    hlerp2<NL>(a0, b0, a1, b1, fx, bias, cur);
#pragma unroll 1
    for (; k < end; ++k)
      emit2<NL, OLK, SPLIT, SIG, VEC, Out>(prev, cur, R.q[k], k, col_thr, KReg{K}, lut, swap, col1, al, out, fix);
  };
  for (uint32_t i = 0; i < nv; i += 2) {
    visit(i, hA, hB);
    if (i + 1 < nv) visit(i + 1, hB, hA);
  }
}

// ------------------------------------------------- staged (cp.async) walk --
// Each visit's source row is new to the warp, so a direct tap load is an L2
// round trip. The staged walk instead copies the row span the warp's columns
// touch into a shared-memory ring kRing - 1 visits ahead with cp.async (16-byte
// chunks, zero-filled past the crop's last byte so nothing beyond the plane is
// read; no registers hold data in flight), and gathers taps from shared memory.
#ifndef FK_RING
#define FK_RING 4
#endif
constexpr uint32_t kRing = FK_RING;  // staged source rows per warp (kRing - 1 visits in flight)
constexpr uint32_t kRingRow = 512;  // bytes per staged row: one slot's span, or two 256-byte halves

__device__ __forceinline__ void cp_async16(uint32_t dst, uint64_t src, uint32_t n) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// The warp's staging plan: whether the span of every plane slot in the warp fits
// its region of a ring row (and is 16-byte aligned), this lane's copy job
// (source chunk at relative row 0, pitch, shared offset, byte count), and this
// lane's tap offsets within a ring row.
struct StagePlan {
  bool ok;
  uint64_t g;            // copy job: source address of the chunk in relative row 0
  uint32_t pitch, dst, n;  // ... row pitch, byte offset in a ring row, bytes (0: none)
  uint32_t ta[2], tb[2];  // byte offsets of tap a / b of columns x, x + 1 in a ring row
};

template <int NL>
__device__ __forceinline__ StagePlan stage_plan(const DSample& s, bool mine, uint32_t hs, const XEnt& e0,
                                                const XEnt& e1) {
  StagePlan S;
  const uint32_t o00 = e0.o0, o11 = e1.o1;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t hA = __shfl_sync(0xffffffffu, hs, 0), hB = __shfl_sync(0xffffffffu, hs, 31);
  const bool first = hs == hA;
  const uint32_t lo = mine ? o00 : 0xffffffffu, hi = mine ? o11 + NL : 0u;
  const uint32_t loA = __reduce_min_sync(0xffffffffu, first ? lo : 0xffffffffu);
  const uint32_t hiA = __reduce_max_sync(0xffffffffu, first ? hi : 0u);
  const uint32_t loB = __reduce_min_sync(0xffffffffu, first ? 0xffffffffu : lo);
  const uint32_t hiB = __reduce_max_sync(0xffffffffu, first ? 0u : hi);
  const uint32_t cap = hA == hB ? kRingRow : kRingRow / 2;
  const uint32_t spA = loA & ~15u, spB = loB & ~15u;
  const uint32_t nA = hiA > loA ? (hiA - spA + 15) / 16 : 0, nB = hiB > loB ? (hiB - spB + 15) / 16 : 0;
  const uint64_t origin = s.src + uint64_t(s.y0) * s.pitch;
  const bool al16 = ((origin | s.pitch) & 15) == 0;
  S.ok = __all_sync(0xffffffffu, al16 || !mine) && nA * 16 <= cap && nB * 16 <= cap;
  // this lane's taps: offsets from its slot's span start, in its slot's region
  // (lanes without columns read offset 0)
  const uint32_t sp = first ? spA : spB, reg = first ? 0u : kRingRow / 2;
  S.ta[0] = mine ? reg + e0.o0 - sp : 0u;
  S.tb[0] = mine ? reg + e0.o1 - sp : 0u;
  S.ta[1] = mine ? reg + e1.o0 - sp : 0u;
  S.tb[1] = mine ? reg + e1.o1 - sp : 0u;
  // copy job: chunks [0, nA) of the first slot, then [0, nB) of the second
  const bool jobA = lane < nA, jobB = !jobA && lane < nA + nB;
  const uint32_t src_lane = jobA ? 0u : 31u;
  const uint64_t org = __shfl_sync(0xffffffffu, origin, src_lane);
  const uint32_t pit = __shfl_sync(0xffffffffu, uint32_t(s.pitch), src_lane);
  const uint32_t vend = __shfl_sync(0xffffffffu, (s.x0 + s.rect_w) * NL, src_lane);  // last tap byte + 1
  const uint32_t c = jobA ? lane : lane - nA, csp = jobA ? spA : spB;
  const uint32_t start = csp + 16 * c;
  S.g = org + start;
  S.pitch = pit;
  S.dst = (jobA ? 0u : kRingRow / 2) * (hA == hB ? 0u : 1u) + 16 * c;
  S.n = (jobA || jobB) ? min(16u, vend - start) : 0u;
  return S;
}

// A 32-bit value the compiler must keep in a register (not rematerialise in the loop)
__device__ __forceinline__ uint32_t pin(uint32_t v) {
  asm volatile("" : "+r"(v));
  return v;
}

// Every lane copies a 16-byte chunk of the visit's row span with cp.async
// (zero-filled past the crop) kRing - 1 visits ahead.
template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG, bool VEC, class Out, class KS>
__device__ __forceinline__ void pair_bilinear_staged(const DWrite& w, const BandRows& R, const Visits& V,
                                                     uint8_t* ring, const StagePlan& S,
                                                     const XEnt& e0, const XEnt& e1, bool active, uint32_t x,
                                                     bool col1, uint32_t y0, bool swap, bool al, const KS& ks,
                                                     const Out* lut, FixList& fix) {
  const uint64_t fx = f2::pack(float(e0.f), float(e1.f));
  const float col_thr = (coord_exact8(e0.f) && coord_exact8(e1.f)) ? 0.5f : 0.5f - kNearTol;
  const uint32_t bias = pin(bias_reg());
  // shared addresses, computed once: ring slot 0 + this lane's tap words, the
  // visit list, the row table, the copy destination
  const uint32_t base = pin(uint32_t(__cvta_generic_to_shared(ring)));
  const uint32_t a0 = pin(base + (S.ta[0] & ~3u)), b0 = pin(base + (S.tb[0] & ~3u));
  const uint32_t a1 = pin(base + (S.ta[1] & ~3u)), b1 = pin(base + (S.tb[1] & ~3u));
  const uint32_t sa0 = 8 * (S.ta[0] & 3u), sb0 = 8 * (S.tb[0] & 3u), sa1 = 8 * (S.ta[1] & 3u),
                 sb1 = 8 * (S.tb[1] & 3u);
  const uint32_t cdst = pin(base + S.dst);
  uint32_t vp = pin(uint32_t(__cvta_generic_to_shared(V.v)));
  uint32_t qp = pin(uint32_t(__cvta_generic_to_shared(R.q)));
  using Cur = typename std::conditional<VEC, VecOut, PairOut<NL, OLK, SPLIT>>::type;
  Cur out(w, x, y0, swap);
  const uint32_t nv = V.n;
  const uint32_t lane = threadIdx.x & 31u;
  // prologue: visits 0 .. kRing - 2 in flight (one commit group per visit)
#pragma unroll
  for (uint32_t j = 0; j < kRing - 1; ++j) {
    if (j < nv && S.n) cp_async16(cdst + j * kRingRow, at_row(S.g, visit_row(lds32(vp + 4 * j)), S.pitch), S.n);
    cp_commit();
  }
  uint64_t hA[3] = {0, 0, 0}, hB[3] = {0, 0, 0};
  uint32_t k = 0;
  // visit i = i0 + U (ring slot U, compile-time): H-lerp its row into `cur`,
  // start the copy of visit i + kRing - 1, emit the output rows it completes
  auto visit = [&](auto U, uint32_t i, uint64_t (&cur)[3], const uint64_t (&prev)[3]) {
    constexpr uint32_t u = decltype(U)::value;
    constexpr uint32_t slot = u * kRingRow, aslot = ((u + kRing - 1) % kRing) * kRingRow;
    cp_wait<kRing - 2>();  // visit i's row has landed (this lane's chunk) ...
    __syncwarp();           // ... and every lane's; every lane is also done with visit i - 1's slot
    if (i + kRing - 1 < nv && S.n)
      cp_async16(cdst + aslot, at_row(S.g, visit_row(lds32(vp + 4 * (u + kRing - 1))), S.pitch), S.n);
    cp_commit();
    const uint32_t ta0 = __funnelshift_r(lds32(a0 + slot), lds32(a0 + slot + 4), sa0);
    const uint32_t tb0 = __funnelshift_r(lds32(b0 + slot), lds32(b0 + slot + 4), sb0);
    const uint32_t ta1 = __funnelshift_r(lds32(a1 + slot), lds32(a1 + slot + 4), sa1);
    const uint32_t tb1 = __funnelshift_r(lds32(b1 + slot), lds32(b1 + slot + 4), sb1);
    hlerp2<NL>(ta0, tb0, ta1, tb1, fx, bias, cur);
    const uint32_t end = visit_end(lds32(vp + 4 * u));
    if (active) {
#pragma unroll 1
      for (; k < end; ++k, qp += 8) {
        float2 q;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(q.x), "=f"(q.y) : "r"(qp));
        emit2<NL, OLK, SPLIT, SIG, VEC, Out>(prev, cur, q, k, col_thr, ks, lut, swap, col1, al, out, fix);
      }
    }
  };
  for (uint32_t i0 = 0; i0 < nv; i0 += kRing, vp += 4 * kRing) {
    static_assert(kRing == 4 || kRing == 8, "the walk is unrolled by the ring size");
    visit(std::integral_constant<uint32_t, 0>(), i0, hA, hB);
    if (i0 + 1 >= nv) break;
    visit(std::integral_constant<uint32_t, 1>(), i0 + 1, hB, hA);
    if (i0 + 2 >= nv) break;
    visit(std::integral_constant<uint32_t, 2>(), i0 + 2, hA, hB);
    if (i0 + 3 >= nv) break;
    visit(std::integral_constant<uint32_t, 3>(), i0 + 3, hB, hA);
    if (kRing == 4 || i0 + 4 >= nv) continue;
    visit(std::integral_constant<uint32_t, 4 % kRing>(), i0 + 4, hA, hB);
    if (i0 + 5 >= nv) break;
    visit(std::integral_constant<uint32_t, 5 % kRing>(), i0 + 5, hB, hA);
    if (i0 + 6 >= nv) break;
    visit(std::integral_constant<uint32_t, 6 % kRing>(), i0 + 6, hA, hB);
    if (i0 + 7 >= nv) break;
    visit(std::integral_constant<uint32_t, 7 % kRing>(), i0 + 7, hB, hA);
  }
  cp_wait<0>();
  __syncwarp();  // the ring and its barriers are reused by the next slice
}

// Nearest / non-resizing planes: one tap per output pixel, the chain in scalar form.
template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG, class Out>
__device__ __forceinline__ void pair_tap(const DSample& s, const DWrite& w, const BandRows& R, uint32_t x, bool col1,
                                         uint32_t y0, uint32_t y1, bool swap, bool al, const AffConsts& K,
                                         const Out* lut) {
  constexpr bool AFFINE = SIG != kSigLut;
  uint32_t oc[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const uint32_t xc = c && col1 ? x + 1 : x;
    oc[c] = s.mode == RD_DIRECT ? (s.x0 + xc) * NL : dev::x_entry(s, xc, NL).o0;
  }
  const uint8_t* base = reinterpret_cast<const uint8_t*>(s.src);
  PairOut<NL, OLK, SPLIT> out(w, x, y0, swap);
  for (uint32_t y = y0; y < y1; ++y) {
    const uint8_t* row = base + uint64_t(s.y0 + (R.s[y - y0] & 0xffffu)) * s.pitch;
    out.next();
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (c == 1 && !col1) break;
      Out o[NL];
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const uint32_t u = __ldg(row + oc[c] + l);
        if constexpr (AFFINE) {
          float cl[4], rl[4];
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) { cl[kk] = K.c[l][kk]; rl[kk] = K.r[l][kk]; }
          o[l] = Out(__float_as_uint(sig_apply<SIG>(float(u), cl, rl)));
        } else {
          o[l] = lut[l * 256 + u];
        }
      }
      if constexpr (NL == 3 && !SPLIT) {
        if (swap) { const Out t = o[0]; o[0] = o[2]; o[2] = t; }
      }
      out.put_col(c, o, al);
    }
  }
}

}  // namespace

// One CTA = ONE warp, an independent unit of work: 32 column pairs of a band of
// output rows of the planes of one z slice (horizontal fusion). A slice is one
// plane, or two planes with equal rect_h, read mode and lane swap laid side by
// side (pair slots [0, T) and [T, 2T)), so a 224-wide plane (112 pairs) plus its
// partner fill exactly 7 warps. The warp builds its own row coordinates and visit
// list (they depend only on rect_h / out_h; rows are relative to each plane's
// y0), walks, and fixes its flagged pixels, synchronising only with __syncwarp:
// no CTA barrier couples warps that the schedulers progress at different rates.
// SIG = a registered AFFINE chain (constants in registers, packed FP32
// evaluation), or kSigLut (a table per slot, the plane's folded unaries + the
// compute program interpreted over the 256 byte values).
template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG, bool STAGED>
__global__ void __launch_bounds__(32, FK_SEP_MINB) fk_resample_sep(const __grid_constant__ DPlan P) {
  constexpr bool AFFINE = SIG != kSigLut;
  using Out = typename std::conditional<OLK == FK_F64, uint64_t, uint32_t>::type;
  __shared__ BandRows R;
  __shared__ Visits vis;
  __shared__ FixShared fixs;
  __shared__ Out lut[AFFINE ? 1 : 2 * NL * 256];
  __shared__ alignas(16) uint8_t ring[STAGED ? kRing * kRingRow : 16];
  __shared__ float kscr[24];
  const uint32_t lane = threadIdx.x;
  const uint32_t T = P.slot_threads;  // column pairs per plane slot
  const uint32_t spc = P.slots ? P.slots_per_cta : 1u;
  const uint32_t ts = blockIdx.x * 32 + lane;  // pair slot within the slice
  const uint32_t hs = ts / T;                   // this lane's plane slot
  const uint32_t x = 2 * (ts - hs * T);
  const uint32_t y_begin = blockIdx.y * P.tiles_per_cta;  // tiles_per_cta = band rows for this kernel
  const uint32_t y_end = min(y_begin + P.tiles_per_cta, P.height);
  const uint32_t nslices = P.slots ? P.slices : P.batch;
  auto plane_of = [&](uint32_t c, uint32_t h) -> uint32_t {
    if (h >= spc) return kNoPlane;
    if (P.slots) return __ldg(P.slots + c * spc + h);
    return P.order ? __ldg(P.order + c) : c;
  };
  for (uint32_t c = blockIdx.z; c < nslices; c += gridDim.z) {
    const uint32_t z0 = plane_of(c, 0);
    const uint32_t zm = plane_of(c, hs);
    const bool slot_on = zm != kNoPlane;
    const uint32_t z = slot_on ? zm : z0;
    const DSample s0 = P.reads[z0];  // the slice's row coordinates
    __syncwarp();
    if (lane == 0) fixs.n = 0;
    for (uint32_t j = lane; j < y_end - y_begin; j += 32) {
      uint32_t r0, r1;
      double f;
      if (s0.mode != RD_DIRECT) {  // y_entry gives row byte offsets; keep source rows relative to y0
        const YEnt ye = dev::y_entry(s0, y_begin + j);
        r0 = uint32_t(ye.r0 / s0.pitch) - s0.y0;
        r1 = uint32_t(ye.r1 / s0.pitch) - s0.y0;
        f = ye.f;
      } else {
        r0 = r1 = y_begin + j;
        f = 0.0;
      }
      R.q[j] = make_float2(float(f), coord_exact8(f) ? 0.5f : 0.5f - kNearTol);
      R.s[j] = r0 | (r1 << 16);
    }
    if constexpr (!AFFINE) {
      for (uint32_t h = 0; h < spc; ++h) {  // each slot's chain over every byte value
        const uint32_t zh = plane_of(c, h);
        if (zh == kNoPlane) continue;
        const DSample sh = P.reads[zh];
        const bool swh = ((sh.flags & SF_POST_SWAP) != 0) != (P.prog_swap != 0);
        for (uint32_t t = lane; t < 256; t += 32) {
          uint64_t v[1][3] = {{t, t, t}};
          dev::run_ops(P, sh.post_off, sh.post_len, zh, v);
          dev::run_ops(P, P.op_base, P.n_ops, zh, v);
#pragma unroll
          for (int m = 0; m < NL; ++m) lut[(h * NL + m) * 256 + t] = Out(v[0][(NL == 3 && swh) ? 2 - m : m]);
        }
      }
    }
    const Out* my_lut = lut + (AFFINE ? 0 : (hs < spc ? hs : 0) * NL * 256);
    __syncwarp();
    const bool bilinear = s0.mode == RD_BILINEAR;  // slice-uniform (slots share the mode)
    if (bilinear) {
      build_visits_warp(R, y_end - y_begin, vis);
      __syncwarp();
    }
    FixList fix{&fixs, false};
    {
      const DSample s = P.reads[z];
      const DWrite w = P.writes[z];
      const bool swap = ((s.flags & SF_POST_SWAP) != 0) != (P.prog_swap != 0);
      // BatchWrite z >= active_count / past the row / empty slot: no stores
      const bool active = slot_on && (w.flags & WF_ACTIVE) && x < P.width;
      const bool col1 = x + 1 < P.width;
      const bool al = (w.flags & WF_LANE_ALIGNED) != 0;
      bool vec = false;
      if constexpr (SPLIT && OLK == FK_F32) {
        vec = col1 && w.pitch[1] == w.pitch[0] && w.pitch[2] == w.pitch[0];
#pragma unroll
        for (int d = 0; d < 3; ++d) vec = vec && ((w.dst[d] | w.pitch[d]) & 7) == 0;
      }
      if (bilinear && STAGED) {  // warp-uniform: the staged walk needs every lane (copies, shuffles)
        const bool mine = slot_on && x < P.width;
        const XEnt e0 = dev::x_entry(s, mine ? x : 0, NL);
        const XEnt e1 = dev::x_entry(s, mine && col1 ? x + 1 : (mine ? x : 0), NL);
        const StagePlan S = stage_plan<NL>(s, mine, hs, e0, e1);
        if (!S.ok) __trap();  // the host checked spans and alignment (sep_stage_ok)
        if (__all_sync(0xffffffffu, vec || !active)) {
          // slots share their lane swap, so `swap` is warp-uniform
          if (AFFINE && P.aff_inline && !swap) {
            pair_bilinear_staged<NL, OLK, SPLIT, SIG, true, Out>(w, R, vis, ring, S, e0, e1, active, x,
                                                                        col1, y_begin, swap, al,
                                                                        KPin<NL, SIG, false>(P, kscr), my_lut, fix);
          } else if (AFFINE && P.aff_inline) {
            pair_bilinear_staged<NL, OLK, SPLIT, SIG, true, Out>(w, R, vis, ring, S, e0, e1, active, x,
                                                                        col1, y_begin, swap, al,
                                                                        KPin<NL, SIG, true>(P, kscr), my_lut, fix);
          } else {
            AffConsts K;
            if constexpr (AFFINE) load_affine<NL, SIG>(P, z, swap, K);
            pair_bilinear_staged<NL, OLK, SPLIT, SIG, true, Out>(w, R, vis, ring, S, e0, e1, active, x,
                                                                        col1, y_begin, swap, al, KReg{K}, my_lut, fix);
          }
        } else {
          AffConsts K;
          if constexpr (AFFINE) load_affine<NL, SIG>(P, z, swap, K);
          pair_bilinear_staged<NL, OLK, SPLIT, SIG, false, Out>(w, R, vis, ring, S, e0, e1, active, x,
                                                                       col1, y_begin, swap, al, KReg{K}, my_lut, fix);
        }
      } else if (bilinear && active) {
        AffConsts K;
        if constexpr (AFFINE) load_affine<NL, SIG>(P, z, swap, K);
        const bool aligned_rows = ((s.src | s.pitch) & 3) == 0;
        if (vec && aligned_rows)
          pair_bilinear<NL, OLK, SPLIT, SIG, true, true, Out>(s, w, R, vis, x, col1, y_begin, swap, al, K, my_lut, fix);
        else if (vec)
          pair_bilinear<NL, OLK, SPLIT, SIG, false, true, Out>(s, w, R, vis, x, col1, y_begin, swap, al, K, my_lut,
                                                              fix);
        else
          pair_bilinear<NL, OLK, SPLIT, SIG, false, false, Out>(s, w, R, vis, x, col1, y_begin, swap, al, K, my_lut,
                                                               fix);
      } else if (active && !bilinear) {
        AffConsts K;
        if constexpr (AFFINE) load_affine<NL, SIG>(P, z, swap, K);
        pair_tap<NL, OLK, SPLIT, SIG, Out>(s, w, R, x, col1, y_begin, y_end, swap, al, K, my_lut);
      }
    }
    if (bilinear) {  // the filter's flagged pixels, exactly (__syncwarp orders them after the walk's stores)
      __syncwarp();
      const uint32_t n = min(fixs.n, kFixCap);
      for (uint32_t i = lane; i < n; i += 32) {
        const uint32_t ent = fixs.e[i], y = y_begin + (ent >> 5);
        const uint32_t tse = blockIdx.x * 32 + (ent & 31u), he = tse / T, ze = plane_of(c, he);
        const uint32_t xp = 2 * (tse - he * T);
        fix_pair<NL, OLK, SPLIT, SIG, Out>(P, ze, xp, y, lut + (AFFINE ? 0 : he * NL * 256));
      }
      if (fix.ovf)
        for (uint32_t y = y_begin; y < y_end; ++y) fix_pair<NL, OLK, SPLIT, SIG, Out>(P, z, x, y, my_lut);
    }
  }
}

}  // namespace fk
