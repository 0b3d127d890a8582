// fk_crop.cu — the planar crop kernel: a batch of crops of u8x3 frames,
// bilinear-resized (ops.cpp:259-299), [SwapRB], cast to f32, an f32 chain
// (sub mean / div std, ...) and split into three f32 planes, one fused launch
// (configs[1], [3], [4]; blockIdx.x = plane x row band: horizontal fusion).
//
// Bilinear is separable, and the kernel computes it vertical-first, in two
// phases per tile of 7 output rows, through shared memory:
//
//  phase 1  one warp per output row: the vertical lerp of the two source rows
//           over the crop's whole source span, EXACTLY, in integers — one
//           dp2a per lane value: K (den - ny) a + K ny b with the reference's
//           fy = ny / den (den = 2 out_h; see CropRow). The sum lands in the
//           mantissa of the biased float 2^17 (bias added by the dp2a), so the
//           V row holds exact values as floats. Loads are coalesced 4-byte
//           words of the source rows; stores are 16-byte, conflict-free.
//  phase 2  one thread per output quad (4 columns) and row: the horizontal
//           lerp in FP32 (two columns per FFMA2), the exact-result filter, the
//           cast + chain in packed FP32 and one 128-bit streaming store per
//           destination plane.
//
// Exact-result filter. The FP32 value v of a lane differs from the exact
// rational bilinear result R by at most 4.6e-5 (hb rounding 2^-7 + fx rounding
// 2^-25 |d| in V units of 1/(K den / 64) pixel; the scale s rounded, 2^-24 v;
// the final rounding 2^-17), and the reference's double result differs from R
// by < 1e-12. So when |v - rint(v)| <= 0.5 - E (E = 2^-13) the reference's
// nearbyint(res) is rint(v). Lanes within E of a half-integer are flagged and
// their quad is recomputed after the tile with the reference's double
// arithmetic op for op. When fx and fy are multiples of 2^-8 and 1/64 every
// FP32 step is exact (CropRow: den = 64, K = 256), v == R, and the check is
// off (threshold 0.5): exact ties (e.g. 448 -> 224) then round to even like
// the double does.
#include <cuda_runtime.h>

#include "fk_crop.hpp"
#include "fk_stages.cuh"
#include "fk_sig.cuh"

#ifndef FK_CROP_MINB
#define FK_CROP_MINB 3
#endif
namespace fk {

namespace {

// ---------------------------------------------------------- packed FP32 --
// Two f32 lanes in one 64-bit register pair: FADD2 / FMUL2 / FFMA2 on sm_100,
// each lane rounded exactly like the scalar op.
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
}  // namespace p2

constexpr float kE = 1.0f / 16384.0f;         // 2^-14 (> the 4.5e-5 bound, see the header)
constexpr float kRound = 12582912.0f;         // 1.5 * 2^23: x + kRound rounds x to an integer (ties to even)

// The chain's constants for input lane m, op k, as pairs: c, and for a
// division either (r_hi, r_lo) [two-op form] or (RN(1/c), -c) [three-op form].
struct KInl {
  const CropPlan& P;
  __device__ __forceinline__ uint64_t c(int k, int m) const { return p2::of(P.kc[k][m]); }
  __device__ __forceinline__ uint64_t h(int k, int m) const { return p2::of(P.kh[k][m]); }
  __device__ __forceinline__ uint64_t l(int k, int m) const { return p2::of(P.kl[k][m]); }
};
template <uint32_t SIG>
struct KReg {
  uint64_t cc[4][3], hh[4][3], ll[4][3];
  __device__ __forceinline__ KReg(const float4* kz) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        if (k < sig_n(SIG)) {
          const float4 v = __ldg(kz + 3 * k + m);
          cc[k][m] = p2::pack(v.x, v.x);
          hh[k][m] = p2::pack(v.y, v.y);
          ll[k][m] = p2::pack(v.z, v.z);
        } else {
          cc[k][m] = hh[k][m] = ll[k][m] = 0;
        }
      }
  }
  __device__ __forceinline__ uint64_t c(int k, int m) const { return cc[k][m]; }
  __device__ __forceinline__ uint64_t h(int k, int m) const { return hh[k][m]; }
  __device__ __forceinline__ uint64_t l(int k, int m) const { return ll[k][m]; }
};

__host__ __device__ constexpr bool div2(uint32_t sig, int k) { return (sig >> (kCropDiv2 + k)) & 1u; }

// The registered chain on a column pair (same IEEE ops, same order as the
// reference's arith ops, ops.cpp:88-159; divisions in a host-verified form).
template <uint32_t SIG, int K, class KS>
__device__ __forceinline__ uint64_t chain_op2(uint64_t x, const KS& ks, int m) {
  constexpr uint32_t fn = sig_fn(SIG, K);
  if constexpr (fn == AF_MUL) return p2::mul(x, ks.c(K, m));
  else if constexpr (fn == AF_ADD) return p2::add(x, ks.c(K, m));
  else if constexpr (fn == AF_SUB) return p2::sub(x, ks.c(K, m));
  else if constexpr (div2(SIG, K)) return p2::fma(x, ks.h(K, m), p2::mul(x, ks.l(K, m)));
  else if constexpr (sig_fast(SIG, K)) {  // q = x r; e = fma(-q, c, x) [l holds -c]; q + e r
    const uint64_t q = p2::mul(x, ks.h(K, m));
    const uint64_t e = p2::fma(q, ks.l(K, m), x);
    return p2::fma(e, ks.h(K, m), q);
  } else {
    const float c = p2::lo(ks.c(K, m));
    return p2::pack(__fdiv_rn(p2::lo(x), c), __fdiv_rn(p2::hi(x), c));
  }
}
template <uint32_t SIG, class KS>
__device__ __forceinline__ uint64_t chain2(uint64_t x, const KS& ks, int m) {
  if constexpr (sig_n(SIG) > 0) x = chain_op2<SIG, 0>(x, ks, m);
  if constexpr (sig_n(SIG) > 1) x = chain_op2<SIG, 1>(x, ks, m);
  if constexpr (sig_n(SIG) > 2) x = chain_op2<SIG, 2>(x, ks, m);
  if constexpr (sig_n(SIG) > 3) x = chain_op2<SIG, 3>(x, ks, m);
  return x;
}

// The same chain on one value, in plain IEEE ops (the fix path).
template <uint32_t SIG, class KS>
__device__ __forceinline__ float chain1(float v, const KS& ks, int m) {
#pragma unroll
  for (int k = 0; k < sig_n(SIG); ++k) {
    const float c = p2::lo(ks.c(k, m));
    switch (sig_fn(SIG, k)) {
      case AF_MUL: v = __fmul_rn(v, c); break;
      case AF_ADD: v = __fadd_rn(v, c); break;
      case AF_SUB: v = __fsub_rn(v, c); break;
      default: v = __fdiv_rn(v, c); break;
    }
  }
  return v;
}

// The reference's bilinear value of one lane in double, op for op
// (ops.cpp:250,283-296), rounded like round_clamp_u8 (nearbyint; the value is
// in [0, 255]), returned as the float of the u8 result.
__device__ __forceinline__ float exact_lane(uint32_t a, uint32_t b, uint32_t c, uint32_t d, double fx, double fy) {
  const double top = __dadd_rn(double(a), __dmul_rn(__dsub_rn(double(b), double(a)), fx));
  const double bot = __dadd_rn(double(c), __dmul_rn(__dsub_rn(double(d), double(c)), fx));
  const double res = __dadd_rn(top, __dmul_rn(__dsub_rn(bot, top), fy));
  return float(uint32_t(__double2loint(__dadd_rn(res, 6755399441055744.0))) & 0xffu);
}

// Scalar constants of the fix path (per-plane block or the kernel parameters).
struct K1 {
  const CropPlan& P;
  const float4* kz;
  __device__ __forceinline__ uint64_t c(int k, int m) const {
    return kz ? p2::pack(__ldg(kz + 3 * k + m).x, 0.f) : p2::of(P.kc[k][m]);
  }
};

// One lane value of output pixel (x, y) of plane z exactly as the reference
// computes it (bilinear_sample in double, ops.cpp:259-299, round_clamp_u8, the
// chain in IEEE f32), stored to its destination plane. The flagged quads of a
// tile are fixed by whole warps, lane = (column, channel) of the quad.
template <uint32_t SIG, bool PERZ>
__device__ __noinline__ void fix_value(const CropPlan& P, uint32_t z, uint32_t x, uint32_t y, int m) {
  const DSample s = P.reads[z];
  const CropAux A = P.aux[z];
  const DWrite& w = P.writes[z];
  const K1 ks{P, PERZ ? P.kz + 12ull * A.kz : nullptr};
  const YEnt ye = dev::y_entry(s, y);
  const XEnt xe = dev::x_entry(s, x, 3);
  const uint8_t* r0 = reinterpret_cast<const uint8_t*>(s.src) + ye.r0;
  const uint8_t* r1 = reinterpret_cast<const uint8_t*>(s.src) + ye.r1;
  const float u = exact_lane(__ldg(r0 + xe.o0 + m), __ldg(r0 + xe.o1 + m), __ldg(r1 + xe.o0 + m),
                             __ldg(r1 + xe.o1 + m), xe.f, ye.f);
  const int d = A.swap ? 2 - m : m;
  __stcs(reinterpret_cast<float*>(w.dst[d] + uint64_t(y) * w.pitch[d]) + x, chain1<SIG>(u, ks, m));
}

// ------------------------------------------------------- bulk copies (TMA) --
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra.uni WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

// Per tile row (prepared one tile ahead by warp 0): staged-row byte offsets of
// the two source rows, the dp2a weights, the exact-row flag.
struct TileRow {
  uint32_t pa, pb, wts, exact;
};

// ------------------------------------------------------------------ kernel --
// One CTA = one plane (blockIdx.x / bands, in P.order) x one band of output
// rows, walked in tiles of 7 rows. Per tile:
//   stage   warp 0 copies the tile's source rows [iy0(first), iy1(last)]
//           (relative to y0) into shared memory with one cp.async.bulk (TMA)
//           per row, one tile AHEAD (completion on an mbarrier), and writes
//           the tile's row table;
//   phase 1 (warp = output row) staged rows -> V row (exact vertical lerp);
//   phase 2 (thread = quad x row lane) V -> horizontal lerp, filter, chain,
//           three 128-bit streaming stores; flagged quads are appended to the
//           tile's fix list;
//   fix     flagged quads in the reference's double arithmetic, two per warp pass.
template <uint32_t SIG, bool PERZ>
__global__ void __launch_bounds__(kCropThreads, FK_CROP_MINB) fk_crop(const __grid_constant__ CropPlan P) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* V = smem;                                         // kCropTileRows x v_stride
  unsigned char* ST = smem + kCropTileRows * P.v_stride;           // stage_rows x stage_stride
  float4* rowc = reinterpret_cast<float4*>(ST + P.stage_rows * P.stage_stride);  // [2][8] (s, s, c, c)
  TileRow* trow = reinterpret_cast<TileRow*>(rowc + 2 * kCropTileRows);            // [2][8]
  uint32_t* fixn = reinterpret_cast<uint32_t*>(trow + 2 * kCropTileRows);          // [2] counts
  uint64_t* mbar = reinterpret_cast<uint64_t*>(fixn + 2);                          // 8-byte aligned
  uint32_t* fixe = reinterpret_cast<uint32_t*>(mbar + 1);                          // [2][7 quads]: never overflows

  const uint32_t plane = blockIdx.x / P.bands, band = blockIdx.x - plane * P.bands;
  const uint32_t z = P.order ? P.order[plane] : plane;
  const DSample s = P.reads[z];
  const CropAux A = P.aux[z];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, wi = tid >> 5;
  const uint32_t quads = P.quads, nrl = kCropThreads / quads, fixcap = kCropTileRows * quads;
  const uint32_t q = tid % quads, rl = tid / quads;
  const uint32_t RS = A.nwords * 16u;
  const uint32_t SS = P.stage_stride;
  const uint32_t y_lo = band * P.band_rows, y_hi = min(P.out_h, y_lo + P.band_rows);
  const uint32_t bar = uint32_t(__cvta_generic_to_shared(mbar));

  // warp 0: stage tile ty into the buffer (one bulk copy per source row, one
  // row per lane) and its row table into slot b
  auto stage = [&](uint32_t ty, uint32_t b) {
    const uint32_t nr = min(kCropTileRows, y_hi - ty);
    const uint32_t lo = __ldg(&P.rows[A.rowtab + ty].iy) & 0x7fffu;
    const uint32_t hi = (__ldg(&P.rows[A.rowtab + ty + nr - 1].iy) >> 16) & 0x7fffu;
    const uint32_t full = A.nwords * 4u;
    const uint32_t lastb = min(full, A.rlim & ~15u);  // the crop's last row may end early
    if (lane == 0) mbar_expect_tx(bar, (hi - lo + 1) * full - (hi == s.rect_h - 1 ? full - lastb : 0u));
    __syncwarp();
    const uint32_t st = uint32_t(__cvta_generic_to_shared(ST));
    for (uint32_t r = lane; r <= hi - lo; r += 32) {
      const uint32_t n = lo + r == s.rect_h - 1 ? lastb : full;
      if (n) bulk_copy(st + r * SS, reinterpret_cast<const unsigned char*>(s.src) + A.wb + uint64_t(s.y0 + lo + r) * s.pitch,
                       n, bar);
    }
    if (lane < nr) {
      const CropRow R = P.rows[A.rowtab + ty + lane];
      trow[b * kCropTileRows + lane] =
          TileRow{((R.iy & 0x7fffu) - lo) * SS, (((R.iy >> 16) & 0x7fffu) - lo) * SS, R.wts, R.iy & kCropExact};
      rowc[b * kCropTileRows + lane] = make_float4(R.s, R.s, R.c, R.c);
    }
  };

  // per-thread column constants of quad q (once per plane)
  uint32_t offA[4];
  float fx[4], cthr[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t x = min(4 * q + c, P.out_w - 1);
    const CropCol C = P.cols[A.coltab + x];
    offA[c] = 4u * (3u * (s.x0 + (C.ix & ~kCropExact)) - A.wb);
    cthr[c] = (C.ix & kCropExact) ? 0.5f : 0.5f - kE;
    fx[c] = C.fx;
  }
  const uint64_t fxp[2] = {p2::pack(fx[0], fx[1]), p2::pack(fx[2], fx[3])};
  uint64_t dst[3];
  uint32_t dpitch;
  {
    const DWrite& w = P.writes[z];
    dpitch = uint32_t(w.pitch[0]);
#pragma unroll
    for (int m = 0; m < 3; ++m) dst[m] = w.dst[A.swap ? 2 - m : m] + 16ull * q;
  }
  using KS = typename std::conditional<PERZ, KReg<SIG>, KInl>::type;
  const KS ks = [&]() {
    if constexpr (PERZ) return KReg<SIG>(P.kz + 12ull * A.kz);
    else return KInl{P};
  }();

  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fixn[0] = fixn[1] = 0;
  }
  __syncthreads();
  if (wi == 0) stage(y_lo, 0);
  __syncthreads();  // tile 0's row table
  uint32_t t = 0;
  for (uint32_t ty = y_lo; ty < y_hi; ty += kCropTileRows, ++t) {
    const uint32_t nrows = min(kCropTileRows, y_hi - ty);
    const uint32_t tb = t & 1u;
    mbar_wait(bar, tb);  // tile t's source rows have landed
    // ---- phase 1: the V rows of the tile (exact vertical lerp): warp wi -> row wi,
    // the whole CTA -> row 7 (8 rows over 7 warps, balanced)
    auto vrow = [&](uint32_t r, uint32_t k0, uint32_t step) {
      const TileRow R = trow[tb * kCropTileRows + r];
      const uint32_t* pa = reinterpret_cast<const uint32_t*>(ST + R.pa);
      const uint32_t* pb = reinterpret_cast<const uint32_t*>(ST + R.pb);
      uint4* out = reinterpret_cast<uint4*>(V + r * RS);
#pragma unroll 4
      for (uint32_t k = k0; k < A.nwords; k += step) {
        const uint32_t a = pa[k], b = pb[k];
        const uint32_t q0 = __byte_perm(a, b, 0x5140), q1 = __byte_perm(a, b, 0x7362);
        uint4 v;
        v.x = __dp2a_lo(R.wts, q0, kCropBias);
        v.y = __dp2a_hi(R.wts, q0, kCropBias);
        v.z = __dp2a_lo(R.wts, q1, kCropBias);
        v.w = __dp2a_hi(R.wts, q1, kCropBias);
        out[k] = v;
      }
    };
    if (wi < nrows) vrow(wi, lane, 32);
    if (nrows > kCropWarps) vrow(kCropWarps, tid, kCropThreads);
    __syncthreads();  // V ready; the stage buffer is free
    if (tid == 0) fixn[tb ^ 1u] = 0;  // the next tile's list (last read before this barrier)
    if (wi == 0 && ty + kCropTileRows < y_hi) stage(ty + kCropTileRows, tb ^ 1u);
    // ---- phase 2: thread (rl, q) -> output quad q of rows ty + rl, ty + rl + nrl, ...
    if (rl < nrl) {
      for (uint32_t r = rl; r < nrows; r += nrl) {
        const float4 sc = rowc[tb * kCropTileRows + r];
        const uint64_t s2 = p2::pack(sc.x, sc.y), c2 = p2::pack(sc.z, sc.w);
        const float rthr = trow[tb * kCropTileRows + r].exact ? 0.5f : 0.5f - kE;
        const unsigned char* Vr = V + r * RS;
        const uint32_t y = ty + r;
        bool near = false;
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          uint64_t o[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const unsigned char* pa = Vr + offA[2 * j];
            const unsigned char* pb = Vr + offA[2 * j + 1];
            const uint64_t a = p2::pack(*reinterpret_cast<const float*>(pa + 4 * m),
                                        *reinterpret_cast<const float*>(pb + 4 * m));
            const uint64_t b = p2::pack(*reinterpret_cast<const float*>(pa + 12 + 4 * m),
                                        *reinterpret_cast<const float*>(pb + 12 + 4 * m));
            const uint64_t hb = p2::fma(p2::sub(b, a), fxp[j], a);   // biased: 2^17 + (K den / 64) h
            const uint64_t v = p2::fma(hb, s2, c2);                     // pixel units
            const uint64_t t2 = p2::add(v, p2::pack(kRound, kRound));
            const uint64_t k = p2::sub(t2, p2::pack(kRound, kRound));  // rint(v): the u8, as f32
            const uint64_t e = p2::sub(v, k);
            near |= fabsf(p2::lo(e)) > fminf(rthr, cthr[2 * j]);
            near |= fabsf(p2::hi(e)) > fminf(rthr, cthr[2 * j + 1]);
            o[j] = chain2<SIG>(k, ks, m);
          }
          float4* d = reinterpret_cast<float4*>(dst[m] + uint64_t(y) * dpitch);
          __stcs(d, make_float4(p2::lo(o[0]), p2::hi(o[0]), p2::lo(o[1]), p2::hi(o[1])));
        }
        if (near) fixe[tb * fixcap + atomicAdd(fixn + tb, 1u)] = (y << 8) | q;
      }
    }
    __syncthreads();  // V free; the fix list complete
    // ---- flagged quads: warp passes over the list, two quads per pass (lane = quad, column, channel)
    const uint32_t nf = fixn[tb];
    for (uint32_t i = 2 * wi; i < nf; i += 2 * kCropWarps) {
      const uint32_t e = i + lane / 12;
      const uint32_t ent = lane < 24 && e < nf ? fixe[tb * fixcap + e] : 0xffffffffu;
      const uint32_t l12 = lane % 12, x = 4 * (ent & 0xffu) + l12 / 3;
      if (ent != 0xffffffffu && x < P.out_w) fix_value<SIG, PERZ>(P, z, x, ent >> 8, int(l12 % 3));
    }
  }
}

}  // namespace

// Registered chains: the AFFINE signatures of fk_sig.cuh, with the two-op
// division variants of the normalising ones.
#define FK_CROP_SIGS(X)                                                              \
  X(sig_make(0))                                                                     \
  X(sig_make(1, AF_MUL)) X(sig_make(1, AF_ADD)) X(sig_make(1, AF_SUB))              \
  X(sig_make(1, AF_DIV)) X(sig_make(1, AF_DIV, 0, 0, 0, 1))                        \
  X(sig_make(1, AF_DIV) | (1u << kCropDiv2))                                         \
  X(sig_make(2, AF_SUB, AF_DIV)) X(sig_make(2, AF_SUB, AF_DIV, 0, 0, 2))            \
  X(sig_make(2, AF_SUB, AF_DIV) | (2u << kCropDiv2))                                 \
  X(sig_make(2, AF_MUL, AF_ADD)) X(sig_make(2, AF_SUB, AF_MUL))                     \
  X(sig_make(3, AF_MUL, AF_SUB, AF_DIV)) X(sig_make(3, AF_MUL, AF_SUB, AF_DIV, 0, 4)) \
  X(sig_make(3, AF_MUL, AF_SUB, AF_DIV) | (4u << kCropDiv2))

bool crop_registered(uint32_t sig) {
#define FK_CASE(S) if (sig == (S)) return true;
  FK_CROP_SIGS(FK_CASE)
#undef FK_CASE
  return false;
}

size_t crop_smem_bytes(uint32_t v_stride, uint32_t stage_rows, uint32_t stage_stride, uint32_t quads) {
  return size_t(kCropTileRows) * v_stride + size_t(stage_rows) * stage_stride +
         2 * kCropTileRows * (sizeof(float4) + sizeof(TileRow)) + 2 * sizeof(uint32_t) + sizeof(uint64_t) +
         2 * kCropTileRows * quads * sizeof(uint32_t);
}

cudaError_t launch_crop(uint32_t sig, bool per_plane, const CropPlan& P, uint32_t ctas, cudaStream_t st) {
  if (ctas == 0) return cudaSuccess;
  const size_t smem = crop_smem_bytes(P.v_stride, P.stage_rows, P.stage_stride, P.quads);
#define FK_RUN(S, PZ)                                                                  \
  do {                                                                                 \
    auto k = fk_crop<S, PZ>;                                                           \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));   \
    k<<<ctas, kCropThreads, smem, st>>>(P);                                            \
  } while (0)
#define FK_CASE(S)                        \
  if (sig == (S)) {                       \
    if (per_plane) FK_RUN(S, true);       \
    else FK_RUN(S, false);                \
    return cudaGetLastError();            \
  }
  FK_CROP_SIGS(FK_CASE)
#undef FK_CASE
#undef FK_RUN
  return cudaErrorInvalidValue;
}

}  // namespace fk
