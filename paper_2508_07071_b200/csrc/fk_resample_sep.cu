// fk_resample_sep.cu — column-streaming kernel for batched u8 crop/resize
// pipelines (configs[1], [3], [4]; the cvGS / FastNPP preprocessing family,
// PAPER.md:695-703).
//
// The reference's bilinear sample (ops.cpp:259-299) is
//     top = lerp(a, b, fx)   taps of source row sy0
//     bot = lerp(c, d, fx)   taps of source row sy1
//     res = lerp(top, bot, fy)
// and `top`/`bot` depend only on (source row, output column). So each thread
// owns ONE output column and walks down a band of output rows, holding the
// horizontal lerps of the two current source rows in registers: a source row's
// H-lerp is computed once however many output rows use it, and the V-lerp is
// the only per-pixel double work. Same double ops in the same order: bit-exact.
//
//   CTA = a strip of up to 256 consecutive output columns x a band of rows of
//   one plane z (blockIdx.z, horizontal fusion). Per CTA and plane: the rows'
//   coordinates in shared memory, the chain's constants in registers (AFFINE:
//   Cast u8->f32 + a registered f32 chain) or its 256-entry table (LUT: any
//   lane-wise chain). The plane's mode (bilinear / one tap) and whether its rows
//   are 4-byte aligned are resolved once per CTA into specialised loop bodies.
#include <cuda_runtime.h>

#include <type_traits>

#include "fk_launch.hpp"
#include "fk_sig.cuh"
#include "fk_stages.cuh"

namespace fk {

namespace {

constexpr uint32_t kBandMax = 64;  // output rows per CTA (host picks <= this)

struct RowEnt {                    // one output row: source rows (absolute) and fy
  uint32_t s0, s1;
  double f;
};

// Per-column gather geometry for 4-byte-aligned source rows: the taps' bytes
// [o0, o1 + 3) lie in words w[0..2] from (row + (o0 & ~3)); a word is loaded only
// if it holds one of those bytes (so nothing past the plane is touched).
struct ColGeom {
  uint32_t woff;         // byte offset of the first word within the row
  uint32_t sa, sb;       // funnel-shift amounts of tap 0 / tap 1 (bits)
  uint32_t need1, need2; // load word 1 / word 2
};

__device__ __forceinline__ ColGeom col_geom(uint32_t o0, uint32_t o1) {
  const uint32_t r = o0 & 3u, last = r + (o1 - o0) + 2;
  return ColGeom{o0 & ~3u, 8 * r, 8 * (r + (o1 - o0)), last >= 4 ? 1u : 0u, last >= 8 ? 1u : 0u};
}

// Load *p only if `need` (the value is unspecified otherwise; callers use only
// bytes of words they need).
__device__ __forceinline__ uint32_t ld_if(const uint32_t* p, uint32_t need) {
  uint32_t v;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.u32 %0, [%1];\n\t}"
               : "=r"(v) : "l"(p), "r"(need));
  return v;
}

// the two 3-byte taps of one source row (aligned-row fast path)
__device__ __forceinline__ void taps_aligned(const uint8_t* row, const ColGeom& g, uint32_t& a, uint32_t& b) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(row + g.woff);
  const uint32_t w0 = __ldg(w), w1 = ld_if(w + 1, g.need1), w2 = ld_if(w + 2, g.need2);
  a = __funnelshift_r(w0, w1, g.sa);
  b = g.sb < 32 ? __funnelshift_r(w0, w1, g.sb) : __funnelshift_r(w1, w2, g.sb - 32);
}

// byte l of v as a double: 2^52 + v is exact and its low word is v
__device__ __forceinline__ double byte_as_biased_double(uint32_t v, int l) {
  return __hiloint2double(0x43300000, int(__byte_perm(v, 0, 0x4440 | l)));
}

// Horizontal lerp a + (b - a) * fx of one source row, per lane (ops.cpp:283-284).
template <int NL>
__device__ __forceinline__ void hlerp(uint32_t a, uint32_t b, double fx, double (&h)[3]) {
  constexpr double kTwo52 = 4503599627370496.0;
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const double A = byte_as_biased_double(a, l), B = byte_as_biased_double(b, l);
    h[l] = __dadd_rn(__dsub_rn(A, kTwo52), __dmul_rn(__dsub_rn(B, A), fx));
  }
}

template <int NL, bool ALIGNED>
__device__ __forceinline__ void row_taps(const uint8_t* row, const ColGeom& g, uint32_t o0, uint32_t o1,
                                         uint32_t& a, uint32_t& b) {
  if constexpr (NL == 3) {
    if constexpr (ALIGNED) taps_aligned(row, g, a, b);
    else dev::load_u8x3_taps(row, o0, o1, a, b);
  } else {
    a = __ldg(row + o0);
    b = __ldg(row + o1);
  }
}

// The chain after the u8 read, on the lanes of one output pixel.
template <int NL, uint32_t OLK, uint32_t SIG, class Out>
__device__ __forceinline__ void chain(uint32_t (&u)[3], bool swap, const float (&acst)[4][3], const float (&arcp)[4][3],
                                      const Out* lut, Out (&o)[NL]) {
  if constexpr (NL == 3) {
    if (swap) { const uint32_t t = u[0]; u[0] = u[2]; u[2] = t; }
  }
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    if constexpr (SIG != kSigLut) {
      float c[4], r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        c[k] = k < sig_n(SIG) ? acst[k][l] : 0.f;
        r[k] = k < sig_n(SIG) ? arcp[k][l] : 0.f;
      }
      o[l] = Out(__float_as_uint(sig_apply<SIG>(float(u[l]), c, r)));  // Cast u8 -> f32, chain
    } else {
      o[l] = lut[l * 256 + u[l]];
    }
  }
}

// Destination cursor of one output column: the byte address of (x, y) in each
// destination plane, advanced by the pitch per output row.
template <int NL, uint32_t OLK, bool SPLIT>
struct ColOut {
  static constexpr int OB = OLK == FK_U8 ? 1 : (OLK == FK_F32 ? 4 : 8);
  static constexpr int ND = SPLIT ? 3 : 1;
  uint8_t* p[ND];
  uint64_t pitch[ND];
  __device__ __forceinline__ ColOut(const DWrite& w, uint32_t x, uint32_t y) {
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      pitch[d] = w.pitch[d];
      p[d] = reinterpret_cast<uint8_t*>(w.dst[d]) + uint64_t(y) * w.pitch[d] + uint64_t(x) * OB * (SPLIT ? 1 : NL);
    }
  }
  // split_block (ops.cpp:402-424) / store_block (:396-400) of one pixel, then next row
  template <bool AL, class Out>
  __device__ __forceinline__ void put(const Out (&o)[NL]) {
    if constexpr (SPLIT) {
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        if constexpr (OLK == FK_F32 && AL) __stcs(reinterpret_cast<float*>(p[l]), __uint_as_float(uint32_t(o[l])));
        else dev::store_lane<OLK, Out>(p[l], o[l], AL);
        p[l] += pitch[l];
      }
    } else {
#pragma unroll
      for (int l = 0; l < NL; ++l) dev::store_lane<OLK, Out>(p[0] + l * OB, o[l], AL);
      p[0] += pitch[0];
    }
  }
};

// V-lerp top + (bot - top) * fy per lane (ops.cpp:296), round_clamp_u8 (res is
// in [0, 255]), the chain, the store.
template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG, bool AL, class Out>
__device__ __forceinline__ void emit(const double (&top)[3], const double (&bot)[3], double fy, bool swap,
                                     const float (&acst)[4][3], const float (&arcp)[4][3], const Out* lut,
                                     ColOut<NL, OLK, SPLIT>& out) {
  uint32_t u[3];
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const double res = __dadd_rn(top[l], __dmul_rn(__dsub_rn(bot[l], top[l]), fy));
    u[l] = uint32_t(__double2loint(__dadd_rn(res, 6755399441055744.0)));
  }
  Out o[NL];
  chain<NL, OLK, SIG, Out>(u, swap, acst, arcp, lut, o);
  out.template put<AL>(o);
}

// Walk output rows [y0, y1) of column x (bilinear). hA / hB hold the H-lerps of
// source rows rA / rB; in state 0 hA is the top row, in state 1 hB is. When the
// next output row moves down by one source row (the common case for scales in
// (0.5, 2)) the old bottom becomes the new top by flipping the state, and only
// the new bottom row's H-lerp is computed — no register copies.
template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG, bool ALIGNED, bool AL, class Out>
__device__ __forceinline__ void column_bilinear(const DSample& s, const DWrite& w, const RowEnt* rows, uint32_t x,
                                                uint32_t y0, uint32_t y1, bool swap, const float (&acst)[4][3],
                                                const float (&arcp)[4][3], const Out* lut) {
  const XEnt xe = dev::x_entry(s, x, NL);
  const ColGeom g = col_geom(xe.o0, xe.o1);
  const uint8_t* base = reinterpret_cast<const uint8_t*>(s.src);
  ColOut<NL, OLK, SPLIT> out(w, x, y0);
  auto load = [&](uint32_t row, double (&h)[3]) {
    uint32_t a, b;
    row_taps<NL, ALIGNED>(base + uint64_t(row) * s.pitch, g, xe.o0, xe.o1, a, b);
    hlerp<NL>(a, b, xe.f, h);
  };
  uint32_t rA = 0xffffffffu, rB = 0xffffffffu;
  double hA[3] = {0, 0, 0}, hB[3] = {0, 0, 0};
  bool state1 = false;
  for (uint32_t y = y0; y < y1; ++y) {
    const RowEnt re = rows[y - y0];
    if (!state1) {  // top = A, bottom = B
      if (re.s0 == rA && re.s1 == rB) {
      } else if (re.s0 == rB && re.s1 != rB) {  // moved down one row: B becomes the top
        load(re.s1, hA);
        rA = re.s1;
        state1 = true;
        emit<NL, OLK, SPLIT, SIG, AL, Out>(hB, hA, re.f, swap, acst, arcp, lut, out);
        continue;
      } else {
        if (re.s0 != rA) { load(re.s0, hA); rA = re.s0; }
        if (re.s1 == re.s0) {
#pragma unroll
          for (int l = 0; l < 3; ++l) hB[l] = hA[l];
        } else if (re.s1 != rB) {
          load(re.s1, hB);
        }
        rB = re.s1;
      }
      emit<NL, OLK, SPLIT, SIG, AL, Out>(hA, hB, re.f, swap, acst, arcp, lut, out);
    } else {        // top = B, bottom = A
      if (re.s0 == rB && re.s1 == rA) {
      } else if (re.s0 == rA && re.s1 != rA) {  // moved down one row: A becomes the top
        load(re.s1, hB);
        rB = re.s1;
        state1 = false;
        emit<NL, OLK, SPLIT, SIG, AL, Out>(hA, hB, re.f, swap, acst, arcp, lut, out);
        continue;
      } else {
        if (re.s0 != rB) { load(re.s0, hB); rB = re.s0; }
        if (re.s1 == re.s0) {
#pragma unroll
          for (int l = 0; l < 3; ++l) hA[l] = hB[l];
        } else if (re.s1 != rA) {
          load(re.s1, hA);
        }
        rA = re.s1;
      }
      emit<NL, OLK, SPLIT, SIG, AL, Out>(hB, hA, re.f, swap, acst, arcp, lut, out);
    }
  }
}

// Nearest / non-resizing planes: one tap per output pixel.
template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG, bool AL, class Out>
__device__ __forceinline__ void column_tap(const DSample& s, const DWrite& w, const RowEnt* rows, uint32_t x,
                                           uint32_t y0, uint32_t y1, bool swap, const float (&acst)[4][3],
                                           const float (&arcp)[4][3], const Out* lut) {
  const uint32_t o0 = s.mode == RD_DIRECT ? (s.x0 + x) * NL : dev::x_entry(s, x, NL).o0;
  const uint8_t* base = reinterpret_cast<const uint8_t*>(s.src) + o0;
  ColOut<NL, OLK, SPLIT> out(w, x, y0);
  for (uint32_t y = y0; y < y1; ++y) {
    const uint8_t* p = base + uint64_t(rows[y - y0].s0) * s.pitch;
    uint32_t u[3];
#pragma unroll
    for (int l = 0; l < NL; ++l) u[l] = __ldg(p + l);
    Out o[NL];
    chain<NL, OLK, SIG, Out>(u, swap, acst, arcp, lut, o);
    out.template put<AL>(o);
  }
}

}  // namespace

template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG>
__global__ void __launch_bounds__(256, 4) fk_resample_sep(const __grid_constant__ DPlan P) {
  constexpr bool AFFINE = SIG != kSigLut;
  using Out = typename std::conditional<OLK == FK_F64, uint64_t, uint32_t>::type;
  __shared__ RowEnt rows[kBandMax];
  __shared__ Out lut[AFFINE ? 1 : NL * 256];
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t y_begin = blockIdx.y * P.tiles_per_cta;  // tiles_per_cta = band rows for this kernel
  const uint32_t y_end = min(y_begin + P.tiles_per_cta, P.height);
  for (uint32_t zi = blockIdx.z; zi < P.batch; zi += gridDim.z) {
    const uint32_t z = P.order ? __ldg(P.order + zi) : zi;
    const DSample s = P.reads[z];
    const DWrite w = P.writes[z];
    const bool swap = ((s.flags & SF_POST_SWAP) != 0) != (P.prog_swap != 0);
    float acst[4][3], arcp[4][3];
    if constexpr (AFFINE) {
#pragma unroll
      for (int k = 0; k < sig_n(SIG); ++k) {
        const DOp op = dev::prog_op(P, P.op_base + k);
        uint64_t c[3] = {op.c[0], op.c[1], op.c[2]};
        if (op.per_z) {
          const uint64_t* row = reinterpret_cast<const uint64_t*>(op.per_z) + 3ull * (z < op.per_z_n ? z : op.per_z_n - 1);
          c[0] = __ldg(row); c[1] = __ldg(row + 1); c[2] = __ldg(row + 2);
        }
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          acst[k][l] = __uint_as_float(uint32_t(c[op.nl == 3 ? l : 0]));
          arcp[k][l] = __frcp_rn(acst[k][l]);
        }
      }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < y_end - y_begin; j += blockDim.x) {
      RowEnt e;
      if (s.mode != RD_DIRECT) {  // y_entry gives row byte offsets; keep the source row numbers
        const YEnt ye = dev::y_entry(s, y_begin + j);
        e.s0 = uint32_t(ye.r0 / s.pitch);
        e.s1 = uint32_t(ye.r1 / s.pitch);
        e.f = ye.f;
      } else {
        e.s0 = e.s1 = s.y0 + y_begin + j;
        e.f = 0.0;
      }
      rows[j] = e;
    }
    if constexpr (!AFFINE) {
      for (uint32_t t = threadIdx.x; t < 256; t += blockDim.x) {  // the chain over every byte value
        uint64_t v[1][3] = {{t, t, t}};
        dev::run_ops(P, s.post_off, s.post_len, z, v);
        dev::run_ops(P, P.op_base, P.n_ops, z, v);
#pragma unroll
        for (int l = 0; l < NL; ++l) lut[l * 256 + t] = Out(v[0][l]);
      }
    }
    __syncthreads();
    if (!(w.flags & WF_ACTIVE) || x >= P.width) continue;  // BatchWrite z >= active_count / past the row
    const bool al = (w.flags & WF_LANE_ALIGNED) != 0;
    const bool aligned_rows = ((s.src | s.pitch) & 3) == 0;
    if (s.mode == RD_BILINEAR) {
      if (aligned_rows && al)
        column_bilinear<NL, OLK, SPLIT, SIG, true, true, Out>(s, w, rows, x, y_begin, y_end, swap, acst, arcp, lut);
      else if (al)
        column_bilinear<NL, OLK, SPLIT, SIG, false, true, Out>(s, w, rows, x, y_begin, y_end, swap, acst, arcp, lut);
      else
        column_bilinear<NL, OLK, SPLIT, SIG, false, false, Out>(s, w, rows, x, y_begin, y_end, swap, acst, arcp, lut);
    } else if (al) {
      column_tap<NL, OLK, SPLIT, SIG, true, Out>(s, w, rows, x, y_begin, y_end, swap, acst, arcp, lut);
    } else {
      column_tap<NL, OLK, SPLIT, SIG, false, Out>(s, w, rows, x, y_begin, y_end, swap, acst, arcp, lut);
    }
  }
}

uint32_t resample_sep_band_max() { return kBandMax; }

cudaError_t launch_resample_sep(int src_lanes, uint32_t out_lane_kind, bool split, uint32_t sig, const DPlan& P,
                                uint32_t block, cudaStream_t st) {
  if (P.width == 0 || P.height == 0 || P.batch == 0) return cudaSuccess;
  const dim3 grid((P.width + block - 1) / block, (P.height + P.tiles_per_cta - 1) / P.tiles_per_cta,
                  P.batch < 65535u ? P.batch : 65535u);
#define FK_RS(NL, OLK, SP, S) fk_resample_sep<NL, OLK, SP, S><<<grid, block, 0, st>>>(P)
  if (sig != kSigLut) {
#define FK_CASE(S)                                          \
  if (sig == (S)) {                                         \
    if (src_lanes == 3 && split) FK_RS(3, FK_F32, true, S); \
    else if (src_lanes == 3) FK_RS(3, FK_F32, false, S);    \
    else FK_RS(1, FK_F32, false, S);                        \
    return cudaGetLastError();                              \
  }
    FK_AFFINE_SIGS(FK_CASE)
#undef FK_CASE
    return cudaErrorInvalidValue;
  }
  if (src_lanes == 3) {
    if (split) {
      if (out_lane_kind == FK_U8) FK_RS(3, FK_U8, true, kSigLut);
      else if (out_lane_kind == FK_F32) FK_RS(3, FK_F32, true, kSigLut);
      else FK_RS(3, FK_F64, true, kSigLut);
    } else {
      if (out_lane_kind == FK_U8) FK_RS(3, FK_U8, false, kSigLut);
      else if (out_lane_kind == FK_F32) FK_RS(3, FK_F32, false, kSigLut);
      else FK_RS(3, FK_F64, false, kSigLut);
    }
  } else {
    if (out_lane_kind == FK_U8) FK_RS(1, FK_U8, false, kSigLut);
    else if (out_lane_kind == FK_F32) FK_RS(1, FK_F32, false, kSigLut);
    else FK_RS(1, FK_F64, false, kSigLut);
  }
#undef FK_RS
  return cudaGetLastError();
}

}  // namespace fk
