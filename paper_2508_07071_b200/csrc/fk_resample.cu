// fk_resample.cu — compiled kernel for batched u8 crop/resize pipelines
// (the cvGS / FastNPP preprocessing family: PAPER.md:695-703, configs[1,3,4]).
//
//   BatchRead(Crop -> Resize{nearest,bilinear}) of u8 / u8x3 sources
//     -> any lane-wise chain (folded unaries + Cast / Mul / Add / Sub / Div /
//        SwapRB / StaticLoop / per-plane BatchArith)
//     -> Write (packed) or SplitWrite (planar)
//
// One CTA walks a contiguous tile range of one plane z (blockIdx.z, horizontal
// fusion). Per CTA and plane it builds, in shared memory,
//   * the sampling coordinates of every output column and of its rows (the
//     reference recomputes center_coord per pixel, ops.cpp:259-270), and
//   * the chain's value for each of the 256 u8 inputs per lane: the chain
//     after a u8 read is a lane-wise function of one byte, so evaluating it
//     once per byte value (with the same device ops as the interpreter) and
//     looking it up is bit-exact by construction.
// The per-pixel work is then: 2 tap gathers, the reference's double-precision
// lerps, one LUT load per lane, and 128-bit streaming stores.
#include <cuda_runtime.h>

#include "fk_launch.hpp"
#include "fk_stages.cuh"

namespace fk {

namespace {

constexpr int kE = 4;  // output pixels per tile (one 16-byte f32 store per planar lane)

// The sampled u8 lanes of output pixel (x, row entry ye) of plane s.
template <int NL>
__device__ __forceinline__ void sample_u8(const DSample& s, const uint8_t* base, const YEnt& ye, const XEnt& xe,
                                          uint32_t (&out)[3]) {
  const uint8_t* r0 = base + ye.r0;
  if (s.mode == RD_BILINEAR) {
    const uint8_t* r1 = base + ye.r1;
    uint32_t ta[3], tb[3], tc[3], td[3];
    if constexpr (NL == 3) {
      uint32_t a, b, c, d;
      dev::load_u8x3_taps(r0, xe.o0, xe.o1, a, b);
      dev::load_u8x3_taps(r1, xe.o0, xe.o1, c, d);
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        ta[l] = (a >> (8 * l)) & 0xffu;
        tb[l] = (b >> (8 * l)) & 0xffu;
        tc[l] = (c >> (8 * l)) & 0xffu;
        td[l] = (d >> (8 * l)) & 0xffu;
      }
    } else {
      ta[0] = __ldg(r0 + xe.o0);
      tb[0] = __ldg(r0 + xe.o1);
      tc[0] = __ldg(r1 + xe.o0);
      td[0] = __ldg(r1 + xe.o1);
    }
    constexpr double kTwo52 = 4503599627370496.0;  // 2^52
    constexpr double kRound = 6755399441055744.0;  // 1.5 * 2^52
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      // bilinear_sample, ops.cpp:283-296: a + (b - a) * fx, c + (d - c) * fx, top + (bot - top) * fy
      const double A = __hiloint2double(0x43300000, int(ta[l]));
      const double B = __hiloint2double(0x43300000, int(tb[l]));
      const double C = __hiloint2double(0x43300000, int(tc[l]));
      const double D = __hiloint2double(0x43300000, int(td[l]));
      const double top = __dadd_rn(__dsub_rn(A, kTwo52), __dmul_rn(__dsub_rn(B, A), xe.f));
      const double bot = __dadd_rn(__dsub_rn(C, kTwo52), __dmul_rn(__dsub_rn(D, C), xe.f));
      const double res = __dadd_rn(top, __dmul_rn(__dsub_rn(bot, top), ye.f));
      out[l] = uint32_t(__double2loint(__dadd_rn(res, kRound)));  // round_clamp_u8 (res in [0, 255])
    }
  } else {  // nearest / direct: one tap
    const uint8_t* p = r0 + xe.o0;
#pragma unroll
    for (int l = 0; l < NL; ++l) out[l] = __ldg(p + l);
  }
}

// Coordinates of a direct (non-resizing) read: source (x0 + x, y0 + y).
__device__ __forceinline__ XEnt direct_x(const DSample& s, uint32_t x, uint32_t bpe) {
  XEnt e;
  e.o0 = e.o1 = (s.x0 + x) * bpe;
  e.f = 0.0;
  return e;
}
__device__ __forceinline__ YEnt direct_y(const DSample& s, uint32_t y) {
  YEnt e;
  e.r0 = e.r1 = uint64_t(s.y0 + y) * s.pitch;
  e.f = 0.0;
  return e;
}

}  // namespace

template <int NL, uint32_t OLK, bool SPLIT>
__global__ void __launch_bounds__(kBlock, 3) fk_resample_lut(const __grid_constant__ DPlan P) {
  using Out = typename std::conditional<OLK == FK_F64, uint64_t, uint32_t>::type;
  constexpr int OB = OLK == FK_U8 ? 1 : (OLK == FK_F32 ? 4 : 8);  // bytes per output lane
  __shared__ XEnt xt[kXCap];
  __shared__ YEnt yt[kYCap];
  __shared__ Out lut[NL][256];
  const uint32_t t_begin = blockIdx.x * P.tiles_per_cta;
  if (t_begin >= P.tiles) return;
  const uint32_t t_end = min(t_begin + P.tiles_per_cta, P.tiles);
  const uint32_t y_first = dev::fastdiv(t_begin, P.tpr);
  const uint32_t rows = dev::fastdiv(t_end - 1, P.tpr) - y_first + 1;
  const bool tab = P.width <= kXCap && rows <= kYCap;
  for (uint32_t z = blockIdx.z; z < P.batch; z += gridDim.z) {
    const DSample s = P.reads[z];
    const DWrite w = P.writes[z];
    const bool swap = ((s.flags & SF_POST_SWAP) != 0) != (P.prog_swap != 0);
    const uint8_t* base = reinterpret_cast<const uint8_t*>(s.src);
    __syncthreads();
    if (tab && s.mode != RD_DIRECT) dev::build_tables(s, P.width, y_first, rows, xt, yt);
    for (uint32_t t = threadIdx.x; t < 256; t += kBlock) {  // the chain over every byte value
      uint64_t v[1][3] = {{t, t, t}};
      dev::run_ops(P, s.post_off, s.post_len, z, v);
      dev::run_ops(P, P.op_base, P.n_ops, z, v);
#pragma unroll
      for (int l = 0; l < NL; ++l) lut[l][t] = Out(v[0][l]);
    }
    __syncthreads();
    if (!(w.flags & WF_ACTIVE)) continue;  // BatchWrite z >= active_count
    for (uint32_t t = t_begin + threadIdx.x; t < t_end; t += kBlock) {
      const uint32_t y = dev::fastdiv(t, P.tpr);
      const uint32_t x = (t - y * P.tiles_per_row) * kE;
      const int n = (P.width - x) < uint32_t(kE) ? int(P.width - x) : kE;
      const YEnt ye = s.mode == RD_DIRECT ? direct_y(s, y) : (tab ? yt[y - y_first] : dev::y_entry(s, y));
      Out o[kE][NL];
#pragma unroll
      for (int e = 0; e < kE; ++e) {
        const uint32_t xi = x + uint32_t(e < n ? e : 0);
        const XEnt xe = s.mode == RD_DIRECT ? direct_x(s, xi, NL) : (tab ? xt[xi] : dev::x_entry(s, xi, NL));
        uint32_t u[3];
        sample_u8<NL>(s, base, ye, xe, u);
        if constexpr (NL == 3) {
          o[e][0] = lut[0][swap ? u[2] : u[0]];
          o[e][1] = lut[1][u[1]];
          o[e][2] = lut[2][swap ? u[0] : u[2]];
        } else {
          o[e][0] = lut[0][u[0]];
        }
      }
      const bool st = (w.flags & WF_STREAM) != 0;
      if constexpr (SPLIT) {  // split_block, ops.cpp:402-424: lane l -> plane l
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          uint8_t* p = reinterpret_cast<uint8_t*>(w.dst[l]) + uint64_t(y) * w.pitch[l] + uint64_t(x) * OB;
          if (n == kE && (reinterpret_cast<uintptr_t>(p) & 3) == 0) {
            Out s4[kE][1];
#pragma unroll
            for (int e = 0; e < kE; ++e) s4[e][0] = o[e][l];
            uint32_t wd[kE * OB / 4];
            dev::encode<OLK, Out, 1, kE>(s4, wd);
            dev::store_words<kE * OB / 4>(p, wd, st);
          } else {
            for (int e = 0; e < n; ++e) dev::store_lane<OLK, Out>(p + e * OB, o[e][l], (w.flags & WF_LANE_ALIGNED) != 0);
          }
        }
      } else {  // store_block, ops.cpp:396-400: packed NL-lane elements
        constexpr uint32_t K = NL == 3 ? OLK + 3 : OLK;
        uint8_t* p = reinterpret_cast<uint8_t*>(w.dst[0]) + uint64_t(y) * w.pitch[0] + uint64_t(x) * OB * NL;
        if (n == kE && (kE * OB * NL) % 4 == 0 && (reinterpret_cast<uintptr_t>(p) & 3) == 0) {
          uint32_t wd[(kE * OB * NL + 3) / 4];
          dev::encode<K, Out, NL, kE>(o, wd);
          dev::store_words<(kE * OB * NL + 3) / 4>(p, wd, st);
        } else {
          for (int e = 0; e < n; ++e)
            for (int l = 0; l < NL; ++l)
              dev::store_lane<OLK, Out>(p + (e * NL + l) * OB, o[e][l], (w.flags & WF_LANE_ALIGNED) != 0);
        }
      }
    }
  }
}

int resample_elems() { return kE; }

cudaError_t launch_resample(int src_lanes, uint32_t out_lane_kind, bool split, const DPlan& P, cudaStream_t st) {
  if (P.tiles == 0 || P.batch == 0) return cudaSuccess;
  const dim3 grid((P.tiles + P.tiles_per_cta - 1) / P.tiles_per_cta, 1, P.batch < 65535u ? P.batch : 65535u);
#define FK_RS(NL, OLK, SP) fk_resample_lut<NL, OLK, SP><<<grid, kBlock, 0, st>>>(P)
  if (src_lanes == 3) {
    if (split) {
      if (out_lane_kind == FK_U8) FK_RS(3, FK_U8, true);
      else if (out_lane_kind == FK_F32) FK_RS(3, FK_F32, true);
      else FK_RS(3, FK_F64, true);
    } else {
      if (out_lane_kind == FK_U8) FK_RS(3, FK_U8, false);
      else if (out_lane_kind == FK_F32) FK_RS(3, FK_F32, false);
      else FK_RS(3, FK_F64, false);
    }
  } else {
    if (out_lane_kind == FK_U8) FK_RS(1, FK_U8, false);
    else if (out_lane_kind == FK_F32) FK_RS(1, FK_F32, false);
    else FK_RS(1, FK_F64, false);
  }
#undef FK_RS
  return cudaGetLastError();
}

}  // namespace fk
