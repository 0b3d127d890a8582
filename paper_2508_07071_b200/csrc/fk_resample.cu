// fk_resample.cu — compiled kernel for batched u8 crop/resize pipelines
// (the cvGS / FastNPP preprocessing family: PAPER.md:695-703, configs[1,3,4]).
//
//   BatchRead(Crop -> Resize{nearest,bilinear} | Crop | PerThreadRead) of u8 / u8x3
//     -> a lane-wise chain -> Write (packed) or SplitWrite (planar)
//
// One CTA walks a contiguous tile range of one plane z (blockIdx.z: horizontal
// fusion); everything between the read and the write stays in registers
// (vertical fusion). Per CTA and plane, shared memory holds the sampling
// coordinates of every output column (struct-of-arrays, read with 128-bit
// loads) and of the CTA's rows, so center_coord/floor/clamp (ops.cpp:253-270)
// run once per column/row instead of once per pixel.
//
// Two chain modes, picked on the host:
//  * AFFINE: Cast(u8 -> f32) [+ SwapRB] then a registered straight-line chain of
//    f32 Mul/Add/Sub/Div (fk_sig.cuh), compiled into the kernel as a template
//    signature, constants per lane (and optionally per plane) in registers —
//    the normalisation chain of configs[1,3,4]. A division whose reciprocal form
//    the host verified on all 256 reachable inputs uses it (3 FP32 ops).
//  * LUT: any lane-wise chain (folded unaries + Cast / arith / SwapRB /
//    StaticLoop / BatchArith, any length): after a u8 read each output lane is
//    a function of one byte, so the chain is evaluated once per byte value
//    (by the same device ops as the interpreter) into a 256-entry table.
// Both are bit-exact with the reference by construction.
#include <cuda_runtime.h>

#include <type_traits>

#include "fk_launch.hpp"
#include "fk_sig.cuh"
#include "fk_stages.cuh"

namespace fk {

namespace {

constexpr int kE = 4;  // output pixels per tile (one 16-byte f32 store per planar lane)

// The sampled u8 lanes of one output pixel: taps at byte offsets o0/o1 of the
// rows r0/r1 (bilinear_sample, ops.cpp:259-299) or one tap at o0 of r0.
template <int NL>
__device__ __forceinline__ void sample_u8(bool bilinear, const uint8_t* r0, const uint8_t* r1, uint32_t o0,
                                          uint32_t o1, double fx, double fy, uint32_t (&out)[3]) {
  if (bilinear) {
    uint32_t ta[3], tb[3], tc[3], td[3];
    if constexpr (NL == 3) {
      uint32_t a, b, c, d;
      dev::load_u8x3_taps(r0, o0, o1, a, b);
      dev::load_u8x3_taps(r1, o0, o1, c, d);
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
    constexpr double kTwo52 = 4503599627370496.0;  // 2^52: (2^52 + v) has v in its low word
    constexpr double kRound = 6755399441055744.0;  // 1.5 * 2^52: adding it rounds to an integer, ties-to-even
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      // a + (b - a) * fx, c + (d - c) * fx, top + (bot - top) * fy in double (ops.cpp:283-296)
      const double A = __hiloint2double(0x43300000, int(ta[l]));
      const double B = __hiloint2double(0x43300000, int(tb[l]));
      const double C = __hiloint2double(0x43300000, int(tc[l]));
      const double D = __hiloint2double(0x43300000, int(td[l]));
      const double top = __dadd_rn(__dsub_rn(A, kTwo52), __dmul_rn(__dsub_rn(B, A), fx));
      const double bot = __dadd_rn(__dsub_rn(C, kTwo52), __dmul_rn(__dsub_rn(D, C), fx));
      const double res = __dadd_rn(top, __dmul_rn(__dsub_rn(bot, top), fy));
      out[l] = uint32_t(__double2loint(__dadd_rn(res, kRound)));  // round_clamp_u8: res is in [0, 255]
    }
  } else {  // nearest / direct: one tap
    const uint8_t* p = r0 + o0;
#pragma unroll
    for (int l = 0; l < NL; ++l) out[l] = __ldg(p + l);
  }
}

}  // namespace

template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG>
__global__ void __launch_bounds__(kBlock, 3) fk_resample(const __grid_constant__ DPlan P) {
  constexpr bool AFFINE = SIG != kSigLut;
  using Out = typename std::conditional<OLK == FK_F64, uint64_t, uint32_t>::type;
  constexpr int OB = OLK == FK_U8 ? 1 : (OLK == FK_F32 ? 4 : 8);  // bytes per output lane
  __shared__ XTab xt;
  __shared__ YEnt yt[kYCap];
  __shared__ Out lut[AFFINE ? 1 : NL][AFFINE ? 1 : 256];
  const uint32_t t_begin = blockIdx.x * P.tiles_per_cta;
  if (t_begin >= P.tiles) return;
  const uint32_t t_end = min(t_begin + P.tiles_per_cta, P.tiles);
  const uint32_t y_first = dev::fastdiv(t_begin, P.tpr);
  const uint32_t rows = dev::fastdiv(t_end - 1, P.tpr) - y_first + 1;
  const bool tab = P.width <= kXCap && rows <= kYCap;
  for (uint32_t zi = blockIdx.z; zi < P.batch; zi += gridDim.z) {
    const uint32_t z = P.order ? __ldg(P.order + zi) : zi;
    const DSample s = P.reads[z];
    const DWrite w = P.writes[z];
    const bool swap = ((s.flags & SF_POST_SWAP) != 0) != (P.prog_swap != 0);
    const uint8_t* base = reinterpret_cast<const uint8_t*>(s.src);
    const bool resampling = s.mode != RD_DIRECT;
    const bool bilinear = s.mode == RD_BILINEAR;
    // AFFINE: the chain's constants (and reciprocals) of plane z in registers
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
    if (tab && resampling) dev::build_tables(s, P.width, y_first, rows, xt, yt);
    if constexpr (!AFFINE) {
      for (uint32_t t = threadIdx.x; t < 256; t += kBlock) {  // the chain over every byte value
        uint64_t v[1][3] = {{t, t, t}};
        dev::run_ops(P, s.post_off, s.post_len, z, v);
        dev::run_ops(P, P.op_base, P.n_ops, z, v);
#pragma unroll
        for (int l = 0; l < NL; ++l) lut[l][t] = Out(v[0][l]);
      }
    }
    __syncthreads();
    if (!(w.flags & WF_ACTIVE)) continue;  // BatchWrite z >= active_count
    const bool st = (w.flags & WF_STREAM) != 0;
    for (uint32_t t = t_begin + threadIdx.x; t < t_end; t += kBlock) {
      const uint32_t y = dev::fastdiv(t, P.tpr);
      const uint32_t x = (t - y * P.tiles_per_row) * kE;
      const int n = (P.width - x) < uint32_t(kE) ? int(P.width - x) : kE;
      // row and column coordinates of this tile
      YEnt ye;
      uint32_t o[kE];
      double f[kE];
      if (!resampling) {
        ye.r0 = ye.r1 = uint64_t(s.y0 + y) * s.pitch;
        ye.f = 0.0;
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          o[e] = (s.x0 + x + uint32_t(e < n ? e : 0)) * NL | kEdge;
          f[e] = 0.0;
        }
      } else if (tab) {
        ye = yt[y - y_first];
        dev::load_xtab<kE>(xt, x, o, f);
      } else {
        ye = dev::y_entry(s, y);
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          const XEnt xe = dev::x_entry(s, x + uint32_t(e < n ? e : 0), NL);
          o[e] = xe.o0 | (xe.o1 == xe.o0 ? kEdge : 0u);
          f[e] = xe.f;
        }
      }
      Out out[kE][NL];
#pragma unroll
      for (int e = 0; e < kE; ++e) {
        const uint32_t o0 = o[e] & ~kEdge, o1 = (o[e] & kEdge) ? o0 : o0 + NL;
        uint32_t u[3];
        sample_u8<NL>(bilinear, base + ye.r0, base + ye.r1, o0, o1, f[e], ye.f, u);
        if constexpr (NL == 3) {
          if (swap) { const uint32_t tmp = u[0]; u[0] = u[2]; u[2] = tmp; }
        }
        if constexpr (AFFINE) {
#pragma unroll
          for (int l = 0; l < NL; ++l) {
            float c[4], r[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              c[k] = k < sig_n(SIG) ? acst[k][l] : 0.f;
              r[k] = k < sig_n(SIG) ? arcp[k][l] : 0.f;
            }
            // Cast u8 -> f32 (exact), then the compiled chain
            out[e][l] = Out(__float_as_uint(sig_apply<SIG>(float(u[l]), c, r)));
          }
        } else {
#pragma unroll
          for (int l = 0; l < NL; ++l) out[e][l] = lut[l][u[l]];
        }
      }
      if constexpr (SPLIT) {  // split_block, ops.cpp:402-424: lane l -> plane l
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          uint8_t* p = reinterpret_cast<uint8_t*>(w.dst[l]) + uint64_t(y) * w.pitch[l] + uint64_t(x) * OB;
          if (n == kE && (reinterpret_cast<uintptr_t>(p) & 3) == 0) {
            Out s4[kE][1];
#pragma unroll
            for (int e = 0; e < kE; ++e) s4[e][0] = out[e][l];
            uint32_t wd[kE * OB / 4];
            dev::encode<OLK, Out, 1, kE>(s4, wd);
            dev::store_words<kE * OB / 4>(p, wd, st);
          } else {
            for (int e = 0; e < n; ++e)
              dev::store_lane<OLK, Out>(p + e * OB, out[e][l], (w.flags & WF_LANE_ALIGNED) != 0);
          }
        }
      } else {  // store_block, ops.cpp:396-400: packed NL-lane elements
        constexpr uint32_t K = NL == 3 ? OLK + 3 : OLK;
        constexpr int NB = kE * OB * NL;
        uint8_t* p = reinterpret_cast<uint8_t*>(w.dst[0]) + uint64_t(y) * w.pitch[0] + uint64_t(x) * OB * NL;
        if (NB % 4 == 0 && n == kE && (reinterpret_cast<uintptr_t>(p) & 3) == 0) {
          uint32_t wd[(NB + 3) / 4];
          dev::encode<K, Out, NL, kE>(out, wd);
          dev::store_words<(NB + 3) / 4>(p, wd, st);
        } else {
          for (int e = 0; e < n; ++e)
            for (int l = 0; l < NL; ++l)
              dev::store_lane<OLK, Out>(p + (e * NL + l) * OB, out[e][l], (w.flags & WF_LANE_ALIGNED) != 0);
        }
      }
    }
  }
}

int resample_elems() { return kE; }

bool resample_affine_registered(uint32_t sig) {
#define FK_CASE(S) if (sig == (S)) return true;
  FK_AFFINE_SIGS(FK_CASE)
#undef FK_CASE
  return false;
}

cudaError_t launch_resample(int src_lanes, uint32_t out_lane_kind, bool split, uint32_t sig, const DPlan& P,
                            cudaStream_t st) {
  if (P.tiles == 0 || P.batch == 0) return cudaSuccess;
  const dim3 grid((P.tiles + P.tiles_per_cta - 1) / P.tiles_per_cta, 1, P.batch < 65535u ? P.batch : 65535u);
#define FK_RS(NL, OLK, SP, S) fk_resample<NL, OLK, SP, S><<<grid, kBlock, 0, st>>>(P)
  if (sig != kSigLut) {  // AFFINE: f32 outputs
#define FK_CASE(S)                                   \
  if (sig == (S)) {                                  \
    if (src_lanes == 3 && split) FK_RS(3, FK_F32, true, S);        \
    else if (src_lanes == 3) FK_RS(3, FK_F32, false, S);           \
    else FK_RS(1, FK_F32, false, S);                                \
    return cudaGetLastError();                       \
  }
    FK_AFFINE_SIGS(FK_CASE)
#undef FK_CASE
    return cudaErrorInvalidValue;  // unregistered signature: the host picks LUT mode instead
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
