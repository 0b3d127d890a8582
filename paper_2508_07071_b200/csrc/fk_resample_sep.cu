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
// H-lerp is computed once however many output rows use it, the V-lerp is the
// only per-pixel double work. Same double ops, same order: bit-exact.
//
//   CTA = a strip of up to 256 consecutive output columns x a band of rows of
//   one plane z (blockIdx.z, horizontal fusion). Per CTA and plane: the rows'
//   coordinates in shared memory, the chain's constants in registers (AFFINE:
//   Cast u8->f32 + a registered f32 chain) or its 256-entry table (LUT: any
//   lane-wise chain). Nearest and non-resizing planes take the same path with
//   one tap.
#include <cuda_runtime.h>

#include <type_traits>

#include "fk_launch.hpp"
#include "fk_sig.cuh"
#include "fk_stages.cuh"

namespace fk {

namespace {

constexpr uint32_t kBandMax = 64;  // output rows per CTA (host picks <= this)

// u8 lanes of the two taps of one source row (bytes at row + o0 and row + o1).
template <int NL>
__device__ __forceinline__ void taps_u8(const uint8_t* row, uint32_t o0, uint32_t o1, uint32_t& a, uint32_t& b) {
  if constexpr (NL == 3) {
    dev::load_u8x3_taps(row, o0, o1, a, b);
  } else {
    a = __ldg(row + o0);
    b = __ldg(row + o1);
  }
}

// Horizontal lerp of one source row for this column: a + (b - a) * fx in
// double per lane (ops.cpp:283-284), with 2^52 + v as the exact int->double.
template <int NL>
__device__ __forceinline__ void hlerp(const uint8_t* row, uint32_t o0, uint32_t o1, double fx, bool lerp,
                                      double (&h)[3]) {
  uint32_t a, b;
  taps_u8<NL>(row, o0, o1, a, b);
  constexpr double kTwo52 = 4503599627370496.0;
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const double A = __hiloint2double(0x43300000, int((a >> (8 * l)) & 0xffu));
    if (lerp) {
      const double B = __hiloint2double(0x43300000, int((b >> (8 * l)) & 0xffu));
      h[l] = __dadd_rn(__dsub_rn(A, kTwo52), __dmul_rn(__dsub_rn(B, A), fx));
    } else {
      h[l] = __dsub_rn(A, kTwo52);  // nearest / direct: the tap itself
    }
  }
}

}  // namespace

template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG>
__global__ void __launch_bounds__(256) fk_resample_sep(const __grid_constant__ DPlan P) {
  constexpr bool AFFINE = SIG != kSigLut;
  using Out = typename std::conditional<OLK == FK_F64, uint64_t, uint32_t>::type;
  constexpr int OB = OLK == FK_U8 ? 1 : (OLK == FK_F32 ? 4 : 8);
  __shared__ YEnt yt[kBandMax];
  __shared__ Out lut[AFFINE ? 1 : NL][AFFINE ? 1 : 256];
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t y_begin = blockIdx.y * P.tiles_per_cta;  // tiles_per_cta = band rows for this kernel
  const uint32_t y_end = min(y_begin + P.tiles_per_cta, P.height);
  for (uint32_t zi = blockIdx.z; zi < P.batch; zi += gridDim.z) {
    const uint32_t z = P.order ? __ldg(P.order + zi) : zi;
    const DSample s = P.reads[z];
    const DWrite w = P.writes[z];
    const bool swap = ((s.flags & SF_POST_SWAP) != 0) != (P.prog_swap != 0);
    const bool resampling = s.mode != RD_DIRECT;
    const bool bilinear = s.mode == RD_BILINEAR;
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
      if (resampling) {
        yt[j] = dev::y_entry(s, y_begin + j);
      } else {
        YEnt e;
        e.r0 = e.r1 = uint64_t(s.y0 + y_begin + j) * s.pitch;
        e.f = 0.0;
        yt[j] = e;
      }
    }
    if constexpr (!AFFINE) {
      for (uint32_t t = threadIdx.x; t < 256; t += blockDim.x) {  // the chain over every byte value
        uint64_t v[1][3] = {{t, t, t}};
        dev::run_ops(P, s.post_off, s.post_len, z, v);
        dev::run_ops(P, P.op_base, P.n_ops, z, v);
#pragma unroll
        for (int l = 0; l < NL; ++l) lut[l][t] = Out(v[0][l]);
      }
    }
    __syncthreads();
    if (!(w.flags & WF_ACTIVE) || x >= P.width) continue;  // BatchWrite z >= active_count / past the row
    // this column's taps
    uint32_t o0, o1;
    double fx = 0.0;
    if (resampling) {
      const XEnt xe = dev::x_entry(s, x, NL);
      o0 = xe.o0;
      o1 = xe.o1;
      fx = xe.f;
    } else {
      o0 = o1 = (s.x0 + x) * NL;
    }
    const uint8_t* base = reinterpret_cast<const uint8_t*>(s.src);
    const bool st = (w.flags & WF_STREAM) != 0;
    // horizontal lerps of the source rows used by the previous output row
    uint64_t held0 = ~uint64_t(0), held1 = ~uint64_t(0);
    double h0[3] = {0, 0, 0}, h1[3] = {0, 0, 0};
    for (uint32_t y = y_begin; y < y_end; ++y) {
      const YEnt ye = yt[y - y_begin];
      // rows advance monotonically: reuse a held row, else compute its H-lerp once
      double n0[3], n1[3];
      if (ye.r0 == held0) {
#pragma unroll
        for (int l = 0; l < 3; ++l) n0[l] = h0[l];
      } else if (ye.r0 == held1) {
#pragma unroll
        for (int l = 0; l < 3; ++l) n0[l] = h1[l];
      } else {
        hlerp<NL>(base + ye.r0, o0, o1, fx, bilinear, n0);
      }
      if (bilinear) {
        if (ye.r1 == ye.r0) {
#pragma unroll
          for (int l = 0; l < 3; ++l) n1[l] = n0[l];
        } else if (ye.r1 == held1) {
#pragma unroll
          for (int l = 0; l < 3; ++l) n1[l] = h1[l];
        } else {
          hlerp<NL>(base + ye.r1, o0, o1, fx, true, n1);
        }
      }
      held0 = ye.r0;
      held1 = bilinear ? ye.r1 : ye.r0;
      uint32_t u[3];
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        h0[l] = n0[l];
        h1[l] = bilinear ? n1[l] : n0[l];
      }
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        if (bilinear) {  // top + (bot - top) * fy, then round_clamp_u8 (res is in [0, 255])
          const double res = __dadd_rn(h0[l], __dmul_rn(__dsub_rn(h1[l], h0[l]), ye.f));
          u[l] = uint32_t(__double2loint(__dadd_rn(res, 6755399441055744.0)));
        } else {
          u[l] = uint32_t(__double2loint(__dadd_rn(h0[l], 4503599627370496.0)));  // exact small integer
        }
      }
      if constexpr (NL == 3) {
        if (swap) { const uint32_t t = u[0]; u[0] = u[2]; u[2] = t; }
      }
      Out o[NL];
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        if constexpr (AFFINE) {
          float c[4], r[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            c[k] = k < sig_n(SIG) ? acst[k][l] : 0.f;
            r[k] = k < sig_n(SIG) ? arcp[k][l] : 0.f;
          }
          o[l] = Out(__float_as_uint(sig_apply<SIG>(float(u[l]), c, r)));  // Cast u8 -> f32, chain
        } else {
          o[l] = lut[l][u[l]];
        }
      }
      const bool al = (w.flags & WF_LANE_ALIGNED) != 0;
      if constexpr (SPLIT) {  // split_block, ops.cpp:402-424
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          uint8_t* p = reinterpret_cast<uint8_t*>(w.dst[l]) + uint64_t(y) * w.pitch[l] + uint64_t(x) * OB;
          if constexpr (OLK == FK_F32) {
            if (al) {
              if (st) __stcs(reinterpret_cast<float*>(p), __uint_as_float(uint32_t(o[l])));
              else *reinterpret_cast<uint32_t*>(p) = uint32_t(o[l]);
              continue;
            }
          }
          dev::store_lane<OLK, Out>(p, o[l], al);
        }
      } else {  // store_block, ops.cpp:396-400
        uint8_t* p = reinterpret_cast<uint8_t*>(w.dst[0]) + uint64_t(y) * w.pitch[0] + uint64_t(x) * OB * NL;
#pragma unroll
        for (int l = 0; l < NL; ++l) dev::store_lane<OLK, Out>(p + l * OB, o[l], al);
      }
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
