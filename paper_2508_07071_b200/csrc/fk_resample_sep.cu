// fk_resample_sep.cu — instantiations and launch of the column-streaming
// kernel (fk_resample_sep.cuh): the registered AFFINE chains and LUT mode.
#include "fk_resample_sep.cuh"

namespace fk {

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
