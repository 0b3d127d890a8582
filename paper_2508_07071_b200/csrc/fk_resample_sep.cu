// fk_resample_sep.cu — instantiations of the column-streaming kernel
// (fk_resample_sep.cuh): AFFINE chains with their constants in the kernel
// parameters, and LUT mode. Per-plane (BatchArith) AFFINE chains are in
// fk_resample_sep_pz.cu.
#include "fk_resample_sep.cuh"

namespace fk {

uint32_t resample_sep_band_max() { return kBandMax; }

cudaError_t launch_resample_sep(int src_lanes, uint32_t out_lane_kind, bool split, uint32_t sig, const DPlan& P,
                                uint32_t block, cudaStream_t st) {
  if (P.width == 0 || P.height == 0 || P.batch == 0) return cudaSuccess;
  const dim3 grid = sep_grid(P, block);
  if (sig != kSigLut) {
    if (!P.aff_inline) return launch_resample_sep_pz(src_lanes, split, sig, P, grid, block, st);
#define FK_CASE(S) \
  if (sig == (S)) return launch_sep_affine<S, false>(src_lanes, split, P, grid, block, st);
    FK_AFFINE_SIGS(FK_CASE)
#undef FK_CASE
    return cudaErrorInvalidValue;
  }
#define FK_RS(NL, OLK, SP) fk_resample_sep<NL, OLK, SP, kSigLut, false><<<grid, block, 0, st>>>(P)
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
