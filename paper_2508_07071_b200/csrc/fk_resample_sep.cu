// fk_resample_sep.cu — instantiations and launch of the column-streaming
// kernel (fk_resample_sep.cuh): the registered AFFINE chains and LUT mode.
#include "fk_resample_sep.cuh"

namespace fk {

uint32_t resample_sep_band_max() { return kBandMax; }
uint32_t resample_sep_ring_row() { return kRingRow; }

cudaError_t launch_resample_sep(int src_lanes, uint32_t out_lane_kind, bool split, uint32_t sig, const DPlan& P,
                                bool staged, cudaStream_t st) {
  if (P.width == 0 || P.height == 0 || P.batch == 0) return cudaSuccess;
  // one warp per CTA: 32 pair slots of a slice (P.slot_threads pairs per plane slot)
  const uint32_t spc = P.slots ? P.slots_per_cta : 1u;
  const uint32_t slices = P.slots ? P.slices : P.batch;
  const dim3 grid((spc * P.slot_threads + 31) / 32, (P.height + P.tiles_per_cta - 1) / P.tiles_per_cta,
                  slices < 65535u ? slices : 65535u);
  const uint32_t block = 32;
#define FK_RS(NL, OLK, SP, S)                                                     \
  do {                                                                            \
    if (staged) fk_resample_sep<NL, OLK, SP, S, true><<<grid, block, 0, st>>>(P); \
    else fk_resample_sep<NL, OLK, SP, S, false><<<grid, block, 0, st>>>(P);       \
  } while (0)
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
