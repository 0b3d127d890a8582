// fk_resample_sep_pz.cu — the column-streaming kernel's AFFINE instantiations
// whose constants vary per plane (BatchArith, e.g. per-crop normalisation):
// each CTA loads its plane's row of constants into registers.
#include "fk_resample_sep.cuh"

namespace fk {

cudaError_t launch_resample_sep_pz(int src_lanes, bool split, uint32_t sig, const DPlan& P, dim3 grid,
                                   uint32_t block, cudaStream_t st) {
#define FK_CASE(S) \
  if (sig == (S)) return launch_sep_affine<S, true>(src_lanes, split, P, grid, block, st);
  FK_AFFINE_SIGS(FK_CASE)
#undef FK_CASE
  return cudaErrorInvalidValue;
}

}  // namespace fk
