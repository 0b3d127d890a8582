// fk_launch.hpp — host entry points of the kernel families.
#pragma once

#include <cuda_runtime.h>

#include "fk_devprog.hpp"

namespace fk {

// interpreted-chain kernel (fk_generic.cu)
int generic_state_class(bool wide, int lanes);  // 0..3
int generic_elems(int cls);                     // E: consecutive x per thread
cudaError_t launch_generic(int cls, const DPlan& P, cudaStream_t st);

}  // namespace fk

namespace fk {

// compiled batched u8 crop/resize -> lane-wise chain (LUT) -> write/split kernel (fk_resample.cu)
int resample_elems();
// compiled f32 element-wise chain kernel (fk_direct.cu)
int direct_elems();
bool direct_registered(uint32_t sig);
// exhaustive 2^32-input device check, cached per divisor: 0 = use IEEE division,
// 1 = the guarded reciprocal form is exact, 2 = the unguarded one is too
int recip_div_verified(float d);
cudaError_t launch_direct(uint32_t sig, bool to_u8, const DPlan& P, cudaStream_t st);

// compiled column-streaming u8 resample kernel (fk_resample_sep.cu); P.tiles_per_cta = band rows
uint32_t resample_sep_band_max();
// staged: every warp's source span fits the cp.async ring and source rows are
// 16-byte aligned (the host checks, sep_stage_ok), so the kernel is built without
// the direct-load walk
cudaError_t launch_resample_sep(int src_lanes, uint32_t out_lane_kind, bool split, uint32_t sig, const DPlan& P,
                                bool staged, cudaStream_t st);
uint32_t resample_sep_ring_row();

bool resample_affine_registered(uint32_t sig);  // fk_sig.cuh FK_AFFINE_SIGS
// sig == kSigLut: LUT mode; else the registered AFFINE chain signature
cudaError_t launch_resample(int src_lanes, uint32_t out_lane_kind, bool split, uint32_t sig, const DPlan& P,
                            cudaStream_t st);

}  // namespace fk
