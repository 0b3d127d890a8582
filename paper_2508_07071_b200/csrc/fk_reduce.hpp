// fk_reduce.hpp — device-side form of ReduceDPP specs (dpp.hpp:37-41) and the
// launch entry of fk_reduce.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "fk_devprog.hpp"

namespace fk {

constexpr int kMaxReduceSpecs = 4;     // specs folded per traversal (more: further traversals)
constexpr uint32_t kNoOp = 0xffffffffu;

struct RSpecDev {
  uint32_t op;          // index of the transform in the DPlan program table, kNoOp = identity
  uint32_t combine;     // fk_reducer
  uint32_t lane_kind;   // FK_U8 / FK_F32 / FK_F64 of the value kind
  uint32_t lanes;       // 1 or 3
  uint32_t dsum;        // float Sum: accumulate in double (dpp.cpp:116-127)
  uint32_t pad;
  uint64_t ident[3];       // reducer_identity(combine, value kind), lane bits (dpp.cpp:48-73)
  uint64_t user_ident[3];  // the spec's identity: lane bits, or (dsum) lane values as double bits
};

struct RSpecsDev {
  uint32_t n;
  uint32_t pad;
  RSpecDev s[kMaxReduceSpecs];
};

// a plain read: one plane of u8 / f32 / u8x3 rows, 16-byte aligned, no
// default values or folded unaries, walked as 16-byte vectors
struct PlainRows {
  uint64_t base;   // address of element (0, 0)
  uint64_t pitch;  // bytes per row (multiple of 16)
  uint32_t width;  // elements per row
  uint32_t vpr;    // vectors per row
  uint32_t vecs;   // rows * vpr (< 2^32)
  uint32_t kind;   // FK_U8 / FK_F32 (16-byte vectors) / FK_U8X3 (16 pixels, 48 bytes)
  uint32_t vb;     // bytes per vector
  FastDiv vdiv;    // / vpr
};

// cls: generic_state_class (32/64-bit lanes x 1/3 lanes); out: 3 lane-bit words per spec (device)
cudaError_t launch_reduce(int cls, const DPlan& P, const RSpecsDev& S, void* scratch, uint32_t nblocks, uint64_t* out,
                          cudaStream_t st);
// second pass when a float Max / Min came out zero: first +0 / -0 index per
// (spec, lane) in zmask (bit 3 * spec + lane); first[6 * spec + 2 * lane + neg]
cudaError_t launch_reduce_zero_sign(int cls, const DPlan& P, const RSpecsDev& S, uint32_t zmask, uint32_t nblocks,
                                    unsigned long long* first, cudaStream_t st);
cudaError_t launch_reduce_plain(const DPlan& P, const RSpecsDev& S, const PlainRows& R, void* scratch,
                                uint32_t nblocks, uint64_t* out, cudaStream_t st);
// zero-sign pass over plain u8 / f32 rows (single-lane specs: zmask bits 3 * spec)
cudaError_t launch_reduce_plain_zero_sign(const DPlan& P, const RSpecsDev& S, const PlainRows& R, uint32_t zmask,
                                          uint32_t nblocks, unsigned long long* first, cudaStream_t st);
uint32_t reduce_plain_blocks(uint32_t kind, int sms);  // resident CTAs on the device
size_t reduce_scratch_bytes(uint32_t nblocks);
int reduce_tile_elems();

}  // namespace fk
