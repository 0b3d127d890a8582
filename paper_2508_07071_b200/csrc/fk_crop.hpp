// fk_crop.hpp — host/device contract of the planar crop kernel (fk_crop.cu):
// batched crop -> bilinear resize of u8x3 frames -> [SwapRB] -> cast f32 ->
// f32 chain -> split into three f32 planes (configs[1], [3], [4]; the cvGS
// preprocessing family). Built once per pipeline (fk_exec.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "fk_devprog.hpp"

namespace fk {

constexpr uint32_t kCropThreads = 224;             // 7 warps
constexpr uint32_t kCropWarps = kCropThreads / 32;
constexpr uint32_t kCropTileRows = 8;              // output rows per tile (2 quads per thread at 56 quads a row)
constexpr uint32_t kCropMaxQuads = kCropThreads;   // out_w <= 4 * 224
constexpr uint32_t kCropBias = 0x48000000u;        // bit pattern of 2^17: V values are biased floats

// One output row y of a (rect_h, out_h) table. The reference's center_coord /
// floor / clamp (ops.cpp:253-275) in exact integer form: cy = P / den with
// P = (2y + 1) rect_h - out_h, den = 2 out_h, iy = floor(P / den),
// ny = P - iy den; the vertical lerp of a lane is exactly
//   (K (den - ny) a + K ny b) / (K den)            (dp2a on the two source rows)
// and phase 2 maps the biased float 2^17 + M 2^-6 (M the dp2a sum) back to
// pixel units with v = hb * s + c, s = 64 / (K den), c = -2^17 s.
// Rows whose fy is a multiple of 1/64 use den = 64, K = 256: every step is then
// exact in FP32 (kCropExact).
struct CropRow {
  uint32_t iy;    // iy0 | iy1 << 16 relative to the crop's y0, clamped to [0, rect_h); bit 31: exact row
  uint32_t wts;   // dp2a weights K (den - ny) | K ny << 16
  float s, c;
};
// One output column x of a (rect_w, out_w) table: the left tap ix0 relative to
// x0 (clamped) and fx rounded to f32; fx = 0 where both taps clamp to the same
// source column (the lerp of equal taps is that tap, for any fx).
struct CropCol {
  uint32_t ix;    // ix0 | bit 31: fx is a multiple of 2^-8 (exact column)
  float fx;
};
constexpr uint32_t kCropExact = 0x80000000u;

// Per plane: its table offsets and phase-1 source span.
struct CropAux {
  uint32_t rowtab;   // CropRow index of output row 0
  uint32_t coltab;   // CropCol index of output column 0
  uint32_t wb;       // first source byte of the span, relative to the row start (16-byte aligned)
  uint32_t nwords;   // 4-byte words of the span, a multiple of 4 (V row = 4 nwords values)
  uint32_t rlim;     // bytes readable from wb in the crop's last source row (staging zero-fills past it)
  uint32_t swap;     // 1: input lane m lands in output lane 2 - m (folded SwapRB)
  uint32_t kz;       // per-plane constant block index (CropPlan::kz)
  uint32_t pad;
};

struct CropPlan {
  const DSample* reads;
  const DWrite* writes;
  const CropAux* aux;
  const CropRow* rows;
  const CropCol* cols;
  const uint32_t* order;   // CTA -> plane (cost-descending), or null
  const float4* kz;        // per-plane constants [kz][op][lane] = (c, r_hi, r_lo, r), input-lane order; or null
  uint32_t out_w, out_h, quads;
  uint32_t bands;          // CTAs per plane (row bands)
  uint32_t band_rows;      // output rows per band (multiple of kCropTileRows)
  uint32_t v_stride;       // bytes per V row in shared memory (16-byte multiple)
  uint32_t n_planes;
  uint32_t stage_rows;     // staged source rows per tile (max over planes and tiles)
  uint32_t stage_stride;   // bytes per staged row (max span, 16-byte multiple)
  uint32_t pad[3];
  // inline chain constants (every plane shares them, swap uniform), input-lane order,
  // duplicated into pairs for the packed FP32 ops: c, RN(1/c) and the low part of 1/c
  float2 kc[4][3], kh[4][3], kl[4][3];
};

// Chain signature of the planar kernel: fk_sig.cuh's sig_make bits plus, per
// op k, bit 20 + k: the two-op reciprocal division q = fma(x, r_hi, x r_lo)
// equals IEEE x / c on every value the op can see (host-verified).
constexpr uint32_t kCropDiv2 = 20;

bool crop_registered(uint32_t sig);
size_t crop_smem_bytes(uint32_t v_stride, uint32_t stage_rows, uint32_t stage_stride, uint32_t quads);
cudaError_t launch_crop(uint32_t sig, bool per_plane, const CropPlan& P, uint32_t ctas, cudaStream_t st);

}  // namespace fk
