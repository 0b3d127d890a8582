// fk_walk.hpp — host/device contract of the column-walk crop kernel (fk_walk.cu):
// a batch of bilinear crops of u8x3 frames -> [SwapRB] -> cast f32 -> f32 chain
// -> split into three f32 planes, one fused launch (configs[1], [3], [4]; the
// cvGS preprocessing family). Tables, units and TMA tensor
// maps are built once per pipeline (fk_exec.cu build_walk) and uploaded with it.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "fk_devprog.hpp"

namespace fk {

constexpr uint32_t kWalkWarps = 4;               // warps per CTA (independent: no CTA barrier)
#ifndef FK_WALK_GROUP
#define FK_WALK_GROUP 6  // 6 vs 8: 1.346 vs 1.366 ms on C5 (smaller ring)
#endif
constexpr uint32_t kWalkGroup = FK_WALK_GROUP;   // source rows per TMA box (one copy per group of visits; even)
constexpr uint32_t kWalkSlots = 2;               // box slots per half in the ring (8-16 rows staged ahead)
static_assert(kWalkSlots == 2, "fk_walk steps between two ring slots");
constexpr uint32_t kWalkHalfLanes = 16;          // lanes per half-warp strip (2 output columns per lane)
#ifndef FK_WALK_MAXROWS
#define FK_WALK_MAXROWS 80  // 80 (75-row bands at out_h 224): 1.149 ms on C5 vs 1.161 (112, balanced), 1.158 (64)
#endif
constexpr uint32_t kWalkMaxRows = FK_WALK_MAXROWS;  // output rows per unit (bounds the fix masks)
constexpr uint32_t kWalkSinkLines = 4096;         // one 256-byte line per warp (mod): no shared hot line
constexpr uint32_t kWalkBias = 0x4B000000u;      // bit pattern of 2^23: H values are biased floats
constexpr float kWalkThr = 0.5f - 1.0f / 8192.0f;  // exact-result filter: 0.5 - E, E = 2^-13
// The filter squared: a value is flagged when fma(e, e, -T) >= 0 (e = v - rint(v)),
// i.e. |e| >= sqrt(T). T = kWalkThr^2 = 1/4 - 2^-13 + 2^-26 is exact in f32
// (0x3e7fe001); an exact column of an exact row uses T = RN_up(1/4) (never flagged).
constexpr uint32_t kWalkThr2Bits = 0x3e7fe001u;
constexpr uint32_t kWalkOff2Bits = 0x3e800001u;

// One output column x of a (rect_w, out_w) table. Horizontal lerp of source row
// r as ONE exact integer per lane: H = wa * a + wb * b (dp2a), with
//   exact column  (fx = j / 2^m, m <= 7, or both taps clamped to one column):
//                 wa + wb = 2^14, H in units of 2^-14 pixel, s = 2^-14, c = -512
//   other columns (fx = nx / den, den = 2 out_w):
//                 wa = K (den - nx), wb = K nx, K = floor((2^23 - 1) / (255 den)),
//                 H in units of 1 / (K den), s = RN(1 / (K den)), c = RN(-2^23 / (K den))
// so H < 2^23 and the dp2a accumulating into the bits of 2^23 yields the float
// 2^23 + H exactly. The finish maps a vertically lerped value p to pixel units
// with v = fma(p, s, c).
struct WalkCol {
  uint32_t tap;   // 3 * ix0 (clamped), bytes from the crop's left edge
  uint32_t wts;   // dp2a weights wa | wb << 16 (wb = 0 when both taps clamp to one column)
  float s, c;     // pixel scale of H, see above
  float thr;      // -T of the exact-result filter on an exact row: -kWalkOff2 (exact column) or -kWalkThr2
  uint32_t d1;    // bytes from the left to the right tap: 3, or 0 when both clamp to one column
  double fx;      // the reference's fx (center_coord - floor, ops.cpp:259-270): the exact recompute
};
// One output row y of a (rect_h, out_h) table: the row completes when the walk
// has visited source row r1 (relative to y0, clamped); r0 = r1 - 1, or r0 = r1
// at a clamped edge (then fy = 1: the lerp of the rows r1 - 1 and r1 with
// weight 1 is row r1 exactly). Each table ends with a sentinel row (r1 =
// kWalkRowMask, never visited) so the walk may read one row past out_h.
struct WalkRow {
  uint32_t r1;    // r1 | same << 31 (r0 == r1) | exact << 30 (fy = j / 2^m, m <= 7, or same)
  float fy;       // RN(ny / den) (1 when clamped)
  double fyd;     // the reference's fy (center_coord - floor): the exact recompute
};
constexpr uint32_t kWalkSame = 0x80000000u;
constexpr uint32_t kWalkExactRow = 0x40000000u;
constexpr uint32_t kWalkRowMask = 0x3fffffffu;

// Per plane (BatchRead/BatchWrite entry z).
struct WalkAux {
  uint64_t dst[3];    // output planes in INPUT-lane order (SwapRB folded into the pointers)
  uint32_t dpitch;    // destination row pitch (bytes, shared by the 3 planes)
  uint32_t x3;        // 3 * x0
  uint32_t coltab;    // WalkCol index of output column 0
  uint32_t kz;        // per-plane constant block (WalkPlan::kz)
};

// One warp's work: two half strips of up to 32 output columns — columns
// [x, x + 2 n) of plane z for each half (lanes [0, n0) and [n0, n0 + n1)) — and
// output rows [y_lo, y_hi). The halves (of one plane, or of two planes with the
// same rect_h) share the row table and the visit walk; each has its own TMA box.
struct WalkUnit {
  uint32_t z[2];
  uint32_t y0[2];       // TMA y of each half's source row 0 (the crop's top row in its frame)
  uint16_t bx[2];       // TMA box x (in elements): the staged span starts at byte elem * bx of the frame row
  uint16_t x[2];        // first output column of each half
  uint16_t n[2];        // lanes of each half (n[1] = 0: one plane)
  uint16_t map[2];      // tensor map (WalkPlan::maps) of each half's source frame and box width
  uint16_t bw[2];       // box width of each half in bytes (a multiple of 32): its staged row stride;
                        // bw[1] = 0: adjacent halves of one crop share ONE box (bx[1] = bx[0])
  uint16_t y_lo, y_hi;  // output rows
  uint16_t r_first, r_last;  // source rows visited (relative to y0)
  uint32_t rowtab;      // WalkRow index of output row 0
};

struct WalkPlan {
  const WalkUnit* units;
  const WalkAux* aux;
  const WalkCol* cols;
  const WalkRow* rows;
  const CUtensorMap* maps;  // per source frame (buffer and pitch): its rows as a 2D tensor of elem-byte elements
  const DSample* reads;     // exact-fix path (reference arithmetic)
  const float4* kz;         // per-plane constants [kz][op][lane] = (c, r_hi, r_lo, 0), input-lane order; or null
  uint32_t n_units;
  uint32_t row_bytes;       // the widest box (bytes per staged row): sizes the ring
  uint32_t max_rows;        // output rows of the largest unit (fix-mask capacity)
  uint32_t elem;            // tensor-map element bytes (2, 4 or 8)
  uint64_t negz;            // kNegZero2 (fk_pack2.cuh): a product's runtime -0 addend
  uint64_t dst_base;        // added to every WalkAux::dst (0: absolute; the unfused pass 0: its intermediate)
  uint64_t sink;            // kWalkSinkLines x 256-byte scratch the idle lanes of a unit store to (no
                            // store predicate): warp u's idle lanes write line u % kWalkSinkLines
  // inline chain constants (shared by every plane), input-lane order, as pairs
  float2 kc[4][3], kh[4][3], kl[4][3];
};

// Chain signature: fk_sig.cuh's sig_make bits plus, per op k, bit 20 + k: the
// two-op reciprocal division q = fma(x, r_hi, x r_lo) equals IEEE x / c on
// every value the op can see (host-verified).
constexpr uint32_t kWalkDiv2 = 20;

bool walk_registered(uint32_t sig);
size_t walk_smem_bytes(uint32_t row_bytes, uint32_t max_rows);
cudaError_t launch_walk(uint32_t sig, bool per_plane, const WalkPlan& P, cudaStream_t st);
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
bool walk_encode_map(CUtensorMap* map, uint64_t base, uint64_t width_elems, uint64_t rows, uint64_t pitch,
                     uint32_t elem, uint32_t box_w, uint32_t box_h);

}  // namespace fk
