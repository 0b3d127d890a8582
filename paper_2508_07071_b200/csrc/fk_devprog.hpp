// fk_devprog.hpp — the device-resident form of a validated pipeline.
//
// Built once per Pipeline (fk_exec.cu) and uploaded to HBM: per-plane read
// params (the BatchRead array indexed by z, ops.cpp:369-378), per-plane write
// params (BatchWrite, ops.cpp:437-445), and the compute program. Kernels get a
// DPlan by value (kernel parameter space) and index the arrays by z.
#pragma once

#include <cstdint>

namespace fk {

// read modes, resolved on the host from SampleReadParams::resizing()/mode (ops.cpp:327-344)
enum : uint32_t { RD_DIRECT = 0, RD_NEAREST = 1, RD_BILINEAR = 2 };
// DSample::flags. SF_LUT_SRC: u8 lanes and a lane-wise folded-unary program, so
// post+compute can be tabulated over the 256 possible lane values.
// SF_POST_SWAP: the folded unaries swap lanes 0/2 an odd number of times.
enum : uint32_t { SF_DEFAULT = 1u, SF_LANE_ALIGNED = 2u, SF_LUT_SRC = 4u, SF_POST_SWAP = 8u };
// DWrite::flags
enum : uint32_t { WF_ACTIVE = 1u, WF_LANE_ALIGNED = 2u, WF_STREAM = 4u };
// write modes
enum : uint32_t { WR_DIRECT = 0, WR_SPLIT = 1 };
// compute op classes
enum : uint32_t { OC_NOP = 0, OC_ARITH = 1, OC_SWAP = 2, OC_CAST = 3, OC_GRAY = 4 };
// arith functions (same order as fk_op_id MUL..DIV)
enum : uint32_t { AF_MUL = 0, AF_ADD = 1, AF_SUB = 2, AF_DIV = 3 };

struct DSample {             // one plane's read (SampleReadParams, ops.hpp:78-91)
  uint64_t src;              // device address of source element (0,0)
  uint64_t pitch;            // bytes per source row
  uint32_t x0, y0, rect_w, rect_h;
  uint32_t out_w, out_h;
  uint32_t kind;             // source ScalarKind
  uint32_t mode;             // RD_*
  uint32_t post_off, post_len;  // folded unaries: absolute index into the DPlan program table
  uint32_t flags;            // SF_*
  uint32_t tail_bytes;       // bytes readable from the start of the crop's last source row
                             // (pitch when the view has a row below it, else the row's width)
};

struct DWrite {              // one plane's write (WriteParams / SplitWriteParams)
  uint64_t dst[3];
  uint64_t pitch[3];         // bytes per destination row, per destination plane
  uint32_t flags;            // WF_*
  uint32_t pad;
};

struct DOp {                 // one compute op of the program
  uint32_t cls;              // OC_*
  uint32_t fn;               // AF_* for OC_ARITH
  uint32_t lk_in, lk_out;    // lane kinds (FK_U8/FK_F32/FK_F64)
  uint32_t nl;               // lanes (1 or 3)
  uint32_t repeat;           // StaticLoop count (1 otherwise)
  uint64_t c[3];             // raw lane constants (u8 value / f32 bits / f64 bits)
  uint64_t per_z;            // BatchArith: device array of 24-byte Elements, else 0
  uint32_t per_z_n;
  uint32_t pad;
};

struct FastDiv {             // n / d for 32-bit n (Granlund-Montgomery round-up)
  uint32_t d, m, s;
};

// Per-CTA resample tables in shared memory: the sampling coordinates depend only
// on the output column (x) or row (y), so center_coord/floor/clamp (ops.cpp:253-270)
// run once per column and row of the CTA instead of once per pixel.
struct XEnt { uint32_t o0, o1; double f; };  // tap byte offsets in the row (x0 + clamp) * bpe, fx
struct YEnt { uint64_t r0, r1; double f; };  // tap row byte offsets (y0 + clamp) * pitch, fy
constexpr uint32_t kBlock = 256;             // threads per CTA
constexpr uint32_t kXCap = 1024;             // table path when out_w <= kXCap
constexpr uint32_t kYCap = 160;              // rows one CTA may span (host keeps tiles_per_cta within it)
constexpr uint32_t kEdge = 0x80000000u;      // XTab::o flag: the second tap equals the first (clamped edge)
struct XTab {                                // shared-memory column table, struct-of-arrays
  alignas(16) uint32_t o[kXCap + 8];         // byte offset of tap 0 within the row | kEdge
  alignas(16) double f[kXCap + 8];           // fx (bilinear), 0 (nearest)
};

constexpr uint32_t kProg = 24;  // ops carried in kernel-parameter space (constant bank)

struct DPlan {
  uint32_t width, height, batch;  // iteration space (flattened to height 1 when contiguous)
  uint32_t tiles_per_row;
  FastDiv tpr;
  uint32_t tiles;            // tiles per plane = height * tiles_per_row
  uint32_t tiles_per_cta;    // contiguous tile range one CTA walks (multiple of the block size)
  uint32_t n_ops;            // compute program length
  uint32_t prog_inline;      // 1: program table is prog[] below (kernel params), else `table`
  uint32_t lut_ok;           // compute program is lane-wise (LUT-able for u8 sources)
  uint32_t prog_swap;        // compute program swaps lanes 0/2 an odd number of times
  const DOp* table;          // [compute ops..., folded-unary programs...] in HBM (long programs)
  DOp prog[kProg];           // same layout, inline
  const uint32_t* order;     // visiting order of the planes (blockIdx.z -> z), nullptr = identity:
                             // planes sharing a source are adjacent so it stays L2-resident
  const DSample* reads;      // batch entries; nullptr -> affine read below
  const DWrite* writes;      // batch entries; nullptr -> affine write below
  DSample rd;                // affine read: plane z at rd.src + z * rd_zstride
  DWrite wr;                 // affine write: plane z at wr.dst + z * wr_zstride
  uint64_t rd_zstride, wr_zstride;
  uint32_t write_kind;       // element kind reaching the write op
  uint32_t write_mode;       // WR_*
  uint32_t def_kind;         // kind of the BatchRead default value
  uint32_t op_base;          // compute ops are table[op_base, op_base + n_ops); post ops at DSample::post_off
  uint64_t def[3];           // BatchRead default Element (ops.hpp:111), lane-encoded
  float aff_c[4][3];         // AFFINE chain constants per op and lane when no op is per-plane
  float aff_r[4][3];         // ... and their reciprocals RN(1 / c)
  uint32_t aff_inline;       // 1: aff_c / aff_r hold the chain's constants
  // column-streaming kernel (fk_resample_sep): CTA slice blockIdx.z runs planes
  // slots[blockIdx.z * slots_per_cta + h] (h < slots_per_cta, kNoPlane = none) with
  // threads [h * slot_threads, (h + 1) * slot_threads); slots == nullptr: plane
  // order[blockIdx.z], one per CTA
  const uint32_t* slots;
  uint32_t slots_per_cta;    // 1, or 2 planes sharing one row/visit table (equal rect_h, mode, swap)
  uint32_t slot_threads;     // threads per plane slot
  uint32_t slices;           // CTA slices along z (slots != nullptr)
  uint32_t no_stage;         // 1: column-streaming kernel uses direct tap loads (spans the ring cannot hold)
  uint32_t dir_rep[4];       // fk_direct: repeat count of chain op k (its constant / reciprocal in aff_c / aff_r [k][0])
  FastDiv zdiv;              // fk_reduce: n / tiles (plane of a linear tile index)
  uint64_t negz;             // (-0.0f, -0.0f) at run time: packed products as fma(a, b, negz) (fk_pack2.cuh)
};
constexpr uint32_t kNoPlane = 0xffffffffu;

}  // namespace fk
