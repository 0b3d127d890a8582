// fk_exec.cu — pipeline -> device program, and the two executors.
//
// execute_fused (executor.cpp:63-85) becomes ONE kernel launch over the whole
// (x, y, z) space; execute_unfused (executor.cpp:134-217) becomes one launch per
// compute op through stream-ordered intermediates (cudaMallocAsync, freed after
// the consuming pass) plus a final write launch — the in-repo comparator.
// Counters follow the reference's accounting exactly (fk_core.cpp:analytic_traffic).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "fk_core.hpp"
#include "fk_pack2.cuh"
#include "fk_stream.hpp"
#include "fk_walk.hpp"
#include "fk_reduce.hpp"
#include "fk_exec.hpp"
#include "fk_launch.hpp"
#include "fk_sig.cuh"

namespace fk {

namespace {
thread_local const char* t_last_kernel = "";  // kernel family of this thread's last fused execute

std::atomic<uint64_t> g_launches{0};

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(FK_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Lane-encode an Element (scalar.hpp:94-121) the way DOp::c / DPlan::def hold it.
void encode_element(uint32_t kind, const Element& e, uint64_t (&c)[3]) {
  c[0] = c[1] = c[2] = 0;
  for (int l = 0; l < lanes_of(kind); ++l) {
    switch (lane_kind(kind)) {
      case FK_U8: c[l] = e.raw[l]; break;
      case FK_F32: { uint32_t b; std::memcpy(&b, e.raw + 4 * l, 4); c[l] = b; break; }
      default: { uint64_t b; std::memcpy(&b, e.raw + 8 * l, 8); c[l] = b; break; }
    }
  }
}

DOp arith_op(uint32_t fn, uint32_t kind, const Element& value, uint32_t repeat) {
  DOp d{};
  d.cls = OC_ARITH;
  d.fn = fn;
  d.lk_in = d.lk_out = lane_kind(kind);
  d.nl = uint32_t(lanes_of(kind));
  d.repeat = repeat;
  encode_element(kind, value, d.c);
  return d;
}

// compute_exec_block dispatch (ops.cpp:214-235) -> one device op
DOp encode_compute(const Op& op) {
  DOp d{};
  const uint32_t in = uint32_t(op.in_kind), out = uint32_t(op.out_kind);
  switch (op.id) {
    case FK_OP_MUL: case FK_OP_ADD: case FK_OP_SUB: case FK_OP_DIV:
      return arith_op(op.id - FK_OP_MUL, in, op.value, 1);
    case FK_OP_BATCH_ARITH:
      return arith_op(op.inner_id - FK_OP_MUL, in, Element{}, 1);  // per_z attached by caller
    case FK_OP_STATIC_LOOP:  // static_loop_block, ops.cpp:200-210
      switch (op.inner_id) {
        case FK_OP_MUL: case FK_OP_ADD: case FK_OP_SUB: case FK_OP_DIV:
          return arith_op(op.inner_id - FK_OP_MUL, op.value_kind, op.value, op.repeat);
        case FK_OP_SWAP_RB:
          d.cls = OC_SWAP;
          d.repeat = op.repeat;
          return d;
        default:
          d.cls = OC_NOP;  // kind-preserving cast: identity
          return d;
      }
    case FK_OP_CAST:
      if (in == out) { d.cls = OC_NOP; return d; }
      d.cls = OC_CAST;
      d.lk_in = lane_kind(in);
      d.lk_out = lane_kind(out);
      d.nl = uint32_t(lanes_of(in));
      return d;
    case FK_OP_SWAP_RB:
      d.cls = OC_SWAP;
      d.repeat = 1;
      return d;
    case FK_OP_TO_GRAY:
      d.cls = OC_GRAY;
      d.lk_in = lane_kind(in);
      d.lk_out = FK_F32;
      d.nl = 3;
      return d;
  }
  fail(FK_E_INVALID_ARGUMENT, "not a compute op");
}

DOp encode_unary(const Folded& f) {
  Op op;
  op.id = f.id;
  op.in_kind = int32_t(f.in);
  op.out_kind = int32_t(f.out);
  return encode_compute(op);
}

// The fused program: drop identities, merge runs of the same op into one
// repeat count (semantically n-fold application, exactly what StaticLoop is).
std::vector<DOp> compress(const std::vector<DOp>& ops) {
  std::vector<DOp> out;
  for (const DOp& d : ops) {
    if (d.cls == OC_NOP) continue;
    if (!out.empty()) {
      DOp& b = out.back();
      const bool same_arith = d.cls == OC_ARITH && b.cls == OC_ARITH && !d.per_z && !b.per_z && d.fn == b.fn &&
                              d.lk_in == b.lk_in && d.nl == b.nl && std::memcmp(d.c, b.c, sizeof d.c) == 0;
      const bool same_swap = d.cls == OC_SWAP && b.cls == OC_SWAP;
      if ((same_arith || same_swap) && uint64_t(b.repeat) + d.repeat <= 0xffffffffull) {
        b.repeat += d.repeat;
        continue;
      }
    }
    out.push_back(d);
  }
  return out;
}

uint64_t pitch_of(const fk_plane& p) { return uint64_t(p.row_stride) * bpe(p.kind); }

bool lane_aligned(const fk_plane& p) {
  const uint64_t lb = lane_bytes(p.kind);
  return (reinterpret_cast<uintptr_t>(p.data) % lb) == 0 && (pitch_of(p) % lb) == 0;
}

template <class T>
T* upload(const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  void* d = nullptr;
  cuda_check(cudaMalloc(&d, v.size() * sizeof(T)), "cudaMalloc(program)");
  cuda_check(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy(program)");
  return static_cast<T*>(d);
}

FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  uint32_t s = 0;
  while ((uint64_t(1) << s) < d) ++s;
  f.s = s;
  f.m = uint32_t(((uint64_t(1) << 32) * ((uint64_t(1) << s) - d)) / d + 1);
  return f;
}

void add_kind(uint32_t k, bool& wide, int& lanes) {
  if (lane_kind(k) == FK_F64) wide = true;
  if (lanes_of(k) == 3) lanes = 3;
}

}  // namespace

struct DeviceProgram {
  int device = -1;
  // program table: [fused (compressed) ops | 1:1 ops (unfused pass i) | folded-unary programs]
  std::vector<DOp> table;
  DOp* d_table = nullptr;
  uint32_t n_fused = 0, n_ops = 0;
  bool fused_lut_ok = true;      // every fused op is lane-wise
  bool fused_swap = false;       // odd number of lane swaps in the fused program
  bool resample_ok = false;      // the compiled u8 resample/LUT kernel can run the fused pass
  bool sep_ok = false;           // ... and the column-streaming variant (32-bit source pitches)
  int resample_lanes = 0;
  bool affine_ok = false;        // ... in AFFINE mode: cast u8->f32 then a registered f32 chain
  uint32_t aff_base = 0, aff_n = 0, aff_sig = 0;
  bool aff_inline = false;       // no AFFINE op is per-plane: constants go in the kernel parameters
  float aff_c[4][3] = {}, aff_r[4][3] = {};
  bool direct_ok = false;        // the compiled f32 element-wise kernel can run the fused pass
  bool direct_u8 = false;        // ... ending in Cast f32 -> u8
  uint32_t dir_base = 0, dir_sig = 0;
  std::map<uint64_t, std::vector<uint64_t>> per_z_host;  // BatchArith rows by device address
  DSample* d_reads = nullptr;
  DWrite* d_writes = nullptr;
  uint32_t* d_order = nullptr;   // plane visiting order (grouped by source), or null
  uint32_t* d_slots2 = nullptr;  // column-streaming kernel: planes paired by (mode, rect_h, swap), kNoPlane = none
  uint32_t n_slices2 = 0;        // ... number of pairs
  bool stage_ok[2] = {false, false};  // staged column walk valid for [single, dual] slices (set at build)
  std::vector<void*> extra;      // BatchArith constant tables
  std::vector<DSample> reads;    // host copies
  bool read_flat = false, write_flat = false;
  bool fused_wide = false;
  int fused_lanes = 1;
  bool read_wide = false;        // kinds touched by the read stage alone
  int read_lanes = 1;
  uint64_t def[3] = {0, 0, 0};
  uint32_t def_kind = 0;
  Traffic traffic;               // analytic ExecReport counters (computed once)
  // column-walk crop kernel (fk_walk.cu): crop -> bilinear -> [swap] -> f32 chain -> split f32
  bool walk_ok = false;
  bool walk_perz = false;        // per-plane chain constants (BatchArith or per-plane lane swaps)
  uint32_t walk_sig = 0;
  WalkPlan walk{};               // units, tables, inline constants (reads set at launch)
  // roofline-grade unfused comparator (fk_stream.cu): pass 0 = fk_walk over the
  // first op into a planar intermediate, or a stream pass; then one stream pass
  // per op and the write pass (src / dst pointers set per execute)
  bool unf_fast = false;
  bool unf_walk = false;
  WalkPlan unf_walk_plan{};
  uint32_t unf_walk_sig = 0;
  bool unf_walk_perz = false;
  std::vector<StreamPass> unf_pass;  // [0, n]: pass i (pass 0 unused when unf_walk), n = the write pass
  std::vector<uint64_t> unf_bytes;   // intermediate bytes after pass i

  ~DeviceProgram() {
    for (void* p : {static_cast<void*>(d_table), static_cast<void*>(d_reads), static_cast<void*>(d_writes),
                    static_cast<void*>(d_order), static_cast<void*>(d_slots2)})
      if (p) cudaFree(p);
    for (void* p : extra) cudaFree(p);
  }
};

Pipeline::~Pipeline() = default;

namespace {

bool lane_wise(const DOp& d) { return d.cls != OC_GRAY; }
bool odd_swap(const DOp& d) { return d.cls == OC_SWAP && (d.repeat & 1u); }

float f32_bits(uint64_t v) {
  float f;
  const uint32_t b = uint32_t(v);
  std::memcpy(&f, &b, 4);
  return f;
}
bool same_f32(float a, float b) {
  if (a != a && b != b) return true;
  return std::memcmp(&a, &b, 4) == 0;
}

// The AFFINE chain's op k is a division: does the reciprocal form (fk_sig.cuh
// div_by_recip) equal IEEE division on every value op k can receive? After a u8
// read those are prefix_k(t) for t in 0..255, per lane and — with BatchArith
// constants — per plane: at most 256 * 3 * batch checks, done once per pipeline
// in host IEEE arithmetic (identical to the device's _rn ops).
bool recip_div_exact(const std::vector<DOp>& arith, size_t k, const std::map<uint64_t, std::vector<uint64_t>>& rows,
                     uint32_t batch) {
  bool per_plane = false;
  for (size_t j = 0; j <= k; ++j) per_plane = per_plane || arith[j].per_z;
  const uint32_t planes = per_plane ? batch : 1;
  auto lane_const = [&](const DOp& d, uint32_t z, int l) {
    const int li = d.nl == 3 ? l : 0;
    if (!d.per_z) return f32_bits(d.c[li]);
    const std::vector<uint64_t>& r = rows.at(d.per_z);
    const uint32_t zz = z < d.per_z_n ? z : d.per_z_n - 1;
    return f32_bits(r[3 * size_t(zz) + li]);
  };
  for (uint32_t z = 0; z < planes; ++z)
    for (int l = 0; l < int(arith[k].nl); ++l) {
      const float d = lane_const(arith[k], z, l);
      const float r = 1.0f / d;
      for (int t = 0; t < 256; ++t) {
        float v = float(t);
        for (size_t j = 0; j < k; ++j) {
          const float c = lane_const(arith[j], z, l);
          switch (arith[j].fn) {
            case AF_MUL: v = v * c; break;
            case AF_ADD: v = v + c; break;
            case AF_SUB: v = v - c; break;
            default: v = v / c; break;
          }
        }
        const float q = v * r;
        const float e = std::fmaf(-q, d, v);
        if (!same_f32(std::fmaf(e, r, q), v / d)) return false;
      }
    }
  return true;
}

// The unfused comparator allocates stream-ordered intermediates every execute
// (executor.cpp:112-118 allocates fresh planes per pass); keep freed blocks in
// the device pool instead of returning them to the driver at each sync.
void keep_pool_memory(int device) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lock(mu);
  for (int d : done)
    if (d == device) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = ~uint64_t(0);
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  done.push_back(device);
}


// ------------------------------------------------------ planar crop kernel --
// floor(a / b) for b > 0
int64_t floor_div(int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// WalkRow for output row y (fk_walk.hpp): center_coord / floor / clamp of
// ops.cpp:253-275 in exact integers: cy = P / den, P = (2y + 1) rect_h - out_h,
// den = 2 out_h, iy = floor(P / den), fy = (P - iy den) / den.
WalkRow walk_row(uint32_t y, uint32_t rect_h, uint32_t out_h) {
  const int64_t den = 2 * int64_t(out_h);
  const int64_t P = (2 * int64_t(y) + 1) * rect_h - out_h;
  const int64_t iy = floor_div(P, den), ny = P - iy * den;
  const int64_t maxy = int64_t(rect_h) - 1;
  const uint32_t iy0 = uint32_t(std::min(std::max<int64_t>(iy, 0), maxy));
  const uint32_t iy1 = uint32_t(std::min(std::max<int64_t>(iy + 1, 0), maxy));
  WalkRow r{};
  const bool same = iy0 == iy1;
  r.r1 = iy1 | (same ? kWalkSame : 0u) | ((same || (ny * 128) % den == 0) ? kWalkExactRow : 0u);
  r.fy = same ? 1.0f : float(double(ny) / double(den));  // clamped: both taps are row r1 (fk_walk: Ha + (Hb - Ha) 1 = Hb)
  { // the reference's double coordinate (ops.cpp:253-257 center_coord, floor): fk_walk's exact recompute
    const double cy = ((double(y) + 0.5) * double(rect_h)) / double(out_h) - 0.5;
    r.fyd = cy - std::floor(cy);
  }
  return r;
}

// WalkCol for output column x: the left tap (clamped) and the dp2a weights /
// pixel scale of the horizontal lerp (fk_walk.hpp).
WalkCol walk_col(uint32_t x, uint32_t rect_w, uint32_t out_w) {
  const int64_t den = 2 * int64_t(out_w);
  const int64_t P = (2 * int64_t(x) + 1) * rect_w - out_w;
  const int64_t ix = floor_div(P, den), nx = P - ix * den;
  const int64_t maxx = int64_t(rect_w) - 1;
  const uint32_t ix0 = uint32_t(std::min(std::max<int64_t>(ix, 0), maxx));
  const uint32_t ix1 = uint32_t(std::min(std::max<int64_t>(ix + 1, 0), maxx));
  WalkCol c{};
  c.tap = 3 * ix0;
  c.d1 = 3 * (ix1 - ix0);
  {
    const double cx = ((double(x) + 0.5) * double(rect_w)) / double(out_w) - 0.5;
    c.fx = cx - std::floor(cx);
  }
  if (ix0 == ix1 || (nx * 128) % den == 0) {  // exact: units of 2^-14 pixel
    const uint32_t j = ix0 == ix1 ? 0u : uint32_t(nx * 16384 / den);
    c.wts = (16384u - j) | (j << 16);
    c.s = 1.0f / 16384.0f;
    c.c = -512.0f;
    c.thr = -__builtin_bit_cast(float, kWalkOff2Bits);
  } else {
    const uint32_t K = uint32_t(8388607 / (255 * den));
    c.wts = uint32_t(K * (den - nx)) | (uint32_t(K * nx) << 16);
    c.s = float(1.0 / double(K * den));
    c.c = float(-8388608.0 / double(K * den));
    c.thr = -__builtin_bit_cast(float, kWalkThr2Bits);
  }
  return c;
}

// Two-op division q = fma(x, r_hi, RN(x r_lo)): equal to IEEE x / d on every value op k of
// the AFFINE chain can receive (prefix_k of the 256 u8 values, per lane and plane)?
bool recip2_div_exact(const std::vector<DOp>& arith, size_t k, const std::map<uint64_t, std::vector<uint64_t>>& rows,
                      uint32_t batch) {
  bool per_plane = false;
  for (size_t j = 0; j <= k; ++j) per_plane = per_plane || arith[j].per_z;
  const uint32_t planes = per_plane ? batch : 1;
  auto lane_const = [&](const DOp& d, uint32_t z, int l) {
    const int li = d.nl == 3 ? l : 0;
    if (!d.per_z) return f32_bits(d.c[li]);
    const std::vector<uint64_t>& r = rows.at(d.per_z);
    return f32_bits(r[3 * size_t(z < d.per_z_n ? z : d.per_z_n - 1) + li]);
  };
  for (uint32_t z = 0; z < planes; ++z)
    for (int l = 0; l < 3; ++l) {
      const float d = lane_const(arith[k], z, l);
      const float rh = 1.0f / d;
      const float rl = float(1.0 / double(d) - double(rh));
      for (int t = 0; t < 256; ++t) {
        float v = float(t);
        for (size_t j = 0; j < k; ++j) {
          const float c = lane_const(arith[j], z, l);
          switch (arith[j].fn) {
            case AF_MUL: v = v * c; break;
            case AF_ADD: v = v + c; break;
            case AF_SUB: v = v - c; break;
            default: v = v / c; break;
          }
        }
        if (!same_f32(std::fmaf(v, rh, v * rl), v / d)) return false;
      }
    }
  return true;
}

// Eligibility, tables, units, TMA tensor maps and constants of the
// column-walk crop kernel (fk_walk.cu): every plane a bilinear crop (or a crop
// of the output size) of a u8x3 frame with 16-byte aligned rows, an AFFINE
// chain, a split write of three f32 planes sharing one 8-byte multiple pitch,
// an even output width.
bool build_walk(DeviceProgram& dp, const Pipeline& p, const std::vector<DOp>& arith, uint32_t sig,
                const std::vector<DWrite>& writes, WalkPlan& P, uint32_t& wsig_out, bool& perz_out) {
  const uint32_t W = p.space.width, H = p.space.height, B = p.space.batch;
  const uint32_t wid = p.write.id == FK_OP_BATCH_WRITE ? p.write.w_inner : p.write.id;
  if (!dp.affine_ok || dp.resample_lanes != 3 || wid != FK_OP_SPLIT_WRITE || B == 0 || W % 2 || W == 0 || H == 0 ||
      W > 65534 || H > 65535 || 255ull * 2 * W > 8388607 /* K >= 1 in walk_col */ ||
      lane_kind(uint32_t(p.write.in_kind)) != FK_F32)
    return false;
  bool ok = true;
  for (const DSample& s : dp.reads) {
    // a crop without resize (rect == out, resizing() false) is the bilinear walk with fx = fy = 0
    ok = ok && (s.mode == RD_BILINEAR || (s.mode == RD_DIRECT && s.rect_w == W && s.rect_h == H)) &&
         s.kind == FK_U8X3 && !(s.flags & SF_DEFAULT) && s.rect_h <= 65535 && s.rect_w <= 65535 &&
         ((s.src | s.pitch) & 15) == 0 && s.pitch < (1ull << 39) && s.out_w == W && s.out_h == H;
  }
  for (const DWrite& w : writes)
    ok = ok && (w.flags & WF_ACTIVE) && w.pitch[0] == w.pitch[1] && w.pitch[0] == w.pitch[2] &&
         (w.pitch[0] & 7) == 0 && w.pitch[0] * H < (1ull << 32) && ((w.dst[0] | w.dst[1] | w.dst[2]) & 7) == 0;
  if (!ok) return false;
  // chain: the AFFINE signature with the verified division forms
  uint32_t fn[4] = {0, 0, 0, 0}, fast = 0, two = 0;
  for (size_t k = 0; k < arith.size(); ++k) {
    fn[k] = arith[k].fn;
    if (fn[k] != AF_DIV) continue;
    if (recip2_div_exact(arith, k, dp.per_z_host, B)) two |= 1u << k;
    else if (sig_fast(sig, int(k))) fast |= 1u << k;
  }
  uint32_t wsig = sig_make(int(arith.size()), fn[0], fn[1], fn[2], fn[3], fast) | (two << kWalkDiv2);
  if (!walk_registered(wsig)) wsig = sig_make(int(arith.size()), fn[0], fn[1], fn[2], fn[3], fast);
  if (!walk_registered(wsig)) wsig = sig_make(int(arith.size()), fn[0], fn[1], fn[2], fn[3], 0);
  if (!walk_registered(wsig)) return false;

  // tables: one per distinct crop height / width (the out extents are uniform)
  std::vector<WalkRow> rows;
  std::vector<WalkCol> cols;
  std::map<uint32_t, uint32_t> row_at, col_at;
  std::vector<WalkAux> aux(B);
  std::vector<bool> swaps(B);
  bool swap0 = false, swap_uniform = true;
  for (uint32_t z = 0; z < B; ++z) {
    const DSample& s = dp.reads[z];
    auto r = row_at.find(s.rect_h);
    if (r == row_at.end()) {
      r = row_at.emplace(s.rect_h, uint32_t(rows.size())).first;
      for (uint32_t y = 0; y < H; ++y) rows.push_back(walk_row(y, s.rect_h, H));
      rows.push_back(WalkRow{kWalkRowMask, 0.0f, 0.0});  // sentinel: the walk reads one row ahead
    }
    auto c = col_at.find(s.rect_w);
    if (c == col_at.end()) {
      c = col_at.emplace(s.rect_w, uint32_t(cols.size())).first;
      for (uint32_t x = 0; x < W; ++x) cols.push_back(walk_col(x, s.rect_w, W));
    }
    WalkAux& a = aux[z];
    const bool swap = ((s.flags & SF_POST_SWAP) != 0) != dp.fused_swap;
    if (z == 0) swap0 = swap;
    swap_uniform = swap_uniform && swap == swap0;
    swaps[z] = swap;
    for (int m = 0; m < 3; ++m) a.dst[m] = writes[z].dst[swap ? 2 - m : m];
    a.dpitch = uint32_t(writes[z].pitch[0]);
    a.x3 = 3 * s.x0;
    a.coltab = c->second;
    a.kz = z;
  }
  // units: two half strips of 32 output columns (16 lanes, 2 columns each) per
  // warp, paired among the halves of planes with the same crop height
  struct Half { uint32_t z, x, n; };
  std::map<uint32_t, std::vector<Half>> by_h;  // rect_h -> half strips, plane order
  for (uint32_t z = 0; z < B; ++z)
    for (uint32_t x = 0; x < W; x += 2 * kWalkHalfLanes)
      by_h[dp.reads[z].rect_h].push_back(Half{z, x, std::min(kWalkHalfLanes, (W - x) / 2)});
  const uint64_t halves = uint64_t(B) * ((W + 2 * kWalkHalfLanes - 1) / (2 * kWalkHalfLanes));
  const uint64_t target = 148ull * 28 * 3;  // three waves of 28 warps per SM
  uint32_t bands = uint32_t(std::min<uint64_t>((2 * target + halves - 1) / halves, (H + 7) / 8));
  bands = std::max({bands, 1u, (H + kWalkMaxRows - 1) / kWalkMaxRows});
  const uint32_t band_rows = (H + bands - 1) / bands;
  std::vector<WalkUnit> units;
  uint32_t row_bytes = 16, box_max = 16;
  // one half: plane z, columns [x, x + 2n): the staged span [2 bx, ...) of each crop row
  auto half = [&](WalkUnit& u, int h, const Half& hf) {
    const DSample& s = dp.reads[hf.z];
    const WalkCol* ct = &cols[aux[hf.z].coltab];
    const uint32_t first = 3 * s.x0 + ct[hf.x].tap, last = 3 * s.x0 + ct[hf.x + 2 * hf.n - 1].tap;
    const uint32_t wb = first & ~15u;
    const uint32_t bw = (last + 6 - wb + 31) & ~31u;  // the half's box width (32-byte classes)
    row_bytes = std::max(row_bytes, bw);
    box_max = std::max(box_max, bw);
    u.bw[h] = uint16_t(std::min(bw, 65504u));
    ok = ok && bw <= 65504;
    u.z[h] = hf.z;
    u.bx[h] = uint16_t(wb / 2);
    u.x[h] = uint16_t(hf.x);
    u.n[h] = uint16_t(hf.n);
    ok = ok && wb / 2 < 65536;
  };
  uint32_t max_rows = 0;
  for (auto& kv : by_h) {
    // A unit costs ~ rows (finishes) + visits = rows (1 + rect_h / H). Where a
    // crop is more than 3x taller than the output (a band's visits are several
    // TMA round trips), its class's band is sized to the cost of a 1:1 band
    // (C2 16.7 -> 15.2 us). Elsewhere uniform bands measure best (C5: 75-row
    // uniform bands 1.149 ms, cost-balanced 112-row bands 1.161, balanced
    // 80-row 1.177; C4 B = 8..1024: shorter bands only add unit start-ups).
    const bool balance = kv.first > 3 * H;
    const uint32_t brk =
        balance ? std::min<uint32_t>(kWalkMaxRows,
                                     std::max<uint32_t>(1, uint32_t(2.0 * band_rows * H / (double(H) + kv.first) + 0.5)))
                : band_rows;
    max_rows = std::max(max_rows, brk);
    for (uint32_t y_lo = 0; y_lo < H; y_lo += brk) {
      const uint32_t y_hi = std::min(H, y_lo + brk);
      const WalkRow* rt = &rows[row_at[kv.first]];
      const std::vector<Half>& hs = kv.second;
      for (size_t i = 0; i < hs.size(); i += 2) {
        WalkUnit u{};
        const bool two = i + 1 < hs.size();
        half(u, 0, hs[i]);
        half(u, 1, two ? hs[i + 1] : hs[i]);
        if (!two) u.n[1] = 0;
        if (two && u.z[0] == u.z[1] && u.x[1] > u.x[0]) {
          // adjacent halves of one crop: ONE box over both spans (bw[1] = 0),
          // in 64-byte classes; the ring's two half slots hold it
          const uint32_t wb0 = 2u * u.bx[0], end1 = 2u * u.bx[1] + u.bw[1];
          const uint32_t bwm = (end1 - wb0 + 63) & ~63u;
          if (bwm <= 65504) {
            u.bw[0] = uint16_t(bwm);
            u.bw[1] = 0;
            u.bx[1] = u.bx[0];
            box_max = std::max(box_max, bwm);
            row_bytes = std::max(row_bytes, ((bwm + 1) / 2 + 15) & ~15u);
          }
        }
        u.y_lo = uint16_t(y_lo);
        u.y_hi = uint16_t(y_hi);
        const uint32_t r1 = rt[y_lo].r1 & kWalkRowMask;
        u.r_first = uint16_t((rt[y_lo].r1 & kWalkSame) ? r1 : r1 - 1);
        u.r_last = uint16_t(rt[y_hi - 1].r1 & kWalkRowMask);
        u.rowtab = row_at[kv.first];
        units.push_back(u);
      }
    }
  }
  // TMA tensor maps: one per source frame (buffer, pitch) and box width class,
  // its rows [0, rows)
  // as elements of 2, 4 or 8 bytes (the smallest whose 256-element box holds a
  // staged row) over [0, width): rows = the lowest crop bottom, width = the
  // widest crop's right edge rounded up to an element. The tensor's last
  // element of a row may extend past a crop, so that byte range must be
  // readable: every row but the frame's last has a row below it (pitch bytes),
  // the last row its crop's tail_bytes. One map per frame and width class
  // keeps the TMA descriptor cache warm (one per crop missed on every copy);
  // per-half box widths stage only the bytes a half needs (one widest box for
  // every half staged ~1.8x the crop bytes).
  const uint32_t elem = box_max <= 512 ? 2 : box_max <= 1024 ? 4 : 8;
  if (!ok || units.empty() || box_max > 256 * elem) return false;
  if (walk_smem_bytes(row_bytes, max_rows) > 200 * 1024) return false;
  struct Frame { uint64_t src = 0, pitch = 0, rows = 0, width = 0, tail = ~0ull; };
  std::map<std::pair<uint64_t, uint64_t>, uint32_t> frame_at;
  std::vector<Frame> frames;
  std::vector<uint32_t> frame_of(B);
  for (uint32_t z = 0; z < B; ++z) {
    const DSample& s = dp.reads[z];
    auto f = frame_at.emplace(std::make_pair(s.src, s.pitch), uint32_t(frames.size())).first;
    if (f->second == frames.size()) frames.push_back(Frame{s.src, s.pitch});
    frame_of[z] = f->second;
    Frame& fr = frames[f->second];
    const uint64_t bottom = uint64_t(s.y0) + s.rect_h, end = 3ull * (s.x0 + s.rect_w);
    if (bottom > fr.rows) fr.rows = bottom, fr.tail = s.tail_bytes;
    else if (bottom == fr.rows) fr.tail = std::min<uint64_t>(fr.tail, s.tail_bytes);
    fr.width = std::max(fr.width, (end + elem - 1) / elem);
    ok = ok && s.pitch <= 0xffffffffull;
  }
  for (size_t f = 0; f < frames.size() && ok; ++f)
    ok = frames[f].width * elem <= std::min<uint64_t>(frames[f].tail, frames[f].pitch);
  std::map<std::pair<uint32_t, uint32_t>, uint32_t> map_at;  // (frame, box width) -> map
  std::vector<CUtensorMap> maps;
  for (WalkUnit& u : units)
    for (int h = 0; h < 2 && ok; ++h) {
      u.bx[h] = uint16_t(u.bx[h] * 2 / elem);  // bx was in 2-byte elements
      u.y0[h] = dp.reads[u.z[h]].y0;
      if (u.bw[h] == 0) {  // merged into half 0's box
        u.map[h] = u.map[0];
        continue;
      }
      const uint32_t f = frame_of[u.z[h]];
      auto m = map_at.emplace(std::make_pair(f, uint32_t(u.bw[h])), uint32_t(maps.size())).first;
      if (m->second == maps.size()) {
        const Frame& fr = frames[f];
        maps.emplace_back();
        ok = maps.size() <= 65536 && walk_encode_map(&maps.back(), fr.src, fr.width, fr.rows, fr.pitch, elem,
                                                     u.bw[h] / elem, kWalkGroup);
      }
      u.map[h] = uint16_t(m->second);
    }
  if (!ok) return false;
  // units of one source frame back to back (the frame stays L2-resident while
  // its crops run), longest first within a frame (walk cost ~ visits + rows)
  std::stable_sort(units.begin(), units.end(), [&](const WalkUnit& a, const WalkUnit& b) {
    const uint64_t sa = dp.reads[a.z[0]].src, sb = dp.reads[b.z[0]].src;
    if (sa != sb) return sa < sb;
    return 2u * (a.r_last - a.r_first) + 5u * (a.y_hi - a.y_lo) > 2u * (b.r_last - b.r_first) + 5u * (b.y_hi - b.y_lo);
  });
  bool perz = !swap_uniform;
  for (const DOp& d : arith) perz = perz || d.per_z;
  // constants, input-lane order: lane m of plane z uses output lane sigma_z(m)
  auto lane_const = [&](const DOp& d, uint32_t z, int l) {
    const int li = d.nl == 3 ? l : 0;
    if (!d.per_z) return f32_bits(d.c[li]);
    const std::vector<uint64_t>& r = dp.per_z_host.at(d.per_z);
    return f32_bits(r[3 * size_t(z < d.per_z_n ? z : d.per_z_n - 1) + li]);
  };
  auto consts = [&](size_t k, uint32_t z, int m, bool swap, float& c, float& h, float& l) {
    c = lane_const(arith[k], z, swap ? 2 - m : m);
    h = l = 0.0f;
    if (arith[k].fn != AF_DIV) return;
    h = 1.0f / c;
    l = (two >> k) & 1u ? float(1.0 / double(c) - double(h)) : -c;
  };
  P = WalkPlan{};
  if (perz) {
    std::vector<float4> kz(size_t(B) * 12, make_float4(0, 0, 0, 0));
    for (uint32_t z = 0; z < B; ++z)
      for (size_t k = 0; k < arith.size(); ++k)
        for (int m = 0; m < 3; ++m) {
          float c, h, l;
          consts(k, z, m, swaps[z], c, h, l);
          kz[size_t(z) * 12 + 3 * k + m] = make_float4(c, h, l, 0.0f);
        }
    P.kz = upload(kz);
    dp.extra.push_back(const_cast<float4*>(P.kz));
  } else {
    for (size_t k = 0; k < arith.size(); ++k)
      for (int m = 0; m < 3; ++m) {
        float c, h, l;
        consts(k, 0, m, swap0, c, h, l);
        P.kc[k][m] = make_float2(c, c);
        P.kh[k][m] = make_float2(h, h);
        P.kl[k][m] = make_float2(l, l);
      }
  }
  P.units = upload(units);
  P.aux = upload(aux);
  P.rows = upload(rows);
  P.cols = upload(cols);
  P.maps = upload(maps);
  for (const void* q : {static_cast<const void*>(P.units), static_cast<const void*>(P.aux),
                        static_cast<const void*>(P.rows), static_cast<const void*>(P.cols),
                        static_cast<const void*>(P.maps)})
    dp.extra.push_back(const_cast<void*>(q));
  P.n_units = uint32_t(units.size());
  P.row_bytes = row_bytes;
  P.elem = elem;
  P.negz = kNegZero2;
  P.max_rows = max_rows;
  P.sink = reinterpret_cast<uint64_t>(upload(std::vector<uint64_t>(kWalkSinkLines * 32, 0)));
  dp.extra.push_back(reinterpret_cast<void*>(P.sink));
  wsig_out = wsig;
  perz_out = perz;
  return true;
}

// The fast unfused comparator's passes (execute_unfused, executor.cpp:134-217),
// when every pass is streamable: f32 / f32x3 arithmetic, a final Cast f32 ->
// u8 on one lane, a split / per-thread write of the last intermediate; pass 0
// through fk_walk (crop batches) or a stream over contiguous f32 sources.
void build_unfused(DeviceProgram& dp, const Pipeline& p, const std::vector<DWrite>& writes) {
  const uint32_t W = p.space.width, H = p.space.height, B = p.space.batch;
  const size_t n = p.compute.size();
  const uint64_t pts = uint64_t(W) * H;
  if (n == 0 || W % 4 || pts % 4 || pts * B * 3 / 4 >= (uint64_t(1) << 32) || dp.reads.empty()) return;
  const DOp* ops = dp.table.data() + dp.n_fused;  // the 1:1 program
  auto plane_div = [&](uint32_t nl) { return make_fastdiv(uint32_t(pts / 4)); };
  std::vector<StreamPass> passes(n + 1);
  std::vector<uint64_t> bytes(n);
  uint32_t kind = uint32_t(p.read.out_kind);
  for (size_t i = 0; i < n; ++i) {
    const DOp& d = ops[i];
    const uint32_t out = uint32_t(p.compute[i].out_kind);
    StreamPass& S = passes[i];
    S = StreamPass{};
    S.nl = uint32_t(lanes_of(kind));
    S.chunks = pts * B * S.nl / 4;
    S.plane_chunks = plane_div(S.nl);
    S.negz = kNegZero2;
    S.repeat = 1;
    if (d.cls == OC_ARITH && lane_kind(kind) == FK_F32 && out == kind) {
      S.op = SP_ARITH;
      S.fn = d.fn;
      S.repeat = d.repeat;
      for (int l = 0; l < 3; ++l) S.c[l] = f32_bits(d.c[d.nl == 3 ? l : 0]);
      S.per_z = reinterpret_cast<const uint64_t*>(d.per_z);
      S.per_z_n = d.per_z_n;
    } else if (d.cls == OC_NOP && lane_kind(kind) == FK_F32 && out == kind) {
      S.op = SP_ARITH;  // an identity cast: a copy pass
      S.fn = AF_ADD;
      S.repeat = 0;
    } else if (d.cls == OC_CAST && kind == FK_F32 && out == FK_U8) {
      S.op = SP_TO_U8;
    } else {
      return;
    }
    bytes[i] = pts * B * bpe(out);
    kind = out;
  }
  // the write pass: the last intermediate through the write op
  const uint32_t wid = p.write.id == FK_OP_BATCH_WRITE ? p.write.w_inner : p.write.id;
  StreamPass& F = passes[n];
  F = StreamPass{};
  F.op = SP_COPY;
  F.nl = uint32_t(lanes_of(kind));
  F.chunks = pts * B * F.nl / 4;
  F.plane_chunks = plane_div(F.nl);
  F.row_chunks = make_fastdiv(W / 4);
  F.width = W;
  F.vbytes = bpe(kind) / F.nl;
  if (!(wid == FK_OP_SPLIT_WRITE && kind == FK_F32X3) && !(wid == FK_OP_PER_THREAD_WRITE && F.nl == 1)) return;
  if (lane_kind(kind) != FK_F32 && kind != FK_U8) return;
  const uint64_t align = F.vbytes == 4 ? 16 : 4;
  for (const DWrite& w : writes)
    for (uint32_t l = 0; l < F.nl; ++l)
      if ((w.flags & WF_ACTIVE) && ((w.dst[l] | w.pitch[l]) % align)) return;
  F.wr = writes[0];  // non-batch; a BatchWrite's table (dp.d_writes) is set at launch
  // pass 0
  const DSample& s0 = dp.reads[0];
  bool direct = uint32_t(p.read.out_kind) == FK_F32;
  for (uint32_t z = 0; z < B && direct; ++z) {
    const DSample& s = dp.reads[z];
    direct = !(s.flags & SF_DEFAULT) && s.mode == RD_DIRECT && s.kind == FK_F32 && s.post_len == 0 && s.x0 == 0 &&
             s.y0 == 0 && s.pitch == uint64_t(W) * 4 && s.src == s0.src + uint64_t(z) * pts * 4 && s.src % 16 == 0;
  }
  if (!direct) {  // fk_walk over op 0 into the planar intermediate [z][lane][H W]
    if (!dp.affine_ok || uint32_t(p.compute[0].out_kind) != FK_F32X3) return;
    std::vector<DOp> one{ops[0]};
    if (ops[0].cls != OC_ARITH || ops[0].repeat != 1) return;
    uint32_t fast = ops[0].fn == AF_DIV && recip_div_exact(one, 0, dp.per_z_host, B) ? 1u : 0u;
    const uint32_t sig = sig_make(1, ops[0].fn, 0, 0, 0, fast);
    std::vector<DWrite> planar(B);
    for (uint32_t z = 0; z < B; ++z) {
      planar[z] = DWrite{};
      for (int l = 0; l < 3; ++l) {
        planar[z].dst[l] = (uint64_t(z) * 3 + l) * pts * 4;  // offsets: WalkPlan::dst_base adds the buffer
        planar[z].pitch[l] = uint64_t(W) * 4;
      }
      planar[z].flags = WF_ACTIVE;
    }
    if (!build_walk(dp, p, one, sig, planar, dp.unf_walk_plan, dp.unf_walk_sig, dp.unf_walk_perz)) return;
    dp.unf_walk = true;
  }
  dp.unf_pass = passes;
  dp.unf_bytes = bytes;
  dp.unf_fast = true;
}

bool sep_stage_ok(const DeviceProgram& dp, uint32_t W, uint32_t T, uint32_t spc);

std::shared_ptr<DeviceProgram> build_program(const Pipeline& p, int device) {
  keep_pool_memory(device);
  auto dp = std::make_shared<DeviceProgram>();
  dp->device = device;
  const uint32_t W = p.space.width, H = p.space.height, B = p.space.batch;

  // compute program (1:1) + BatchArith constant tables
  std::vector<DOp> ops;
  for (const Op& op : p.compute) {
    DOp d = encode_compute(op);
    if (op.id == FK_OP_BATCH_ARITH) {
      std::vector<uint64_t> rows(op.values.size() * 3);
      for (size_t z = 0; z < op.values.size(); ++z) {
        uint64_t c[3];
        encode_element(uint32_t(op.in_kind), op.values[z], c);
        std::memcpy(&rows[3 * z], c, sizeof c);
      }
      uint64_t* t = upload(rows);
      dp->extra.push_back(t);
      dp->per_z_host[reinterpret_cast<uint64_t>(t)] = rows;
      d.per_z = reinterpret_cast<uint64_t>(t);
      d.per_z_n = uint32_t(op.values.size());
    }
    ops.push_back(d);
    add_kind(uint32_t(op.in_kind), dp->fused_wide, dp->fused_lanes);
    add_kind(uint32_t(op.out_kind), dp->fused_wide, dp->fused_lanes);
  }
  const std::vector<DOp> fops = compress(ops);
  dp->n_fused = uint32_t(fops.size());
  dp->n_ops = uint32_t(ops.size());
  for (const DOp& d : fops) {
    dp->fused_lut_ok = dp->fused_lut_ok && lane_wise(d);
    dp->fused_swap ^= odd_swap(d);
  }
  dp->table = fops;
  dp->table.insert(dp->table.end(), ops.begin(), ops.end());
  const uint32_t post_base = uint32_t(dp->table.size());

  // per-plane reads (BatchRead array, ops.cpp:369-378) + deduplicated post programs
  std::map<std::vector<uint32_t>, uint32_t> post_index;
  bool flat = uint64_t(W) * H < (uint64_t(1) << 32);
  dp->def_kind = uint32_t(p.read.out_kind);
  if (p.read.id == FK_OP_BATCH_READ) encode_element(dp->def_kind, p.read.def, dp->def);
  add_kind(dp->def_kind, dp->read_wide, dp->read_lanes);
  for (uint32_t z = 0; z < B; ++z) {
    DSample s{};
    const Sample* sp = read_plane(p, z);
    if (!sp) {
      s.flags = SF_DEFAULT;
      dp->reads.push_back(s);
      continue;
    }
    s.src = reinterpret_cast<uint64_t>(sp->source.data);
    s.pitch = pitch_of(sp->source);
    if (s.pitch >= (uint64_t(1) << 32)) fail(FK_E_CAPACITY_OVERFLOW, "source rows above 4 GiB");
    s.x0 = sp->x0;
    s.y0 = sp->y0;
    s.rect_w = sp->rect_w;
    s.rect_h = sp->rect_h;
    s.out_w = sp->out_w;
    s.out_h = sp->out_h;
    s.kind = sp->source.kind;
    s.mode = !sp->resizing() ? RD_DIRECT : (sp->mode == FK_NEAREST ? RD_NEAREST : RD_BILINEAR);
    s.flags = lane_aligned(sp->source) ? SF_LANE_ALIGNED : 0;
    {  // how far a whole-row bulk copy may read in the crop's last row
      const uint64_t last = uint64_t(sp->y0) + (sp->rect_h ? sp->rect_h : 1) - 1;
      const uint64_t lim = last + 1 < sp->source.height ? s.pitch : uint64_t(sp->source.width) * bpe(sp->source.kind);
      s.tail_bytes = uint32_t(std::min<uint64_t>(lim, 0xffffffffu));
    }
    add_kind(s.kind, dp->read_wide, dp->read_lanes);
    bool post_lane_wise = true, post_swap = false;
    if (!sp->post.empty()) {
      std::vector<uint32_t> key;
      for (const Folded& f : sp->post) {
        key.insert(key.end(), {f.id, f.in, f.out});
        add_kind(f.in, dp->read_wide, dp->read_lanes);
        add_kind(f.out, dp->read_wide, dp->read_lanes);
        const DOp d = encode_unary(f);
        post_lane_wise = post_lane_wise && lane_wise(d);
        post_swap ^= odd_swap(d);
      }
      auto it = post_index.find(key);
      if (it == post_index.end()) {
        const uint32_t off = uint32_t(dp->table.size());
        for (const Folded& f : sp->post) dp->table.push_back(encode_unary(f));
        it = post_index.emplace(key, off).first;
      }
      s.post_off = it->second;
      s.post_len = uint32_t(sp->post.size());
    } else {
      s.post_off = post_base;
    }
    if (lane_kind(s.kind) == FK_U8 && post_lane_wise) s.flags |= SF_LUT_SRC;
    if (post_swap) s.flags |= SF_POST_SWAP;
    // contiguous identity read of whole rows -> the plane is one flat run
    flat = flat && s.mode == RD_DIRECT && s.x0 == 0 && s.y0 == 0 && sp->source.row_stride == W;
    dp->reads.push_back(s);
  }
  dp->read_flat = flat;

  // per-plane writes (BatchWrite array, ops.cpp:437-445)
  std::vector<DWrite> writes;
  const bool batch_w = p.write.id == FK_OP_BATCH_WRITE;
  const uint32_t wid = batch_w ? p.write.w_inner : p.write.id;
  const int per = wid == FK_OP_SPLIT_WRITE ? 3 : 1;
  bool wflat = uint64_t(W) * H < (uint64_t(1) << 32);
  for (uint32_t z = 0; z < B; ++z) {
    DWrite w{};
    const bool active = !batch_w || z < p.write.active;
    w.flags = active ? (WF_ACTIVE | WF_STREAM) : 0;
    bool al = true;
    for (int l = 0; l < per; ++l) {
      const fk_plane& d = batch_w ? p.write.wdest[size_t(z) * per + l] : p.write.dest[l];
      w.dst[l] = reinterpret_cast<uint64_t>(d.data);
      w.pitch[l] = pitch_of(d);
      al = al && lane_aligned(d);
      wflat = wflat && d.row_stride == W;
    }
    if (al) w.flags |= WF_LANE_ALIGNED;
    writes.push_back(w);
  }
  dp->write_flat = wflat;
  add_kind(uint32_t(p.write.in_kind), dp->fused_wide, dp->fused_lanes);
  if (dp->read_wide) dp->fused_wide = true;
  if (dp->read_lanes == 3) dp->fused_lanes = 3;

  // compiled-kernel eligibility: every plane a u8-lane read with lane-wise folded
  // unaries, a lane-wise compute program, lane count preserved to the write
  {
    bool ok = dp->fused_lut_ok && !dp->reads.empty();
    const int nl = dp->reads.empty() ? 0 : lanes_of(dp->reads[0].kind);
    for (const DSample& s : dp->reads)
      ok = ok && !(s.flags & SF_DEFAULT) && (s.flags & SF_LUT_SRC) && lanes_of(s.kind) == nl;
    ok = ok && lanes_of(uint32_t(p.write.in_kind)) == nl;
    for (const DWrite& w : writes)  // the column-streaming kernel keeps 32-bit destination pitches
      for (uint64_t pitch : w.pitch) ok = ok && pitch < (1ull << 32);
    dp->resample_ok = ok;
    dp->resample_lanes = nl;
    // the column-streaming kernel keeps 32-bit source pitches (row addresses are IMAD.WIDE)
    bool sep = true;
    for (const DSample& s : dp->reads)  // ... and 16-bit band-relative source rows
      sep = sep && s.pitch < (1ull << 32) && s.rect_h < 65536 && s.out_h < 65536;
    dp->sep_ok = sep;
    // AFFINE mode: [SwapRB | Cast u8->f32]* (exactly one cast, folded or not), then
    // only f32 Mul/Add/Sub/Div (no swap after the first one), at most 4 of them.
    bool aff = ok && lane_kind(uint32_t(p.write.in_kind)) == FK_F32;
    int post_casts = -1;
    for (const DSample& s : dp->reads) {
      int casts = 0;
      for (uint32_t i = 0; i < s.post_len && aff; ++i) {
        const DOp& d = dp->table[s.post_off + i];
        if (d.cls == OC_CAST && d.lk_in == FK_U8 && d.lk_out == FK_F32) ++casts;
        else if (d.cls != OC_SWAP) aff = false;
      }
      if (post_casts >= 0 && casts != post_casts) aff = false;
      post_casts = casts;
    }
    int casts = post_casts < 0 ? 0 : post_casts;
    std::vector<DOp> arith;
    for (uint32_t i = 0; i < dp->n_fused && aff; ++i) {
      const DOp& d = dp->table[i];
      if (d.cls == OC_CAST && d.lk_in == FK_U8 && d.lk_out == FK_F32 && arith.empty()) ++casts;
      else if (d.cls == OC_SWAP && arith.empty()) continue;
      else if (d.cls == OC_ARITH && d.lk_in == FK_F32) arith.push_back(d);
      else aff = false;
    }
    aff = aff && casts == 1 && arith.size() <= 4;
    for (const DOp& d : arith) aff = aff && d.repeat == 1;
    uint32_t sig = kSigLut;
    if (aff) {
      uint32_t fn[4] = {0, 0, 0, 0}, fast = 0;
      for (size_t k = 0; k < arith.size(); ++k) {
        fn[k] = arith[k].fn;
        if (fn[k] == AF_DIV && recip_div_exact(arith, k, dp->per_z_host, B)) fast |= 1u << k;
      }
      sig = sig_make(int(arith.size()), fn[0], fn[1], fn[2], fn[3], fast);
      if (!resample_affine_registered(sig)) sig = sig_make(int(arith.size()), fn[0], fn[1], fn[2], fn[3], 0);
      aff = resample_affine_registered(sig);
    }
    dp->affine_ok = aff;
    if (aff) {
      dp->aff_sig = sig;
      dp->aff_base = uint32_t(dp->table.size());
      dp->aff_n = uint32_t(arith.size());
      dp->table.insert(dp->table.end(), arith.begin(), arith.end());
      dp->aff_inline = true;
      for (size_t k = 0; k < arith.size(); ++k) {
        dp->aff_inline = dp->aff_inline && !arith[k].per_z;
        for (int l = 0; l < 3; ++l) {
          const uint32_t bits = uint32_t(arith[k].c[arith[k].nl == 3 ? l : 0]);
          float c;
          std::memcpy(&c, &bits, 4);
          dp->aff_c[k][l] = c;
          dp->aff_r[k][l] = 1.0f / c;  // IEEE RN, as __frcp_rn
        }
      }
    }
    dp->walk_ok = build_walk(*dp, p, arith, sig, writes, dp->walk, dp->walk_sig, dp->walk_perz);
    build_unfused(*dp, p, writes);
  }
  // direct f32 kernel: f32 planes read as-is, f32 arith runs (any repeat), an
  // optional final Cast f32 -> u8, a packed write
  {
    bool ok = !dp->reads.empty() && (p.write.id == FK_OP_BATCH_WRITE ? p.write.w_inner : p.write.id) ==
                                        FK_OP_PER_THREAD_WRITE;
    for (const DSample& s : dp->reads)
      ok = ok && !(s.flags & SF_DEFAULT) && s.mode == RD_DIRECT && s.kind == FK_F32 && s.post_len == 0 &&
           (s.flags & SF_LANE_ALIGNED);
    std::vector<DOp> arith;
    bool to_u8 = false;
    for (uint32_t i = 0; i < dp->n_fused && ok; ++i) {
      const DOp& d = dp->table[i];
      if (d.cls == OC_ARITH && d.lk_in == FK_F32 && d.nl == 1 && !d.per_z && !to_u8) arith.push_back(d);
      else if (d.cls == OC_CAST && d.lk_in == FK_F32 && d.lk_out == FK_U8 && d.nl == 1 && i + 1 == dp->n_fused)
        to_u8 = true;
      else ok = false;
    }
    ok = ok && arith.size() <= 4 && uint32_t(p.write.in_kind) == (to_u8 ? FK_U8 : FK_F32);
    if (ok) {
      uint32_t fn[4] = {0, 0, 0, 0}, fast = 0, total = 0;
      for (size_t k = 0; k < arith.size(); ++k) {
        fn[k] = arith[k].fn;
        if (fn[k] == AF_DIV) {
          const int lvl = recip_div_verified(f32_bits(arith[k].c[0]));
          if (lvl >= 1) fast |= 1u << k;
          if (lvl >= 2) total |= 1u << k;
        }
      }
      uint32_t sig = sig_make(int(arith.size()), fn[0], fn[1], fn[2], fn[3], fast, total);
      if (!direct_registered(sig)) sig = sig_make(int(arith.size()), fn[0], fn[1], fn[2], fn[3], fast);
      if (!direct_registered(sig)) sig = sig_make(int(arith.size()), fn[0], fn[1], fn[2], fn[3], 0);
      ok = direct_registered(sig);
      if (ok) {
        dp->direct_ok = true;
        dp->direct_u8 = to_u8;
        dp->dir_sig = sig;
        dp->dir_base = uint32_t(dp->table.size());
        dp->table.insert(dp->table.end(), arith.begin(), arith.end());
      }
    }
  }
  // Visit planes grouped by source buffer (then by crop origin): the crops of one
  // frame run back to back, so the frame stays L2-resident instead of every
  // frame of the batch competing for L2 at once. Any order is correct: planes
  // are independent (ops.cpp:369-378).
  if (B > 1) {
    std::vector<uint32_t> order(B);
    for (uint32_t z = 0; z < B; ++z) order[z] = z;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
      const DSample &x = dp->reads[a], &y = dp->reads[b];
      if (x.src != y.src) return x.src < y.src;
      if (x.y0 != y.y0) return x.y0 < y.y0;
      return x.x0 < y.x0;
    });
    bool identity = true;
    for (uint32_t z = 0; z < B; ++z) identity = identity && order[z] == z;
    if (!identity) dp->d_order = upload(order);
    // Two-plane slots for the column-streaming kernel: planes whose row walk is
    // identical (same read mode, rect_h and lane swap; out_h is uniform over the
    // batch) share one CTA, in the source-grouped order above.
    if (dp->resample_ok && dp->sep_ok) {
      std::map<std::tuple<uint32_t, uint32_t, uint32_t>, uint32_t> open;  // key -> plane waiting for a partner
      std::vector<uint32_t> slots;
      for (uint32_t z : order) {
        const DSample& r = dp->reads[z];
        const auto key = std::make_tuple(r.mode, r.mode == RD_DIRECT ? 0u : r.rect_h, r.flags & SF_POST_SWAP);
        auto it = open.find(key);
        if (it == open.end()) {
          open.emplace(key, uint32_t(slots.size()));
          slots.push_back(z);
          slots.push_back(kNoPlane);
        } else {
          slots[it->second + 1] = z;
          open.erase(it);
        }
      }
      dp->n_slices2 = uint32_t(slots.size() / 2);
      dp->d_slots2 = upload(slots);
    }
  }
  if (dp->resample_ok && dp->sep_ok) {  // staged column walk: every warp's span fits the ring
    const uint32_t pairs = (W + 1) / 2;
    dp->stage_ok[0] = sep_stage_ok(*dp, W, pairs, 1);
    dp->stage_ok[1] = dp->d_slots2 != nullptr && sep_stage_ok(*dp, W, pairs, 2);
  }
  dp->traffic = analytic_traffic(p);
  dp->d_table = upload(dp->table);
  dp->d_reads = upload(dp->reads);
  dp->d_writes = upload(writes);
  return dp;
}

DPlan base_plan(uint32_t W, uint32_t H, uint32_t B, bool flat, int E) {
  DPlan P{};
  P.negz = kNegZero2;
  if (flat) {
    W = W * H;
    H = 1;
  }
  P.width = W;
  P.height = H;
  P.batch = B;
  P.tiles_per_row = (W + uint32_t(E) - 1) / uint32_t(E);
  const uint64_t tiles = uint64_t(H) * P.tiles_per_row;
  if (tiles >= (uint64_t(1) << 32) - 65536) fail(FK_E_CAPACITY_OVERFLOW, "plane too large for one launch");
  P.tiles = uint32_t(tiles);
  P.tpr = make_fastdiv(P.tiles_per_row);
  // Each CTA walks a contiguous tile range: up to 16 tiles per thread, enough
  // CTAs to fill 148 SMs several times over, and few enough rows per CTA that
  // the resample y-table fits (kYCap).
  const uint64_t planes = B;
  uint32_t per_thread = 16;
  while (per_thread > 1 && planes * ((tiles + uint64_t(kBlock) * per_thread - 1) / (uint64_t(kBlock) * per_thread)) < 148u * 8u)
    per_thread /= 2;
  uint64_t tpc = uint64_t(kBlock) * per_thread;
  const uint64_t max_rows_tiles = uint64_t(kYCap - 2) * P.tiles_per_row;
  while (tpc > kBlock && tpc > max_rows_tiles) tpc -= kBlock;
  P.tiles_per_cta = uint32_t(tpc);
  return P;
}

int current_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(FK_E_NO_DEVICE, "no CUDA device visible");
  }
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  int major = 0;
  cuda_check(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev), "cudaDeviceGetAttribute");
  if (major != 10) fail(FK_E_NO_DEVICE, "libfk_cuda.so is built for sm_100a (B200); device " +
                                            std::to_string(dev) + " is sm_" + std::to_string(major) + "x");
  return dev;
}

std::mutex g_build_mu;

// The pipeline's program for the current device, built on first use. The
// returned reference stays valid for the pipeline's lifetime: programs are
// never replaced, and all lazily derived plan state is computed in
// build_program under this lock (execute_* only read it, so concurrent
// executes of one pipeline are safe).
DeviceProgram& ensure_program(const Pipeline& p) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(g_build_mu);
  auto& slot = const_cast<Pipeline&>(p).dev[dev];
  if (!slot) slot = build_program(p, dev);
  return *slot;
}

struct Timer {
  cudaStream_t st;
  bool on;
  cudaEvent_t a = nullptr, b = nullptr;
  Timer(cudaStream_t s, bool enabled) : st(s), on(enabled) {
    if (!on) return;
    cuda_check(cudaEventCreate(&a), "cudaEventCreate");
    cuda_check(cudaEventCreate(&b), "cudaEventCreate");
    cuda_check(cudaEventRecord(a, st), "cudaEventRecord");
  }
  double stop() {
    if (!on) return 0.0;
    cuda_check(cudaEventRecord(b, st), "cudaEventRecord");
    cuda_check(cudaEventSynchronize(b), "cudaEventSynchronize");
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
  }
  ~Timer() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

void launch(int cls, const DPlan& P, cudaStream_t st, uint64_t& count) {
  cuda_check(launch_generic(cls, P, st), "fk_transform_generic launch");
  ++count;
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

uint64_t now_ns() {
  return uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                      std::chrono::steady_clock::now().time_since_epoch()).count());
}

void fill_plan_io(DPlan& P, const DeviceProgram& dp, const Pipeline& p, const fk_exec_config* cfg) {
  P.table = dp.d_table;
  P.order = dp.d_order;
  P.prog_inline = dp.table.size() <= kProg ? 1u : 0u;
  if (P.prog_inline) std::memcpy(P.prog, dp.table.data(), dp.table.size() * sizeof(DOp));
  P.def_kind = dp.def_kind;
  std::memcpy(P.def, dp.def, sizeof P.def);
  P.write_kind = uint32_t(p.write.in_kind);
  const uint32_t wid = p.write.id == FK_OP_BATCH_WRITE ? p.write.w_inner : p.write.id;
  P.write_mode = wid == FK_OP_SPLIT_WRITE ? WR_SPLIT : WR_DIRECT;
  P.lut_ok = 0;
  (void)cfg;
}

bool lut_allowed(const fk_exec_config* cfg) { return !(cfg && (cfg->flags & FK_EXEC_NO_LUT)); }

}  // namespace

namespace {

// Host mirror of x_entry (fk_stages.cuh): tap byte offsets of output column i.
void host_taps(const DSample& s, uint32_t i, uint32_t bpe, uint32_t& o0, uint32_t& o1) {
  const double cx = (double(i) + 0.5) * double(s.rect_w) / double(s.out_w) - 0.5;
  const long long ix = (long long)std::floor(cx), maxx = (long long)s.rect_w - 1;
  o0 = uint32_t((s.x0 + std::min(std::max(ix, 0ll), maxx)) * bpe);
  o1 = uint32_t((s.x0 + std::min(std::max(ix + 1, 0ll), maxx)) * bpe);
}

// Can every warp of the column-streaming kernel use the staged (cp.async ring)
// walk? Source rows 16-byte aligned, and each warp's span of source bytes per
// plane slot fits its ring region (the whole row, or half when the warp holds
// two slots) — the same arithmetic as stage_plan in fk_resample_sep.cuh.
bool sep_stage_ok(const DeviceProgram& dp, uint32_t W, uint32_t T, uint32_t spc) {
  const uint32_t row = resample_sep_ring_row();
  const uint32_t warps = (spc * T + 31) / 32;
  for (const DSample& s : dp.reads) {
    if (s.mode != RD_BILINEAR) continue;
    if (((s.src + uint64_t(s.y0) * s.pitch) | s.pitch) & 15) return false;
    const uint32_t bpe = uint32_t(lanes_of(s.kind));
    for (uint32_t wi = 0; wi < warps; ++wi) {
      const uint32_t t0 = wi * 32, t1 = std::min(t0 + 32, spc * T);
      const bool two = t0 / T != (t1 - 1) / T;
      for (uint32_t h = t0 / T; h <= (t1 - 1) / T; ++h) {
        const uint32_t p0 = std::max(t0, h * T) - h * T, p1 = std::min(t1, (h + 1) * T) - h * T;
        const uint32_t c0 = 2 * p0, c1 = std::min(2 * p1, W);
        if (c0 >= c1) continue;
        uint32_t lo, x1, x2, hi;
        host_taps(s, c0, bpe, lo, x1);
        host_taps(s, c1 - 1, bpe, x2, hi);
        hi += bpe;
        if ((hi - (lo & ~15u) + 15) / 16 * 16 > (two ? row / 2 : row)) return false;
      }
    }
  }
  return true;
}

}  // namespace

void check_config(const fk_exec_config* c) {  // executor.cpp:20-25
  if (!c) return;
  if (c->chunk_rows < 1) fail(FK_E_INVALID_CONFIG, "chunk_rows must be >= 1");
  const int b = c->coarsen_block;
  if (!(b == 1 || b == 2 || b == 4 || b == 8 || b == 16))
    fail(FK_E_INVALID_CONFIG, "coarsening block must be one of 1/2/4/8/16");
  if (c->workers < 0) fail(FK_E_INVALID_CONFIG, "workers must be >= 0");
}

fk_exec_report execute_fused(const Pipeline& p, const fk_exec_config* cfg) {
  check_config(cfg);
  const uint64_t t0 = now_ns();
  DeviceProgram& dp = ensure_program(p);
  cudaStream_t st = cfg ? static_cast<cudaStream_t>(cfg->stream) : nullptr;
  fk_exec_report r{};
  Timer timer(st, cfg && (cfg->flags & FK_EXEC_TIMED));
  const bool generic_only = cfg && (cfg->flags & FK_EXEC_FORCE_GENERIC);
  // kernel selection: a registered compiled chain first, the interpreter otherwise
  const bool direct = dp.direct_ok && !generic_only;
  const bool affine = !direct && dp.affine_ok && !generic_only;
  const bool compiled = affine || (!direct && dp.resample_ok && lut_allowed(cfg) && !generic_only);
  const int cls = generic_state_class(dp.fused_wide, dp.fused_lanes);
  DPlan P = base_plan(p.space.width, p.space.height, p.space.batch, dp.read_flat && dp.write_flat,
                      direct ? direct_elems() : compiled ? resample_elems() : generic_elems(cls));
  fill_plan_io(P, dp, p, cfg);
  P.op_base = affine ? dp.aff_base : direct ? dp.dir_base : 0;
  P.n_ops = affine ? dp.aff_n : dp.n_fused;
  P.lut_ok = (dp.fused_lut_ok && lut_allowed(cfg)) ? 1u : 0u;
  P.prog_swap = dp.fused_swap ? 1u : 0u;
  P.reads = dp.d_reads;
  P.writes = dp.d_writes;
  if (direct) {
    // the chain's constants at fixed parameter offsets: the kernel's FMUL/FADD
    // read them as constant-bank operands
    for (uint32_t k = 0; k < 4 && k < uint32_t(sig_n(dp.dir_sig)); ++k) {
      const DOp& d = dp.table[dp.dir_base + k];
      const float c = f32_bits(d.c[0]);
      P.aff_c[k][0] = c;
      P.aff_r[k][0] = 1.0f / c;  // RN(1/c) on the host: the same value as the device's __frcp_rn
      P.dir_rep[k] = d.repeat;
    }
    cuda_check(launch_direct(dp.dir_sig, dp.direct_u8, P, st), "fk_direct launch");
    t_last_kernel = "fk_direct";
    ++r.kernels_launched;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    r.path = FK_PATH_COMPILED;
  } else if (affine && dp.walk_ok) {
    // column-walk crop kernel: one warp per (64-column strip, row band), source rows visited once
    WalkPlan C = dp.walk;
    C.reads = dp.d_reads;
    cuda_check(launch_walk(dp.walk_sig, dp.walk_perz, C, st), "fk_walk launch");
    t_last_kernel = "fk_walk";
    ++r.kernels_launched;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    r.path = FK_PATH_COMPILED;
  } else if (compiled && dp.sep_ok) {
    // column-streaming kernel: one warp per CTA, 32 column pairs x a band of rows
    // of one z slice (one plane, or two planes of equal row structure side by side)
    const uint32_t W = p.space.width, H = p.space.height, B = p.space.batch;
    const uint32_t pairs = (W + 1) / 2;  // one lane per output column pair
    const uint32_t w1 = (pairs + 31) / 32, w2 = (2 * pairs + 31) / 32;  // warps per slice
    // two planes per slice when that fills the warps better (224 columns: 112
    // pairs -> 7 full warps per two planes instead of 4 warps per plane)
    const bool dual = dp.d_slots2 && double(2 * pairs) / (32.0 * w2) > double(pairs) / (32.0 * w1);
    DPlan S = P;
    S.slots = dual ? dp.d_slots2 : nullptr;
    S.slots_per_cta = dual ? 2u : 1u;
    S.slot_threads = pairs;
    S.slices = dual ? dp.n_slices2 : B;
    S.no_stage = dp.stage_ok[dual ? 1 : 0] ? 0u : 1u;
    // band: whole planes (up to the table size) unless the batch is too small to
    // give ~2 waves of 16 warps per SM
    const uint64_t units = uint64_t(dual ? w2 : w1) * S.slices;
    const uint64_t target = 148ull * 16 * 2;
    uint64_t band = std::min<uint64_t>(H, resample_sep_band_max());
    if (units < target) {
      const uint64_t nb = (target + units - 1) / units;
      band = std::max<uint64_t>(4, std::min<uint64_t>(band, (H + nb - 1) / nb));
    }
    if (affine && dp.aff_inline) {
      S.aff_inline = 1;
      std::memcpy(S.aff_c, dp.aff_c, sizeof S.aff_c);
      std::memcpy(S.aff_r, dp.aff_r, sizeof S.aff_r);
    }
    S.width = W;
    S.height = H;
    S.tiles_per_cta = uint32_t(band);
    cuda_check(launch_resample_sep(dp.resample_lanes, lane_kind(uint32_t(p.write.in_kind)), P.write_mode == WR_SPLIT,
                                   affine ? dp.aff_sig : kSigLut, S, S.no_stage == 0, st),
               "fk_resample_sep launch");
    t_last_kernel = "fk_resample_sep";
    ++r.kernels_launched;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    r.path = FK_PATH_COMPILED;
  } else if (compiled) {
    cuda_check(launch_resample(dp.resample_lanes, lane_kind(uint32_t(p.write.in_kind)), P.write_mode == WR_SPLIT,
                               affine ? dp.aff_sig : kSigLut, P, st),
               "fk_resample launch");
    t_last_kernel = "fk_resample";
    ++r.kernels_launched;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    r.path = FK_PATH_COMPILED;
  } else {
    launch(cls, P, st, r.kernels_launched);
    t_last_kernel = "fk_transform_generic";
    r.path = FK_PATH_GENERIC;
  }
  r.device_ms = timer.stop();
  r.wall_time_ns = now_ns() - t0;
  r.bytes_read = dp.traffic.fused_read;
  r.bytes_written = dp.traffic.fused_written;
  r.passes = 1;
  r.points_visited = uint64_t(p.space.width) * p.space.height * p.space.batch;
  return r;
}

fk_exec_report execute_unfused(const Pipeline& p, const fk_exec_config* cfg) {
  check_config(cfg);
  const uint64_t t0 = now_ns();
  DeviceProgram& dp = ensure_program(p);
  cudaStream_t st = cfg ? static_cast<cudaStream_t>(cfg->stream) : nullptr;
  fk_exec_report r{};
  Timer timer(st, cfg && (cfg->flags & FK_EXEC_TIMED));
  const uint32_t W = p.space.width, H = p.space.height, B = p.space.batch;
  const size_t n = p.compute.size();
  if (dp.unf_fast && !(cfg && (cfg->flags & FK_EXEC_FORCE_GENERIC))) {
    // one compiled streaming pass per op (planar intermediates), then the write pass
    void* prev = nullptr;
    for (size_t i = 0; i <= n; ++i) {
      void* next = nullptr;
      if (i < n) {
        cuda_check(cudaMallocAsync(&next, dp.unf_bytes[i], st), "cudaMallocAsync(intermediate)");
        r.intermediate_bytes_allocated += dp.unf_bytes[i];
      }
      if (i == 0 && dp.unf_walk) {
        WalkPlan C = dp.unf_walk_plan;
        C.reads = dp.d_reads;
        C.dst_base = reinterpret_cast<uint64_t>(next);
        cuda_check(launch_walk(dp.unf_walk_sig, dp.unf_walk_perz, C, st), "fk_walk launch (unfused pass 0)");
      } else {
        StreamPass S = dp.unf_pass[i];
        S.src = static_cast<const uint8_t*>(i == 0 ? reinterpret_cast<void*>(dp.reads[0].src) : prev);
        S.dst = static_cast<uint8_t*>(next);
        if (i == n && p.write.id == FK_OP_BATCH_WRITE) S.writes = dp.d_writes;
        cuda_check(launch_stream(S, st), "fk_stream launch");
      }
      ++r.kernels_launched;
      g_launches.fetch_add(1, std::memory_order_relaxed);
      if (prev) cuda_check(cudaFreeAsync(prev, st), "cudaFreeAsync(intermediate)");
      prev = next;
    }
    t_last_kernel = "fk_stream";
    r.device_ms = timer.stop();
    r.wall_time_ns = now_ns() - t0;
    r.bytes_read = dp.traffic.unfused_read;
    r.bytes_written = dp.traffic.unfused_written;
    r.passes = n + 1;
    r.points_visited = uint64_t(W) * H * B * r.passes;
    r.path = FK_PATH_COMPILED;
    return r;
  }
  if (n == 0) {  // executor.cpp:144-166: one read -> write sweep
    const int cls = generic_state_class(dp.fused_wide, dp.fused_lanes);
    DPlan P = base_plan(W, H, B, dp.read_flat && dp.write_flat, generic_elems(cls));
    fill_plan_io(P, dp, p, cfg);
    P.op_base = 0;
    P.n_ops = 0;
    P.lut_ok = lut_allowed(cfg) ? 1u : 0u;  // folded unaries alone
    P.reads = dp.d_reads;
    P.writes = dp.d_writes;
    launch(cls, P, st, r.kernels_launched);
  } else {
    const uint64_t pts = uint64_t(W) * H;
    void* prev = nullptr;
    uint32_t prev_kind = 0;
    for (size_t i = 0; i <= n; ++i) {
      const bool final_pass = i == n;
      bool wide = false;
      int lanes = 1;
      DSample rd{};
      if (i == 0) {
        wide = dp.read_wide;
        lanes = dp.read_lanes;
      } else {  // load_block of the previous intermediate (executor.cpp:120-124)
        add_kind(prev_kind, wide, lanes);
        rd.src = reinterpret_cast<uint64_t>(prev);
        rd.pitch = uint64_t(W) * bpe(prev_kind);
        rd.rect_w = rd.out_w = W;
        rd.rect_h = rd.out_h = H;
        rd.kind = prev_kind;
        rd.mode = RD_DIRECT;
        rd.post_off = dp.n_fused + dp.n_ops;
        rd.flags = SF_LANE_ALIGNED | (lane_kind(prev_kind) == FK_U8 ? SF_LUT_SRC : 0u);
      }
      void* next = nullptr;
      uint32_t out_kind = 0;
      if (!final_pass) {
        out_kind = uint32_t(p.compute[i].out_kind);
        add_kind(uint32_t(p.compute[i].in_kind), wide, lanes);
        add_kind(out_kind, wide, lanes);
        cuda_check(cudaMallocAsync(&next, pts * B * bpe(out_kind), st), "cudaMallocAsync(intermediate)");
        r.intermediate_bytes_allocated += pts * B * bpe(out_kind);
      } else {
        add_kind(uint32_t(p.write.in_kind), wide, lanes);
      }
      const int cls = generic_state_class(wide, lanes);
      const bool flat = (i == 0 ? dp.read_flat : true) && (final_pass ? dp.write_flat : true);
      DPlan P = base_plan(W, H, B, flat, generic_elems(cls));
      fill_plan_io(P, dp, p, cfg);
      if (i == 0) {
        P.reads = dp.d_reads;
      } else {
        P.rd = rd;
        P.rd_zstride = pts * bpe(prev_kind);
      }
      if (final_pass) {  // final sweep through the write op (executor.cpp:197-213)
        P.writes = dp.d_writes;
        P.n_ops = 0;
      } else {           // store_block_to the fresh intermediate (executor.cpp:126-130)
        const DOp& d = dp.table[dp.n_fused + i];
        P.op_base = dp.n_fused + uint32_t(i);
        P.n_ops = 1;
        P.lut_ok = (lane_wise(d) && lut_allowed(cfg)) ? 1u : 0u;
        P.prog_swap = odd_swap(d) ? 1u : 0u;
        P.wr.dst[0] = reinterpret_cast<uint64_t>(next);
        P.wr.pitch[0] = uint64_t(W) * bpe(out_kind);
        P.wr.flags = WF_ACTIVE | WF_LANE_ALIGNED;
        P.wr_zstride = pts * bpe(out_kind);
        P.write_kind = out_kind;
        P.write_mode = WR_DIRECT;
      }
      launch(cls, P, st, r.kernels_launched);
      if (prev) cuda_check(cudaFreeAsync(prev, st), "cudaFreeAsync(intermediate)");
      prev = next;
      prev_kind = out_kind;
    }
  }
  r.device_ms = timer.stop();
  r.wall_time_ns = now_ns() - t0;
  r.bytes_read = dp.traffic.unfused_read;
  r.bytes_written = dp.traffic.unfused_written;
  r.passes = n + 1;
  r.points_visited = uint64_t(W) * H * B * r.passes;
  r.path = FK_PATH_GENERIC;
  return r;
}

// ----------------------------------------------------------- ReduceDPP --
namespace {

// reducer_identity, dpp.cpp:48-73, as lane bits of the value kind
void reducer_identity_bits(uint32_t r, uint32_t kind, uint64_t (&out)[3]) {
  const uint32_t lk = lane_kind(kind);
  double v = 0.0;
  if (r == FK_REDUCE_MAX) v = lk == FK_U8 ? 0.0 : -INFINITY;
  else if (r == FK_REDUCE_MIN) v = lk == FK_U8 ? 255.0 : INFINITY;
  for (int l = 0; l < 3; ++l) {
    if (lk == FK_U8) out[l] = uint64_t(v);
    else if (lk == FK_F32) {
      const float f = float(v);
      uint32_t b;
      std::memcpy(&b, &f, 4);
      out[l] = b;
    } else {
      std::memcpy(&out[l], &v, 8);
    }
  }
}

void element_bits(uint32_t kind, const Element& e, uint64_t (&out)[3], bool as_double) {
  for (int l = 0; l < 3; ++l) {
    out[l] = 0;
    if (l >= lanes_of(kind)) continue;
    if (as_double) {
      const double d = lane_as_double(kind, e, l);
      std::memcpy(&out[l], &d, 8);
    } else {
      std::memcpy(&out[l], e.raw + l * lane_bytes(kind), lane_bytes(kind));
    }
  }
}

}  // namespace

std::vector<Element> multi_reduce(const Op& read, const std::vector<ReduceSpecHost>& specs, int workers,
                                  cudaStream_t st, uint64_t* elements_read) {
  (void)workers;  // the device fold's partition is its own; only float sums can tell (within 2^-20)
  if (specs.empty()) fail(FK_E_EMPTY_ITER_SPACE, "no reduce specs given");
  if (read.opkind != FK_KIND_READ) fail(FK_E_FIRST_NOT_READ, "iteration space comes from a read op");
  if (!read.dims) fail(FK_E_MISSING_DIMS, std::string(op_name(read.id)) + " has no dims hint");
  const fk_extent3 sp = *read.dims;
  if (uint64_t(sp.width) * sp.height * sp.batch == 0) fail(FK_E_EMPTY_ITER_SPACE, "empty iteration space");
  // the read and every transform as one device program (a chain never executed
  // as such: its write is a placeholder), so the kernel reuses the fused read stage
  Pipeline pl;
  pl.read = read;
  pl.space = sp;
  std::vector<uint32_t> vkind(specs.size()), top(specs.size(), kNoOp);
  for (size_t s = 0; s < specs.size(); ++s) {
    const Op* t = specs[s].transform;
    if (t) {
      if (t->opkind != FK_KIND_UNARY && t->opkind != FK_KIND_BINARY)
        fail(FK_E_INVALID_CONFIG, "reduce transform must be a compute op");
      if (t->in_kind != read.out_kind) fail(FK_E_KIND_MISMATCH, "reduce transform input kind vs read output");
      vkind[s] = uint32_t(t->out_kind >= 0 ? t->out_kind : t->in_kind);
      top[s] = uint32_t(pl.compute.size());
      pl.compute.push_back(*t);
    } else {
      vkind[s] = uint32_t(read.out_kind);
    }
  }
  pl.write.id = FK_OP_PER_THREAD_WRITE;
  pl.write.opkind = FK_KIND_WRITE;
  pl.write.in_kind = read.out_kind;
  pl.write.dest[0] = fk_plane{nullptr, sp.width, sp.height, sp.width, uint32_t(read.out_kind)};
  DeviceProgram& dp = ensure_program(pl);
  // the widest lane state any value passes through
  bool wide = dp.read_wide;
  int lanes = dp.read_lanes;
  for (uint32_t k : vkind) add_kind(k, wide, lanes);
  add_kind(uint32_t(read.out_kind), wide, lanes);
  const int cls = generic_state_class(wide, lanes);
  DPlan P = base_plan(sp.width, sp.height, sp.batch, dp.read_flat, reduce_tile_elems());
  fill_plan_io(P, dp, pl, nullptr);
  P.reads = dp.d_reads;
  P.zdiv = make_fastdiv(P.tiles);
  uint64_t reads_total = 0;
  for (uint32_t z = 0; z < sp.batch; ++z) {  // sample_raw's touched counts (ops.cpp:312-325)
    const Sample* smp = read_plane(pl, z);
    if (!smp) continue;
    reads_total += uint64_t(sp.width) * sp.height * (smp->resizing() && smp->mode == FK_BILINEAR ? 4 : 1);
  }
  if (elements_read) *elements_read = reads_total;

  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dp.device);
  const uint64_t tiles = uint64_t(P.tiles) * sp.batch;
  const uint32_t nblocks = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>((tiles + 255) / 256, uint64_t(sms) * 8)));
  // one plane of 16-byte aligned single-lane u8 / f32 rows read as they are:
  // the vector kernel (resident CTAs only, grid-stride)
  PlainRows R{};
  bool plain = false;
  if (sp.batch == 1 && !dp.reads.empty() && (cls == 0 || (cls == 1 && dp.reads[0].kind == FK_U8X3))) {
    const DSample& r = dp.reads[0];
    const uint32_t ve = r.kind == FK_F32 ? 4u : 16u, eb = r.kind == FK_F32 ? 4u : (r.kind == FK_U8X3 ? 3u : 1u);
    const uint64_t base = r.src + uint64_t(r.y0) * r.pitch + uint64_t(r.x0) * eb;
    const uint64_t vpr = (uint64_t(sp.width) + ve - 1) / ve;
    plain = r.mode == RD_DIRECT && !(r.flags & SF_DEFAULT) && r.post_len == 0 &&
            (r.kind == FK_U8 || r.kind == FK_F32 || r.kind == FK_U8X3) && base % 16 == 0 && r.pitch % 16 == 0 &&
            vpr * sp.height < (uint64_t(1) << 31) && r.pitch * sp.height < (uint64_t(1) << 32);
    if (plain) {
      R.base = base;
      R.pitch = r.pitch;
      R.width = sp.width;
      R.vpr = uint32_t(vpr);
      R.vecs = uint32_t(vpr * sp.height);
      R.kind = r.kind;
      R.vb = ve * eb;
      R.vdiv = make_fastdiv(R.vpr);
    }
  }
  const uint32_t plain_blocks = plain ? std::max<uint32_t>(1, std::min<uint32_t>(reduce_plain_blocks(R.kind, sms),
                                                                                 (R.vecs + 255) / 256))
                                      : 0;
  std::vector<Element> result(specs.size());
  void* scratch = nullptr;
  uint64_t* d_out = nullptr;
  cuda_check(cudaMallocAsync(&scratch, reduce_scratch_bytes(std::max(nblocks, plain_blocks)), st), "cudaMallocAsync");
  cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&d_out), 3 * sizeof(uint64_t) * kMaxReduceSpecs, st),
             "cudaMallocAsync");
  for (size_t base = 0; base < specs.size(); base += kMaxReduceSpecs) {  // kMaxReduceSpecs specs per traversal
    RSpecsDev S{};
    S.n = uint32_t(std::min<size_t>(kMaxReduceSpecs, specs.size() - base));
    for (uint32_t k = 0; k < S.n; ++k) {
      const size_t s = base + k;
      RSpecDev& d = S.s[k];
      d.op = top[s] == kNoOp ? kNoOp : dp.n_fused + top[s];  // the 1:1 ops follow the fused program
      d.combine = specs[s].combine;
      d.lane_kind = lane_kind(vkind[s]);
      d.lanes = uint32_t(lanes_of(vkind[s]));
      d.dsum = specs[s].combine == FK_REDUCE_SUM && d.lane_kind != FK_U8;
      reducer_identity_bits(d.combine, vkind[s], d.ident);
      if (specs[s].has_identity) element_bits(vkind[s], specs[s].identity, d.user_ident, d.dsum);
      else if (d.dsum) element_bits(vkind[s], Element{}, d.user_ident, true);  // identity 0 for sums
      else for (int l = 0; l < 3; ++l) d.user_ident[l] = d.ident[l];
    }
    if (plain) cuda_check(launch_reduce_plain(P, S, R, scratch, plain_blocks, d_out, st), "fk_reduce_plain launch");
    else cuda_check(launch_reduce(cls, P, S, scratch, nblocks, d_out, st), "fk_reduce launch");
    t_last_kernel = !plain ? "fk_reduce_partial"
                           : (R.kind == FK_U8 ? "fk_reduce_plain<u8>"
                                              : (R.kind == FK_U8X3 ? "fk_reduce_plain<u8x3>" : "fk_reduce_plain<f32>"));
    g_launches.fetch_add(2, std::memory_order_relaxed);
    uint64_t h[3 * kMaxReduceSpecs];
    cuda_check(cudaMemcpyAsync(h, d_out, sizeof(uint64_t) * 3 * S.n, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    // a float Max / Min that came out zero: the reference keeps the FIRST zero,
    // whose sign the order-free fold cannot know -> find the first +0 and -0
    uint32_t zmask = 0;
    for (uint32_t k = 0; k < S.n; ++k) {
      const RSpecDev& d = S.s[k];
      if (d.combine == FK_REDUCE_SUM || d.lane_kind == FK_U8) continue;
      for (uint32_t l = 0; l < d.lanes; ++l) {
        const uint64_t mag = d.lane_kind == FK_F32 ? (h[3 * k + l] & 0x7fffffffu) : (h[3 * k + l] << 1);
        const bool ident_zero = d.lane_kind == FK_F32 ? (d.user_ident[l] & 0x7fffffffu) == 0 : (d.user_ident[l] << 1) == 0;
        if (mag == 0 && !ident_zero) zmask |= 1u << (3 * k + l);  // a zero identity comes first and is kept
      }
    }
    if (zmask) {
      unsigned long long* first = nullptr;
      cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&first), 6 * kMaxReduceSpecs * sizeof(unsigned long long), st),
                 "cudaMallocAsync");
      cuda_check(cudaMemsetAsync(first, 0xff, 6 * kMaxReduceSpecs * sizeof(unsigned long long), st), "cudaMemsetAsync");
      if (plain && R.kind != FK_U8X3)
        cuda_check(launch_reduce_plain_zero_sign(P, S, R, zmask, plain_blocks, first, st),
                   "fk_reduce_plain_zero_sign launch");
      else
        cuda_check(launch_reduce_zero_sign(cls, P, S, zmask, nblocks, first, st), "fk_reduce_zero_sign launch");
      g_launches.fetch_add(1, std::memory_order_relaxed);
      unsigned long long hf[6 * kMaxReduceSpecs];
      cuda_check(cudaMemcpyAsync(hf, first, sizeof hf, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
      cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
      cudaFreeAsync(first, st);
      for (uint32_t k = 0; k < S.n; ++k)
        for (uint32_t l = 0; l < 3; ++l) {
          if (!((zmask >> (3 * k + l)) & 1u)) continue;
          const bool neg = hf[6 * k + 2 * l + 1] < hf[6 * k + 2 * l];
          const uint64_t sign = S.s[k].lane_kind == FK_F32 ? 0x80000000ull : 0x8000000000000000ull;
          h[3 * k + l] = neg ? sign : 0;
        }
    }
    for (uint32_t k = 0; k < S.n; ++k) {
      Element e{};
      const uint32_t vk = vkind[base + k];
      for (int l = 0; l < lanes_of(vk); ++l) std::memcpy(e.raw + l * lane_bytes(vk), &h[3 * k + l], lane_bytes(vk));
      result[base + k] = e;
    }
  }
  cudaFreeAsync(scratch, st);
  cudaFreeAsync(d_out, st);
  return result;
}

uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

const char* last_kernel() { return t_last_kernel; }

std::string device_info() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return "no CUDA device";
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, dev);
  return std::string(prop.name) + " sm_" + std::to_string(prop.major) + std::to_string(prop.minor) + " SMs=" +
         std::to_string(prop.multiProcessorCount) + " L2=" + std::to_string(prop.l2CacheSize);
}

}  // namespace fk
