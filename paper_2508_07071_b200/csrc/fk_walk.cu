// fk_walk.cu — the column-walk crop kernel: a batch of crops of u8x3 frames,
// bilinear-resized (ops.cpp:259-299), [SwapRB], cast to f32, an f32 chain
// (sub mean / div std, ...) and split into three f32 planes, ONE fused launch
// (configs[1], [3], [4]; horizontal fusion: the batch index z is a warp's unit).
//
// Structure. Every warp is independent (no CTA barrier): it owns two half
// strips of 32 output columns (two per lane) — of one plane, or of two planes
// with the same crop height, so a 224-wide plane is 3.5 warps without idle
// lanes — and a band of output rows. Bilinear is separable; the warp walks the
// source rows the band needs, top to bottom, each visited ONCE:
//
//   stage   one elected lane copies kWalkGroup source rows at a time into a
//           per-warp shared-memory ring: one 2D TMA tensor copy per half (or
//           one for both halves of one crop), the frame's rows as a tensor map
//           with a box as wide as the half needs, completion on the slot's
//           mbarrier, one group ahead (no LSU traffic, no registers);
//   H       each lane lerps row r horizontally at its two columns as exact
//           integers: three 32-bit shared loads, a funnel shift to the
//           column's byte offset, two byte_perm and three dp2a per column
//           (see WalkCol: H lands in the mantissa of 2^23);
//   finish  every output row whose lower source row is r: vertical lerp of the
//           two H rows in packed FP32 (FFMA2 over the lane's column pair), the
//           exact-result filter, cast + chain in packed FP32, and one 8-byte
//           store per destination plane (a warp writes 2 x 128 contiguous
//           bytes per plane).
//
// Exact-result filter. v (FP32, pixel units) differs from the exact rational
// bilinear value R by less than 6.9e-5 for out_w <= 224 (1.1e-4 for any width
// the walk accepts) on non-exact columns/rows (dp2a exact; the FFMA2 vertical
// lerp <= 0.75 units of 1 / (K den); s and c rounded; the final rounding;
// derivation in DESIGN.md §4.1), and the reference's double result differs
// from R by < 1e-12. So when |v - rint(v)| < 0.5 - E (E = 2^-13) the
// reference's nearbyint(res) is rint(v); the kernel flags e^2 >= (0.5 - E)^2.
// Flagged values are recomputed after the walk in the reference's double
// arithmetic, op for op, and stored over the fast value (same thread, program
// order). Where the column AND row fractions are dyadic with <= 7 bits every
// FP32 step is exact (v == R), so the check is off there and exact ties round
// to even like the reference's nearbyint.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "fk_pack2.cuh"
#include "fk_walk.hpp"
#include "fk_stages.cuh"
#include "fk_sig.cuh"

#ifndef FK_WALK_MINB
#define FK_WALK_MINB 6  // CTAs of 4 warps per SM (80 registers: no spills)
#endif

namespace fk {

namespace {


constexpr float kRound = 12582912.0f;        // 1.5 * 2^23: x + kRound rounds x to an integer (ties to even)

__host__ __device__ constexpr bool div2(uint32_t sig, int k) { return (sig >> (kWalkDiv2 + k)) & 1u; }

// The chain's constants for input lane m, op k, as pairs: c, and for a division
// either (r_hi, r_lo) [two-op form] or (RN(1/c), -c) [three-op form].
template <uint32_t SIG>
struct KInl {
  const WalkPlan& P;
  uint64_t z;  // runtime -0 pair (fk_pack2.cuh)
  __device__ __forceinline__ KInl(const WalkPlan& Pp, uint64_t negz) : P(Pp), z(negz) {}
  __device__ __forceinline__ uint64_t c(int k, int m) const { return p2::of(P.kc[k][m]); }
  __device__ __forceinline__ uint64_t h(int k, int m) const { return p2::of(P.kh[k][m]); }
  __device__ __forceinline__ uint64_t l(int k, int m) const { return p2::of(P.kl[k][m]); }
};
template <uint32_t SIG>
struct KReg {
  uint64_t cc[4][3], hh[4][3], ll[4][3];
  uint64_t z;  // runtime -0 pair (fk_pack2.cuh)
  __device__ __forceinline__ KReg(const float4* kz, uint64_t negz) : z(negz) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        if (k < sig_n(SIG)) {
          const float4 v = __ldg(kz + 3 * k + m);
          cc[k][m] = p2::pack(v.x, v.x);
          hh[k][m] = p2::pack(v.y, v.y);
          ll[k][m] = p2::pack(v.z, v.z);
        } else {
          cc[k][m] = hh[k][m] = ll[k][m] = 0;
        }
      }
  }
  __device__ __forceinline__ uint64_t c(int k, int m) const { return cc[k][m]; }
  __device__ __forceinline__ uint64_t h(int k, int m) const { return hh[k][m]; }
  __device__ __forceinline__ uint64_t l(int k, int m) const { return ll[k][m]; }
};


// The registered chain on a column pair: the reference's arith ops
// (ops.cpp:88-159), same IEEE ops in the same order; divisions in a
// host-verified form.
template <uint32_t SIG, int K, class KS>
__device__ __forceinline__ uint64_t chain_op2(uint64_t x, const KS& ks, int m) {
  constexpr uint32_t fn = sig_fn(SIG, K);
  if constexpr (fn == AF_MUL) return p2::mul_z(x, ks.c(K, m), ks.z);
  else if constexpr (fn == AF_ADD) return p2::add(x, ks.c(K, m));
  else if constexpr (fn == AF_SUB) return p2::sub(x, ks.c(K, m));
  else if constexpr (div2(SIG, K)) return p2::fma(x, ks.h(K, m), p2::mul(x, ks.l(K, m)));
  else if constexpr (sig_fast(SIG, K)) {  // q = x r; e = fma(q, -c, x) [l holds -c]; q + e r
    const uint64_t q = p2::mul(x, ks.h(K, m));
    const uint64_t e = p2::fma(q, ks.l(K, m), x);
    return p2::fma(e, ks.h(K, m), q);
  } else {
    const float c = p2::lo(ks.c(K, m));
    return p2::pack(__fdiv_rn(p2::lo(x), c), __fdiv_rn(p2::hi(x), c));
  }
}
template <uint32_t SIG, class KS>
__device__ __forceinline__ uint64_t chain2(uint64_t x, const KS& ks, int m) {
  if constexpr (sig_n(SIG) > 0) x = chain_op2<SIG, 0>(x, ks, m);
  if constexpr (sig_n(SIG) > 1) x = chain_op2<SIG, 1>(x, ks, m);
  if constexpr (sig_n(SIG) > 2) x = chain_op2<SIG, 2>(x, ks, m);
  if constexpr (sig_n(SIG) > 3) x = chain_op2<SIG, 3>(x, ks, m);
  return x;
}

// ------------------------------------------------------------- fix path --
// The reference's bilinear value of one lane in double, op for op
// (ops.cpp:250,283-296), rounded like round_clamp_u8 (nearbyint; the value is
// in [0, 255]), as the float of the u8 result.
__device__ __forceinline__ float exact_lane(uint32_t a, uint32_t b, uint32_t c, uint32_t d, double fx, double fy) {
  const double top = __dadd_rn(double(a), __dmul_rn(__dsub_rn(double(b), double(a)), fx));
  const double bot = __dadd_rn(double(c), __dmul_rn(__dsub_rn(double(d), double(c)), fx));
  const double res = __dadd_rn(top, __dmul_rn(__dsub_rn(bot, top), fy));
  return float(uint32_t(__double2loint(__dadd_rn(res, 6755399441055744.0))) & 0xffu);
}

// The flagged pair of output row y of lane `owner` of warp unit u — both
// columns (x, x + 1) and the three lanes — recomputed exactly as the reference
// does: bilinear_sample in double op for op (ops.cpp:250,283-296) with the
// reference's own fx / fy and taps (precomputed per column / row in the walk
// tables: no double division here), round_clamp_u8, then the chain on that u8.
// The chain is the walk's own packed form, proven equal to the reference's IEEE
// ops on every u8 input (host-verified divisions), so the stored values are the
// reference's. Runs after the walk for pairs whose fast value came within E of
// a rounding boundary; stores over the fast values (same thread, program order).
// The unit's fields the recompute needs, kept in the warp's shared memory so its
// table loads are one round trip (no unit -> plane -> column chain).
struct UnitFix {
  uint32_t z[2];
  uint32_t coltab[2];
  uint32_t rowtab;
  uint16_t x[2];
  uint16_t n0, pad;
  uint32_t pad2;
};
static_assert(sizeof(UnitFix) == 32, "UnitFix");

template <uint32_t SIG, bool PERZ>
__device__ __forceinline__ void fix_owner(const WalkPlan& P, const UnitFix* uf, uint32_t owner, uint32_t y) {
  const UnitFix F = *uf;
  const bool h = owner >= F.n0;
  const uint32_t z = h ? F.z[1] : F.z[0];
  const uint32_t x = (h ? F.x[1] : F.x[0]) + 2u * (h ? owner - F.n0 : owner);
  const uint32_t ct = (h ? F.coltab[1] : F.coltab[0]) + x;
  const WalkAux A = P.aux[z];
  const DSample s = P.reads[z];
  const WalkRow R = P.rows[F.rowtab + y];
  const WalkCol C0 = P.cols[ct], C1 = P.cols[ct + 1];
  const uint32_t i1 = R.r1 & kWalkRowMask, i0 = (R.r1 & kWalkSame) ? i1 : i1 - 1u;
  const uint8_t* r0 = reinterpret_cast<const uint8_t*>(s.src) + uint64_t(s.y0 + i0) * s.pitch + A.x3;
  const uint8_t* r1 = reinterpret_cast<const uint8_t*>(s.src) + uint64_t(s.y0 + i1) * s.pitch + A.x3;
  float k[2][3];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const WalkCol& C = c ? C1 : C0;
#pragma unroll
    for (int m = 0; m < 3; ++m)
      k[c][m] = exact_lane(__ldg(r0 + C.tap + m), __ldg(r0 + C.tap + C.d1 + m), __ldg(r1 + C.tap + m),
                           __ldg(r1 + C.tap + C.d1 + m), C.fx, R.fyd);
  }
  using KS = typename std::conditional<PERZ, KReg<SIG>, KInl<SIG>>::type;
  const KS ks = [&]() {
    if constexpr (PERZ) return KReg<SIG>(P.kz + 12ull * A.kz, P.negz);
    else return KInl<SIG>(P, P.negz);
  }();
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    const uint64_t o = chain2<SIG>(p2::pack(k[0][m], k[1][m]), ks, m);
    *reinterpret_cast<float2*>(P.dst_base + A.dst[m] + uint64_t(y) * A.dpitch + 4ull * x) =
        make_float2(p2::lo(o), p2::hi(o));
  }
}

// ------------------------------------------------------- TMA tensor copies --
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra.uni WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
// kWalkGroup source rows of one crop (box at element (x, row y)) into shared memory
__device__ __forceinline__ void tma_rows(uint32_t dst, uint64_t map, uint32_t x, uint32_t y, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst), "l"(map), "r"(x), "r"(y), "r"(mbar)
      : "memory");
}
// One elected lane: expect `tx` bytes on mbar, copy half 0's box to dst and, if
// off1 != 0, half 1's box to dst + off1 (all operands warp-uniform). The source
// rows are read with an L2 evict_last policy: the frames stay resident while
// the outputs stream past them (the outputs stream through with the default policy).
__device__ __forceinline__ void tma_group(uint32_t dst, uint64_t m0, uint32_t x0, uint32_t y0, uint64_t m1, uint32_t x1,
                                          uint32_t y1, uint32_t mbar, uint32_t tx, uint32_t off1) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t.reg .b64 pol;\n\t"
      "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.and.u32 q, %9, 0, p;\n\t"
      "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%7], %8;\n\t"
      "@p cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%7], pol;\n\t"
      "@q cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%10], [%4, {%5, %6}], [%7], pol;\n\t"
      "}" ::"r"(dst),
      "l"(m0), "r"(x0), "r"(y0), "l"(m1), "r"(x1), "r"(y1), "r"(mbar), "r"(tx), "r"(off1), "r"(dst + off1)
      : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// H of one visited source row at the lane's two columns (the 12-byte windows at
// shared addresses p[0], p[1]): three exact integers (lanes R, G, B) per column
// as biased floats 2^23 + H.
__device__ __forceinline__ void h_row(const uint32_t (&p)[2], const uint32_t (&sh)[2], const uint32_t (&wts)[2],
                                      float (&H)[2][3]) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const uint32_t a = p[c];
    const uint32_t w0 = lds32(a), w1 = lds32(a + 4), w2 = lds32(a + 8);
    const uint32_t lo = __funnelshift_r(w0, w1, sh[c]), hi = __funnelshift_r(w1, w2, sh[c]);
    const uint32_t rg = __byte_perm(lo, hi, 0x4130);  // (a_R, b_R, a_G, b_G)
    const uint32_t b = __byte_perm(lo, hi, 0x0052);   // (a_B, b_B, -, -)
    H[c][0] = __uint_as_float(__dp2a_lo(wts[c], rg, kWalkBias));
    H[c][1] = __uint_as_float(__dp2a_hi(wts[c], rg, kWalkBias));
    H[c][2] = __uint_as_float(__dp2a_lo(wts[c], b, kWalkBias));
  }
}

// Per-warp shared memory: the ring (kWalkSlots slots x 2 halves x kWalkGroup
// rows), the slots' mbarriers and lane 0's staging arguments (64 bytes), the
// unit's row entries (RowEnt: the walk reads them on its critical path, an L2
// round trip from the table) and a sentinel, the fix masks (one lane mask per
// output row of the unit), slack for the last row's 12-byte window; 128-byte
// aligned (TMA destinations).
struct StageArgs {
  uint64_t map0, map1;  // tensor maps of the two halves' frames
  uint32_t bx0, bx1;    // box x of each half
  uint32_t y0, y1;      // TMA y of each half's source row r_first
  uint32_t two;         // half 1 present
  uint32_t tx;          // bytes a group's boxes deliver (kWalkGroup rows of each half's box width)
};
__host__ __device__ constexpr uint32_t walk_half_bytes(uint32_t rb) { return (kWalkGroup * rb + 127) / 128 * 128; }
__host__ __device__ constexpr uint32_t walk_ring_bytes(uint32_t rb) { return kWalkSlots * 2 * walk_half_bytes(rb); }
struct RowEnt {        // a WalkRow as the walk reads it: one 16-byte shared load
  uint32_t r1;          // source row that completes the output row (kWalkRowMask: sentinel)
  float fy;
  uint32_t exact;       // kWalkExactRow set: the exact-column filter applies
  uint32_t pad;
};
constexpr uint32_t kWalkMeta = 64;  // mbarriers + StageArgs
static_assert(8 * kWalkSlots + sizeof(StageArgs) <= kWalkMeta, "walk meta");
__host__ __device__ constexpr uint32_t walk_warp_bytes(uint32_t rb, uint32_t max_rows) {
  return (walk_ring_bytes(rb) + kWalkMeta + 16 * (max_rows + 1) + 32 + 4 * max_rows + 16 + 127) / 128 * 128;
}

// ------------------------------------------------------------------ kernel --
template <uint32_t SIG, bool PERZ>
__global__ void __launch_bounds__(kWalkWarps * 32, PERZ ? 6 : FK_WALK_MINB) fk_walk(const __grid_constant__ WalkPlan P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t wi = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t u = blockIdx.x * kWalkWarps + wi;
  if (u >= P.n_units) return;  // the whole warp: no CTA-wide synchronisation follows
  const WalkUnit U = P.units[u];
  const uint32_t RB = P.row_bytes, HB = walk_half_bytes(RB), GB = 2 * HB;
  unsigned char* wbase = smem + wi * walk_warp_bytes(RB, P.max_rows);
  const uint32_t ring = uint32_t(__cvta_generic_to_shared(wbase));
  const uint32_t bar = ring + kWalkSlots * GB;
  StageArgs* sa = reinterpret_cast<StageArgs*>(wbase + kWalkSlots * GB + 8 * kWalkSlots);
  RowEnt* rows = reinterpret_cast<RowEnt*>(wbase + kWalkSlots * GB + kWalkMeta);
  UnitFix* ufix = reinterpret_cast<UnitFix*>(rows + P.max_rows + 1);
  uint32_t* fixm = reinterpret_cast<uint32_t*>(ufix + 1);

  // lane role: half h, plane z, output columns x, x + 1 (fields picked with
  // selects: a dynamic index into U would put it in local memory)
  const uint32_t n0 = U.n[0];
  const bool h = lane >= n0;
  const bool active = lane < n0 + U.n[1];
  const uint32_t z = h ? U.z[1] : U.z[0];
  const uint32_t xh = h ? U.x[1] : U.x[0];
  const uint32_t x = xh + 2u * (h ? lane - n0 : lane);
  // the lane reads the second box (else half 0's, or the merged one); idle lanes of a one-half unit read
  // half 0's staged bytes too (finite values: their v = 0 is never flagged)
  const bool h2 = h && U.bw[1] != 0 && U.n[1] != 0;
  const uint32_t bwl = h2 ? U.bw[1] : U.bw[0];  // the lane's box: staged row stride
  const WalkAux A = P.aux[z];
  if (lane == 0 || lane == n0) {  // the recompute's unit record; each half's first lane (n0 < 32) its column table
    if (lane == 0) {
      ufix->z[0] = U.z[0];
      ufix->z[1] = U.z[1];
      ufix->rowtab = U.rowtab;
      ufix->x[0] = U.x[0];
      ufix->x[1] = U.x[1];
      ufix->n0 = uint16_t(n0);
    }
    ufix->coltab[lane == 0 ? 0 : 1] = A.coltab;
  }
  // column constants. An idle lane lerps a valid column with s = c = 0 (v = 0:
  // never flagged) and stores to its warp's line of the plan's sink with a zero
  // row step, so the finish carries no store predicate. (One sink line shared by
  // every warp was an L2 hot spot: B = 1024 crops, odd half counts per crop
  // height, 212 -> 323 us.)
  uint32_t w[2], sh[2], wts[2];
  float s[2], c[2], tc[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const WalkCol C = P.cols[A.coltab + (active ? x + k : xh)];
    const uint32_t rel = A.x3 + C.tap - P.elem * (h ? U.bx[1] : U.bx[0]);
    w[k] = (rel & ~3u) + (h2 ? HB : 0u);
    sh[k] = (rel & 3u) * 8u;
    wts[k] = C.wts;
    s[k] = active ? C.s : 0.0f;
    c[k] = active ? C.c : 0.0f;
    tc[k] = C.thr;
  }
  const uint64_t s2 = p2::pack(s[0], s[1]), c2 = p2::pack(c[0], c[1]);
  const uint64_t kR = p2::pack(kRound, kRound);
  const uint64_t nT_col = p2::pack(tc[0], tc[1]);
  const float nthr = -__uint_as_float(kWalkThr2Bits);
  const uint64_t nT_thr = p2::pack(nthr, nthr);
  const uint32_t y_hi = U.y_hi, y_lo = U.y_lo;
  const uint32_t dstep = active ? A.dpitch : 0u;
  uint64_t dst[3];  // the lane's column pair in row y_lo of each plane; row y at dst + yoff
#pragma unroll
  for (int m = 0; m < 3; ++m)
    dst[m] = active ? P.dst_base + A.dst[m] + 4ull * x + uint64_t(y_lo) * A.dpitch
                    : P.sink + 256ull * (u % kWalkSinkLines) + 8 * lane;
  uint32_t yoff = 0;  // (y - y_lo) * dstep: a plane is < 4 GiB
  using KS = typename std::conditional<PERZ, KReg<SIG>, KInl<SIG>>::type;
  const KS ks = [&]() {
    if constexpr (PERZ) return KReg<SIG>(P.kz + 12ull * A.kz, P.negz);
    else return KInl<SIG>(P, P.negz);
  }();

  // lane 0 stages group g (source rows r_first + kWalkGroup g ...) into ring
  // slot g % 2, both halves on that slot's mbarrier; its arguments wait in
  // shared memory
  const uint32_t r_first = U.r_first;
  const uint32_t nvis = uint32_t(U.r_last) - r_first + 1u, ngroups = (nvis + kWalkGroup - 1) / kWalkGroup;
  if (lane == 0) {
    StageArgs t;
    t.map0 = reinterpret_cast<uint64_t>(P.maps + U.map[0]);
    t.map1 = reinterpret_cast<uint64_t>(P.maps + U.map[1]);
    t.bx0 = U.bx[0];
    t.bx1 = U.bx[1];
    t.y0 = U.y0[0] + r_first;
    t.y1 = U.y0[1] + r_first;
    t.two = U.n[1] != 0 && U.bw[1] != 0;  // a second box (a merged unit has one)
    t.tx = kWalkGroup * (uint32_t(U.bw[0]) + (t.two ? uint32_t(U.bw[1]) : 0u));
    *sa = t;
  }
  // Called by the whole (converged) warp: the arguments are made warp-uniform
  // with shuffles, so one elected lane issues the copies straight from uniform
  // registers (no per-lane issue loop).
  auto stage = [&](uint32_t g) {
    const StageArgs t = *sa;
    const uint64_t m0 = __shfl_sync(0xffffffffu, t.map0, 0), m1 = __shfl_sync(0xffffffffu, t.map1, 0);
    const uint32_t bx0 = __shfl_sync(0xffffffffu, t.bx0, 0), bx1 = __shfl_sync(0xffffffffu, t.bx1, 0);
    const uint32_t two = __shfl_sync(0xffffffffu, t.two, 0);
    const uint32_t slot = g % kWalkSlots;
    const uint32_t y0 = __shfl_sync(0xffffffffu, t.y0, 0) + g * kWalkGroup;
    const uint32_t y1 = __shfl_sync(0xffffffffu, t.y1, 0) + g * kWalkGroup;
    const uint32_t mb = __shfl_sync(0xffffffffu, bar, 0) + 8 * slot;
    const uint32_t dst = __shfl_sync(0xffffffffu, ring, 0) + slot * GB;
    const uint32_t tx = __shfl_sync(0xffffffffu, t.tx, 0);  // the boxes' bytes (zero-filled outside the frame)
    tma_group(dst, m0, bx0, y0, m1, bx1, y1, mb, tx, two ? HB : 0u);
  };
  if (lane == 0) {
#pragma unroll
    for (uint32_t i = 0; i < kWalkSlots; ++i) mbar_init(bar + 8 * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  for (uint32_t g = 0; g < kWalkSlots && g < ngroups; ++g) stage(g);
  // the unit's row entries y_lo .. y_hi - 1 and a sentinel in shared memory
  const uint32_t nrows = y_hi - y_lo;
  for (uint32_t i = lane; i <= nrows; i += 32) {
    const WalkRow& e = P.rows[U.rowtab + y_lo + i];
    const uint32_t r1 = __ldg(&e.r1);
    rows[i] = i < nrows ? RowEnt{r1 & kWalkRowMask, __ldg(&e.fy), r1 & kWalkExactRow, 0u}
                        : RowEnt{kWalkRowMask, 0.0f, 0u, 0u};
  }
  __syncwarp();
  uint32_t ri = 0;  // the next output row's entry (y - y_lo)
  RowEnt R = rows[0];

  // finish the output row of entry (r1, fy) from the H rows of its two source
  // rows (a clamped row has fy = 1: Ha + (Hb - Ha) * 1 == Hb exactly)
  auto finish = [&](const float (&Ha)[2][3], const float (&Hb)[2][3], const RowEnt& E) {
    const uint64_t fy2 = p2::pack(E.fy, E.fy);
    const uint64_t nT = E.exact ? nT_col : nT_thr;
    uint32_t acc = 0xffffffffu;  // AND of the filter values' sign bits: clear = flagged
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const uint64_t a2 = p2::pack(Ha[0][m], Ha[1][m]), b2 = p2::pack(Hb[0][m], Hb[1][m]);
      const uint64_t p = p2::fma(p2::sub(b2, a2), fy2, a2);  // 2^23 + the vertical lerp (units of H)
      const uint64_t v = p2::fma(p, s2, c2);                  // pixel units
      const uint64_t k = p2::sub(p2::add(v, kR), kR);         // rint(v): the u8 result, as f32
      const uint64_t e = p2::sub(v, k);
      const uint64_t q = p2::fma(e, e, nT);                   // e^2 - T
      acc &= uint32_t(q) & uint32_t(q >> 32);
      const uint64_t o = chain2<SIG>(k, ks, m);
      // default write-back policy: 1.2 % faster than evict-first (.cs) or write-through
      *reinterpret_cast<float2*>(dst[m] + yoff) = make_float2(p2::lo(o), p2::hi(o));
    }
    yoff += dstep;
    // the row's flagged lanes (rare; recomputed after the walk): every lane
    // stores the same ballot, the row is finished exactly once
    fixm[ri] = __ballot_sync(0xffffffffu, int32_t(acc) >= 0);
  };

  float HA[2][3], HB2[2][3];
  // visit source row r (staged at `row`): H into Hn, then every output row it completes
  // the lane's two tap windows in the staged row being visited: running shared
  // addresses, one row stride per visit, a slot step per group
  uint32_t pw[2] = {ring + w[0], ring + w[1]};
  auto visit = [&](uint32_t r, float (&Hn)[2][3], float (&Hp)[2][3]) {
    h_row(pw, sh, wts, Hn);
    pw[0] += bwl;
    pw[1] += bwl;
    while (R.r1 == r) {
      finish(Hp, Hn, R);
      R = rows[++ri];
    }
  };
  // visit 0's "previous" row is row 0 itself (only a clamped row completes there)
  mbar_wait(bar, 0);
  h_row(pw, sh, wts, HB2);
  const uint32_t gstep = kWalkGroup * bwl;
  // whole groups: visits past r_last read staged rows but complete nothing (the sentinel)
  for (uint32_t g = 0; g < ngroups; ++g) {
    const uint32_t slot = g % kWalkSlots;
    mbar_wait(bar + 8 * slot, (g / kWalkSlots) & 1u);
    const uint32_t r = r_first + g * kWalkGroup;
#pragma unroll
    for (uint32_t q = 0; q < kWalkGroup; q += 2) {
      visit(r + q, HA, HB2);
      visit(r + q + 1, HB2, HA);
    }
    // to the next slot's row 0 (kWalkSlots = 2: slot 0 -> 1 is + GB, 1 -> 0 is - GB)
    const uint32_t step = (slot == 0 ? GB : 0u - GB) - gstep;
    pw[0] += step;
    pw[1] += step;
    __syncwarp();  // every lane is done with the slot
    if (g + kWalkSlots < ngroups) stage(g + kWalkSlots);
  }
  // values near a rounding boundary (rare), recomputed in the reference's
  // arithmetic: the flagged (row, lane) pairs are dealt to the warp's lanes,
  // 32 at a time, so the double-precision path runs with full warps
  __syncwarp();  // the fast values and the masks are stored
  {
    uint32_t pend = 0, my_row = 0, my_owner = 0;
    for (uint32_t i0 = 0; i0 < y_hi - y_lo; i0 += 32) {
      const uint32_t mi = i0 + lane < y_hi - y_lo ? fixm[i0 + lane] : 0u;
      uint32_t rows_set = __ballot_sync(0xffffffffu, mi != 0);
      while (rows_set) {
        const uint32_t j = __ffs(rows_set) - 1;
        rows_set &= rows_set - 1;
        uint32_t mask = __shfl_sync(0xffffffffu, mi, j);
        while (mask) {
          const uint32_t take = min(uint32_t(__popc(mask)), 32u - pend);
          if (lane >= pend && lane < pend + take) {
            my_row = i0 + j;
            my_owner = __fns(mask, 0, int(lane - pend) + 1);
          }
          for (uint32_t t = 0; t < take; ++t) mask &= mask - 1;
          pend += take;
          if (pend == 32) {
            fix_owner<SIG, PERZ>(P, ufix, my_owner, y_lo + my_row);
            pend = 0;
          }
        }
      }
    }
    if (lane < pend) fix_owner<SIG, PERZ>(P, ufix, my_owner, y_lo + my_row);
  }
}

}  // namespace

// Registered chains: the AFFINE signatures of fk_sig.cuh, with the two-op
// division variants of the normalising ones.
#define FK_WALK_SIGS(X)                                                              \
  X(sig_make(0))                                                                     \
  X(sig_make(1, AF_MUL)) X(sig_make(1, AF_ADD)) X(sig_make(1, AF_SUB))              \
  X(sig_make(1, AF_DIV)) X(sig_make(1, AF_DIV, 0, 0, 0, 1))                        \
  X(sig_make(1, AF_DIV) | (1u << kWalkDiv2))                                         \
  X(sig_make(2, AF_SUB, AF_DIV)) X(sig_make(2, AF_SUB, AF_DIV, 0, 0, 2))            \
  X(sig_make(2, AF_SUB, AF_DIV) | (2u << kWalkDiv2))                                 \
  X(sig_make(2, AF_MUL, AF_ADD)) X(sig_make(2, AF_SUB, AF_MUL))                     \
  X(sig_make(3, AF_MUL, AF_SUB, AF_DIV)) X(sig_make(3, AF_MUL, AF_SUB, AF_DIV, 0, 4)) \
  X(sig_make(3, AF_MUL, AF_SUB, AF_DIV) | (4u << kWalkDiv2))

bool walk_registered(uint32_t sig) {
#define FK_CASE(S) if (sig == (S)) return true;
  FK_WALK_SIGS(FK_CASE)
#undef FK_CASE
  return false;
}

size_t walk_smem_bytes(uint32_t row_bytes, uint32_t max_rows) {
  return size_t(kWalkWarps) * walk_warp_bytes(row_bytes, max_rows);
}

cudaError_t launch_walk(uint32_t sig, bool per_plane, const WalkPlan& P, cudaStream_t st) {
  if (P.n_units == 0) return cudaSuccess;
  const size_t smem = walk_smem_bytes(P.row_bytes, P.max_rows);
  const uint32_t ctas = (P.n_units + kWalkWarps - 1) / kWalkWarps;
#define FK_RUN(S, PZ)                                                                  \
  do {                                                                                 \
    auto k = fk_walk<S, PZ>;                                                           \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));   \
    k<<<ctas, kWalkWarps * 32, smem, st>>>(P);                                         \
  } while (0)
#define FK_CASE(S)                        \
  if (sig == (S)) {                       \
    if (per_plane) FK_RUN(S, true);       \
    else FK_RUN(S, false);                \
    return cudaGetLastError();            \
  }
  FK_WALK_SIGS(FK_CASE)
#undef FK_CASE
#undef FK_RUN
  return cudaErrorInvalidValue;
}

bool walk_encode_map(CUtensorMap* map, uint64_t base, uint64_t width_elems, uint64_t rows, uint64_t pitch,
                     uint32_t elem, uint32_t box_w, uint32_t box_h) {
  static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    cudaGetLastError();
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return false;
  const cuuint64_t dims[2] = {width_elems, rows};
  const cuuint64_t strides[1] = {pitch};
  const cuuint32_t box[2] = {box_w, box_h};
  const cuuint32_t es[2] = {1, 1};
  const CUtensorMapDataType type = elem == 2   ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                   : elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                                               : CU_TENSOR_MAP_DATA_TYPE_UINT64;
  return encode(map, type, 2, reinterpret_cast<void*>(base), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace fk
