// fk_resample_sep.cuh — column-streaming kernel for batched u8 crop/resize
// pipelines (configs[1], [3], [4]; the cvGS / FastNPP preprocessing family,
// PAPER.md:695-703).
//
// The reference's bilinear sample (ops.cpp:259-299) is
//     top = lerp(a, b, fx)   taps of source row sy0
//     bot = lerp(c, d, fx)   taps of source row sy1
//     res = lerp(top, bot, fy)
// and `top`/`bot` depend only on (source row, output column). So each thread
// owns ONE output column and walks down a band of output rows, holding the
// horizontal lerps of the two current source rows in registers: a source row's
// H-lerp is computed once however many output rows use it, and the V-lerp is
// the only per-pixel double work. Same double ops in the same order: bit-exact.
//
//   CTA = a strip of up to 256 consecutive output columns x a band of rows of
//   one plane z (blockIdx.z, horizontal fusion). Per CTA and plane: the rows'
//   coordinates in shared memory, the chain's constants in registers (AFFINE:
//   Cast u8->f32 + a registered f32 chain) or its 256-entry table (LUT: any
//   lane-wise chain). The plane's mode (bilinear / one tap) and whether its rows
//   are 4-byte aligned are resolved once per CTA into specialised loop bodies.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

#include "fk_launch.hpp"
#include "fk_sig.cuh"
#include "fk_stages.cuh"

namespace fk {

namespace {

#ifndef FK_SEP_MINB
#define FK_SEP_MINB 4  // resident CTAs per SM (64 registers per thread)
#endif
constexpr uint32_t kBandMax = 64;  // output rows per CTA (host picks <= this)

struct RowEnt {                    // one output row: source rows (absolute) and fy
  uint32_t s0, s1;
  double f;
};

// Per-column gather geometry for 4-byte-aligned source rows: the taps' bytes
// [o0, o1 + 3) lie in words w[0..2] from (row + (o0 & ~3)); a word is loaded only
// if it holds one of those bytes (so nothing past the plane is touched).
struct ColGeom {
  uint32_t woff;         // byte offset of the first word within the row
  uint32_t sa, sb;       // funnel-shift amounts of tap 0 / tap 1 (bits)
  uint32_t need1, need2; // load word 1 / word 2
};

__device__ __forceinline__ ColGeom col_geom(uint32_t o0, uint32_t o1) {
  const uint32_t r = o0 & 3u, last = r + (o1 - o0) + 2;
  return ColGeom{o0 & ~3u, 8 * r, 8 * (r + (o1 - o0)), last >= 4 ? 1u : 0u, last >= 8 ? 1u : 0u};
}

// Load *p only if `need` (the value is unspecified otherwise; callers use only
// bytes of words they need).
__device__ __forceinline__ uint32_t ld_if(const uint32_t* p, uint32_t need) {
  uint32_t v;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.u32 %0, [%1];\n\t}"
               : "=r"(v) : "l"(p), "r"(need));
  return v;
}

// the two 3-byte taps of one source row (aligned-row fast path)
__device__ __forceinline__ void taps_aligned(const uint8_t* row, const ColGeom& g, uint32_t& a, uint32_t& b) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(row + g.woff);
  const uint32_t w0 = __ldg(w), w1 = ld_if(w + 1, g.need1), w2 = ld_if(w + 2, g.need2);
  a = __funnelshift_r(w0, w1, g.sa);
  b = g.sb < 32 ? __funnelshift_r(w0, w1, g.sb) : __funnelshift_r(w1, w2, g.sb - 32);
}

// byte l of v as a double: 2^52 + v is exact and its low word is v
__device__ __forceinline__ double byte_as_biased_double(uint32_t v, int l) {
  return __hiloint2double(0x43300000, int(__byte_perm(v, 0, 0x4440 | l)));
}

// Horizontal lerp a + (b - a) * fx of one source row, per lane (ops.cpp:283-284).
template <int NL>
__device__ __forceinline__ void hlerp(uint32_t a, uint32_t b, double fx, double (&h)[3]) {
  constexpr double kTwo52 = 4503599627370496.0;
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const double A = byte_as_biased_double(a, l), B = byte_as_biased_double(b, l);
    h[l] = __dadd_rn(__dsub_rn(A, kTwo52), __dmul_rn(__dsub_rn(B, A), fx));
  }
}

template <int NL, bool ALIGNED>
__device__ __forceinline__ void row_taps(const uint8_t* row, const ColGeom& g, uint32_t o0, uint32_t o1,
                                         uint32_t& a, uint32_t& b) {
  if constexpr (NL == 3) {
    if constexpr (ALIGNED) taps_aligned(row, g, a, b);
    else dev::load_u8x3_taps(row, o0, o1, a, b);
  } else {
    a = __ldg(row + o0);
    b = __ldg(row + o1);
  }
}

// The chain after the u8 read, on the lanes of one output pixel: one table
// lookup per lane (the table holds the chain over all 256 byte values, slot m
// = output lane sigma(m) from input lane m; see build_affine_table / the LUT
// build in the kernel). Packed outputs put lane sigma(m) in place here; split
// outputs swap their destination planes instead (ColOut).
template <int NL, bool SPLIT, class Out>
__device__ __forceinline__ void chain(const uint32_t (&u)[3], bool swap, const Out* lut, Out (&o)[NL]) {
#pragma unroll
  for (int l = 0; l < NL; ++l) o[l] = lut[l * 256 + u[l]];
  if constexpr (NL == 3 && !SPLIT) {
    if (swap) { const Out t = o[0]; o[0] = o[2]; o[2] = t; }
  }
}

// Destination cursor of one output column: the byte address of (x, y) in each
// destination plane, advanced by the pitch per output row.
template <int NL, uint32_t OLK, bool SPLIT>
struct ColOut {
  static constexpr int OB = OLK == FK_U8 ? 1 : (OLK == FK_F32 ? 4 : 8);
  static constexpr int ND = SPLIT ? 3 : 1;
  uint8_t* p[ND];
  uint32_t pitch[ND];  // < 2^32 (checked by the host)
  __device__ __forceinline__ ColOut(const DWrite& w, uint32_t x, uint32_t y, bool swap) {
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      const int e = (SPLIT && swap) ? 2 - d : d;  // split + lane swap: lane m goes to plane sigma(m)
      pitch[d] = uint32_t(w.pitch[e]);
      // one row above (x, y): put() advances first, then stores
      p[d] = reinterpret_cast<uint8_t*>(w.dst[e]) + (uint64_t(y) - 1) * w.pitch[e] + uint64_t(x) * OB * (SPLIT ? 1 : NL);
    }
  }
  // split_block (ops.cpp:402-424) / store_block (:396-400) of one pixel, then next row
  template <bool AL, class Out>
  __device__ __forceinline__ void put(const Out (&o)[NL]) {
    if constexpr (SPLIT) {
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        p[l] += pitch[l];
        if constexpr (OLK == FK_F32 && AL) __stcs(reinterpret_cast<float*>(p[l]), __uint_as_float(uint32_t(o[l])));
        else dev::store_lane<OLK, Out>(p[l], o[l], AL);
      }
    } else {
      p[0] += pitch[0];
#pragma unroll
      for (int l = 0; l < NL; ++l) dev::store_lane<OLK, Out>(p[0] + l * OB, o[l], AL);
    }
  }
};

// V-lerp top + (bot - top) * fy per lane (ops.cpp:296), round_clamp_u8 (res is
// in [0, 255]), the chain, the store.
template <int NL, uint32_t OLK, bool SPLIT, bool AL, class Out>
__device__ __forceinline__ void emit(const double (&top)[3], const double (&bot)[3], double fy, bool swap,
                                     const Out* lut, ColOut<NL, OLK, SPLIT>& out) {
  uint32_t u[3];
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const double res = __dadd_rn(top[l], __dmul_rn(__dsub_rn(bot[l], top[l]), fy));
    u[l] = uint32_t(__double2loint(__dadd_rn(res, 6755399441055744.0)));
  }
  Out o[NL];
  chain<NL, SPLIT, Out>(u, swap, lut, o);
  out.template put<AL>(o);
}

// One source row's two taps, split into issue (the loads) and use (the byte
// extraction) so the next row's loads are in flight while this row is lerped.
// `at` is the column's gather address in that row: the first tap word for
// aligned rows, the row start otherwise.
template <int NL, bool ALIGNED>
struct RowFetch {
  uint32_t w[3];
  const uint8_t* row;
  __device__ __forceinline__ void issue(const uint8_t* at, const ColGeom& g) {
    if constexpr (NL == 3 && ALIGNED) {
      const uint32_t* p = reinterpret_cast<const uint32_t*>(at);
      w[0] = __ldg(p);
      w[1] = ld_if(p + 1, g.need1);
      w[2] = ld_if(p + 2, g.need2);
    } else {
      row = at;
    }
  }
  __device__ __forceinline__ void taps(const ColGeom& g, uint32_t o0, uint32_t o1, uint32_t& a, uint32_t& b) const {
    if constexpr (NL == 3 && ALIGNED) {
      a = __funnelshift_r(w[0], w[1], g.sa);
      b = g.sb < 32 ? __funnelshift_r(w[0], w[1], g.sb) : __funnelshift_r(w[1], w[2], g.sb - 32);
    } else {
      row_taps<NL, false>(row, g, o0, o1, a, b);
    }
  }
};

// The source rows a band visits, in order (byte offsets voff[]), and the output
// rows each visit completes: output row k (source rows s0, s1) is emitted right
// after the visits s0, s1 — the last two visits are always exactly (s0, s1),
// so an edge row whose s0 == s1 (clamped) visits that row twice. Output rows
// [vend[v - 1], vend[v]) are emitted at visit v. voff[nv] repeats voff[nv - 1]
// (the walk prefetches one visit ahead).
struct Visits {
  uint64_t voff[2 * kBandMax + 1];
  uint32_t vend[2 * kBandMax];
  uint32_t n;
};

// Built by warp 0 for the band's n output rows. Output row k adds no visit when
// (s0, s1) equals row k - 1's, one visit (s1) when its s0 is row k - 1's s1,
// two (s0, s1) otherwise; a warp scan places them.
__device__ __forceinline__ void build_visits_warp(const RowEnt* rows, uint32_t n, uint64_t pitch, Visits& V) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t base = 0;
  for (uint32_t c = 0; c < n; c += 32) {
    const uint32_t k = c + lane;
    const bool in = k < n;
    const uint32_t s0 = in ? rows[k].s0 : 0, s1 = in ? rows[k].s1 : 0;
    const bool first = k == 0;
    const uint32_t p0 = (in && !first) ? rows[k - 1].s0 : 0, p1 = (in && !first) ? rows[k - 1].s1 : 0;
    const uint32_t cnt = !in ? 0u : (!first && s0 == p0 && s1 == p1) ? 0u : (!first && s0 == p1) ? 1u : 2u;
    uint32_t incl = cnt;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    const uint32_t pos = base + incl - cnt;
    if (cnt == 2) {
      V.voff[pos] = uint64_t(s0) * pitch;
      V.vend[pos] = k;
    }
    if (cnt != 0) V.voff[pos + cnt - 1] = uint64_t(s1) * pitch;
    __syncwarp();
    // the last output row attached to a visit closes it
    if (in && (k + 1 == n || rows[k + 1].s0 != s0 || rows[k + 1].s1 != s1)) V.vend[pos + cnt - 1] = k + 1;
    base += __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();
  }
  if (lane == 0) {
    V.voff[base] = V.voff[base - 1];
    V.n = base;
  }
}

// Walk the band's visits for column x (bilinear). Each visit H-lerps ONE source
// row (a source row's H-lerp is computed once however many output rows use it)
// and emits the output rows it completes. hA / hB alternate as the current row
// by unrolling the walk by two, so no H-lerp is ever copied between registers.
template <int NL, uint32_t OLK, bool SPLIT, bool ALIGNED, bool AL, class Out>
__device__ __forceinline__ void column_bilinear(const DSample& s, const DWrite& w, const RowEnt* rows,
                                                const Visits& V, uint32_t x, uint32_t y0, bool swap,
                                                const Out* lut) {
  const XEnt xe = dev::x_entry(s, x, NL);
  const ColGeom g = col_geom(xe.o0, xe.o1);
  const uint8_t* col = reinterpret_cast<const uint8_t*>(s.src) + (NL == 3 && ALIGNED ? g.woff : 0u);
  ColOut<NL, OLK, SPLIT> out(w, x, y0, swap);
  RowFetch<NL, ALIGNED> F;
  F.issue(col + V.voff[0], g);
  double hA[3] = {0, 0, 0}, hB[3] = {0, 0, 0};
  uint32_t k = 0;
  const uint32_t nv = V.n;
  // visit v: H-lerp its row into `cur`, prefetch visit v + 1, emit its outputs
  auto visit = [&](uint32_t v, double (&cur)[3], const double (&prev)[3]) {
    uint32_t a, b;
    F.taps(g, xe.o0, xe.o1, a, b);
    F.issue(col + V.voff[v + 1], g);
    hlerp<NL>(a, b, xe.f, cur);
#pragma unroll 1
    for (const uint32_t e = V.vend[v]; k < e; ++k)
      emit<NL, OLK, SPLIT, AL, Out>(prev, cur, rows[k].f, swap, lut, out);
  };
  for (uint32_t v = 0; v < nv; v += 2) {
    visit(v, hA, hB);
    if (v + 1 < nv) visit(v + 1, hB, hA);
  }
}

// Nearest / non-resizing planes: one tap per output pixel.
template <int NL, uint32_t OLK, bool SPLIT, bool AL, class Out>
__device__ __forceinline__ void column_tap(const DSample& s, const DWrite& w, const RowEnt* rows, uint32_t x,
                                           uint32_t y0, uint32_t y1, bool swap, const Out* lut) {
  const uint32_t o0 = s.mode == RD_DIRECT ? (s.x0 + x) * NL : dev::x_entry(s, x, NL).o0;
  const uint8_t* base = reinterpret_cast<const uint8_t*>(s.src) + o0;
  ColOut<NL, OLK, SPLIT> out(w, x, y0, swap);
  for (uint32_t y = y0; y < y1; ++y) {
    const uint8_t* p = base + uint64_t(rows[y - y0].s0) * s.pitch;
    uint32_t u[3];
#pragma unroll
    for (int l = 0; l < NL; ++l) u[l] = __ldg(p + l);
    Out o[NL];
    chain<NL, SPLIT, Out>(u, swap, lut, o);
    out.template put<AL>(o);
  }
}

// AFFINE table: slot m, entry t = the registered f32 chain (constants of output
// lane sigma(m)) applied to float(t) — Cast u8 -> f32 then the chain, exactly
// the per-pixel arithmetic, tabulated. Constants from the kernel parameters, or
// the plane's BatchArith rows.
template <int NL, uint32_t SIG, class Out>
__device__ __forceinline__ void build_affine_table(const DPlan& P, uint32_t z, bool swap, Out* lut) {
  float c[4][3], r[4][3];
#pragma unroll
  for (int k = 0; k < sig_n(SIG); ++k) {
    if (P.aff_inline) {
#pragma unroll
      for (int l = 0; l < 3; ++l) { c[k][l] = P.aff_c[k][l]; r[k][l] = P.aff_r[k][l]; }
    } else {
      const DOp op = dev::prog_op(P, P.op_base + k);
      uint64_t v[3] = {op.c[0], op.c[1], op.c[2]};
      if (op.per_z) {
        const uint64_t* row = reinterpret_cast<const uint64_t*>(op.per_z) + 3ull * (z < op.per_z_n ? z : op.per_z_n - 1);
        v[0] = __ldg(row); v[1] = __ldg(row + 1); v[2] = __ldg(row + 2);
      }
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        c[k][l] = __uint_as_float(uint32_t(v[op.nl == 3 ? l : 0]));
        r[k][l] = __frcp_rn(c[k][l]);
      }
    }
  }
  for (uint32_t t = threadIdx.x; t < 256; t += blockDim.x) {
#pragma unroll
    for (int m = 0; m < NL; ++m) {
      const int l = (NL == 3 && swap) ? 2 - m : m;
      float cl[4], rl[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        cl[k] = k < sig_n(SIG) ? c[k][l] : 0.f;
        rl[k] = k < sig_n(SIG) ? r[k][l] : 0.f;
      }
      lut[m * 256 + t] = Out(__float_as_uint(sig_apply<SIG>(float(t), cl, rl)));
    }
  }
}

}  // namespace

// One CTA = a strip of output columns x a band of rows, for the planes
// blockIdx.z, blockIdx.z + gridDim.z, ... (horizontal fusion). SIG = a
// registered AFFINE chain (table built from the compiled chain: once per CTA
// when its constants are plane-independent), or kSigLut (table built per plane
// by interpreting the plane's folded unaries + the compute program).
template <int NL, uint32_t OLK, bool SPLIT, uint32_t SIG>
__global__ void __launch_bounds__(256, FK_SEP_MINB) fk_resample_sep(const __grid_constant__ DPlan P) {
  constexpr bool AFFINE = SIG != kSigLut;
  using Out = typename std::conditional<OLK == FK_F64, uint64_t, uint32_t>::type;
  __shared__ RowEnt rows[kBandMax];
  __shared__ Visits vis;
  __shared__ Out lut[NL * 256];
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t y_begin = blockIdx.y * P.tiles_per_cta;  // tiles_per_cta = band rows for this kernel
  const uint32_t y_end = min(y_begin + P.tiles_per_cta, P.height);
  int table_swap = -1;  // AFFINE with plane-independent constants: the swap the table was built for
  for (uint32_t zi = blockIdx.z; zi < P.batch; zi += gridDim.z) {
    const uint32_t z = P.order ? __ldg(P.order + zi) : zi;
    const DSample s = P.reads[z];
    const DWrite w = P.writes[z];
    const bool swap = ((s.flags & SF_POST_SWAP) != 0) != (P.prog_swap != 0);
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < y_end - y_begin; j += blockDim.x) {
      RowEnt e;
      if (s.mode != RD_DIRECT) {  // y_entry gives row byte offsets; keep the source row numbers
        const YEnt ye = dev::y_entry(s, y_begin + j);
        e.s0 = uint32_t(ye.r0 / s.pitch);
        e.s1 = uint32_t(ye.r1 / s.pitch);
        e.f = ye.f;
      } else {
        e.s0 = e.s1 = s.y0 + y_begin + j;
        e.f = 0.0;
      }
      rows[j] = e;
    }
    if constexpr (AFFINE) {
      if (!P.aff_inline || table_swap != int(swap)) {
        build_affine_table<NL, SIG, Out>(P, z, swap, lut);
        table_swap = P.aff_inline ? int(swap) : -1;
      }
    } else {
      for (uint32_t t = threadIdx.x; t < 256; t += blockDim.x) {  // the chain over every byte value
        uint64_t v[1][3] = {{t, t, t}};
        dev::run_ops(P, s.post_off, s.post_len, z, v);
        dev::run_ops(P, P.op_base, P.n_ops, z, v);
#pragma unroll
        for (int m = 0; m < NL; ++m) lut[m * 256 + t] = Out(v[0][(NL == 3 && swap) ? 2 - m : m]);
      }
    }
    __syncthreads();
    if (s.mode == RD_BILINEAR) {
      if (threadIdx.x < 32) build_visits_warp(rows, y_end - y_begin, s.pitch, vis);
      __syncthreads();
    }
    if (!(w.flags & WF_ACTIVE) || x >= P.width) continue;  // BatchWrite z >= active_count / past the row
    const bool al = (w.flags & WF_LANE_ALIGNED) != 0;
    const bool aligned_rows = ((s.src | s.pitch) & 3) == 0;
    if (s.mode == RD_BILINEAR) {
      if (aligned_rows && al)
        column_bilinear<NL, OLK, SPLIT, true, true, Out>(s, w, rows, vis, x, y_begin, swap, lut);
      else if (al)
        column_bilinear<NL, OLK, SPLIT, false, true, Out>(s, w, rows, vis, x, y_begin, swap, lut);
      else
        column_bilinear<NL, OLK, SPLIT, false, false, Out>(s, w, rows, vis, x, y_begin, swap, lut);
    } else if (al) {
      column_tap<NL, OLK, SPLIT, true, Out>(s, w, rows, x, y_begin, y_end, swap, lut);
    } else {
      column_tap<NL, OLK, SPLIT, false, Out>(s, w, rows, x, y_begin, y_end, swap, lut);
    }
  }
}

}  // namespace fk
