// fk_generic.cu — the interpreted-chain fused kernel (TransformDPP).
//
// One launch runs Read -> Compute* -> Write for every point of the iteration
// space: blockIdx.z is the batch plane z (horizontal fusion),
// each thread owns E consecutive x of one row (thread coarsening) and keeps all
// intermediates in registers (vertical fusion). The compute chain is a device
// program walked with warp-uniform dispatch, so ANY validated chain runs fused
// in one kernel; chains the registry knows run the compiled kernels instead
// (fk_compiled.cu). Four instantiations cover every chain: 32/64-bit lanes x 1/3 lanes.
#include <cuda_runtime.h>

#include "fk_launch.hpp"
#include "fk_stages.cuh"

#ifndef FK_MIN_BLOCKS
#define FK_MIN_BLOCKS 3  // CTAs per SM the register budget must allow
#endif

namespace fk {

template <class Lane, int L, int E>
__global__ void __launch_bounds__(kBlock, FK_MIN_BLOCKS) fk_transform_generic(const __grid_constant__ DPlan P) {
  __shared__ XTab xt;
  __shared__ YEnt yt[kYCap];
  __shared__ Lane lut[L][256];
  // this CTA walks tiles [t_begin, t_end) of plane z; a tile is E consecutive x of one row
  const uint32_t t_begin = blockIdx.x * P.tiles_per_cta;
  if (t_begin >= P.tiles) return;
  const uint32_t t_end = min(t_begin + P.tiles_per_cta, P.tiles);
  const uint32_t y_first = dev::fastdiv(t_begin, P.tpr);
  const uint32_t rows = dev::fastdiv(t_end - 1, P.tpr) - y_first + 1;
  for (uint32_t zi = blockIdx.z; zi < P.batch; zi += gridDim.z) {
    const uint32_t z = P.order ? __ldg(P.order + zi) : zi;
    DSample s;
    if (P.reads) {
      s = P.reads[z];
    } else {
      s = P.rd;
      s.src += uint64_t(z) * P.rd_zstride;
    }
    DWrite w;
    if (P.writes) {
      w = P.writes[z];
    } else {
      w = P.wr;
      w.dst[0] += uint64_t(z) * P.wr_zstride;
    }
    // CTA-uniform setup: resample coordinate tables and the u8 chain LUT
    const bool tab = s.mode != RD_DIRECT && !(s.flags & SF_DEFAULT) && P.width <= kXCap && rows <= kYCap;
    const bool use_lut = P.lut_ok && (s.flags & SF_LUT_SRC) && (P.n_ops + s.post_len) > 0;
    const bool swap = ((s.flags & SF_POST_SWAP) != 0) != (P.prog_swap != 0);
    if (tab || use_lut) {
      __syncthreads();
      if (tab) dev::build_tables(s, P.width, y_first, rows, xt, yt);
      if (use_lut) dev::build_lut<Lane, L, E>(P, s, z, lut);
      __syncthreads();
    }
    for (uint32_t t = t_begin + threadIdx.x; t < t_end; t += kBlock) {
      const uint32_t y = dev::fastdiv(t, P.tpr);
      const uint32_t x = (t - y * P.tiles_per_row) * E;
      const int n = (P.width - x) < uint32_t(E) ? int(P.width - x) : E;
      Lane v[E][L];
      dev::read_raw(P, s, x, y, n, v, tab ? &xt : nullptr, tab ? yt + (y - y_first) : nullptr);
      if (use_lut) {
        dev::apply_lut(lut, swap, v);
      } else {
        if (!(s.flags & SF_DEFAULT)) dev::run_ops(P, s.post_off, s.post_len, z, v);
        dev::run_ops(P, P.op_base, P.n_ops, z, v);
      }
      dev::write_tile(P, w, x, y, n, v);
    }
  }
}

int generic_state_class(bool wide, int lanes) { return (wide ? 2 : 0) + (lanes == 3 ? 1 : 0); }

int generic_elems(int cls) { return cls == 0 ? 8 : 4; }

cudaError_t launch_generic(int cls, const DPlan& P, cudaStream_t st) {
  if (P.tiles == 0 || P.batch == 0) return cudaSuccess;
  const dim3 grid((P.tiles + P.tiles_per_cta - 1) / P.tiles_per_cta, 1, P.batch < 65535u ? P.batch : 65535u);
  switch (cls) {
    case 0: fk_transform_generic<uint32_t, 1, 8><<<grid, kBlock, 0, st>>>(P); break;
    case 1: fk_transform_generic<uint32_t, 3, 4><<<grid, kBlock, 0, st>>>(P); break;
    case 2: fk_transform_generic<uint64_t, 1, 4><<<grid, kBlock, 0, st>>>(P); break;
    default: fk_transform_generic<uint64_t, 3, 4><<<grid, kBlock, 0, st>>>(P); break;
  }
  return cudaGetLastError();
}

}  // namespace fk
