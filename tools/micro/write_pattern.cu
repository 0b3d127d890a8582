// Microbenchmark: DRAM write patterns of the C5 planar-split output (8192 crops x 3 planes of 224x224 f32,
// 4.93 GB), 8-byte stores per lane, CTA = one crop band of 112 rows (4 warps), 2 bands per crop.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a write_pattern.cu -o write_pattern && ./write_pattern
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int W = 224, H = 224, B = 8192, ROWS = 112;
constexpr size_t PLANE = size_t(W) * H * 4;

template <int MODE>
__global__ void __launch_bounds__(128) wp(unsigned char* out) {
  const int cta = blockIdx.x, band = cta & 1;
  // MODE 4: the real pattern with CTAs in frame order (crop z uses frame z % 16, as C5's units run)
  const int z = MODE == 4 ? ((cta >> 1) % 512) * 16 + (cta >> 1) / 512 : cta >> 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float2 v = make_float2(1.0f, 2.0f);
  for (int r = 0; r < ROWS; ++r) {
    const int y = band * ROWS + r;
    for (int m = 0; m < 3; ++m) {
      unsigned char* plane = out + (size_t(z) * 3 + m) * PLANE;
      if (MODE == 0 || MODE == 1 || MODE == 4) {  // real: warp w owns columns [64w, 64w + 64)
        const int x = 64 * warp + 2 * lane;
        if (x < W) *reinterpret_cast<float2*>(plane + size_t(y) * W * 4 + x * 4) = v;
      } else if (MODE == 2) {  // CTA row-major: threads 0..111 write the 896-byte row contiguously
        if (threadIdx.x < W / 2) *reinterpret_cast<float2*>(plane + size_t(y) * W * 4 + threadIdx.x * 8) = v;
      } else {  // per-warp sequential region (same bytes per warp)
        const size_t wid = size_t(cta) * 4 + warp;
        const size_t per_warp = size_t(ROWS) * 3 * 256;
        if (!(warp == 3 && lane >= 16))
          *reinterpret_cast<float2*>(out + wid * per_warp - (wid / 4) * size_t(ROWS) * 3 * 128 + (size_t(r) * 3 + m) * (warp == 3 ? 128 : 256) + lane * 8) = v;
      }
    }
    if (MODE == 1) __syncthreads();
  }
}

int main() {
  unsigned char* out;
  const size_t bytes = size_t(B) * 3 * PLANE;
  if (cudaMalloc(&out, bytes + (64 << 20)) != cudaSuccess) return 1;
  unsigned char* flush;
  cudaMalloc(&flush, 512 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[5] = {"real (warp column strips)", "real + __syncthreads per row", "CTA row-major (896 B rows)",
                          "per-warp sequential", "real, CTAs in frame order"};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 5; ++mode) {
      float best = 1e9;
      for (int it = 0; it < 5; ++it) {
        cudaMemsetAsync(flush, it, 512 << 20);
        cudaEventRecord(a);
        switch (mode) {
          case 0: wp<0><<<B * 2, 128>>>(out); break;
          case 1: wp<1><<<B * 2, 128>>>(out); break;
          case 2: wp<2><<<B * 2, 128>>>(out); break;
          case 3: wp<3><<<B * 2, 128>>>(out); break;
          default: wp<4><<<B * 2, 128>>>(out); break;
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      printf("%-32s %.3f ms  %.0f GB/s\n", names[mode], best, bytes / (best * 1e-3) / 1e9);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
