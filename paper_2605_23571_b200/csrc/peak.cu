// Roofline denominators measured on the box (MEASURED_PEAKS.json has HBM and
// bf16 only): an fp64 FMA-pipe loop (DFMA) and an fp64 tensor-pipe loop
// (DMMA.8x8x4), each with 8 independent dependency chains per thread/warp.
#include "common.cuh"

namespace edak {

__global__ void __launch_bounds__(256) k_peak_dfma(double* sink, int iters) {
  double a[8];
  const double b = 1.0000001, c = 1e-9;
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-7 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.678) sink[0] = s;  // keeps the chains alive
}

__global__ void __launch_bounds__(256) k_peak_dmma(double* sink, int iters) {
  double c[8][2];
  const double a = 1.0000001 + threadIdx.x * 1e-9, b = 0.9999999;
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) sink[0] = s;
}

}  // namespace edak

extern "C" {

// flops per launch: DFMA 2*8*iters*256*blocks; DMMA 512*8*iters*(256/32)*blocks
int edak_peak_dfma(double* sink, int iters, int blocks, void* stream) {
  edak::k_peak_dfma<<<blocks, 256, 0, edak::as_stream(stream)>>>(sink, iters);
  return edak::check_launch("k_peak_dfma");
}

int edak_peak_dmma(double* sink, int iters, int blocks, void* stream) {
  edak::k_peak_dmma<<<blocks, 256, 0, edak::as_stream(stream)>>>(sink, iters);
  return edak::check_launch("k_peak_dmma");
}

}  // extern "C"
