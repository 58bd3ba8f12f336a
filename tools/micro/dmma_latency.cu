// DMMA.8x8x4 (mma.sync m8n8k4 f64) throughput vs warps per SM and independent
// accumulator chains per warp on B200 (one CTA per SM, clock64 inside).
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void chains(double* out, long long* cyc, int iters) {
  double c[K][2];
  const double a = 1.0000001 + threadIdx.x * 1e-9, b = 0.9999999;
#pragma unroll
  for (int j = 0; j < K; ++j) c[j][0] = c[j][1] = j;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < K; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < K; ++j) s += c[j][0] + c[j][1];
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K>
void run(int warps) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 1024;
  chains<K><<<148, 32 * warps>>>(out, cyc, iters);
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  const double dm = (double)iters * K * warps;  // DMMAs per SM
  printf("chains %2d warps/SM %2d: %.1f cyc per dependent DMMA, %.3f DMMA/clk/SM, %.1f TF at 1.965 GHz\n", K,
         warps, c / iters, dm / c, dm / c * 512 * 148 * 1.965e9 / 1e12);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16, 32}) {
    run<4>(w);
    run<8>(w);
    run<16>(w);
  }
  return 0;
}
