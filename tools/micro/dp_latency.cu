// fp64 pipe micro-benchmark on B200: latency of dependent DADD/DFMA chains and
// throughput vs warps per SM and independent chains per thread (clock64 inside
// the kernel; one CTA per SM).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void chains(double* out, long long* cyc, int iters, double b) {
  double a[K];
#pragma unroll
  for (int j = 0; j < K; ++j) a[j] = threadIdx.x * 1e-7 + j;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < K; ++j) a[j] = fma(a[j], b, 1e-9);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < K; ++j) s += a[j];
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K>
__global__ void chains_add(double* out, long long* cyc, int iters, double b) {
  double a[K];
#pragma unroll
  for (int j = 0; j < K; ++j) a[j] = threadIdx.x * 1e-7 + j;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < K; ++j) a[j] = __dadd_rn(a[j], b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < K; ++j) s += a[j];
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K, bool ADD>
void run(int warps) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  if (ADD) chains_add<K><<<148, 32 * warps>>>(out, cyc, iters, 1.0000001);
  else chains<K><<<148, 32 * warps>>>(out, cyc, iters, 1.0000001);
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  const double ops = (double)iters * K * warps;  // warp-instructions per SM
  printf("%s chains/thread %2d warps/SM %2d: %.2f cyc per dependent op, %.3f warp-DP/clk/SM (peak 2.0)\n",
         ADD ? "DADD" : "DFMA", K, warps, c / iters, ops / c);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<1, false>(1);
  run<1, true>(1);
  for (int w : {4, 8, 16}) {
    run<4, false>(w);
    run<8, false>(w);
    run<16, false>(w);
  }
  run<8, true>(8);
  run<16, true>(8);
  return 0;
}
