// fp64 pipe throughput vs register operand count on B200: DFMA/DADD/DMUL
// chains whose operands are all distinct live registers (no reuse cache
// hits, no immediates) against the 1-register-operand form.
#include <cstdio>
#include <cuda_runtime.h>

// MODE 0: a = fma(a, b, imm) ; 1: a = fma(a, b_j, c_j) (3 distinct regs) ;
// 2: a = a + b_j (DADD, 2 regs) ; 3: a = fma(b_j, c_j, a) with b/c rotating
template <int K, int MODE>
__global__ void k(double* out, long long* cyc, int iters) {
  double a[K], b[K], c[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    a[j] = threadIdx.x * 1e-7 + j;
    b[j] = 1.0 + 1e-9 * (j + threadIdx.x);
    c[j] = 1e-9 * (j + 1);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (MODE == 0) a[j] = fma(a[j], 1.0000001, 1e-9);
      if (MODE == 1) a[j] = fma(a[j], b[j], c[j]);
      if (MODE == 2) a[j] = __dadd_rn(a[j], b[j]);
      if (MODE == 3) a[j] = fma(b[(j + 1) % K], c[(j + 3) % K], a[j]);
    }
    if (MODE == 3) {
      double t = b[0];
#pragma unroll
      for (int j = 0; j < K - 1; ++j) b[j] = b[j + 1];
      b[K - 1] = t;
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < K; ++j) s += a[j] + b[j] + c[j];
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K, int MODE>
void run(int warps) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 2048;
  k<K, MODE><<<148, 32 * warps>>>(out, cyc, iters);
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  printf("mode %d chains %2d warps/SM %2d: %.3f warp-DP/clk/SM (peak 2.0)\n", MODE, K, warps,
         (double)iters * K * warps / c);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {8, 16}) {
    run<16, 0>(w);
    run<16, 1>(w);
    run<16, 2>(w);
    run<16, 3>(w);
  }
  return 0;
}
