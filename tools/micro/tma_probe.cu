// Probe: a 3-D tensor map {16, rows, 8} with strides {128 B, 16 B} (rows
// overlapping: dim 2 shifts the window by 16 B) so that ONE TMA load can
// fetch a 65-row x 128-B window starting at any even element, SWIZZLE_128B.
// Checks encode status and the landed smem layout.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap tm, int c1, int c2, double* out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  double* buf = reinterpret_cast<double*>(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t mbar;
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(65 * 128));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(buf)),
        "l"((uint64_t)&tm), "r"(0), "r"(c1), "r"(c2), "r"(mb)
        : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                 : "=r"(done) : "r"(mb) : "memory");
  for (int i = threadIdx.x; i < 65 * 16; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const size_t total = 1 << 16;
  std::vector<double> h(total);
  for (size_t i = 0; i < total; ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, total * 8);
  cudaMalloc(&o, 65 * 16 * 8);
  cudaMemcpy(d, h.data(), total * 8, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no entry point\n"); return 1; }
  CUtensorMap tm;
  cuuint64_t dims[3] = {16, (total - 30) / 16 + 1, 8};
  cuuint64_t strides[2] = {128, 16};
  cuuint32_t box[3] = {16, 65, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode (overlapping strides) -> %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 2;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65 * 128 + 1024);
  int bad_total = 0;
  for (int c1 : {0, 3, 100}) for (int c2 : {0, 1, 5, 7}) {
    k<<<1, 128, 65 * 128 + 1024>>>(tm, c1, c2, o);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("kernel error %s\n", cudaGetErrorString(e)); return 3; }
    std::vector<double> g(65 * 16);
    cudaMemcpy(g.data(), o, g.size() * 8, cudaMemcpyDeviceToHost);
    const long E = 16L * c1 + 2L * c2;
    int bad = 0;
    for (int row = 0; row < 65; ++row)
      for (int p = 0; p < 8; ++p) {
        const int c = p ^ (row & 7);
        for (int u = 0; u < 2; ++u)
          if (g[row * 16 + 2 * p + u] != (double)(E + 16 * row + 2 * c + u)) ++bad;
      }
    printf("c1=%d c2=%d: %d mismatches (first row: %g %g %g %g)\n", c1, c2, bad, g[0], g[1], g[2], g[3]);
    bad_total += bad;
  }
  printf(bad_total ? "FAIL\n" : "OK\n");
  return bad_total ? 4 : 0;
}
