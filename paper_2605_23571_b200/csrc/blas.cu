// Dense fp64 pieces of the Nystrom / LMP / PCG stages on sm_100a.
//
//  * k_gemm_tn  : C = A^T B with the long dim K contiguous -- Gram Y^T Y
//                 (CholeskyQR2, replacing np.linalg.qr nystrom.py:118), W =
//                 Phi^T Y (nystrom.py:125), S^T R (lmp.py:63).  DMMA
//                 (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4) 64x64 tiles,
//                 deterministic split-K: fixed-slice partials + a fixed-order
//                 reduction (no atomics).
//  * k_gemm_nn  : D = beta*Cin + A diag(bscale) B with short inner dim --
//                 Q = Y R^-1, S = Q U_T (nystrom.py:131), S (c o S^T r)
//                 (lmp.py:65).  DMMA 64x64 tiles.
//  * column dots, fixed order (PCG r.z, p.Hp; krylov.py:72,81,87).
#include "common.cuh"

namespace edak {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ----------------------------------------------------------------- TN ----
// CTA: 256 threads (8 warps as 2 x 4), C tile 64 (a) x 64 (b); warp tile 32 x 16.
constexpr int TN_BM = 64, TN_BN = 64, TN_BK = 32, TN_PAD = 4;

__global__ void __launch_bounds__(256) k_gemm_tn(const double* __restrict__ A, int64_t lda,
                                                 const double* __restrict__ B, int64_t ldb, int m, int nb,
                                                 int64_t K, int64_t kslice, double* __restrict__ part) {
  __shared__ double sA[TN_BM][TN_BK + TN_PAD];
  __shared__ double sB[TN_BN][TN_BK + TN_PAD];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wa = (warp >> 2) * 32, wb = (warp & 3) * 16;
  const int a0 = blockIdx.x * TN_BM, b0 = blockIdx.y * TN_BN;
  const int64_t k_begin = (int64_t)blockIdx.z * kslice;
  const int64_t k_end = min(K, k_begin + kslice);
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int64_t k0 = k_begin; k0 < k_end; k0 += TN_BK) {
    // 64 columns x 32 contiguous k for each operand: 2048 doubles, 8 per thread
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = t + q * 256;
      const int col = idx >> 5, kk = idx & 31;
      const int64_t k = k0 + kk;
      const bool kin = k < k_end;
      sA[col][kk] = (kin && a0 + col < m) ? __ldg(A + k + (int64_t)(a0 + col) * lda) : 0.0;
      sB[col][kk] = (kin && b0 + col < nb) ? __ldg(B + k + (int64_t)(b0 + col) * ldb) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < TN_BK; ks += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = sA[wa + i * 8 + (lane >> 2)][ks + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = sB[wb + j * 8 + (lane >> 2)][ks + (lane & 3)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  // partial tile (m x nb, column-major with ld = m) for this K slice
  double* P = part + (size_t)blockIdx.z * m * nb;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = a0 + wa + i * 8 + (lane >> 2);
        const int b = b0 + wb + j * 8 + 2 * (lane & 3) + h;
        if (a < m && b < nb) P[a + (size_t)b * m] = acc[i][j][h];
      }
}

__global__ void k_reduce_parts(const double* __restrict__ part, int nsplit, int m, int nb, double* __restrict__ C,
                               int ldc) {
  const int64_t tot = (int64_t)m * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < nsplit; ++z) s += part[(size_t)z * tot + e];  // fixed order
    const int a = (int)(e % m), b = (int)(e / m);
    C[a + (size_t)b * ldc] = s;
  }
}

static int tn_nsplit(int m, int nb, int64_t K, int64_t& kslice) {
  const int tiles = ((m + TN_BM - 1) / TN_BM) * ((nb + TN_BN - 1) / TN_BN);
  int64_t want = (2 * 148 + tiles - 1) / tiles;  // >= ~2 waves of CTAs
  int64_t maxs = (K + 255) / 256;                // slices of >= 256 rows
  int64_t s = want < maxs ? want : maxs;
  if (s < 1) s = 1;
  kslice = (K + s - 1) / s;
  kslice = (kslice + TN_BK - 1) / TN_BK * TN_BK;
  s = (K + kslice - 1) / kslice;
  return (int)s;
}

int64_t gemm_tn_partials(int m, int nb, int64_t K) {
  int64_t ks;
  return (int64_t)tn_nsplit(m, nb, K, ks) * m * nb;
}

int launch_gemm_tn(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int ldc, int m, int nb,
                   int64_t K, double* part, cudaStream_t st) {
  int64_t ks;
  const int s = tn_nsplit(m, nb, K, ks);
  dim3 grid((m + TN_BM - 1) / TN_BM, (nb + TN_BN - 1) / TN_BN, s);
  k_gemm_tn<<<grid, 256, 0, st>>>(A, lda, B, ldb, m, nb, K, ks, part);
  int64_t tot = (int64_t)m * nb;
  int nblk = (int)((tot + 255) / 256);
  k_reduce_parts<<<nblk < 1024 ? nblk : 1024, 256, 0, st>>>(part, s, m, nb, C, ldc);
  count_launch(2);
  return check_launch("k_gemm_tn");
}

// ----------------------------------------------------------------- NN ----
constexpr int NN_BM = 64, NN_BN = 64, NN_BK = 32, NN_PAD = 4;

__global__ void __launch_bounds__(256) k_gemm_nn(const double* __restrict__ A, int64_t lda,
                                                 const double* __restrict__ B, int ldb,
                                                 const double* __restrict__ bscale, const double* Cin,
                                                 int64_t ldc, double beta, double* D, int64_t ldd, int64_t M,
                                                 int N, int kk) {
  __shared__ double sA[NN_BK][NN_BM + NN_PAD];
  __shared__ double sB[NN_BN][NN_BK + NN_PAD];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wi = (warp >> 2) * 32, wj = (warp & 3) * 16;
  const int64_t i0 = (int64_t)blockIdx.x * NN_BM;
  const int j0 = blockIdx.y * NN_BN;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int l0 = 0; l0 < kk; l0 += NN_BK) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = t + q * 256;
      // A chunk: 32 (l) x 64 (i), i contiguous in memory
      {
        const int l = idx >> 6, i = idx & 63;
        const int64_t gi = i0 + i;
        sA[l][i] = (l0 + l < kk && gi < M) ? __ldg(A + gi + (int64_t)(l0 + l) * lda) : 0.0;
      }
      // B chunk: 64 (j) x 32 (l), l contiguous in memory
      {
        const int j = idx >> 5, l = idx & 31;
        double bv = 0.0;
        if (l0 + l < kk && j0 + j < N) {
          bv = __ldg(B + (l0 + l) + (int64_t)(j0 + j) * ldb);
          if (bscale) bv *= __ldg(bscale + l0 + l);
        }
        sB[j][l] = bv;
      }
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < NN_BK; ks += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = sA[ks + (lane & 3)][wi + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = sB[wj + j * 8 + (lane >> 2)][ks + (lane & 3)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gi = i0 + wi + i * 8 + (lane >> 2);
        const int gj = j0 + wj + j * 8 + 2 * (lane & 3) + h;
        if (gi < M && gj < N) {
          double v = acc[i][j][h];
          if (Cin) v += beta * Cin[gi + gj * ldc];
          D[gi + gj * ldd] = v;
        }
      }
}

int launch_gemm_nn(const double* A, int64_t lda, const double* B, int ldb, const double* bscale, const double* Cin,
                   int64_t ldc, double beta, double* D, int64_t ldd, int64_t M, int N, int kk, cudaStream_t st) {
  dim3 grid((unsigned)((M + NN_BM - 1) / NN_BM), (N + NN_BN - 1) / NN_BN);
  k_gemm_nn<<<grid, 256, 0, st>>>(A, lda, B, ldb, bscale, Cin, ldc, beta, D, ldd, M, N, kk);
  count_launch();
  return check_launch("k_gemm_nn");
}

// ------------------------------------------------------- column dots ----
template <int NT>
__global__ void __launch_bounds__(NT) k_col_dots(int n, const double* __restrict__ a, const double* __restrict__ b,
                                                 double* __restrict__ out) {
  __shared__ double sh[32];
  const int col = blockIdx.x;
  const double* x = a + (size_t)col * n;
  const double* y = b + (size_t)col * n;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += NT) s += x[i] * y[i];
  s = block_sum<NT>(s, sh);
  if (threadIdx.x == 0) out[col] = s;
}

int launch_col_dots(int n, int ncols, const double* a, const double* b, double* out, cudaStream_t st) {
  k_col_dots<256><<<ncols, 256, 0, st>>>(n, a, b, out);
  count_launch();
  return check_launch("k_col_dots");
}

}  // namespace edak
