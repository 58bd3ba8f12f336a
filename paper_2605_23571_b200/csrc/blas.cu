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
#include <cstdlib>

namespace edak {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// cp.async 8-byte copy with zero-fill (src_bytes = 0 writes zeros)
__device__ __forceinline__ void cpa8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 8 : 0));
}
// 16-byte variant (cp.async.cg, L2 only): nbytes of 0, 8 or 16 valid source
// bytes, the rest zero-filled
__device__ __forceinline__ void cpa16(double* dst, const double* src, int nbytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(nbytes));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Both kernels: 8 warps as WM x (8 / WM), each warp FM x FN DMMA.8x8x4
// fragments, so the CTA tile is BM = 8 WM FM rows by BN = 8 (8 / WM) FN
// columns; K chunks of 32 staged by a 2-deep cp.async pipeline so the next
// chunk's loads overlap this chunk's DMMAs.  Two tilings:
//   <2, 4, 2>: 64 x 64 (general shapes)
//   <4, 2, 7>: 64 x 112 -- one N tile for the 65..112-member groups of the
//              batched PCG (100 at cfg4: 13 live fragments of 14, against
//              128 columns for two 64-wide tiles), 14 DMMAs per 9 fragment
//              loads; fragments wholly past N are skipped (warp-uniform).
constexpr int G_BK = 32, G_PAD = 4;

template <int WM, int FM, int FN>
struct GTile {
  static constexpr int WN = 8 / WM, BM = 8 * WM * FM, BN = 8 * WN * FN;
  static constexpr size_t smem_tn = (2 * (size_t)(BM + BN) * (G_BK + G_PAD)) * sizeof(double);
  static constexpr size_t smem_nn =
      (2 * (size_t)G_BK * (BM + G_PAD) + 2 * (size_t)BN * (G_BK + G_PAD) + 2 * G_BK) * sizeof(double);
};

// ----------------------------------------------------------------- TN ----
// sA[stage][col a][k], sB[stage][col b][k]  (both operands K-contiguous)
template <int WM, int FM, int FN, bool V16 = false>
__global__ void __launch_bounds__(256) k_gemm_tn(const double* __restrict__ A, int64_t lda,
                                                 const double* __restrict__ B, int64_t ldb, int m, int nb,
                                                 int64_t K, int64_t kslice, double* __restrict__ part) {
  using GT = GTile<WM, FM, FN>;
  constexpr int BM = GT::BM, BN = GT::BN;
  extern __shared__ __align__(16) double gsm[];
  double (*sA)[BM][G_BK + G_PAD] = reinterpret_cast<double (*)[BM][G_BK + G_PAD]>(gsm);
  double (*sB)[BN][G_BK + G_PAD] = reinterpret_cast<double (*)[BN][G_BK + G_PAD]>(gsm + 2 * BM * (G_BK + G_PAD));
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wa = (warp % WM) * 8 * FM, wb = (warp / WM) * 8 * FN;
  const int a0 = blockIdx.x * BM, b0 = blockIdx.y * BN;
  const int64_t k_begin = (int64_t)blockIdx.z * kslice;
  const int64_t k_end = min(K, k_begin + kslice);
  const int nch = (int)((k_end - k_begin + G_BK - 1) / G_BK);
  auto load = [&](int stg, int64_t k0) {
    if constexpr (V16) {  // 16-byte pairs along K (even lda/ldb/k0, 16-byte aligned operands)
#pragma unroll
      for (int q = 0; q < (BM + BN) * G_BK / 512; ++q) {
        const int idx = t + q * 256;
        const int col = idx >> 4, kk = 2 * (idx & 15);
        const int64_t k = k0 + kk;
        const int nbytes = k < k_end ? (k + 1 < k_end ? 16 : 8) : 0;
        if (col < BM) {
          const bool va = a0 + col < m;
          cpa16(&sA[stg][col][kk], va ? A + k + (int64_t)(a0 + col) * lda : A, va ? nbytes : 0);
        } else {
          const int c = col - BM;
          const bool vb = b0 + c < nb;
          cpa16(&sB[stg][c][kk], vb ? B + k + (int64_t)(b0 + c) * ldb : B, vb ? nbytes : 0);
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < (BM + BN) * G_BK / 256; ++q) {
        const int idx = t + q * 256;
        const int col = idx >> 5, kk = idx & 31;
        const int64_t k = k0 + kk;
        const bool kin = k < k_end;
        if (col < BM) {
          const bool va = kin && a0 + col < m;
          cpa8(&sA[stg][col][kk], va ? A + k + (int64_t)(a0 + col) * lda : A, va);
        } else {
          const int c = col - BM;
          const bool vb = kin && b0 + c < nb;
          cpa8(&sB[stg][c][kk], vb ? B + k + (int64_t)(b0 + c) * ldb : B, vb);
        }
      }
    }
    cpa_commit();
  };
  // fragments wholly past nb are skipped (warp-uniform)
  int nfr = (nb - b0 - wb + 7) / 8;
  nfr = nfr < 0 ? 0 : (nfr > FN ? FN : nfr);
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (nch > 0) load(0, k_begin);
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      load((c + 1) & 1, k_begin + (int64_t)(c + 1) * G_BK);
      cpa_wait<1>();
    } else {
      cpa_wait<0>();
    }
    __syncthreads();
    const int stg = c & 1;
#pragma unroll
    for (int ks = 0; ks < G_BK; ks += 4) {
      double af[FM], bf[FN];
#ifdef EDAK_EXP_NOFRAG  // timing ablation (wrong results): DMMAs without their fragment loads
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = 1.0 + i * 1e-3 + ks;
#pragma unroll
      for (int j = 0; j < FN; ++j) bf[j] = 1.0 + j * 1e-3 + ks;
#else
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = sA[stg][wa + i * 8 + (lane >> 2)][ks + (lane & 3)];
#pragma unroll
      for (int j = 0; j < FN; ++j)
        if (j < nfr) bf[j] = sB[stg][wb + j * 8 + (lane >> 2)][ks + (lane & 3)];
#endif
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
          if (j < nfr) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  double* P = part + (size_t)blockIdx.z * m * nb;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = a0 + wa + i * 8 + (lane >> 2);
        const int b = b0 + wb + j * 8 + 2 * (lane & 3) + h;
        if (a < m && b < nb) P[a + (size_t)b * m] = acc[i][j][h];
      }
}

// Fixed-order split-K reduction: 8 lanes per output, lane q sums splits
// q, q+8, q+16, ... in order, then the 8 lane sums are combined in a fixed
// butterfly order -- deterministic, and 8x the memory-level parallelism of
// one thread per output (the reduction was latency-bound: 50 CTAs).
// sym: the partials hold only the upper-triangle 128 x 128 tiles of a
// symmetric product (launch_big_tn); outputs of the other tiles are read
// from their mirror image.
__global__ void __launch_bounds__(256) k_reduce_parts(const double* __restrict__ part, int nsplit, int m, int nb,
                                                      double* __restrict__ C, int ldc, int sym = 0) {
  const int64_t tot = (int64_t)m * nb;
  const int q = threadIdx.x & 7;
  for (int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3; e < tot;
       e += ((int64_t)gridDim.x * blockDim.x) >> 3) {
    int64_t src = e;
    if (sym) {
      const int a = (int)(e % m), b = (int)(e / m);
      if ((a >> 7) > (b >> 7)) src = b + (int64_t)a * m;
    }
    double s = 0.0;
    for (int z = q; z < nsplit; z += 8) s += part[(size_t)z * tot + src];
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (q == 0) {
      const int a = (int)(e % m), b = (int)(e / m);
      C[a + (size_t)b * ldc] = s;
    }
  }
}

int launch_reduce_parts(const double* part, int nsplit, int m, int nb, double* C, int ldc, cudaStream_t st) {
  const int64_t tot = (int64_t)m * nb;
  const int nblk = (int)((tot * 8 + 255) / 256);
  k_reduce_parts<<<nblk < 4096 ? nblk : 4096, 256, 0, st>>>(part, nsplit, m, nb, C, ldc);
  count_launch();
  return check_launch("k_reduce_parts");
}

// tiling for N columns: 64 x 112 for 65..112 (EDAK_GEMM_WIDE=0: always 64 x 64)
static bool gemm_wide(int nb) {
  const char* e = getenv("EDAK_GEMM_WIDE");
  if (e && atoi(e) == 0) return false;
  return nb > 64 && nb <= 112;
}

static int tn_nsplit(int m, int nb, int64_t K, int64_t& kslice) {
  const int bn = gemm_wide(nb) ? GTile<4, 2, 7>::BN : GTile<2, 4, 2>::BN;
  const int tiles = ((m + 63) / 64) * ((nb + bn - 1) / bn);
  static const int waves = [] {  // A/B knob: CTAs per SM targeted by the split
    const char* e = getenv("EDAK_TN_WAVES");
    return e ? atoi(e) : 2;
  }();
  int64_t want = (waves * 148 + tiles - 1) / tiles;
  int64_t maxs = (K + 127) / 128;                // slices of >= 128 rows
  int64_t s = want < maxs ? want : maxs;
  if (s < 1) s = 1;
  kslice = (K + s - 1) / s;
  kslice = (kslice + G_BK - 1) / G_BK * G_BK;
  s = (K + kslice - 1) / kslice;
  return (int)s;
}

bool big_tn_ok(const double* A, int64_t lda, const double* B, int64_t ldb, int m, int nb, int64_t K);
bool big_tn_sym(const double* A, int64_t lda, const double* B, int64_t ldb, int m, int nb);
int64_t big_tn_partials(int m, int nb, int64_t K);
int launch_big_tn(const double* A, int64_t lda, const double* B, int64_t ldb, int m, int nb, int64_t K, double* part,
                  cudaStream_t st);

int64_t gemm_tn_partials(int m, int nb, int64_t K) {
  if (m < 1 || nb < 1 || K < 1) return 0;  // empty block: no partials
  int64_t ks;
  const int64_t a = (int64_t)tn_nsplit(m, nb, K, ks) * m * nb;
  const int64_t b = m >= 128 && nb >= 128 ? big_tn_partials(m, nb, K) : 0;
  return a > b ? a : b;
}

// split-K partials only (the consumer reduces them): returns the split count
int launch_gemm_tn_parts(const double* A, int64_t lda, const double* B, int64_t ldb, int m, int nb, int64_t K,
                         double* part, cudaStream_t st) {
  using G0 = GTile<2, 4, 2>;
  using G1 = GTile<4, 2, 7>;
  if (big_tn_ok(A, lda, B, ldb, m, nb, K)) return launch_big_tn(A, lda, B, ldb, m, nb, K, part, st);
  int64_t ks;
  const int s = tn_nsplit(m, nb, K, ks);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_tn<2, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G0::smem_tn);
    cudaFuncSetAttribute(k_gemm_tn<4, 2, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G1::smem_tn);
    cudaFuncSetAttribute(k_gemm_tn<2, 4, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G0::smem_tn);
    cudaFuncSetAttribute(k_gemm_tn<4, 2, 7, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G1::smem_tn);
    attr = true;
  }
  const char* ev = getenv("EDAK_GEMM_V16");
  const bool v16 = !(ev && atoi(ev) == 0) && lda % 2 == 0 && ldb % 2 == 0 && ks % 2 == 0 &&
                   ((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0;
  if (gemm_wide(nb) && v16) {
    dim3 grid((m + G1::BM - 1) / G1::BM, (nb + G1::BN - 1) / G1::BN, s);
    k_gemm_tn<4, 2, 7, true><<<grid, 256, G1::smem_tn, st>>>(A, lda, B, ldb, m, nb, K, ks, part);
  } else if (gemm_wide(nb)) {
    dim3 grid((m + G1::BM - 1) / G1::BM, (nb + G1::BN - 1) / G1::BN, s);
    k_gemm_tn<4, 2, 7><<<grid, 256, G1::smem_tn, st>>>(A, lda, B, ldb, m, nb, K, ks, part);
  } else if (v16) {
    dim3 grid((m + G0::BM - 1) / G0::BM, (nb + G0::BN - 1) / G0::BN, s);
    k_gemm_tn<2, 4, 2, true><<<grid, 256, G0::smem_tn, st>>>(A, lda, B, ldb, m, nb, K, ks, part);
  } else {
    dim3 grid((m + G0::BM - 1) / G0::BM, (nb + G0::BN - 1) / G0::BN, s);
    k_gemm_tn<2, 4, 2><<<grid, 256, G0::smem_tn, st>>>(A, lda, B, ldb, m, nb, K, ks, part);
  }
  count_launch();
  return s;
}

int launch_gemm_tn(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int ldc, int m, int nb,
                   int64_t K, double* part, cudaStream_t st) {
  const int s = launch_gemm_tn_parts(A, lda, B, ldb, m, nb, K, part, st);
  const int sym = big_tn_ok(A, lda, B, ldb, m, nb, K) && big_tn_sym(A, lda, B, ldb, m, nb);
  int64_t tot = (int64_t)m * nb;
  int nblk = (int)((tot * 8 + 255) / 256);
  k_reduce_parts<<<nblk < 4096 ? nblk : 4096, 256, 0, st>>>(part, s, m, nb, C, ldc, sym);
  count_launch();
  return check_launch("k_gemm_tn");
}

// ----------------------------------------------------------------- NN ----
// sA[stage][l][i] (A is M-contiguous), sB[stage][j][l] (B is K-contiguous)
template <int WM, int FM, int FN, bool V16 = false>
__global__ void __launch_bounds__(256, 2) k_gemm_nn(const double* __restrict__ A, int64_t lda,
                                                 const double* __restrict__ B, int ldb,
                                                 const double* __restrict__ bscale, const double* Cin,
                                                 int64_t ldc, double beta, double* D, int64_t ldd, int64_t M,
                                                 int N, int kk, const double* __restrict__ colscale,
                                                 const double* C2) {
  using GT = GTile<WM, FM, FN>;
  constexpr int BM = GT::BM, BN = GT::BN;
  extern __shared__ __align__(16) double gsm[];
  double (*sA)[G_BK][BM + G_PAD] = reinterpret_cast<double (*)[G_BK][BM + G_PAD]>(gsm);
  double (*sB)[BN][G_BK + G_PAD] = reinterpret_cast<double (*)[BN][G_BK + G_PAD]>(gsm + 2 * G_BK * (BM + G_PAD));
  double (*sS)[G_BK] =
      reinterpret_cast<double (*)[G_BK]>(gsm + 2 * G_BK * (BM + G_PAD) + 2 * BN * (G_BK + G_PAD));
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wi = (warp % WM) * 8 * FM, wj = (warp / WM) * 8 * FN;
  const int64_t i0 = (int64_t)blockIdx.x * BM;
  const int j0 = blockIdx.y * BN;
  const int nch = (kk + G_BK - 1) / G_BK;
  auto load = [&](int stg, int l0) {
    if constexpr (V16) {  // 16-byte pairs (even M offsets / lda / ldb, 16-byte aligned operands)
#pragma unroll
      for (int q = 0; q < BM * G_BK / 512; ++q) {
        const int idx = t + q * 256;
        const int l = idx / (BM / 2), i = 2 * (idx % (BM / 2));
        const int nb_ = l0 + l < kk ? (i0 + i + 1 < M ? 16 : (i0 + i < M ? 8 : 0)) : 0;
        cpa16(&sA[stg][l][i], nb_ ? A + (i0 + i) + (int64_t)(l0 + l) * lda : A, nb_);
      }
#pragma unroll
      for (int q = 0; q < BN * G_BK / 512; ++q) {
        const int idx = t + q * 256;
        const int j = idx >> 4, l = 2 * (idx & 15);
        const int nb_ = j0 + j < N ? (l0 + l + 1 < kk ? 16 : (l0 + l < kk ? 8 : 0)) : 0;
        cpa16(&sB[stg][j][l], nb_ ? B + (l0 + l) + (int64_t)(j0 + j) * ldb : B, nb_);
      }
    } else {
#pragma unroll
      for (int q = 0; q < BM * G_BK / 256; ++q) {
        const int idx = t + q * 256;
        const int l = idx / BM, i = idx % BM;
        const bool v = l0 + l < kk && i0 + i < M;
        cpa8(&sA[stg][l][i], v ? A + (i0 + i) + (int64_t)(l0 + l) * lda : A, v);
      }
#pragma unroll
      for (int q = 0; q < BN * G_BK / 256; ++q) {
        const int idx = t + q * 256;
        const int j = idx >> 5, l = idx & 31;
        const bool v = l0 + l < kk && j0 + j < N;
        cpa8(&sB[stg][j][l], v ? B + (l0 + l) + (int64_t)(j0 + j) * ldb : B, v);
      }
    }
    if (bscale && t < G_BK) {
      const bool v = l0 + t < kk;
      cpa8(&sS[stg][t], v ? bscale + l0 + t : bscale, v);
    }
    cpa_commit();
  };
  int nfr = (N - j0 - wj + 7) / 8;  // live fragments of this warp (warp-uniform)
  nfr = nfr < 0 ? 0 : (nfr > FN ? FN : nfr);
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  load(0, 0);
  // the epilogue operands (PCG p-update: r and p) are fetched now, so their
  // latency hides behind the K loop instead of ending every CTA (K is only
  // 4 chunks for the LMP shapes); the wide tiling has no registers to spare
  constexpr bool PRE = FM * FN <= 8;
  double ec[FM][FN][2], e2[FM][FN][2];
#pragma unroll
  for (int i = 0; i < (PRE ? FM : 0); ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gi = i0 + wi + i * 8 + (lane >> 2);
        const int gj = j0 + wj + j * 8 + 2 * (lane & 3) + h;
        const bool in = gi < M && gj < N;
        ec[i][j][h] = Cin && in ? Cin[gi + gj * ldc] : 0.0;
        e2[i][j][h] = C2 && in ? C2[gi + gj * ldd] : 0.0;  // C2 may alias D: read before any write
      }
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      load((c + 1) & 1, (c + 1) * G_BK);
      cpa_wait<1>();
    } else {
      cpa_wait<0>();
    }
    __syncthreads();
    const int stg = c & 1;
#pragma unroll
    for (int ks = 0; ks < G_BK; ks += 4) {
      double af[FM], bf[FN];
#ifdef EDAK_EXP_NOFRAG
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = 1.0 + i * 1e-3 + ks;
#pragma unroll
      for (int j = 0; j < FN; ++j) bf[j] = 1.0 + j * 1e-3 + ks;
#else
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = sA[stg][ks + (lane & 3)][wi + i * 8 + (lane >> 2)];
      const double sc = bscale ? sS[stg][ks + (lane & 3)] : 1.0;
#pragma unroll
      for (int j = 0; j < FN; ++j)
        if (j < nfr) bf[j] = sc * sB[stg][wj + j * 8 + (lane >> 2)][ks + (lane & 3)];
#endif
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
          if (j < nfr) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gi = i0 + wi + i * 8 + (lane >> 2);
        const int gj = j0 + wj + j * 8 + 2 * (lane & 3) + h;
        if (gi < M && gj < N) {
          double v = acc[i][j][h];
          if (Cin) v += beta * (PRE ? ec[i][j][h] : Cin[gi + gj * ldc]);
          if (C2) v += colscale[gj] * (PRE ? e2[i][j][h] : C2[gi + gj * ldd]);  // C2 may alias D
          D[gi + gj * ldd] = v;
        }
      }
}

int launch_gemm_nn(const double* A, int64_t lda, const double* B, int ldb, const double* bscale, const double* Cin,
                   int64_t ldc, double beta, double* D, int64_t ldd, int64_t M, int N, int kk, cudaStream_t st,
                   const double* colscale, const double* C2) {
  using G0 = GTile<2, 4, 2>;
  using G1 = GTile<4, 2, 7>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_nn<2, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G0::smem_nn);
    cudaFuncSetAttribute(k_gemm_nn<4, 2, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G1::smem_nn);
    cudaFuncSetAttribute(k_gemm_nn<2, 4, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G0::smem_nn);
    attr = true;
  }
  // the p-update (K = 128) keeps the 64 x 64 tiling: its epilogue-operand
  // prefetch needs the registers the wide tiling spends on accumulators
  // (measured: 35.5 us narrow vs 35.8 us wide per 100-member group)
  const char* ew = getenv("EDAK_GEMM_WIDE_NN");
  if (ew && atoi(ew) != 0 && gemm_wide(N)) {
    dim3 grid((unsigned)((M + G1::BM - 1) / G1::BM), (N + G1::BN - 1) / G1::BN);
    k_gemm_nn<4, 2, 7><<<grid, 256, G1::smem_nn, st>>>(A, lda, B, ldb, bscale, Cin, ldc, beta, D, ldd, M, N, kk,
                                                       colscale, C2);
  } else {
    const char* ev = getenv("EDAK_GEMM_V16");
    const bool v16 = !(ev && atoi(ev) == 0) && lda % 2 == 0 && ldb % 2 == 0 && ((uintptr_t)A & 15) == 0 &&
                     ((uintptr_t)B & 15) == 0;
    dim3 grid((unsigned)((M + G0::BM - 1) / G0::BM), (N + G0::BN - 1) / G0::BN);
    if (v16)
      k_gemm_nn<2, 4, 2, true><<<grid, 256, G0::smem_nn, st>>>(A, lda, B, ldb, bscale, Cin, ldc, beta, D, ldd, M,
                                                               N, kk, colscale, C2);
    else
      k_gemm_nn<2, 4, 2><<<grid, 256, G0::smem_nn, st>>>(A, lda, B, ldb, bscale, Cin, ldc, beta, D, ldd, M, N, kk,
                                                         colscale, C2);
  }
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
