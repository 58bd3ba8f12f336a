// The two DMMA GEMMs of the spectral-LMP step of the batched PCG, shaped
// for the rank-k (k <= 128) factor S and a member group of <= 112 columns
// (lmp.py:62-74 applied to every member's residual; krylov.py:89-95):
//
//   k_lmp_tn : W = S^T R, split-K over n -- each CTA owns ALL k x M outputs
//              of its slice of n, so S and R are each read once;
//   k_lmp_nn : D = Cin + colscale o C2 + S diag(coef) W over an n-tile of
//              128 rows and all members -- the PCG p-update
//              p = r + beta p + S (c o W) (or z = r + S (c o W)), with the
//              whole coef o W (<= 112 x 128) resident in shared memory.
//
// Both use DMMA.8x8x4 (mma.sync m8n8k4 f64) with 8 warps as 4 x 2, each warp
// 4 x 7 fragments (32 x 56 outputs): 28 accumulator chains per warp and 11
// fragment loads per 28 DMMAs, against 2 x 2 chains / 6 loads per 8 DMMAs
// of the generic 64 x 64 tiles in blas.cu (which measured 13.6 / 10.1
// TFLOP/s on these shapes at cfg4, profiles/r1_cfg4_gemm_ncu_summary.txt).
// One CTA per SM (up to ~200 KB of staged operands), 3-stage (TN) / 2-stage
// (NN) cp.async pipelines, deterministic (fixed split-K slices, reduced in
// a fixed order by k_pcg_reduce_rz / k_reduce_parts).
#include "common.cuh"

namespace edak {

namespace lmpg {

constexpr int BK = 32, PAD = 4, LD = BK + PAD;  // K chunk and padded row stride (doubles)
constexpr int KMAX = 128, MMAX = 112;           // rank and member-group limits
constexpr int FM = 4, FN = 7;                   // fragments per warp
constexpr int NST_TN = 3;
constexpr size_t SMEM_TN = (size_t)NST_TN * (KMAX + MMAX) * LD * sizeof(double);
constexpr int BI = 112;                          // NN: n rows per CTA (7 warps x 16)
constexpr int NW_NN = 7, FM_NN = 2, FN_NN = 14;  // NN: warps, fragments per warp (16 x 112)
constexpr int LDW = KMAX + PAD;                  // NN: resident coef o W row stride
constexpr int LDA = BI + PAD;                    // NN: S chunk row stride
constexpr size_t SMEM_NN = ((size_t)MMAX * LDW + 2 * (size_t)BK * LDA) * sizeof(double);

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cpa16(double* dst, const double* src, int nbytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(nbytes));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

}  // namespace lmpg

// W-partials: part[z][b * k + a] = sum over CTA z's n-slice of S[a][i] R[b][i]
// (K chunks of TBK columns through an NST-stage cp.async ring)
template <int TBK, int NST>
__global__ void __launch_bounds__(256, 1) k_lmp_tn(const double* __restrict__ S, const double* __restrict__ R,
                                                   int64_t n, int k, int M, int nchunks,
                                                   double* __restrict__ part, int ldp, int col0) {
  using namespace lmpg;
  constexpr int TLD = TBK + PAD;
  extern __shared__ __align__(16) double sm[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wa = (warp & 3) * 32, wb = (warp >> 2) * 56;
  // this CTA's chunks [c0, c1) of the K = n dimension (fixed slices)
  const int c0 = (int)((int64_t)nchunks * blockIdx.x / gridDim.x);
  const int c1 = (int)((int64_t)nchunks * (blockIdx.x + 1) / gridDim.x);
  auto sA = [&](int st) { return sm + (size_t)st * (KMAX + MMAX) * TLD; };
  auto load = [&](int st, int c) {
    const int64_t k0 = (int64_t)c * TBK;
    double* a = sA(st);
    constexpr int PR = TBK / 2;  // 16-byte pairs per row
    constexpr int NP = (KMAX + MMAX) * PR;
#pragma unroll
    for (int q = 0; q < (NP + 255) / 256; ++q) {
      const int idx = t + q * 256;
      if (NP % 256 && idx >= NP) continue;
      const int row = idx / PR, kk = 2 * (idx % PR);
      const int64_t kg = k0 + kk;
      const int nb = kg < n ? (kg + 1 < n ? 16 : 8) : 0;
      if (row < KMAX) {
        const bool v = row < k;
        cpa16(a + row * TLD + kk, v ? S + kg + (int64_t)row * n : S, v ? nb : 0);
      } else {
        const int b = row - KMAX;
        const bool v = b < M;
        cpa16(a + row * TLD + kk, v ? R + kg + (int64_t)b * n : R, v ? nb : 0);
      }
    }
    commit();
  };
  // member fragments past M are computed on the zero-filled rows: no
  // warp-dependent guards in the unrolled loop (they measured 50% slower)
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nch = c1 - c0;
  for (int p = 0; p < NST - 1; ++p) {
    if (p < nch) load(p, c0 + p);
    else commit();
  }
  for (int c = 0; c < nch; ++c) {
    wait<NST - 2>();
    __syncthreads();  // chunk c landed for everyone; chunk c-1's stage is free
    if (c + NST - 1 < nch) load((c + NST - 1) % NST, c0 + c + NST - 1);
    else commit();
    const double* a = sA(c % NST);
    const double* b = a + (size_t)KMAX * TLD;
#pragma unroll 2
    for (int ks = 0; ks < TBK; ks += 4) {
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = a[(wa + i * 8 + (lane >> 2)) * TLD + ks + (lane & 3)];
#pragma unroll
      for (int j = 0; j < FN; ++j)
        bf[j] = b[(wb + j * 8 + (lane >> 2)) * TLD + ks + (lane & 3)];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
          dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  // partial z of column col0 + b at part[z * k * ldp + (col0 + b) * k + a]
  double* P = part + (size_t)blockIdx.x * k * ldp + (size_t)col0 * k;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ai = wa + i * 8 + (lane >> 2);
        const int bj = wb + j * 8 + 2 * (lane & 3) + h;
        if (ai < k && bj < M) P[(size_t)bj * k + ai] = acc[i][j][h];
      }
}

// D[b][i] = Cin[b][i] + colscale[b] C2[b][i] + sum_a S[a][i] coef[a] W[b][a]
// (C2 may alias D: every element is read before its own write; Cin, C2
// optional).  7 warps, each 16 rows of the 112-row n-tile x all 112 member
// columns (2 x 14 fragments): 147 CTAs cover a 16384 ring, one per SM.
__global__ void __launch_bounds__(lmpg::NW_NN * 32, 1)
    k_lmp_nn(const double* __restrict__ S, const double* __restrict__ W, const double* __restrict__ coef, int64_t n,
             int k, int M, const double* __restrict__ Cin, const double* __restrict__ colscale, const double* C2,
             double* D) {
  using namespace lmpg;
  constexpr int NT = NW_NN * 32, FM = FM_NN, FN = FN_NN;
  extern __shared__ __align__(16) double sm[];
  double* sW = sm;                          // [MMAX][LDW]: coef o W, row b
  double* sAbase = sm + (size_t)MMAX * LDW;  // [2][BK][LDA]: S chunk, row a, n contiguous
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wi = warp * 16;
  const int64_t i0 = (int64_t)blockIdx.x * BI;
  const int nch = (k + BK - 1) / BK;
  auto loadA = [&](int st, int c) {
    double* a = sAbase + (size_t)st * BK * LDA;
#pragma unroll
    for (int q = 0; q < BK * BI / 2 / NT; ++q) {  // 8 16-byte copies per thread
      const int idx = t + q * NT;
      const int row = idx / (BI / 2), ii = 2 * (idx % (BI / 2));
      const int ag = c * BK + row;
      const int64_t ig = i0 + ii;
      const int nb = ag < k ? (ig + 1 < n ? 16 : (ig < n ? 8 : 0)) : 0;
      cpa16(a + row * LDA + ii, nb ? S + ig + (int64_t)ag * n : S, nb);
    }
    commit();
  };
  // resident coef o W (zero beyond k, M): one group with chunk 0 of S
  for (int idx = t; idx < MMAX * KMAX / 2; idx += NT) {
    const int b = idx / (KMAX / 2), a = 2 * (idx % (KMAX / 2));
    const int nb = b < M ? (a + 1 < k ? 16 : (a < k ? 8 : 0)) : 0;
    cpa16(sW + b * LDW + a, nb ? W + a + (size_t)b * k : W, nb);
  }
  loadA(0, 0);
  wait<0>();
  // scale the resident W rows by coef (each thread its own copies' bytes)
  for (int idx = t; idx < MMAX * KMAX / 2; idx += NT) {
    const int b = idx / (KMAX / 2), a = 2 * (idx % (KMAX / 2));
    double* w = sW + b * LDW + a;
    w[0] *= a < k ? __ldg(coef + a) : 0.0;
    w[1] *= a + 1 < k ? __ldg(coef + a + 1) : 0.0;
  }
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int c = 0; c < nch; ++c) {
    if (c > 0) wait<0>();
    __syncthreads();  // chunk c (and, first, the scaled W) visible; the other stage free
    if (c + 1 < nch) loadA((c + 1) & 1, c + 1);
    const double* a = sAbase + (size_t)(c & 1) * BK * LDA;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = a[(ks + (lane & 3)) * LDA + wi + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < FN; ++j)
        bf[j] = sW[(j * 8 + (lane >> 2)) * LDW + c * BK + ks + (lane & 3)];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  // epilogue, one fragment row at a time: its 28 r operands, then its 28 p
  // operands (just written by the preceding PCG kernels, so L2 hits) are
  // loaded together, combined in the reference's order z = r + S(c o W),
  // p = z + beta p (lmp.py:64-65, krylov.py:95)
#pragma unroll
  for (int i = 0; i < FM; ++i) {
    const int64_t gi = i0 + wi + i * 8 + (lane >> 2);
    double e[FN][2];
    if (Cin) {
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gb = j * 8 + 2 * (lane & 3) + h;
          e[j][h] = gi < n && gb < M ? Cin[gi + gb * n] : 0.0;
        }
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[i][j][h] += e[j][h];
    }
    if (C2) {  // C2 may alias D: every element is read before its own write
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gb = j * 8 + 2 * (lane & 3) + h;
          e[j][h] = gi < n && gb < M ? C2[gi + gb * n] : 0.0;
        }
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gb = j * 8 + 2 * (lane & 3) + h;
          if (gb < M) acc[i][j][h] += colscale[gb] * e[j][h];
        }
    }
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gb = j * 8 + 2 * (lane & 3) + h;
        if (gi < n && gb < M) D[gi + gb * n] = acc[i][j][h];
      }
  }
}

// ------------------------------------------------------------ launchers --
bool lmp_gemm_ok(int64_t n, int k, int M) {
  const char* e = getenv("EDAK_LMP_GEMM");
  if (e && atoi(e) == 0) return false;
  // member groups beyond one 112-column tile take the generic kernels: at
  // cfg5 (128 per group) 692 us per LMP apply vs 1290 us as 112 + 16 blocks
  // or 3 x 655 us as three 86-member groups (profiles/r2_lmp_gemm_ab.txt)
  return k >= 1 && k <= lmpg::KMAX && k % 2 == 0 && M >= 1 && M <= lmpg::MMAX && n % 2 == 0 && n >= 4096;
}

// 148 CTAs (one per SM), fewer for short rings
static int lmp_tn_ctas(int64_t n) {
  const int64_t nch = (n + 15) / 16;
  return (int)(nch < 148 ? nch : 148);
}

int64_t lmp_tn_partials(int64_t n, int k, int M) { return (int64_t)lmp_tn_ctas(n) * k * M; }  // any M

template <int TBK, int NST>
static int go_tn(const double* S, const double* R, int64_t n, int k, int M, double* part, int ldp, int col0,
                 cudaStream_t st) {
  constexpr size_t smem = (size_t)NST * (lmpg::KMAX + lmpg::MMAX) * (TBK + lmpg::PAD) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_lmp_tn<TBK, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int g = lmp_tn_ctas(n);
  const int nch = (int)((n + TBK - 1) / TBK);
  k_lmp_tn<TBK, NST><<<g, 256, smem, st>>>(S, R, n, k, M, nch, part, ldp, col0);
  count_launch();
  return g;
}

// split-K partials of W = S^T R (layout part[z][b * k + a], b < M) for any
// M: column blocks of <= MMAX, each through k_lmp_tn (a column's partials do
// not depend on the block it is in); returns the split count, or 0 when the
// generic split-K GEMM should run instead (EDAK_LMP_TN: 0 generic, 1 chunks
// of 32 x 3 stages, 2 (default) chunks of 16 x 5)
int launch_lmp_tn(const double* S, const double* R, int64_t n, int k, int M, double* part, cudaStream_t st) {
  static const int mode = [] {
    const char* e = getenv("EDAK_LMP_TN");
    return e ? atoi(e) : 2;
  }();
  if (mode != 1 && mode != 2) return 0;
  int g = 0;
  for (int c0 = 0; c0 < M; c0 += lmpg::MMAX) {
    const int m = M - c0 < lmpg::MMAX ? M - c0 : lmpg::MMAX;
    g = mode == 1 ? go_tn<32, 3>(S, R + (size_t)c0 * n, n, k, m, part, M, c0, st)
                  : go_tn<16, 5>(S, R + (size_t)c0 * n, n, k, m, part, M, c0, st);
  }
  return g;
}

// column blocks of <= MMAX members (each column's result is independent of
// its block)
int launch_lmp_nn(const double* S, const double* W, const double* coef, int64_t n, int k, int M, const double* Cin,
                  const double* colscale, const double* C2, double* D, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_lmp_nn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lmpg::SMEM_NN);
    attr = true;
  }
  const unsigned g = (unsigned)((n + lmpg::BI - 1) / lmpg::BI);
  for (int c0 = 0; c0 < M; c0 += lmpg::MMAX) {
    const int m = M - c0 < lmpg::MMAX ? M - c0 : lmpg::MMAX;
    const size_t off = (size_t)c0 * n;
    k_lmp_nn<<<g, lmpg::NW_NN * 32, lmpg::SMEM_NN, st>>>(S, W + (size_t)c0 * k, coef, n, k, m,
                                                          Cin ? Cin + off : nullptr, colscale ? colscale + c0 : nullptr,
                                                          C2 ? C2 + off : nullptr, D + off);
    count_launch();
  }
  return check_launch("k_lmp_nn");
}

}  // namespace edak
