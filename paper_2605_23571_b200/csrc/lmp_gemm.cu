// The two DMMA GEMMs of the spectral-LMP step of the batched PCG, shaped
// for the rank-k (k <= 128) factor S and a member group of <= 128 columns
// (lmp.py:62-74 applied to every member's residual; krylov.py:89-95):
//
//   k_lmp_tn : W = S^T R, split-K over n -- each CTA owns ALL k x M outputs
//              of its slice of n, so S and R are each read once;
//   k_lmp_nn : D = Cin + colscale o C2 + S diag(coef) W over an n-tile of
//              112 / 128 rows and all members -- the PCG p-update
//              p = r + beta p + S (c o W) (or z = r + S (c o W)), with the
//              whole coef o W (<= 128 x 128) resident in shared memory.
//
// Both use DMMA.8x8x4 (mma.sync m8n8k4 f64).  TN: 8 warps as 4 x 2, each warp
// 4 x 7 fragments (32 x 56 outputs, 112-member tiles) or 4 x 8 (128-member
// tiles; also the cfg5 Nystrom Grams): 28-32 accumulator chains per warp and
// 11-12 fragment loads per 28-32 DMMAs, against 2 x 2 chains / 6 loads per 8 DMMAs
// of the generic 64 x 64 tiles in blas.cu (which measured 13.6 / 10.1
// TFLOP/s on these shapes at cfg4, profiles/r1_cfg4_gemm_ncu_summary.txt).
// One CTA per SM (up to ~200 KB of staged operands), 3-stage (TN) / 2-stage
// (NN) cp.async pipelines, deterministic (fixed split-K slices, reduced in
// a fixed order by k_pcg_reduce_rz / k_reduce_parts).
#include "common.cuh"

namespace edak {

namespace lmpg {

constexpr int BK = 32, PAD = 4;  // NN K chunk; row padding (doubles)
constexpr int KMAX = 128;                       // rank (rows of the A tile)
constexpr int FM = 4;                           // TN: fragments per warp along A

// NN: 16 rows per warp, NW warps, FN member fragments (MM = 8 FN columns)
template <int NW, int FN>
struct NnShape {
  static constexpr int BI = 16 * NW, MM = 8 * FN, NT = 32 * NW;
  static constexpr int LDW = KMAX + PAD, LDA = BI + PAD;
  static constexpr size_t SMEM = ((size_t)MM * LDW + 2 * (size_t)BK * LDA) * sizeof(double);
};

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

// Split-K partials of C = A^T B for K-contiguous row blocks A (m_tot rows,
// stride lda) and B (nb_tot rows, stride ldb), tiles of KMAX x MM outputs:
// part[z][b * m_tot + a] = sum over CTA z's K-slice of A[a][i] B[b][i]
// (K chunks of TBK through an NST-stage cp.async ring).  blockIdx.y picks
// the tile: (ta, tb) = (y % nta, y / nta), or for a symmetric product
// (A == B, sym = 1) the y-th tile of the upper triangle ta <= tb (the
// reduction mirrors the rest).  The LMP step's W = S^T R is one tile (k x
// M); the cfg5 Nystrom Grams Y^T Y (256 x 256) three.
template <int TBK, int NST, int MM>
__global__ void __launch_bounds__(256, 1)
    k_lmp_tn(const double* __restrict__ A, int64_t lda, const double* __restrict__ B, int64_t ldb, int64_t n,
             int m_tot, int nb_tot, int nchunks, int nta, int sym, double* __restrict__ part) {
  using namespace lmpg;
  constexpr int TLD = TBK + PAD, FN = MM / 16;
  extern __shared__ __align__(16) double sm[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wa = (warp & 3) * 32, wb = (warp >> 2) * (MM / 2);
  int ta, tb;
  if (sym) {  // upper-triangle tile y: row-major over ta <= tb
    int y = blockIdx.y;
    ta = 0;
    while (y >= nta - ta) y -= nta - ta++;
    tb = ta + y;
  } else {
    ta = blockIdx.y % nta;
    tb = blockIdx.y / nta;
  }
  const int a0 = ta * KMAX, b0 = tb * MM;
  const int k = min(KMAX, m_tot - a0), M = min(MM, nb_tot - b0);
  const double* At = A + (int64_t)a0 * lda;
  const double* Bt = B + (int64_t)b0 * ldb;
  // this CTA's chunks [c0, c1) of the K = n dimension (fixed slices)
  const int c0 = (int)((int64_t)nchunks * blockIdx.x / gridDim.x);
  const int c1 = (int)((int64_t)nchunks * (blockIdx.x + 1) / gridDim.x);
  auto sA = [&](int st) { return sm + (size_t)st * (KMAX + MM) * TLD; };
  auto load = [&](int st, int c) {
    const int64_t k0 = (int64_t)c * TBK;
    double* a = sA(st);
    constexpr int PR = TBK / 2;  // 16-byte pairs per row
    constexpr int NP = (KMAX + MM) * PR;
#pragma unroll
    for (int q = 0; q < (NP + 255) / 256; ++q) {
      const int idx = t + q * 256;
      if (NP % 256 && idx >= NP) continue;
      const int row = idx / PR, kk = 2 * (idx % PR);
      const int64_t kg = k0 + kk;
      const int nb = kg < n ? (kg + 1 < n ? 16 : 8) : 0;
      if (row < KMAX) {
        const bool v = row < k;
        cpa16(a + row * TLD + kk, v ? At + kg + (int64_t)row * lda : A, v ? nb : 0);
      } else {
        const int b = row - KMAX;
        const bool v = b < M;
        cpa16(a + row * TLD + kk, v ? Bt + kg + (int64_t)b * ldb : B, v ? nb : 0);
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
  double* P = part + (size_t)blockIdx.x * m_tot * nb_tot + (size_t)b0 * m_tot + a0;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ai = wa + i * 8 + (lane >> 2);
        const int bj = wb + j * 8 + 2 * (lane & 3) + h;
        if (ai < k && bj < M) P[(size_t)bj * m_tot + ai] = acc[i][j][h];
      }
}

// D[b][i] = Cin[b][i] + colscale[b] C2[b][i] + sum_a S[a][i] coef[a] W[b][a]
// (C2 may alias D: every element is read before its own write; Cin, C2
// optional).  NW warps, each 16 rows of the 16 NW-row n-tile x all MM = 8 FN
// member columns (2 x FN fragments): <112, 7 warps> puts 147 CTAs on a
// 16384 ring (cfg4, one per SM), <128, 8 warps> serves 128-member groups
// (cfg5).
template <int NW, int FN>
__global__ void __launch_bounds__(NW * 32, 1)
    k_lmp_nn(const double* __restrict__ S, const double* __restrict__ W, const double* __restrict__ coef, int64_t n,
             int k, int M, const double* __restrict__ Cin, const double* __restrict__ colscale, const double* C2,
             double* D) {
  using namespace lmpg;
  using SH = NnShape<NW, FN>;
  constexpr int NT = SH::NT, FMN = 2, BI = SH::BI, MM = SH::MM, LDW = SH::LDW, LDA = SH::LDA;
  extern __shared__ __align__(16) double sm[];
  double* sW = sm;                          // [MM][LDW]: coef o W, row b
  double* sAbase = sm + (size_t)MM * LDW;   // [2][BK][LDA]: S chunk, row a, n contiguous
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wi = warp * 16;
  const int64_t i0 = (int64_t)blockIdx.x * BI;
  const int nch = (k + BK - 1) / BK;
  auto loadA = [&](int st, int c) {
    double* a = sAbase + (size_t)st * BK * LDA;
    static_assert(BK * BI / 2 % NT == 0, "whole copies per thread");
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
  for (int idx = t; idx < MM * KMAX / 2; idx += NT) {
    const int b = idx / (KMAX / 2), a = 2 * (idx % (KMAX / 2));
    const int nb = b < M ? (a + 1 < k ? 16 : (a < k ? 8 : 0)) : 0;
    cpa16(sW + b * LDW + a, nb ? W + a + (size_t)b * k : W, nb);
  }
  loadA(0, 0);
  wait<0>();
  // scale the resident W rows by coef (each thread its own copies' bytes);
  // coef NULL: W arrives scaled (k_pcg_reduce_rz's prescale)
  if (coef) {
    for (int idx = t; idx < MM * KMAX / 2; idx += NT) {
      const int b = idx / (KMAX / 2), a = 2 * (idx % (KMAX / 2));
      double* w = sW + b * LDW + a;
      w[0] *= a < k ? __ldg(coef + a) : 0.0;
      w[1] *= a + 1 < k ? __ldg(coef + a + 1) : 0.0;
    }
  }
  double acc[FMN][FN][2];
#pragma unroll
  for (int i = 0; i < FMN; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int c = 0; c < nch; ++c) {
    if (c > 0) wait<0>();
    __syncthreads();  // chunk c (and, first, the scaled W) visible; the other stage free
    if (c + 1 < nch) loadA((c + 1) & 1, c + 1);
    const double* a = sAbase + (size_t)(c & 1) * BK * LDA;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double af[FMN], bf[FN];
#pragma unroll
      for (int i = 0; i < FMN; ++i) af[i] = a[(ks + (lane & 3)) * LDA + wi + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < FN; ++j)
        bf[j] = sW[(j * 8 + (lane >> 2)) * LDW + c * BK + ks + (lane & 3)];
#pragma unroll
      for (int i = 0; i < FMN; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  // epilogue, one fragment row at a time: its r operands, then its p
  // operands (just written by the preceding PCG kernels, so L2 hits) are
  // loaded together, combined in the reference's order z = r + S(c o W),
  // p = z + beta p (lmp.py:64-65, krylov.py:95)
  constexpr int FH = FN;
#pragma unroll
  for (int i = 0; i < FMN; ++i) {
    const int64_t gi = i0 + wi + i * 8 + (lane >> 2);
#pragma unroll
    for (int j0 = 0; j0 < FN; j0 += FH) {
      double e[FH][2];
      if (Cin) {
#pragma unroll
        for (int j = 0; j < FH; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gb = (j0 + j) * 8 + 2 * (lane & 3) + h;
            e[j][h] = gi < n && gb < M ? Cin[gi + gb * n] : 0.0;
          }
#pragma unroll
        for (int j = 0; j < FH; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) acc[i][j0 + j][h] += e[j][h];
      }
      if (C2) {  // C2 may alias D: every element is read before its own write
#pragma unroll
        for (int j = 0; j < FH; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gb = (j0 + j) * 8 + 2 * (lane & 3) + h;
            e[j][h] = gi < n && gb < M ? C2[gi + gb * n] : 0.0;
          }
#pragma unroll
        for (int j = 0; j < FH; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gb = (j0 + j) * 8 + 2 * (lane & 3) + h;
            if (gb < M) acc[i][j0 + j][h] += colscale[gb] * e[j][h];
          }
      }
#pragma unroll
      for (int j = 0; j < FH; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gb = (j0 + j) * 8 + 2 * (lane & 3) + h;
          if (gi < n && gb < M) D[gi + gb * n] = acc[i][j0 + j][h];
        }
    }
  }
}

// ------------------------------------------------------------ launchers --
// the member-tile width for a group of M columns: 112 (7 + 7 fragments per
// warp pair, cfg4's 100-member groups) or 128 (cfg5's 128-member groups)
static int lmp_mm(int M) { return M <= 112 ? 112 : 128; }

bool lmp_gemm_ok(int64_t n, int k, int M) {
  const char* e = getenv("EDAK_LMP_GEMM");
  if (e && atoi(e) == 0) return false;
  return k >= 1 && k <= lmpg::KMAX && k % 2 == 0 && M >= 1 && n % 2 == 0 && n >= 4096;
}

// the p-update through k_lmp_nn for member groups of <= 112 (cfg4); wider
// groups take the generic k_gemm_nn: the one-CTA-per-SM 128-member tiles,
// each re-staging the whole 131 KB coef o W, measured 8 ms slower per cfg5
// pass (EDAK_LMP_NN: 0 never, 2 always)
bool lmp_nn_ok(int M) {
  const char* e = getenv("EDAK_LMP_NN");
  const int mode = e ? atoi(e) : 1;
  return mode == 2 || (mode == 1 && M <= 112);
}

// 148 CTAs (one per SM) over the tiles, fewer for short rings
// (EDAK_LMP_TN_CTAS: another CTA budget, A/B)
static int tn_ctas() {
  const char* e = getenv("EDAK_LMP_TN_CTAS");
  const int v = e ? atoi(e) : 148;
  return v >= 1 ? v : 148;
}
static int tn_splits(int64_t n, int tiles) {
  const int64_t nch = (n + 15) / 16;
  int s = tn_ctas() / tiles;
  if (s < 1) s = 1;
  return (int)(nch < s ? nch : s);
}

int64_t lmp_tn_partials(int64_t n, int k, int M) {
  return (int64_t)tn_splits(n, M <= 112 ? 1 : (M + 127) / 128) * k * M;
}

template <int TBK, int NST, int MM>
static int go_tn(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t n, int m_tot, int nb_tot,
                 int nta, int ntiles, int sym, double* part, cudaStream_t st) {
  constexpr size_t smem = (size_t)NST * (lmpg::KMAX + MM) * (TBK + lmpg::PAD) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_lmp_tn<TBK, NST, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int g = tn_splits(n, ntiles);
  const int nch = (int)((n + TBK - 1) / TBK);
  k_lmp_tn<TBK, NST, MM><<<dim3(g, ntiles), 256, smem, st>>>(A, lda, B, ldb, n, m_tot, nb_tot, nch, nta, sym, part);
  count_launch();
  return g;
}

// split-K partials of W = S^T R (layout part[z][b * k + a]) through one
// 112-member k_lmp_tn tile (M <= 112) or ceil(M / 128) 128-member tiles
// sharing the 148 CTAs; returns the split count, or 0 when the generic
// split-K GEMM should run instead (EDAK_LMP_TN: 0 generic, 1 chunks of 32 x
// 3 stages, 2 (default) chunks of 16 x 5)
int launch_lmp_tn(const double* S, const double* R, int64_t n, int k, int M, double* part, cudaStream_t st) {
  const char* e = getenv("EDAK_LMP_TN");  // read per launch (A/B in one process)
  const int mode = e ? atoi(e) : 2;
  if (mode != 1 && mode != 2) return 0;
  if (lmp_mm(M) == 112)
    return mode == 1 ? go_tn<32, 3, 112>(S, n, R, n, n, k, M, 1, 1, 0, part, st)
                     : go_tn<16, 5, 112>(S, n, R, n, n, k, M, 1, 1, 0, part, st);
  return go_tn<16, 5, 128>(S, n, R, n, n, k, M, 1, (M + 127) / 128, 0, part, st);
}

// the big-K Gram / cross products of the Nystrom stage (cfg5: 256 x 256
// over n = 262144) as 128 x 128 k_lmp_tn tiles (the generic 64 x 64
// split-K tiles ran at ~21 TF/s there); symmetric products (A == B) compute
// the upper-triangle tiles only
bool big_tn_ok(const double* A, int64_t lda, const double* B, int64_t ldb, int m, int nb, int64_t K) {
  const char* e = getenv("EDAK_BIG_TN");
  if (e && atoi(e) == 0) return false;
  return m >= 128 && nb >= 128 && K >= 65536 && lda % 2 == 0 && ldb % 2 == 0 && ((uintptr_t)A & 15) == 0 &&
         ((uintptr_t)B & 15) == 0;
}
bool big_tn_sym(const double* A, int64_t lda, const double* B, int64_t ldb, int m, int nb) {
  return A == B && lda == ldb && m == nb;
}
static int big_tn_tiles(int m, int nb, bool sym, int& nta) {
  nta = (m + 127) / 128;
  const int ntb = (nb + 127) / 128;
  return sym ? nta * (nta + 1) / 2 : nta * ntb;
}
int64_t big_tn_partials(int m, int nb, int64_t K) {
  int nta;  // the symmetric product has fewer tiles, so more splits
  const int t = big_tn_tiles(m, nb, m == nb, nta);
  return (int64_t)tn_splits(K, t) * m * nb;
}
int launch_big_tn(const double* A, int64_t lda, const double* B, int64_t ldb, int m, int nb, int64_t K, double* part,
                  cudaStream_t st) {
  const bool sym = big_tn_sym(A, lda, B, ldb, m, nb);
  int nta;
  const int tiles = big_tn_tiles(m, nb, sym, nta);
  return go_tn<16, 5, 128>(A, lda, B, ldb, K, m, nb, nta, tiles, sym ? 1 : 0, part, st);
}

// column blocks of <= 128 members (each column's result is independent of
// its block)
template <int NW, int FN>
static int go_nn(const double* S, const double* W, const double* coef, int64_t n, int k, int M, const double* Cin,
                 const double* colscale, const double* C2, double* D, cudaStream_t st) {
  using SH = lmpg::NnShape<NW, FN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_lmp_nn<NW, FN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SH::SMEM);
    attr = true;
  }
  const unsigned g = (unsigned)((n + SH::BI - 1) / SH::BI);
  for (int c0 = 0; c0 < M; c0 += SH::MM) {
    const int m = M - c0 < SH::MM ? M - c0 : SH::MM;
    const size_t off = (size_t)c0 * n;
    k_lmp_nn<NW, FN><<<g, SH::NT, SH::SMEM, st>>>(S, W + (size_t)c0 * k, coef, n, k, m, Cin ? Cin + off : nullptr,
                                                  colscale ? colscale + c0 : nullptr, C2 ? C2 + off : nullptr,
                                                  D + off);
    count_launch();
  }
  return check_launch("k_lmp_nn");
}

int launch_lmp_nn(const double* S, const double* W, const double* coef, int64_t n, int k, int M, const double* Cin,
                  const double* colscale, const double* C2, double* D, cudaStream_t st) {
  if (lmp_mm(M) == 112) return go_nn<7, 14>(S, W, coef, n, k, M, Cin, colscale, C2, D, st);
  return go_nn<8, 16>(S, W, coef, n, k, M, Cin, colscale, C2, D, st);
}

}  // namespace edak
