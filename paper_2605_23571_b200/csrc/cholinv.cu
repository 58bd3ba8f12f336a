// Blocked Cholesky with the reference shift schedule, fused with the
// triangular inverse, for the (l x l) Gram matrices of the Nystrom stage
// (nystrom.py:67-93 shifted_cholesky; the C^-1 of nystrom.py:129 and the
// R^-1 of every CholeskyQR pass).
//
// One CTA of 256 threads.  The lower factor L (W = L L^T, C = L^T) lives in
// shared memory for l <= CI_SMEM_MAX, else in a global work buffer (L1/L2
// resident at l <= 256).  Right-looking with 32-wide panels:
//   * panel: one warp, warp-synchronous (no block barrier per pivot);
//   * trailing update: all threads, 4x4 register blocks;
//   * dpotrf's breakdown test (pivot <= 0 or NaN) at every pivot.
// The inverse M = L^-1 is formed in place: the 32x32 diagonal blocks by one
// warp each (forward substitution in registers), then block columns from the
// last to the first: M[j+1:, j] = -(M[j+1:, j+1:] L[j+1:, j]) M[j, j].
// Outputs C = L^T and Ci = C^-1 = M^T (column-major, zero lower parts).
#include "common.cuh"
#include <cstdlib>

namespace edak {

constexpr int CI_NT = 256, CI_B = 32, CI_SMEM_MAX = 128;

static __device__ __forceinline__ void tri_index(int b, int& bi, int& bj) {
  // b -> (bi, bj), bi >= bj, row-major over the lower triangle of blocks
  int r = (int)((sqrt(8.0 * b + 1.0) - 1.0) * 0.5);
  while ((r + 1) * (r + 2) / 2 <= b) ++r;
  while (r * (r + 1) / 2 > b) --r;
  bi = r;
  bj = b - r * (r + 1) / 2;
}

__global__ void __launch_bounds__(CI_NT) k_chol_inv(const double* __restrict__ W, int l, double* __restrict__ Cm,
                                                    double* __restrict__ Ci, int mode, double scale,
                                                    double* __restrict__ nu_out, int32_t* __restrict__ info,
                                                    double* __restrict__ gbuf) {
  extern __shared__ __align__(16) double csm[];
  double* A = gbuf ? gbuf : csm;                           // l x l, column-major
  double* Tm = gbuf ? gbuf + (size_t)l * l : csm + (size_t)l * l;  // (l - 32) x 32 temp
  __shared__ int fail;
  __shared__ double red[CI_NT / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double sc = scale;
  if (mode == 1) {  // np.trace(w): sequential, as the old kernels (nu must match bit for bit)
    if (t == 0) {
      double s = 0.0;
      for (int j = 0; j < l; ++j) s += W[j + (size_t)j * l];
      red[0] = s;
    }
    __syncthreads();
    sc = red[0];
  }
  double nu = 0.0;
  int attempt = 0;
  bool ok = false;
  for (; attempt < 6; ++attempt) {
    if (attempt == 1) {
      nu = 2.220446049250313e-16 * sc;
      if (mode == 0 || !(nu > 0.0)) break;
    } else if (attempt > 1) {
      nu *= 10.0;
    }
    // lower triangle from W's upper triangle (dpotrf 'U' reads only it)
    for (int e = t; e < l * l; e += CI_NT) {
      const int i = e % l, j = e / l;
      if (i >= j) A[e] = i == j ? W[j + (size_t)i * l] + nu : W[j + (size_t)i * l];
    }
    if (t == 0) fail = 0;
    __syncthreads();
    for (int kb = 0; kb < l; kb += CI_B) {
      const int nb = min(CI_B, l - kb);
      if (warp == 0) {
        for (int j = kb; j < kb + nb; ++j) {
          const double d = A[j + (size_t)j * l];
          if (!(d > 0.0)) {  // uniform: every lane read the same pivot
            if (lane == 0) fail = 1;
            break;
          }
          const double ljj = sqrt(d);
          const double inv = 1.0 / ljj;
          __syncwarp();
          if (lane == 0) A[j + (size_t)j * l] = ljj;
          for (int i = j + 1 + lane; i < l; i += 32) A[i + (size_t)j * l] *= inv;
          __syncwarp();
          for (int jj = j + 1; jj < kb + nb; ++jj) {
            const double f = A[jj + (size_t)j * l];
            for (int i = jj + lane; i < l; i += 32)
              A[i + (size_t)jj * l] = fma(-A[i + (size_t)j * l], f, A[i + (size_t)jj * l]);
          }
          __syncwarp();
        }
      }
      __syncthreads();
      if (fail) break;
      const int r0 = kb + nb, m = l - r0;
      if (m > 0) {  // A22 -= L21 L21^T (lower), 4x4 register blocks
        const int nbk = (m + 3) / 4, nblk = nbk * (nbk + 1) / 2;
        for (int b = t; b < nblk; b += CI_NT) {
          int bi, bj;
          tri_index(b, bi, bj);
          const int i0 = r0 + 4 * bi, j0 = r0 + 4 * bj;
          double acc[4][4];
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[p][q] = 0.0;
          for (int k = kb; k < kb + nb; ++k) {
            double a[4], c[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              a[p] = i0 + p < l ? A[i0 + p + (size_t)k * l] : 0.0;
              c[p] = j0 + p < l ? A[j0 + p + (size_t)k * l] : 0.0;
            }
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], c[q], acc[p][q]);
          }
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int i = i0 + p, j = j0 + q;
              if (i < l && j < l && i >= j) A[i + (size_t)j * l] -= acc[p][q];
            }
        }
      }
      __syncthreads();
    }
    if (!fail) {
      ok = true;
      break;
    }
    __syncthreads();
  }
  ok = ok && !(attempt >= 1 && mode == 0);
  if (t == 0) {
    info[0] = attempt;
    info[1] = ok ? 0 : 1;
    nu_out[0] = ok ? nu : 0.0;
  }
  // C = L^T (zero strict lower part), also on failure (caller raises)
  for (int e = t; e < l * l; e += CI_NT) {
    const int r = e % l, c = e / l;  // C[r][c], upper: r <= c -> L[c][r]
    Cm[e] = (ok && r <= c) ? A[c + (size_t)r * l] : 0.0;
  }
  if (!Ci) return;
  if (!ok) {
    for (int e = t; e < l * l; e += CI_NT) Ci[e] = 0.0;
    return;
  }
  __syncthreads();
  // diagonal blocks inverted in place, one warp each (lane = column)
  const int nbl = (l + CI_B - 1) / CI_B;
  for (int jb = warp; jb < nbl; jb += CI_NT / 32) {
    const int b0 = jb * CI_B, nb = min(CI_B, l - b0);
    double x[CI_B];
#pragma unroll
    for (int r = 0; r < CI_B; ++r) {
      double v = 0.0;
      if (r < nb && r >= lane && lane < nb) {
        double s = r == lane ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < CI_B; ++k)
          if (k < r && k >= lane) s = fma(-A[b0 + r + (size_t)(b0 + k) * l], x[k], s);
        v = s / A[b0 + r + (size_t)(b0 + r) * l];
      }
      x[r] = v;
    }
    __syncwarp();
    if (lane < nb)
#pragma unroll
      for (int r = 0; r < CI_B; ++r)
        if (r < nb && r >= lane) A[b0 + r + (size_t)(b0 + lane) * l] = x[r];
    __syncwarp();
  }
  __syncthreads();
  // block columns, last to first: M[j+1:, j] = -(M[j+1:, j+1:] L[j+1:, j]) M_jj
  for (int jb = nbl - 2; jb >= 0; --jb) {
    const int b0 = jb * CI_B, nb = CI_B;  // every block but the last is full
    const int r0 = b0 + nb, m = l - r0;
    // Tm[i][c] = sum_{k <= i} M[r0+i][r0+k] L[r0+k][b0+c]
    for (int e = t; e < m * nb; e += CI_NT) {
      const int i = e % m, c = e / m;
      double s = 0.0;
      for (int k = 0; k <= i; ++k) s = fma(A[r0 + i + (size_t)(r0 + k) * l], A[r0 + k + (size_t)(b0 + c) * l], s);
      Tm[i + (size_t)c * m] = s;
    }
    __syncthreads();
    // M[r0+i][b0+c] = -sum_{k >= c} Tm[i][k] M_jj[k][c]
    for (int e = t; e < m * nb; e += CI_NT) {
      const int i = e % m, c = e / m;
      double s = 0.0;
      for (int k = c; k < nb; ++k) s = fma(Tm[i + (size_t)k * m], A[b0 + k + (size_t)(b0 + c) * l], s);
      A[r0 + i + (size_t)(b0 + c) * l] = -s;
    }
    __syncthreads();
  }
  // Ci = M^T (upper)
  for (int e = t; e < l * l; e += CI_NT) {
    const int r = e % l, c = e / l;
    Ci[e] = r <= c ? A[c + (size_t)r * l] : 0.0;
  }
}

// Register-resident variant for l <= 128 (the Nystrom Grams at cfg1-4):
// 1024 threads, thread (warp bj, lane bi) owns the 4x4 block rows 4bi..,
// cols 4bj.. of the lower factor.  A pivot is one shuffle (the diagonal
// lives in the column block's warp), a sqrt, the scaled column written to a
// double-buffered smem vector, ONE barrier and a 4x4 rank-1 update in
// registers; the inverse M = L^-1 runs the same way over rows (L parked in
// shared memory).  ~2l barriers in total, against the panel kernel's
// latency-bound warp-serial panels.
constexpr int CR_MAX = 128;

__global__ void __launch_bounds__(1024) k_chol_inv_reg(const double* __restrict__ W, int l, double* __restrict__ Cm,
                                                       double* __restrict__ Ci, int mode, double scale,
                                                       double* __restrict__ nu_out, int32_t* __restrict__ info) {
  extern __shared__ __align__(16) double crs[];
  double* Ls = crs;                       // l x l lower factor (column-major), for the inverse
  double* vec = crs + CR_MAX * CR_MAX;    // [2][CR_MAX] pivot column / row of M
  double* rdiag = vec + 2 * CR_MAX;       // 1 / L_kk
  __shared__ int fail;
  __shared__ double trace_s;
  const int t = threadIdx.x, bj = t >> 5, bi = t & 31;
  const int r0 = 4 * bi, c0 = 4 * bj;
  const bool live = r0 < l && c0 < l && bi >= bj;  // blocks on/below the diagonal
  if (mode == 1) {
    if (t == 0) {
      double s = 0.0;
      for (int j = 0; j < l; ++j) s += W[j + (size_t)j * l];
      trace_s = s;
    }
    __syncthreads();
  }
  const double sc = mode == 1 ? trace_s : scale;
  double nu = 0.0;
  int attempt = 0;
  bool ok = false;
  double a[4][4];
  for (; attempt < 6; ++attempt) {
    if (attempt == 1) {
      nu = 2.220446049250313e-16 * sc;
      if (mode == 0 || !(nu > 0.0)) break;
    } else if (attempt > 1) {
      nu *= 10.0;
    }
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = r0 + p, k = c0 + q;
        double v = 0.0;
        if (live && i < l && k < l && i >= k) v = W[k + (size_t)i * l] + (i == k ? nu : 0.0);  // W's upper
        a[p][q] = v;
      }
    if (t == 0) fail = 0;
    __syncthreads();
    for (int j = 0; j < l; ++j) {
      const int jb = j >> 2, jq = j & 3, buf = j & 1;
      double* colj = vec + buf * CR_MAX;
      if (bj == jb) {  // the pivot column's warp: diagonal from lane jb
        double dloc = 0.0;
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (p == jq && q == jq) dloc = a[p][q];
        const double d = __shfl_sync(0xffffffffu, dloc, jb);
        if (!(d > 0.0)) {
          if (bi == 0) fail = 1;
        } else {
          const double piv = sqrt(d);
          const double inv = 1.0 / piv;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const int i = r0 + p;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q == jq && live && i >= j && i < l) {
                const double v = i == j ? piv : a[p][q] * inv;
                a[p][q] = v;
                colj[i] = v;
              }
          }
        }
      }
      __syncthreads();
      if (fail) break;
      // rank-1 update of the trailing lower triangle: a[i][k] -= l_ij l_kj
      if (live && c0 + 3 > j) {
        double ci[4], ck[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          ci[p] = (r0 + p > j && r0 + p < l) ? colj[r0 + p] : 0.0;
          ck[p] = (c0 + p > j && c0 + p < l) ? colj[c0 + p] : 0.0;
        }
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) a[p][q] = fma(-ci[p], ck[q], a[p][q]);
      }
    }
    __syncthreads();
    if (!fail) {
      ok = true;
      break;
    }
  }
  ok = ok && !(attempt >= 1 && mode == 0);
  if (t == 0) {
    info[0] = attempt;
    info[1] = ok ? 0 : 1;
    nu_out[0] = ok ? nu : 0.0;
  }
  // C = L^T; L parked in smem for the inverse
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = r0 + p, k = c0 + q;  // L[i][k], i >= k: each C entry written once
      if (i < l && k < l && i >= k) {
        const double v = ok ? a[p][q] : 0.0;
        Cm[k + (size_t)i * l] = v;                 // C[k][i] = L[i][k]
        if (i != k) Cm[i + (size_t)k * l] = 0.0;   // strict lower part of C
        Ls[i + (size_t)k * l] = v;
      }
    }
  if (!Ci) return;
  if (!ok) {
    for (int e = t; e < l * l; e += 1024) Ci[e] = 0.0;
    return;
  }
  for (int k = t; k < l; k += 1024) rdiag[k] = 0.0;
  __syncthreads();
  for (int k = t; k < l; k += 1024) rdiag[k] = 1.0 / Ls[k + (size_t)k * l];
  // M = L^-1 by rows: R = I; for k: M[k][:] = R[k][:] / L_kk, then
  // R[i][:] -= L[i][k] M[k][:] for i > k.  Same block ownership.
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) a[p][q] = (live && r0 + p == c0 + q && r0 + p < l) ? 1.0 : 0.0;
  __syncthreads();
  for (int k = 0; k < l; ++k) {
    const int kb = k >> 2, kp = k & 3;
    double* rowk = vec + (k & 1) * CR_MAX;
    if (bi == kb && live) {  // row k's owners: scale and publish
      const double rd = rdiag[k];
#pragma unroll
      for (int p = 0; p < 4; ++p)
        if (p == kp)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = c0 + q;
            if (c <= k && c < l) {
              const double v = a[p][q] * rd;
              a[p][q] = v;
              rowk[c] = v;
            }
          }
    }
    __syncthreads();
    if (live && r0 + 3 > k && c0 <= k) {
      double li[4], mk[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) li[p] = (r0 + p > k && r0 + p < l) ? Ls[r0 + p + (size_t)k * l] : 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) mk[q] = (c0 + q <= k && c0 + q < l) ? rowk[c0 + q] : 0.0;
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) a[p][q] = fma(-li[p], mk[q], a[p][q]);
    }
  }
  // Ci = M^T (upper): Ci[k][i] = M[i][k]
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = r0 + p, k = c0 + q;
      if (i < l && k < l && i >= k) {
        Ci[k + (size_t)i * l] = a[p][q];          // Ci[k][i] = M[i][k]
        if (i != k) Ci[i + (size_t)k * l] = 0.0;
      }
    }
}

int64_t chol_inv_work_doubles(int l) { return l <= CI_SMEM_MAX ? 0 : (int64_t)l * l + (int64_t)l * CI_B; }

int launch_chol_inv(const double* W, int l, double* C, double* Ci, int mode, double scale, double* nu_out,
                    int32_t* info, double* work, cudaStream_t st) {
  if (l < 1) {
    set_error("chol_inv: l < 1");
    return EDAK_EINVAL;
  }
  if (l <= CR_MAX && !getenv("EDAK_CHOL_PANEL")) {
    constexpr size_t crs = ((size_t)CR_MAX * CR_MAX + 3 * CR_MAX) * sizeof(double);
    static bool attr_r = false;
    if (!attr_r) {
      cudaFuncSetAttribute(k_chol_inv_reg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)crs);
      attr_r = true;
    }
    k_chol_inv_reg<<<1, 1024, crs, st>>>(W, l, C, Ci, mode, scale, nu_out, info);
    count_launch();
    return check_launch("k_chol_inv_reg");
  }
  size_t sm = 0;
  if (l <= CI_SMEM_MAX) {
    sm = ((size_t)l * l + (size_t)l * CI_B) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_chol_inv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (CI_SMEM_MAX * CI_SMEM_MAX + CI_SMEM_MAX * CI_B) * (int)sizeof(double));
      attr = true;
    }
    work = nullptr;
  } else if (!work) {
    set_error("chol_inv: work buffer required for l > 128");
    return EDAK_EINVAL;
  }
  k_chol_inv<<<1, CI_NT, sm, st>>>(W, l, C, Ci, mode, scale, nu_out, info, work);
  count_launch();
  return check_launch("k_chol_inv");
}

}  // namespace edak
