// Small dense (l x l, l <= 256) stages of the randomized Nystrom EVD, each a
// single CTA working out of L2 (nystrom.py:67-93,118-131):
//   k_potrf_shifted : upper Cholesky with the reference's shift schedule
//   k_trinv_upper   : explicit inverse of an upper-triangular factor
//   k_svd_jacobi    : one-sided (Hestenes) Jacobi SVD, descending order
#include "common.cuh"
#include <cstdlib>

namespace edak {

// Upper Cholesky W = C^T C reading W's upper triangle (scipy.linalg.cholesky
// lower=False -> LAPACK dpotrf 'U').  Breakdown test is dpotrf's: a pivot
// that is <= 0 or NaN.  Schedule (nystrom.py:77-93): plain; then if mode != 0
// nu = eps * scale (scale = trace(W) when mode == 1, else `scale`), up to 5
// tries with nu *= 10.
__global__ void __launch_bounds__(256) k_potrf_shifted(const double* __restrict__ W, int l, double* __restrict__ Cm,
                                                       int mode, double scale, double* nu_out, int32_t* info) {
  __shared__ double sh[32];
  __shared__ int fail;
  __shared__ double cjj;
  const int t = threadIdx.x;
  double sc = scale;
  if (mode == 1) {  // np.trace(w)
    sc = 0.0;
    for (int j = 0; j < l; ++j) sc += W[j + (size_t)j * l];
  }
  double nu = 0.0;
  int attempt = 0;
  for (; attempt < 6; ++attempt) {
    if (attempt == 1) {
      nu = 2.220446049250313e-16 * sc;
      if (mode == 0 || !(nu > 0.0)) break;
    } else if (attempt > 1) {
      nu *= 10.0;
    }
    if (t == 0) fail = 0;
    __syncthreads();
    for (int j = 0; j < l && !fail; ++j) {
      // pivot: (W[j][j] + nu) - sum_{k<j} C[k][j]^2
      double s = 0.0;
      for (int k = t; k < j; k += 256) {
        const double c = Cm[k + (size_t)j * l];
        s += c * c;
      }
      s = block_sum<256>(s, sh);
      if (t == 0) {
        const double d = (W[j + (size_t)j * l] + nu) - s;
        if (!(d > 0.0)) {
          fail = 1;
        } else {
          cjj = sqrt(d);
          Cm[j + (size_t)j * l] = cjj;
        }
      }
      __syncthreads();
      if (fail) break;
      const double piv = cjj;
      // row j of C: C[j][i] = (W[j][i] - sum_k C[k][j] C[k][i]) / C[j][j]
      for (int i = j + 1 + t; i < l; i += 256) {
        double acc = W[j + (size_t)i * l];
        const double* cj = Cm + (size_t)j * l;
        const double* ci = Cm + (size_t)i * l;
        for (int k = 0; k < j; ++k) acc -= cj[k] * ci[k];
        Cm[j + (size_t)i * l] = acc / piv;
      }
      // zero the strict lower part of column j
      for (int i = j + 1 + t; i < l; i += 256) Cm[i + (size_t)j * l] = 0.0;
      __syncthreads();
    }
    __syncthreads();
    if (!fail) break;
  }
  if (t == 0) {
    const bool ok = attempt < 6 && !fail && !(attempt >= 1 && mode == 0);
    info[0] = attempt;
    info[1] = ok ? 0 : 1;
    nu_out[0] = ok ? nu : 0.0;
  }
}

// Right-looking variant entirely in shared memory (l <= 128): per pivot one
// scaled row and one parallel rank-1 update of the trailing upper triangle;
// same breakdown test and shift schedule as k_potrf_shifted.
constexpr int POTRF_SMEM_MAX = 128;

__global__ void __launch_bounds__(1024) k_potrf_smem(const double* __restrict__ W, int l, double* __restrict__ Cm,
                                                     int mode, double scale, double* nu_out, int32_t* info) {
  extern __shared__ __align__(16) double psm[];
  double* A = psm;            // l x l, column-major, upper triangle live
  double* row = psm + l * l;  // row j of C
  __shared__ int fail;
  const int t = threadIdx.x, NT = blockDim.x;
  double sc = scale;
  if (mode == 1) {  // np.trace(w)
    sc = 0.0;
    for (int j = 0; j < l; ++j) sc += W[j + (size_t)j * l];
  }
  double nu = 0.0;
  int attempt = 0;
  for (; attempt < 6; ++attempt) {
    if (attempt == 1) {
      nu = 2.220446049250313e-16 * sc;
      if (mode == 0 || !(nu > 0.0)) break;
    } else if (attempt > 1) {
      nu *= 10.0;
    }
    for (int e = t; e < l * l; e += NT) {
      const int r = e % l, c = e / l;
      A[e] = r <= c ? W[e] + (r == c ? nu : 0.0) : 0.0;
    }
    if (t == 0) fail = 0;
    __syncthreads();
    for (int j = 0; j < l; ++j) {
      const double d = A[j + j * l];
      if (!(d > 0.0)) {  // dpotrf: pivot <= 0 or NaN
        if (t == 0) fail = 1;
        break;
      }
      const double cjj = sqrt(d);
      for (int c = j + t; c < l; c += NT) row[c] = c == j ? cjj : A[j + c * l] / cjj;
      __syncthreads();
      const int m = l - j - 1;
      for (int e = t; e < m * m; e += NT) {
        const int r = j + 1 + e % m, c = j + 1 + e / m;
        if (r <= c) A[r + c * l] -= row[r] * row[c];
      }
      for (int c = j + t; c < l; c += NT) A[j + c * l] = row[c];  // row j of C is final
      __syncthreads();
    }
    __syncthreads();
    if (!fail) break;
  }
  const bool ok = attempt < 6 && !fail && !(attempt >= 1 && mode == 0);
  if (ok)
    for (int e = t; e < l * l; e += NT) {
      const int r = e % l, c = e / l;
      Cm[e] = r <= c ? A[e] : 0.0;
    }
  if (t == 0) {
    info[0] = attempt;
    info[1] = ok ? 0 : 1;
    nu_out[0] = ok ? nu : 0.0;
  }
}

int launch_potrf_shifted(const double* W, int l, double* C, int mode, double scale, double* nu_out, int32_t* info,
                         cudaStream_t st) {
  if (l <= POTRF_SMEM_MAX) {
    const size_t sm = (size_t)(l * l + l) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_potrf_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (POTRF_SMEM_MAX * POTRF_SMEM_MAX + POTRF_SMEM_MAX) * (int)sizeof(double));
      attr = true;
    }
    k_potrf_smem<<<1, 1024, sm, st>>>(W, l, C, mode, scale, nu_out, info);
    count_launch();
    return check_launch("k_potrf_smem");
  }
  k_potrf_shifted<<<1, 256, 0, st>>>(W, l, C, mode, scale, nu_out, info);
  count_launch();
  return check_launch("k_potrf_shifted");
}

// Rinv = R^-1, R upper triangular: one thread per column, back substitution.
__global__ void k_trinv_upper(const double* __restrict__ R, int l, double* __restrict__ X) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= l) return;
  double* x = X + (size_t)j * l;
  for (int i = l - 1; i > j; --i) x[i] = 0.0;
  x[j] = 1.0 / R[j + (size_t)j * l];
  for (int i = j - 1; i >= 0; --i) {
    double s = 0.0;
    for (int k = i + 1; k <= j; ++k) s += R[i + (size_t)k * l] * x[k];
    x[i] = -s / R[i + (size_t)i * l];
  }
}

// Shared-memory variant (l <= 128): rows of X = R^-1 from the bottom up,
// X[i][c] = -(1/R_ii) sum_{k=i+1..c} R[i][k] X[k][c], one thread per column c.
__global__ void __launch_bounds__(128) k_trinv_smem(const double* __restrict__ R, int l, double* __restrict__ X) {
  extern __shared__ __align__(16) double tsm[];
  const double* Rs = R;  // read as warp-wide broadcasts (L1)
  double* Xs = tsm;      // column-major l x l
  const int t = threadIdx.x;
  for (int e = t; e < l * l; e += blockDim.x) Xs[e] = 0.0;
  __syncthreads();
  for (int i = l - 1; i >= 0; --i) {
    const double rii = Rs[i + i * l];
    for (int c = i + t; c < l; c += blockDim.x) {
      if (c == i) {
        Xs[i + c * l] = 1.0 / rii;
      } else {
        double s = 0.0;
        for (int k = i + 1; k <= c; ++k) s += Rs[i + k * l] * Xs[k + c * l];
        Xs[i + c * l] = -s / rii;
      }
    }
    __syncthreads();
  }
  for (int e = t; e < l * l; e += blockDim.x) X[e] = Xs[e];
}

int launch_trinv_upper(const double* R, int l, double* X, cudaStream_t st) {
  if (l <= POTRF_SMEM_MAX) {
    const size_t sm = (size_t)l * l * sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_trinv_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           POTRF_SMEM_MAX * POTRF_SMEM_MAX * (int)sizeof(double));
      attr = true;
    }
    k_trinv_smem<<<1, 128, sm, st>>>(R, l, X);
    count_launch();
    return check_launch("k_trinv_smem");
  }
  k_trinv_upper<<<(l + 127) / 128, 128, 0, st>>>(R, l, X);
  count_launch();
  return check_launch("k_trinv_upper");
}

// One-sided Jacobi SVD of M (rows x cols, rows >= cols, column-major).
// work: rows*cols (A) + cols*cols (V) + cols doubles.  Outputs, sorted by
// descending singular value: U (rows x cols, unit columns or 0), sig (cols),
// V (cols x cols) if Vout != NULL.
constexpr int JAC_NT = 1024;

// 1/x to full double precision: hardware reciprocal seed + two Newton steps
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// smem_mode: 0 = everything in the global workspace (L2); 1 = A in shared
// memory; 2 = A and V in shared memory (l <= 128 fits: 128 KB)
__global__ void __launch_bounds__(JAC_NT) k_svd_jacobi(const double* __restrict__ M, int rows, int cols,
                                                       double* __restrict__ U, double* __restrict__ sig,
                                                       double* __restrict__ Vout, double* __restrict__ work,
                                                       int smem_mode) {
  __shared__ int rotated;
  extern __shared__ __align__(16) double jsm[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = JAC_NT / 32;
  double* A = smem_mode >= 1 ? jsm : work;
  double* V = smem_mode >= 2 ? jsm + (size_t)rows * cols : work + (size_t)rows * cols;
  double* nrm = work + (size_t)rows * cols + (size_t)cols * cols;
  for (size_t e = t; e < (size_t)rows * cols; e += JAC_NT) A[e] = M[e];
  if (Vout)
    for (size_t e = t; e < (size_t)cols * cols; e += JAC_NT) V[e] = (e % cols == e / cols) ? 1.0 : 0.0;
  __syncthreads();
  const int m = cols + (cols & 1);  // even tournament size (index `cols` = dummy)
  // LAPACK dgesvj's convergence threshold: sqrt(rows) * eps (squared)
  const double tol2 = (double)rows * 2.220446049250313e-16 * 2.220446049250313e-16;
  // one half-warp (16 lanes) per column pair: 64 pairs in flight per pass.
  // Both halves of a warp always run the same loop trip count (shuffles use
  // the full mask); idle halves carry live = false.
  const int hl = t & 15, half = (t >> 4) & 1;
  // squared column norms, recomputed at every sweep start and tracked
  // through the rotations in between (al' = al - t ga, be' = be + t ga), so a
  // pair costs one dot instead of three; the rotation parameters are
  // evaluated once per pair (lane 0 of the half-warp) and broadcast
  double* n2 = nrm;  // cols entries (the final norms reuse it afterwards)
  int sweep = 0;
  for (; sweep < 40; ++sweep) {
    for (int j = warp; j < cols; j += nw) {
      double s2 = 0.0;
      const double* a = A + (size_t)j * rows;
      for (int i = lane; i < rows; i += 32) s2 = fma(a[i], a[i], s2);
      s2 = warp_sum(s2);
      if (lane == 0) n2[j] = s2;
    }
    if (t == 0) rotated = 0;
    __syncthreads();
    for (int rd = 0; rd < m - 1; ++rd) {
      for (int k0 = warp * 2; k0 < m / 2; k0 += nw * 2) {
        const int k = k0 + half;
        int p = 0, q = 0;
        bool live = k < m / 2;
        if (live) {
          if (k != 0) {
            p = k - 1 + rd;
            p = (p >= m - 1 ? p - (m - 1) : p) + 1;
          }
          q = m - 2 - k + rd;
          q = (q >= m - 1 ? q - (m - 1) : q) + 1;
          if (p > q) { int tmp = p; p = q; q = tmp; }
          live = q < cols && p != q;
        }
        double* ap = A + (size_t)p * rows;
        double* aq = A + (size_t)q * rows;
        double ga = 0.0;
        if (live) {
          double g2 = 0.0;
          int i = hl;
          for (; i + 16 < rows; i += 32) {  // two chains
            ga = fma(ap[i], aq[i], ga);
            g2 = fma(ap[i + 16], aq[i + 16], g2);
          }
          if (i < rows) ga = fma(ap[i], aq[i], ga);
          ga += g2;
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) ga += __shfl_xor_sync(0xffffffffu, ga, o);
        double c = 1.0, sn = 0.0, tt = 0.0;
        bool rot = false;
        if (live && hl == 0) {
          const double al = n2[p], be = n2[q];
          // threshold without square roots: |ga| <= tol sqrt(al be)
          rot = al > 0.0 && be > 0.0 && ga * ga > tol2 * (al * be);
          if (rot) {
            // rotation from reciprocals refined by Newton steps instead of
            // IEEE division / sqrt (the angle only has to be accurate to a
            // few ulps; this is the serial part of every Jacobi round)
            const double zeta = (be - al) * fast_rcp(2.0 * ga);
            const double z2 = fma(zeta, zeta, 1.0);
            const double sq = z2 * rsqrt(z2);  // sqrt(1 + zeta^2)
            tt = copysign(fast_rcp(fabs(zeta) + sq), zeta);
            c = rsqrt(fma(tt, tt, 1.0));
            sn = c * tt;
            n2[p] = fma(-tt, ga, al);
            n2[q] = fma(tt, ga, be);
            rotated = 1;
          }
        }
        const int src = half * 16;
        rot = __shfl_sync(0xffffffffu, rot, src);
        c = __shfl_sync(0xffffffffu, c, src);
        sn = __shfl_sync(0xffffffffu, sn, src);
        if (!rot) continue;
        for (int i = hl; i < rows; i += 16) {
          const double x = ap[i], y = aq[i];
          ap[i] = c * x - sn * y;
          aq[i] = sn * x + c * y;
        }
        if (Vout) {
          double* vp = V + (size_t)p * cols;
          double* vq = V + (size_t)q * cols;
          for (int i = hl; i < cols; i += 16) {
            const double x = vp[i], y = vq[i];
            vp[i] = c * x - sn * y;
            vq[i] = sn * x + c * y;
          }
        }
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  if (t == 0) work[(size_t)rows * cols + (size_t)cols * cols + cols] = (double)(sweep + 1);  // diagnostics
  // column norms
  for (int j = warp; j < cols; j += nw) {
    double s = 0.0;
    const double* a = A + (size_t)j * rows;
    for (int i = lane; i < rows; i += 32) s += a[i] * a[i];
    s = warp_sum(s);
    if (lane == 0) nrm[j] = sqrt(s);
  }
  __syncthreads();
  // rank by descending norm (ties by index), scatter
  for (int j = warp; j < cols; j += nw) {
    const double sj = nrm[j];
    int rank = 0;
    for (int i = lane; i < cols; i += 32) {
      const double si = nrm[i];
      rank += (si > sj || (si == sj && i < j)) ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    const double* a = A + (size_t)j * rows;
    double* u = U + (size_t)rank * rows;
    for (int i = lane; i < rows; i += 32) u[i] = a[i] * inv;
    if (Vout) {
      const double* v = V + (size_t)j * cols;
      double* vo = Vout + (size_t)rank * cols;
      for (int i = lane; i < cols; i += 32) vo[i] = v[i];
    }
    if (lane == 0) sig[rank] = sj;
  }
}

int launch_svd_jacobi_cluster(const double*, int, int, double*, double*, double*, double*, cudaStream_t);

int64_t svd_work_doubles(int rows, int cols) { return (int64_t)rows * cols + (int64_t)cols * cols + cols + 1; }

int launch_svd_jacobi(const double* M, int rows, int cols, double* U, double* sig, double* V, double* work,
                      cudaStream_t st) {
  if (rows < cols) {
    set_error("svd_jacobi needs rows >= cols");
    return EDAK_EINVAL;
  }
  const size_t a_bytes = (size_t)rows * cols * sizeof(double);
  const size_t v_bytes = (size_t)cols * cols * sizeof(double);
  const size_t limit = 200 * 1024;
  int mode = 0;
  size_t smem = 0;
  if (a_bytes + (V ? v_bytes : 0) <= limit) {
    mode = 2;
    smem = a_bytes + (V ? v_bytes : 0);
  } else if (a_bytes <= limit) {
    mode = 1;
    smem = a_bytes;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_svd_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)limit);
    attr = true;
  }
  if (!getenv("EDAK_JACOBI_SINGLE")) {  // 8-SM cluster variant (jacobi_cluster.cu)
    const int rc = launch_svd_jacobi_cluster(M, rows, cols, U, sig, V, work, st);
    if (rc >= 0) return rc;
  }
  k_svd_jacobi<<<1, JAC_NT, smem, st>>>(M, rows, cols, U, sig, V, work, mode);
  count_launch();
  return check_launch("k_svd_jacobi");
}

}  // namespace edak
