// Batched PCG across ensemble members (krylov.pcg, krylov.py:49-97).
// One CTA per member column; every reduction is a fixed-order block tree
// (deterministic).  Per-member status mirrors the reference control flow:
//   0 running, 1 stopped ("converged": rz_new <= 0 or residual_rtol met,
//   krylov.py:90-93), 2 breakdown (p.Hp <= 0 -> the reference raises
//   "system matrix is not positive definite (iteration it)", krylov.py:82-84),
//   3 preconditioner not positive definite (krylov.py:73-74).
// The cost trace J(x_it) (krylov.py:108-113 with assim.py:79-82) is carried
// by linearity: m_it = G U_B x_it = m_{it-1} + alpha * (G U_B p), where
// G U_B p is the raw TL observation vector the Hessian apply already made.
#include "common.cuh"

namespace edak {

constexpr int PCG_NT = 256;

__global__ void __launch_bounds__(PCG_NT) k_pcg_init(int n, const double* __restrict__ b,
                                                     const double* __restrict__ z, double* __restrict__ x,
                                                     double* __restrict__ r, double* __restrict__ p,
                                                     double* __restrict__ rz, double* __restrict__ hist_rz,
                                                     int hist_ld, int32_t* __restrict__ status,
                                                     int32_t* __restrict__ iters) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  const size_t o = (size_t)c * n;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += PCG_NT) {
    const double bi = b[o + i], zi = z[o + i];
    x[o + i] = 0.0;
    r[o + i] = bi;
    p[o + i] = zi;
    s += bi * zi;
  }
  s = block_sum<PCG_NT>(s, sh);
  if (threadIdx.x == 0) {
    rz[c] = s;
    hist_rz[(size_t)c * hist_ld] = s;
    status[c] = s < 0.0 ? 3 : 0;
    iters[c] = 0;
  }
}

// php = p.hp; breakdown check; alpha; x += alpha p; r -= alpha hp; cost.
__global__ void __launch_bounds__(PCG_NT) k_pcg_alpha(int n, const double* __restrict__ p,
                                                      const double* __restrict__ hp, double* __restrict__ x,
                                                      double* __restrict__ r, const double* __restrict__ rz,
                                                      int32_t* __restrict__ status, int32_t* __restrict__ iters,
                                                      int it, int np_obs, const double* __restrict__ gp,
                                                      double* __restrict__ m, const double* __restrict__ d,
                                                      double sigma2, double* __restrict__ hist_J, int hist_ld) {
  __shared__ double sh[32];
  __shared__ double s_alpha;
  __shared__ int s_stop;
  const int c = blockIdx.x;
  if (status[c] != 0) return;
  const size_t o = (size_t)c * n;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += PCG_NT) s += p[o + i] * hp[o + i];
  s = block_sum<PCG_NT>(s, sh);
  if (threadIdx.x == 0) {
    s_stop = s <= 0.0;  // krylov.py:82 (NaN does not raise)
    if (s_stop) {
      status[c] = 2;
      iters[c] = it;
    }
    s_alpha = rz[c] / s;
  }
  __syncthreads();
  if (s_stop) return;
  const double alpha = s_alpha;
  double xx = 0.0;
  for (int i = threadIdx.x; i < n; i += PCG_NT) {
    const double xi = x[o + i] + alpha * p[o + i];
    x[o + i] = xi;
    r[o + i] = r[o + i] - alpha * hp[o + i];
    xx += xi * xi;
  }
  if (hist_J) {
    double mm = 0.0;
    const size_t q0 = (size_t)c * np_obs;
    for (int q = threadIdx.x; q < np_obs; q += PCG_NT) {
      const double mq = m[q0 + q] + alpha * gp[q0 + q];
      m[q0 + q] = mq;
      const double e = mq - d[q0 + q];
      mm += e * (e / sigma2);
    }
    xx = block_sum<PCG_NT>(xx, sh);
    mm = block_sum<PCG_NT>(mm, sh);
    if (threadIdx.x == 0) hist_J[(size_t)c * hist_ld + it] = 0.5 * xx + 0.5 * mm;
  }
}

// rz_new = r.z; record; stop test; p = z + (rz_new / rz) p
__global__ void __launch_bounds__(PCG_NT) k_pcg_beta(int n, const double* __restrict__ z,
                                                     const double* __restrict__ r, double* __restrict__ p,
                                                     double* __restrict__ rz, 
                                                     double rtol, double* __restrict__ hist_rz, int hist_ld,
                                                     int32_t* __restrict__ status, int32_t* __restrict__ iters,
                                                     int it) {
  __shared__ double sh[32];
  __shared__ int s_stop;
  __shared__ double s_beta;
  const int c = blockIdx.x;
  if (status[c] != 0) return;
  const size_t o = (size_t)c * n;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += PCG_NT) s += r[o + i] * z[o + i];
  s = block_sum<PCG_NT>(s, sh);
  if (threadIdx.x == 0) {
    hist_rz[(size_t)c * hist_ld + it] = s;
    iters[c] = it;
    const bool stop = s <= 0.0 || (rtol >= 0.0 && sqrt(s) <= rtol * sqrt(hist_rz[(size_t)c * hist_ld]));
    s_stop = stop;
    if (stop) status[c] = 1;
    s_beta = s / rz[c];
    if (!stop) rz[c] = s;
  }
  __syncthreads();
  if (s_stop) return;
  const double beta = s_beta;
  for (int i = threadIdx.x; i < n; i += PCG_NT) p[o + i] = z[o + i] + beta * p[o + i];
}

// initial cost J(0) = 1/2 d.R^-1 d  (misfit = -d, assim.py:81-82) and m = 0
__global__ void __launch_bounds__(PCG_NT) k_pcg_cost0(int np_obs, const double* __restrict__ d,
                                                      double* __restrict__ m, double sigma2,
                                                      double* __restrict__ hist_J, int hist_ld) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  const size_t q0 = (size_t)c * np_obs;
  double mm = 0.0;
  for (int q = threadIdx.x; q < np_obs; q += PCG_NT) {
    m[q0 + q] = 0.0;
    const double e = -d[q0 + q];
    mm += e * (e / sigma2);
  }
  mm = block_sum<PCG_NT>(mm, sh);
  if (threadIdx.x == 0) hist_J[(size_t)c * hist_ld] = 0.5 * mm;
}

int launch_pcg_init(int n, int ncols, const double* b, const double* z, double* x, double* r, double* p, double* rz,
                    double* hist_rz, int hist_ld, int32_t* status, int32_t* iters, cudaStream_t st) {
  k_pcg_init<<<ncols, PCG_NT, 0, st>>>(n, b, z, x, r, p, rz, hist_rz, hist_ld, status, iters);
  count_launch();
  return check_launch("k_pcg_init");
}

int launch_pcg_alpha(int n, int ncols, const double* p, const double* hp, double* x, double* r, const double* rz,
                     int32_t* status, int32_t* iters, int it, int np_obs, const double* gp, double* m,
                     const double* d, double sigma2, double* hist_J, int hist_ld, cudaStream_t st) {
  k_pcg_alpha<<<ncols, PCG_NT, 0, st>>>(n, p, hp, x, r, rz, status, iters, it, np_obs, gp, m, d, sigma2, hist_J,
                                        hist_ld);
  count_launch();
  return check_launch("k_pcg_alpha");
}

int launch_pcg_beta(int n, int ncols, const double* z, const double* r, double* p, double* rz, double rtol, double* hist_rz, int hist_ld, int32_t* status, int32_t* iters, int it,
                    cudaStream_t st) {
  k_pcg_beta<<<ncols, PCG_NT, 0, st>>>(n, z, r, p, rz, rtol, hist_rz, hist_ld, status, iters, it);
  count_launch();
  return check_launch("k_pcg_beta");
}

int launch_pcg_cost0(int np_obs, int ncols, const double* d, double* m, double sigma2, double* hist_J, int hist_ld,
                     cudaStream_t st) {
  k_pcg_cost0<<<ncols, PCG_NT, 0, st>>>(np_obs, d, m, sigma2, hist_J, hist_ld);
  count_launch();
  return check_launch("k_pcg_cost0");
}

// quadratic_cost reduction: J = 1/2 z.z + 1/2 sum (o - d) ((o - d)/sigma2)
__global__ void __launch_bounds__(PCG_NT) k_cost(int n, int np_obs, const double* __restrict__ z,
                                                 const double* __restrict__ obs, const double* __restrict__ d,
                                                 double sigma2, double* __restrict__ J) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  double zz = 0.0, mm = 0.0;
  for (int i = threadIdx.x; i < n; i += PCG_NT) {
    const double v = z[(size_t)c * n + i];
    zz += v * v;
  }
  for (int q = threadIdx.x; q < np_obs; q += PCG_NT) {
    const double e = obs[(size_t)c * np_obs + q] - d[(size_t)c * np_obs + q];
    mm += e * (e / sigma2);
  }
  zz = block_sum<PCG_NT>(zz, sh);
  mm = block_sum<PCG_NT>(mm, sh);
  if (threadIdx.x == 0) J[c] = 0.5 * zz + 0.5 * mm;
}

int launch_cost(int n, int np_obs, int ncols, const double* z, const double* obs, const double* d, double sigma2,
                double* J, cudaStream_t st) {
  k_cost<<<ncols, PCG_NT, 0, st>>>(n, np_obs, z, obs, d, sigma2, J);
  count_launch();
  return check_launch("k_cost");
}

}  // namespace edak
