// Batched PCG across ensemble members (krylov.pcg, krylov.py:49-97).
// Grid = (2048-element tiles) x members; every reduction is a fixed-order
// tree over tile partials that each CTA recomputes identically (deterministic,
// no atomics, no inter-CTA races).  Per-member status mirrors the reference control flow:
//   0 running, 1 stopped ("converged": rz_new <= 0 or residual_rtol met,
//   krylov.py:90-93), 2 breakdown (p.Hp <= 0 -> the reference raises
//   "system matrix is not positive definite (iteration it)", krylov.py:82-84),
//   3 preconditioner not positive definite (krylov.py:73-74).
// The cost trace J(x_it) (krylov.py:108-113 with assim.py:79-82) comes from
// the J identity J(x) = J(0) - 1/2 x.(b + r) (no extra TL sweep).
#include "common.cuh"

namespace edak {

constexpr int PCG_NT = 256;
constexpr int PCG_EPT = 8;                   // elements per thread per tile
constexpr int PCG_TILE = PCG_NT * PCG_EPT;   // 2048 ring elements per CTA

static inline int pcg_tiles(int n) { return (n + PCG_TILE - 1) / PCG_TILE; }

// fixed-order sum of a member's T tile partials: every CTA that needs the
// value computes it identically (lane-strided then a fixed xor tree)
__device__ __forceinline__ double sum_parts(const double* __restrict__ part, int T) {
  double s = 0.0;
  for (int u = threadIdx.x & 31; u < T; u += 32) s += part[u];
  return warp_sum(s);
}

// part[c*T + t] = sum over tile t of a[c][i] * b[c][i]
__global__ void __launch_bounds__(PCG_NT) k_dot_partial(int n, int T, const double* __restrict__ a,
                                                        const double* __restrict__ b, double* __restrict__ part) {
  __shared__ double sh[32];
  const int c = blockIdx.y, t = blockIdx.x;
  const size_t o = (size_t)c * n;
  const int i0 = t * PCG_TILE;
  const int i1 = min(n, i0 + PCG_TILE);
  double s = 0.0;
  for (int i = i0 + threadIdx.x; i < i1; i += PCG_NT) s += a[o + i] * b[o + i];
  s = block_sum<PCG_NT>(s, sh);
  if (threadIdx.x == 0) part[(size_t)c * T + t] = s;
}

// one CTA of 1024 threads per member; each thread keeps four independent
// partial dots (the loads of four strides in flight: a 256-thread loop with
// one chain was latency-bound, 0.5 ms for cfg5's 256 members), combined in
// a fixed order, then the fixed-order block tree
constexpr int PCG_INIT_NT = 1024;
__global__ void __launch_bounds__(PCG_INIT_NT) k_pcg_init(int n, const double* __restrict__ b,
                                                          const double* __restrict__ z, double* __restrict__ x,
                                                          double* __restrict__ r, double* __restrict__ p,
                                                          double* __restrict__ rzb, double* __restrict__ hist_rz,
                                                          int hist_ld, int32_t* __restrict__ status,
                                                          int32_t* __restrict__ iters) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  const size_t o = (size_t)c * n;
  double s4[4] = {0.0, 0.0, 0.0, 0.0};
  for (int i0 = threadIdx.x; i0 < n; i0 += 4 * PCG_INIT_NT) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * PCG_INIT_NT;
      if (i < n) {
        const double bi = b[o + i], zi = z[o + i];
        x[o + i] = 0.0;
        r[o + i] = bi;
        p[o + i] = zi;
        s4[u] += bi * zi;
      }
    }
  }
  double s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  s = block_sum<PCG_INIT_NT>(s, sh);
  if (threadIdx.x == 0) {
    rzb[c] = s;  // buffer 0 = iteration 0
    hist_rz[(size_t)c * hist_ld] = s;
    status[c] = s < 0.0 ? 3 : 0;
    iters[c] = 0;
  }
}

// after p.hp partials: breakdown test, alpha, x += alpha p, r -= alpha hp on
// this tile; if b != NULL also the tile partial of x.(b + r) for the cost:
//   J(x) = 1/2 x.(I+A)x - b.x + 1/2 d.R^-1 d  (the J identity of
//   test_assim.py:52-63) with (I+A)x = b - r  =>  J = J(0) - 1/2 x.(b + r)
__global__ void __launch_bounds__(PCG_NT) k_pcg_upd_x(int n, int T, int M, const double* __restrict__ p,
                                                      const double* __restrict__ hp, double* __restrict__ x,
                                                      double* __restrict__ r, const double* __restrict__ rzb,
                                                      int32_t* __restrict__ status, int32_t* __restrict__ iters,
                                                      int it, const double* __restrict__ part_a, int Ta,
                                                      double* __restrict__ part_x, const double* __restrict__ b,
                                                      double* __restrict__ part_rr) {
  __shared__ double sh[32];
  __shared__ double s_php;
  const int c = blockIdx.y, t = blockIdx.x;
  if (status[c] != 0) return;
  if (threadIdx.x < 32) {
    const double v = sum_parts(part_a + (size_t)c * Ta, Ta);
    if (threadIdx.x == 0) s_php = v;
  }
  __syncthreads();
  const double php = s_php;
  if (php <= 0.0) {  // krylov.py:82-84 (NaN does not raise)
    if (t == 0 && threadIdx.x == 0) {
      status[c] = 2;
      iters[c] = it;
    }
    return;
  }
  const double alpha = rzb[(size_t)((it - 1) & 1) * M + c] / php;
  const size_t o = (size_t)c * n;
  const int i0 = t * PCG_TILE, i1 = min(n, i0 + PCG_TILE);
  double xbr = 0.0, rr = 0.0;
  for (int i = i0 + threadIdx.x; i < i1; i += PCG_NT) {
    const double xi = x[o + i] + alpha * p[o + i];
    const double ri = r[o + i] - alpha * hp[o + i];
    x[o + i] = xi;
    r[o + i] = ri;
    if (b) xbr += xi * (b[o + i] + ri);
    rr += ri * ri;
  }
  if (b) {
    xbr = block_sum<PCG_NT>(xbr, sh);
    if (threadIdx.x == 0) part_x[(size_t)c * T + t] = xbr;
  }
  if (part_rr) {
    rr = block_sum<PCG_NT>(rr, sh);
    if (threadIdx.x == 0) part_rr[(size_t)c * T + t] = rr;
  }
}

// Fused LMP/beta step (single-pass P = I + S diag(coef) S^T): with W = S^T r,
//   rz_new = r.(r + S(coef o W)) = |r|^2 + sum_i coef_i W_i^2  (exact identity),
// recorded and tested here; beta = rz_new / rz_old goes to the p update that
// the LMP GEMM epilogue performs (p = r + beta p + S (coef o W)).
__global__ void __launch_bounds__(128) k_pcg_rz(int T, int M, int k, const double* __restrict__ W,
                                                const double* __restrict__ coef, const double* __restrict__ part_rr,
                                                const double* __restrict__ part_x, double* __restrict__ rzb,
                                                double* __restrict__ beta, double rtol, double* __restrict__ hist_rz,
                                                double* __restrict__ hist_J, int hist_ld,
                                                int32_t* __restrict__ status, int32_t* __restrict__ iters, int it) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  double q = 0.0;
  for (int i = threadIdx.x; i < k; i += 128) {
    const double w = W[i + (size_t)c * k];
    q += coef[i] * (w * w);
  }
  q = block_sum<128>(q, sh);
  if (threadIdx.x < 32) {
    const double rr = sum_parts(part_rr + (size_t)c * T, T);
    const double xbr = hist_J ? sum_parts(part_x + (size_t)c * T, T) : 0.0;
    if (threadIdx.x == 0) {
      if (status[c] != 0) {
        beta[c] = 0.0;
        return;
      }
      const double rz_new = rr + q;
      const double rz_old = rzb[(size_t)((it - 1) & 1) * M + c];
      const bool stop = rz_new <= 0.0 ||
                        (rtol >= 0.0 && sqrt(rz_new) <= rtol * sqrt(hist_rz[(size_t)c * hist_ld]));
      hist_rz[(size_t)c * hist_ld + it] = rz_new;
      if (hist_J) hist_J[(size_t)c * hist_ld + it] = hist_J[(size_t)c * hist_ld] - 0.5 * xbr;
      iters[c] = it;
      rzb[(size_t)(it & 1) * M + c] = rz_new;
      if (stop) status[c] = 1;
      beta[c] = stop ? 0.0 : rz_new / rz_old;
    }
  }
}

// after r.z partials: record, stop test, p = z + beta p on this tile
__global__ void __launch_bounds__(PCG_NT) k_pcg_upd_p(int n, int T, int M, const double* __restrict__ z,
                                                      double* __restrict__ p, double* __restrict__ rzb,
                                                      double rtol, double* __restrict__ hist_rz,
                                                      double* __restrict__ hist_J, int hist_ld,
                                                      int32_t* __restrict__ status, int32_t* __restrict__ iters,
                                                      int it, const double* __restrict__ part_r,
                                                      const double* __restrict__ part_x) {
  __shared__ double s_rz, s_J;
  const int c = blockIdx.y, t = blockIdx.x;
  if (status[c] != 0) return;
  if (threadIdx.x < 32) {
    const double v = sum_parts(part_r + (size_t)c * T, T);
    double J = 0.0;
    if (hist_J && t == 0) {
      const double xbr = sum_parts(part_x + (size_t)c * T, T);
      J = hist_J[(size_t)c * hist_ld] - 0.5 * xbr;
    }
    if (threadIdx.x == 0) {
      s_rz = v;
      s_J = J;
    }
  }
  __syncthreads();
  const double rz_new = s_rz;
  const double rz_old = rzb[(size_t)((it - 1) & 1) * M + c];
  const bool stop = rz_new <= 0.0 ||
                    (rtol >= 0.0 && sqrt(rz_new) <= rtol * sqrt(hist_rz[(size_t)c * hist_ld]));
  if (t == 0 && threadIdx.x == 0) {
    hist_rz[(size_t)c * hist_ld + it] = rz_new;
    if (hist_J) hist_J[(size_t)c * hist_ld + it] = s_J;
    iters[c] = it;
    rzb[(size_t)(it & 1) * M + c] = rz_new;
    if (stop) status[c] = 1;
  }
  if (stop) return;
  const double beta = rz_new / rz_old;
  const size_t o = (size_t)c * n;
  const int i0 = t * PCG_TILE, i1 = min(n, i0 + PCG_TILE);
  for (int i = i0 + threadIdx.x; i < i1; i += PCG_NT) p[o + i] = z[o + i] + beta * p[o + i];
}

// initial cost J(0) = 1/2 d.R^-1 d  (misfit = -d, assim.py:81-82); one
// 1024-thread CTA per member with four partial sums per thread, as k_pcg_init
__global__ void __launch_bounds__(PCG_INIT_NT) k_pcg_cost0(int np_obs, const double* __restrict__ d, double sigma2,
                                                           double* __restrict__ hist_J, int hist_ld) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  const size_t q0 = (size_t)c * np_obs;
  double m4[4] = {0.0, 0.0, 0.0, 0.0};
  for (int b0 = threadIdx.x; b0 < np_obs; b0 += 4 * PCG_INIT_NT) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = b0 + u * PCG_INIT_NT;
      if (q < np_obs) {
        const double e = -d[q0 + q];
        m4[u] += e * (e / sigma2);
      }
    }
  }
  double mm = (m4[0] + m4[1]) + (m4[2] + m4[3]);
  mm = block_sum<PCG_INIT_NT>(mm, sh);
  if (threadIdx.x == 0) hist_J[(size_t)c * hist_ld] = 0.5 * mm;
}

// work layout: part_a | part_x | part_rr | part_r (M*T each) | rzb (2*M) | beta (M)
int64_t pcg_work_doubles(int n, int M) { return 4LL * M * pcg_tiles(n) + 3LL * M; }

int launch_pcg_init(int n, int M, const double* b, const double* z, double* x, double* r, double* p, double* work,
                    double* hist_rz, int hist_ld, int32_t* status, int32_t* iters, cudaStream_t st) {
  double* rzb = work + 4LL * M * pcg_tiles(n);
  k_pcg_init<<<M, PCG_INIT_NT, 0, st>>>(n, b, z, x, r, p, rzb, hist_rz, hist_ld, status, iters);
  count_launch();
  return check_launch("k_pcg_init");
}

int launch_pcg_alpha(int n, int M, const double* p, const double* hp, double* x, double* r, double* work,
                     int32_t* status, int32_t* iters, int it, const double* b, const double* php_part,
                     int php_tiles, cudaStream_t st) {
  const int T = pcg_tiles(n);
  double* part_a = work;
  double* part_x = work + (size_t)M * T;
  double* part_rr = work + 2 * (size_t)M * T;
  double* rzb = work + 4 * (size_t)M * T;
  dim3 grid(T, M);
  if (!php_part) {
    k_dot_partial<<<grid, PCG_NT, 0, st>>>(n, T, p, hp, part_a);
    count_launch();
    php_part = part_a;
    php_tiles = T;
  }
  k_pcg_upd_x<<<grid, PCG_NT, 0, st>>>(n, T, M, p, hp, x, r, rzb, status, iters, it, php_part, php_tiles, part_x, b,
                                       part_rr);
  count_launch();
  return check_launch("k_pcg_upd_x");
}

// k_pcg_rz with the split-K reduction of W = S^T r folded in: one CTA per
// column reduces its k entries from the GEMM's partials, writes W for the
// p-update GEMM, and runs the rz step.  1024 threads: entry i = t % 128 of a 128-entry slab (a warp reads 32
// consecutive entries of one split row: coalesced), split group q = t / 128
// sums splits q, q + 8, ... in order; the 8 group sums are then combined in
// a fixed tree (deterministic).  The split-K GEMM for the 100-member groups
// writes 128 splits, which the former 2-lanes-per-entry form summed as 64
// dependent strided loads per thread (14 us per launch, latency-bound).
__global__ void __launch_bounds__(1024) k_pcg_reduce_rz(int T, int M, int k, const double* __restrict__ part,
                                                       int nsplit, double* __restrict__ W,
                                                       const double* __restrict__ coef,
                                                       const double* __restrict__ part_rr,
                                                       const double* __restrict__ part_x, double* __restrict__ rzb,
                                                       double* __restrict__ beta, double rtol,
                                                       double* __restrict__ hist_rz, double* __restrict__ hist_J,
                                                       int hist_ld, int32_t* __restrict__ status,
                                                       int32_t* __restrict__ iters, int it, int prescale) {
  __shared__ double sh[32];
  __shared__ double gs[8][128];
  const int c = blockIdx.x, t = threadIdx.x;
  const int e = t & 127, g = t >> 7;
  const int64_t tot = (int64_t)k * M;
  double q = 0.0;
  for (int i0 = 0; i0 < k; i0 += 128) {
    const int i = i0 + e;
    double s = 0.0;
    if (i < k) {
      const double* pp = part + i + (size_t)c * k;
      // up to 19 partials per thread (148 splits / 8 groups): all of their
      // loads in flight before the (fixed-order) sum -- the reduction was
      // load-latency bound with four in flight
      double v[19];
#pragma unroll
      for (int u = 0; u < 19; ++u) {
        const int z = g + 8 * u;
        v[u] = z < nsplit ? pp[(size_t)z * tot] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 19; ++u) s += v[u];
      for (int z = g + 8 * 19; z < nsplit; z += 8) s += pp[(size_t)z * tot];
    }
    gs[g][e] = s;
    __syncthreads();
    if (g == 0 && i < k) {
      const double w = ((gs[0][e] + gs[1][e]) + (gs[2][e] + gs[3][e])) +
                       ((gs[4][e] + gs[5][e]) + (gs[6][e] + gs[7][e]));
      // prescale: coef o W for the p-update GEMM (the product it would form
      // on staging, so the same bits), sparing k_lmp_nn its scaling pass
      W[i + (size_t)c * k] = prescale ? coef[i] * w : w;
      q += coef[i] * (w * w);
    }
    __syncthreads();
  }
  q = block_sum<1024>(q, sh);
  if (threadIdx.x < 32) {
    const double rr = sum_parts(part_rr + (size_t)c * T, T);
    const double xbr = hist_J ? sum_parts(part_x + (size_t)c * T, T) : 0.0;
    if (threadIdx.x == 0) {
      if (status[c] != 0) {
        beta[c] = 0.0;
        return;
      }
      const double rz_new = rr + q;
      const double rz_old = rzb[(size_t)((it - 1) & 1) * M + c];
      const bool stop = rz_new <= 0.0 ||
                        (rtol >= 0.0 && sqrt(rz_new) <= rtol * sqrt(hist_rz[(size_t)c * hist_ld]));
      hist_rz[(size_t)c * hist_ld + it] = rz_new;
      if (hist_J) hist_J[(size_t)c * hist_ld + it] = hist_J[(size_t)c * hist_ld] - 0.5 * xbr;
      iters[c] = it;
      rzb[(size_t)(it & 1) * M + c] = rz_new;
      if (stop) status[c] = 1;
      beta[c] = stop ? 0.0 : rz_new / rz_old;
    }
  }
}

int launch_pcg_reduce_rz(int n, int M, int k, const double* part, int nsplit, double* W, const double* coef,
                         double* work, double rtol, double* hist_rz, double* hist_J, int hist_ld, int32_t* status,
                         int32_t* iters, int it, cudaStream_t st, int prescale) {
  const int T = pcg_tiles(n);
  double* part_x = work + (size_t)M * T;
  double* part_rr = work + 2 * (size_t)M * T;
  double* rzb = work + 4 * (size_t)M * T;
  double* beta = rzb + 2 * (size_t)M;
  k_pcg_reduce_rz<<<M, 1024, 0, st>>>(T, M, k, part, nsplit, W, coef, part_rr, part_x, rzb, beta, rtol, hist_rz,
                                     hist_J, hist_ld, status, iters, it, prescale);
  count_launch();
  return check_launch("k_pcg_reduce_rz");
}

int launch_pcg_rz(int n, int M, int k, const double* W, const double* coef, double* work, double rtol,
                  double* hist_rz, double* hist_J, int hist_ld, int32_t* status, int32_t* iters, int it,
                  cudaStream_t st) {
  const int T = pcg_tiles(n);
  double* part_x = work + (size_t)M * T;
  double* part_rr = work + 2 * (size_t)M * T;
  double* rzb = work + 4 * (size_t)M * T;
  double* beta = rzb + 2 * (size_t)M;
  k_pcg_rz<<<M, 128, 0, st>>>(T, M, k, W, coef, part_rr, part_x, rzb, beta, rtol, hist_rz, hist_J, hist_ld, status,
                              iters, it);
  count_launch();
  return check_launch("k_pcg_rz");
}

double* pcg_beta_ptr(int n, int M, double* work) { return work + 4 * (size_t)M * pcg_tiles(n) + 2 * (size_t)M; }

int launch_pcg_beta(int n, int M, const double* z, const double* r, double* p, double* work, double rtol,
                    double* hist_rz, double* hist_J, int hist_ld, int32_t* status, int32_t* iters, int it,
                    cudaStream_t st) {
  const int T = pcg_tiles(n);
  double* part_x = work + (size_t)M * T;
  double* part_r = work + 3 * (size_t)M * T;
  double* rzb = work + 4 * (size_t)M * T;
  dim3 grid(T, M);
  k_dot_partial<<<grid, PCG_NT, 0, st>>>(n, T, r, z, part_r);
  k_pcg_upd_p<<<grid, PCG_NT, 0, st>>>(n, T, M, z, p, rzb, rtol, hist_rz, hist_J, hist_ld, status, iters, it,
                                       part_r, part_x);
  count_launch(2);
  return check_launch("k_pcg_upd_p");
}

int launch_pcg_cost0(int np_obs, int ncols, const double* d, double sigma2, double* hist_J, int hist_ld,
                     cudaStream_t st) {
  k_pcg_cost0<<<ncols, PCG_INIT_NT, 0, st>>>(np_obs, d, sigma2, hist_J, hist_ld);
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
