// Persistent batched LMP-PCG for small rings (n <= 256: BASELINE cfg1/cfg2,
// the reference harness' n = 40 twins).  SURVEY.md §8d: those configs are
// launch- and latency-bound (microseconds of work per Hessian apply), so the
// whole solve of one member -- every iteration's U_B, TL sweep with
// observation capture, AD sweep with R^-1 forcing, U_B (+I), the PCG
// recurrence with the J identity, and the single-pass LMP -- runs inside ONE
// CTA, one ring element per thread, with no kernel boundary at all.
//
// Same recurrence and formulas as the batched path (krylov.py:49-97 via
// edak_hessian_block + edak_pcg_alpha + edak_pcg_lmp_beta); stage
// recompute bit-exact (l96_f / axpy_rn), tendencies with FMA.
#include "common.cuh"

namespace edak {

constexpr int PS_MAXN = 256;

struct SmallArgs {
  edak_problem P;
  const int32_t* col_traj;  // member -> trajectory (NULL: trajectory 0)
  const double* b;          // (M, n) right-hand sides
  const double* d;          // (M, p) innovations (J(0)); NULL: no cost trace
  const double* S;          // (k, n) LMP vectors or NULL (no preconditioner)
  const double* coef;       // (k) theta/(lam+1) - 1
  int k;
  int max_iters;
  double rtol;              // < 0: none
  double* x;                // (M, n)
  double* hist_rz;          // (M, L)
  double* hist_J;           // (M, L) or NULL
  int hist_ld;
  int32_t* status;
  int32_t* iters;
};

__device__ __forceinline__ int rw(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// block sum broadcast to every thread (same summation order in all threads)
template <int NT>
__device__ __forceinline__ double bsum(double v, double* sh) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = sh[0];
#pragma unroll
  for (int w = 1; w < NT / 32; ++w) s += sh[w];
  return s;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_pcg_small(SmallArgs A) {
  __shared__ double sh[32];
  __shared__ double sp_[PS_MAXN], sv[PS_MAXN], su[2][PS_MAXN], sx[2][PS_MAXN], sX[PS_MAXN];
  __shared__ double st4[3][PS_MAXN];  // AD: x2, x3, x4 of the current step
  __shared__ double sg[PS_MAXN], sa[2][PS_MAXN];
  __shared__ double sW[PS_MAXN];
  extern __shared__ double sobs[];    // G * T observations of the current apply
  const edak_problem& P = A.P;
  const int n = P.n, N = P.n_steps, G = P.G, T = P.T, K = P.ntaps, w = P.tap_w;
  const int c = blockIdx.x, i = threadIdx.x;
  const bool own = i < n;
  const int traj = A.col_traj ? A.col_traj[c] : 0;
  const double* tr = P.states + (size_t)traj * P.traj_stride;
  const double dt = P.dt, h = 0.5 * dt, c6 = dt / 6.0, F = P.forcing, inv_s2 = 1.0 / P.sigma2;
  const int gp = own ? __ldg(P.gpos + i) : -1;
  const int L = A.hist_ld;
  const int im1 = rw(i - 1, n), im2 = rw(i - 2, n), ip1 = rw(i + 1, n), ip2 = rw(i + 2, n);

  // U_B applied to the ring in `in` (smem), result for element i
  auto circ = [&](const double* in) {
    double acc = 0.0;
    if (own)
      for (int q = 0; q < K; ++q) acc = fma(__ldg(P.taps + q), in[rw((i + w - q) % n, n)], acc);
    return acc;
  };
  // (I + A) p for p in sp_ -> returns hp_i
  auto hessian = [&]() -> double {
    // v = U_B p
    double v = circ(sp_);
    if (own) sv[i] = v;
    __syncthreads();
    // TL sweep with capture (levels 0..N)
    {
      const int tp0 = __ldg(P.tpos + 0);
      if (own && tp0 >= 0 && gp >= 0) sobs[tp0 * G + gp] = v;
    }
    for (int s = 0; s < N; ++s) {
      const double X = own ? __ldg(tr + (size_t)s * n + i) : 0.0;
      if (own) sX[i] = X;
      __syncthreads();
      double a1 = 0.0, acc = 0.0;
      if (own) {
        const double d1 = __dsub_rn(sX[ip1], sX[im2]);
        a1 = l96_tl_d(sv[ip1], sv[im2], sv[im1], sv[i], d1, sX[im1]);
        su[0][i] = fma(h, a1, sv[i]);
        sx[0][i] = axpy_rn(X, h, l96_f_d(d1, sX[im1], X, F));
        acc = a1;
      }
      __syncthreads();
      double a2 = 0.0;
      if (own) {
        const double d2 = __dsub_rn(sx[0][ip1], sx[0][im2]);
        a2 = l96_tl_d(su[0][ip1], su[0][im2], su[0][im1], su[0][i], d2, sx[0][im1]);
        su[1][i] = fma(h, a2, sv[i]);
        sx[1][i] = axpy_rn(X, h, l96_f_d(d2, sx[0][im1], sx[0][i], F));
        acc = fma(2.0, a2, acc);
      }
      __syncthreads();
      double a3 = 0.0;
      if (own) {
        const double d3 = __dsub_rn(sx[1][ip1], sx[1][im2]);
        a3 = l96_tl_d(su[1][ip1], su[1][im2], su[1][im1], su[1][i], d3, sx[1][im1]);
        su[0][i] = fma(dt, a3, sv[i]);
        sx[0][i] = axpy_rn(X, dt, l96_f_d(d3, sx[1][im1], sx[1][i], F));
        acc = fma(2.0, a3, acc);
      }
      __syncthreads();
      double vn = 0.0;
      if (own) {
        const double d4 = __dsub_rn(sx[0][ip1], sx[0][im2]);
        const double a4 = l96_tl_d(su[0][ip1], su[0][im2], su[0][im1], su[0][i], d4, sx[0][im1]);
        vn = fma(c6, acc + a4, sv[i]);
      }
      __syncthreads();
      if (own) {
        sv[i] = vn;
        const int tp = __ldg(P.tpos + s + 1);
        if (tp >= 0 && gp >= 0) sobs[tp * G + gp] = vn;
      }
      __syncthreads();
    }
    // AD sweep: g = w[N]; for s = N-1..0: g = step_adj(stages(s), g) + w[s]
    auto force = [&](int level) -> double {
      const int tp = __ldg(P.tpos + level);
      return (own && tp >= 0 && gp >= 0) ? sobs[tp * G + gp] * inv_s2 : 0.0;
    };
    double g = force(N);
    for (int s = N - 1; s >= 0; --s) {
      const double X = own ? __ldg(tr + (size_t)s * n + i) : 0.0;
      if (own) {
        sX[i] = X;
        sg[i] = g;
      }
      __syncthreads();
      if (own) st4[0][i] = axpy_rn(X, h, l96_f(sX[ip1], sX[im2], sX[im1], X, F));  // x2
      __syncthreads();
      if (own) st4[1][i] = axpy_rn(X, h, l96_f(st4[0][ip1], st4[0][im2], st4[0][im1], st4[0][i], F));  // x3
      __syncthreads();
      if (own) st4[2][i] = axpy_rn(X, dt, l96_f(st4[1][ip1], st4[1][im2], st4[1][im1], st4[1][i], F));  // x4
      if (own) sa[0][i] = c6 * g;  // a4 = (dt/6) g
      __syncthreads();
      // the AD kernel's stage combination: w = (dt/6) g,
      // b3 = h u4 + w, b2 = h u3' + w, a1 = dt u2' + w
      double vh = 0.0, wv = 0.0;
      if (own) {
        wv = sa[0][i];
        const double* x4 = st4[2];
        const double u4 = l96_ad(x4[im2], x4[im1], x4[ip1], x4[ip2], sa[0][im1], sa[0][i], sa[0][ip1], sa[0][ip2]);
        vh = g + u4;
        sa[1][i] = fma(h, u4, wv);  // b3
      }
      __syncthreads();
      if (own) {
        const double* x3 = st4[1];
        const double u3 = l96_ad(x3[im2], x3[im1], x3[ip1], x3[ip2], sa[1][im1], sa[1][i], sa[1][ip1], sa[1][ip2]);
        vh = fma(2.0, u3, vh);
        sa[0][i] = fma(h, u3, wv);  // b2
      }
      __syncthreads();
      if (own) {
        const double* x2 = st4[0];
        const double u2 = l96_ad(x2[im2], x2[im1], x2[ip1], x2[ip2], sa[0][im1], sa[0][i], sa[0][ip1], sa[0][ip2]);
        vh = fma(2.0, u2, vh);
        sa[1][i] = fma(dt, u2, wv);  // a1
      }
      __syncthreads();
      if (own) {
        const double u1 = l96_ad(sX[im2], sX[im1], sX[ip1], sX[ip2], sa[1][im1], sa[1][i], sa[1][ip1], sa[1][ip2]);
        g = vh + u1 + force(s);
      }
      __syncthreads();
    }
    // hp = p + U_B g
    if (own) sg[i] = g;
    __syncthreads();
    const double hp = own ? sp_[i] + circ(sg) : 0.0;
    __syncthreads();
    return hp;
  };
  // z = P r (single-pass LMP; identity when S == NULL), W = S^T r in sW
  auto lmp_w = [&](double r_i) {
    if (own) sg[i] = r_i;
    __syncthreads();
    for (int q = i; q < A.k; q += NT) {
      double s = 0.0;
      for (int e = 0; e < n; ++e) s = fma(__ldg(A.S + (size_t)q * n + e), sg[e], s);
      sW[q] = s;
    }
    __syncthreads();
  };
  auto lmp_apply = [&](double r_i) -> double {  // after lmp_w
    double z = r_i;
    if (own)
      for (int q = 0; q < A.k; ++q) z = fma(__ldg(A.S + (size_t)q * n + i), __ldg(A.coef + q) * sW[q], z);
    return z;
  };

  // ---- init (krylov.py:63-73) ----------------------------------------------
  const double b_i = own ? A.b[(size_t)c * n + i] : 0.0;
  double x_i = 0.0, r_i = b_i, z_i = b_i;
  if (A.S) {
    lmp_w(r_i);
    z_i = lmp_apply(r_i);
  }
  double rz = bsum<NT>(own ? r_i * z_i : 0.0, sh);
  double J0 = 0.0;
  if (A.d) {
    const int p = G * T;
    double m2 = 0.0;
    for (int q = i; q < p; q += NT) {
      const double e = -A.d[(size_t)c * p + q];
      m2 += e * (e / P.sigma2);
    }
    J0 = 0.5 * bsum<NT>(m2, sh);
  }
  const double rz0 = rz;
  int status = rz < 0.0 ? 3 : 0, done_it = 0;
  if (i == 0) {
    A.hist_rz[(size_t)c * L] = rz;
    if (A.hist_J) A.hist_J[(size_t)c * L] = J0;
  }
  double p_i = z_i;
  for (int it = 1; it <= A.max_iters && status == 0; ++it) {
    if (own) sp_[i] = p_i;
    __syncthreads();
    const double hp_i = hessian();
    const double php = bsum<NT>(own ? p_i * hp_i : 0.0, sh);
    if (php <= 0.0) {  // krylov.py:82-84 (NaN does not raise)
      status = 2;
      done_it = it;
      break;
    }
    const double alpha = rz / php;
    x_i = fma(alpha, p_i, x_i);
    r_i = fma(-alpha, hp_i, r_i);
    const double xbr = A.hist_J ? bsum<NT>(own ? x_i * (b_i + r_i) : 0.0, sh) : 0.0;
    double rz_new;
    if (A.S) {
      lmp_w(r_i);
      double q = 0.0;
      for (int j = i; j < A.k; j += NT) q += __ldg(A.coef + j) * (sW[j] * sW[j]);
      const double rr = bsum<NT>(own ? r_i * r_i : 0.0, sh);
      rz_new = rr + bsum<NT>(q, sh);
    } else {
      rz_new = bsum<NT>(own ? r_i * r_i : 0.0, sh);
    }
    done_it = it;
    if (i == 0) {
      A.hist_rz[(size_t)c * L + it] = rz_new;
      if (A.hist_J) A.hist_J[(size_t)c * L + it] = J0 - 0.5 * xbr;
    }
    if (rz_new <= 0.0 || (A.rtol >= 0.0 && sqrt(rz_new) <= A.rtol * sqrt(rz0))) {
      status = 1;
      break;
    }
    const double beta = rz_new / rz;
    const double zr = A.S ? lmp_apply(r_i) : r_i;
    p_i = fma(beta, p_i, zr);
    rz = rz_new;
  }
  if (own) A.x[(size_t)c * n + i] = x_i;
  if (i == 0) {
    A.status[c] = status;
    A.iters[c] = done_it;
  }
}

int launch_pcg_small(const SmallArgs& A, int M, cudaStream_t st) {
  const int n = A.P.n;
  if (A.k > PS_MAXN) {
    set_error("pcg_small: more than 256 LMP vectors");
    return EDAK_EUNSUPPORTED;
  }
  if (n > PS_MAXN || n < 8) {
    set_error("pcg_small: n outside [8, 256]");
    return EDAK_EUNSUPPORTED;
  }
  if (A.P.stage_mode != 0) {
    set_error("pcg_small: needs stage_mode recompute");
    return EDAK_EUNSUPPORTED;
  }
  const size_t obs = (size_t)A.P.G * A.P.T * sizeof(double);
  if (obs > 64 * 1024) {
    set_error("pcg_small: too many observations for shared memory");
    return EDAK_EUNSUPPORTED;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_pcg_small<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_pcg_small<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_pcg_small<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    attr = true;
  }
  if (n <= 64)
    k_pcg_small<64><<<M, 64, obs, st>>>(A);
  else if (n <= 128)
    k_pcg_small<128><<<M, 128, obs, st>>>(A);
  else
    k_pcg_small<256><<<M, 256, obs, st>>>(A);
  count_launch();
  return check_launch("k_pcg_small");
}

int launch_pcg_small_c(const edak_problem* P, const int32_t* col_traj, int M, const double* b, const double* d,
                       const double* S, const double* coef, int k, int max_iters, double rtol, double* x,
                       double* hist_rz, double* hist_J, int hist_ld, int32_t* status, int32_t* iters,
                       cudaStream_t st) {
  SmallArgs A{*P, col_traj, b, d, S, coef, S ? k : 0, max_iters, rtol, x, hist_rz, hist_J, hist_ld, status, iters};
  return launch_pcg_small(A, M, st);
}

}  // namespace edak
