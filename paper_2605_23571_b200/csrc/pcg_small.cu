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
// recompute as in the sweeps (stg_f / stg_axpy, common.cuh), tendencies with FMA.
#include "common.cuh"

namespace edak {

constexpr int PS_MAXN = 256;
constexpr int PS_MAXDYN = 160 * 1024;  // dynamic shared memory bytes

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

// three block sums with one pair of barriers
template <int NT>
__device__ __forceinline__ double3 bsum3(double a, double b, double c, double* sh) {
  a = warp_sum(a);
  b = warp_sum(b);
  c = warp_sum(c);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    sh[threadIdx.x >> 5] = a;
    sh[8 + (threadIdx.x >> 5)] = b;
    sh[16 + (threadIdx.x >> 5)] = c;
  }
  __syncthreads();
  double3 r = make_double3(sh[0], sh[8], sh[16]);
#pragma unroll
  for (int w = 1; w < NT / 32; ++w) {
    r.x += sh[w];
    r.y += sh[8 + w];
    r.z += sh[16 + w];
  }
  return r;
}

// dynamic shared memory (doubles): trajectory states N x n | observations
// G*T | taps K | LMP vectors k x n | coef k | tpos (N+1 ints)
__host__ __device__ inline size_t small_smem_doubles(int n, int N, int p, int K, int k) {
  return (size_t)N * n + p + K + (size_t)k * n + k + (N + 2) / 2;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_pcg_small(SmallArgs A) {
  __shared__ double sh[32];
  __shared__ double sp_[PS_MAXN], sv[2][PS_MAXN], su[2][PS_MAXN], sx[2][PS_MAXN];
  __shared__ double st4[2][3][PS_MAXN];  // AD: x2, x3, x4 of steps s (cur) and s-1 (next)
  __shared__ double sg[PS_MAXN], sa[2][PS_MAXN];
  __shared__ double sW[PS_MAXN];
  extern __shared__ double dyn[];
  const edak_problem& P = A.P;
  const int n = P.n, N = P.n_steps, G = P.G, T = P.T, K = P.ntaps, w = P.tap_w, k = A.k;
  double* sTr = dyn;
  double* sobs = sTr + (size_t)N * n;
  double* sTap = sobs + G * T;
  double* sS = sTap + K;
  double* sC = sS + (size_t)k * n;
  int* sTp = reinterpret_cast<int*>(sC + k);
  const int c = blockIdx.x, i = threadIdx.x;
  const bool own = i < n;
  {
    const int traj = A.col_traj ? A.col_traj[c] : 0;
    const double* tr = P.states + (size_t)traj * P.traj_stride;
    for (int e = i; e < N * n; e += NT) sTr[e] = tr[e];
    for (int e = i; e < K; e += NT) sTap[e] = P.taps[e];
    for (int e = i; e < k * n; e += NT) sS[e] = A.S[e];
    for (int e = i; e < k; e += NT) sC[e] = A.coef[e];
    for (int e = i; e <= N; e += NT) sTp[e] = P.tpos[e];
  }
  const double dt = P.dt, h = 0.5 * dt, c6 = dt / 6.0, F = P.forcing, inv_s2 = 1.0 / P.sigma2;
  const int gp = own ? __ldg(P.gpos + i) : -1;
  const int L = A.hist_ld;
  const int im1 = rw(i - 1, n), im2 = rw(i - 2, n), ip1 = rw(i + 1, n), ip2 = rw(i + 2, n);
  const int j0 = own ? (i + w) % n : 0;
  __syncthreads();

  // U_B applied to the ring in `in` (smem), result for element i
  auto circ = [&](const double* in) {
    double acc = 0.0;
    if (own) {
      int j = j0;
      for (int q = 0; q < K; ++q) {
        acc = fma(sTap[q], in[j], acc);
        j = j == 0 ? n - 1 : j - 1;
      }
    }
    return acc;
  };
  // x2, x3, x4 of step s into st4[buf]: three neighbour exchanges; the
  // caller places a barrier after each (they overlap the adjoint phases)
  auto stage = [&](int s, int buf, int which) {
    if (!own) return;
    const double* X = sTr + (size_t)s * n;
    const double* y = which == 0 ? X : st4[buf][which - 1];
    st4[buf][which][i] = stg_axpy(X[i], which == 2 ? dt : h, stg_f(y[ip1], y[im2], y[im1], y[i], F));
  };
  // (I + A) p for p in sp_ (barrier after its write) -> returns hp_i
  auto hessian = [&]() -> double {
    // v = U_B p
    double v = circ(sp_);
    int cb = 0;
    if (own) {
      sv[0][i] = v;
      const int tp0 = sTp[0];
      if (tp0 >= 0 && gp >= 0) sobs[tp0 * G + gp] = v;
    }
    __syncthreads();
    // TL sweep with capture (levels 1..N): four exchanges per step
    for (int s = 0; s < N; ++s) {
      const double* X = sTr + (size_t)s * n;
      const double* V = sv[cb];
      double acc = 0.0;
      if (own) {
        const double x0 = X[i];
        const double d1 = __dsub_rn(X[ip1], X[im2]);
        const double a1 = l96_tl_d(V[ip1], V[im2], V[im1], v, d1, X[im1]);
        su[0][i] = fma(h, a1, v);
        sx[0][i] = stg_axpy(x0, h, stg_f_d(d1, X[im1], x0, F));
        acc = a1;
      }
      __syncthreads();
      if (own) {
        const double x0 = X[i];
        const double d2 = __dsub_rn(sx[0][ip1], sx[0][im2]);
        const double a2 = l96_tl_d(su[0][ip1], su[0][im2], su[0][im1], su[0][i], d2, sx[0][im1]);
        su[1][i] = fma(h, a2, v);
        sx[1][i] = stg_axpy(x0, h, stg_f_d(d2, sx[0][im1], sx[0][i], F));
        acc = fma(2.0, a2, acc);
      }
      __syncthreads();
      if (own) {
        const double x0 = X[i];
        const double d3 = __dsub_rn(sx[1][ip1], sx[1][im2]);
        const double a3 = l96_tl_d(su[1][ip1], su[1][im2], su[1][im1], su[1][i], d3, sx[1][im1]);
        su[0][i] = fma(dt, a3, v);
        sx[0][i] = stg_axpy(x0, dt, stg_f_d(d3, sx[1][im1], sx[1][i], F));
        acc = fma(2.0, a3, acc);
      }
      __syncthreads();
      if (own) {
        const double d4 = __dsub_rn(sx[0][ip1], sx[0][im2]);
        const double a4 = l96_tl_d(su[0][ip1], su[0][im2], su[0][im1], su[0][i], d4, sx[0][im1]);
        v = fma(c6, acc + a4, v);
        sv[cb ^ 1][i] = v;
        const int tp = sTp[s + 1];
        if (tp >= 0 && gp >= 0) sobs[tp * G + gp] = v;
      }
      cb ^= 1;
      __syncthreads();
    }
    // AD sweep: g = w[N]; for s = N-1..0: g = step_adj(stages(s), g) + w[s].
    // The stages of step s-1 are recomputed during step s's adjoint phases.
    auto force = [&](int level) -> double {
      const int tp = sTp[level];
      return (own && tp >= 0 && gp >= 0) ? sobs[tp * G + gp] * inv_s2 : 0.0;
    };
    double g = force(N);
    int sb = 0;
    stage(N - 1, 0, 0);
    if (own) sa[0][i] = c6 * g;
    __syncthreads();
    stage(N - 1, 0, 1);
    __syncthreads();
    stage(N - 1, 0, 2);
    __syncthreads();
    for (int s = N - 1; s >= 0; --s) {
      // the AD kernel's stage combination: w = (dt/6) g,
      // b3 = h u4 + w, b2 = h u3' + w, a1 = dt u2' + w
      const double wv = c6 * g;
      const double* x4 = st4[sb][2];
      const double* x3 = st4[sb][1];
      const double* x2 = st4[sb][0];
      double vh = 0.0;
      if (own) {
        const double u4 = l96_ad(x4[im2], x4[im1], x4[ip1], x4[ip2], sa[0][im1], sa[0][i], sa[0][ip1], sa[0][ip2]);
        vh = g + u4;
        sa[1][i] = fma(h, u4, wv);  // b3
      }
      if (s > 0) stage(s - 1, sb ^ 1, 0);
      __syncthreads();
      if (own) {
        const double u3 = l96_ad(x3[im2], x3[im1], x3[ip1], x3[ip2], sa[1][im1], sa[1][i], sa[1][ip1], sa[1][ip2]);
        vh = fma(2.0, u3, vh);
        sa[0][i] = fma(h, u3, wv);  // b2
      }
      if (s > 0) stage(s - 1, sb ^ 1, 1);
      __syncthreads();
      if (own) {
        const double u2 = l96_ad(x2[im2], x2[im1], x2[ip1], x2[ip2], sa[0][im1], sa[0][i], sa[0][ip1], sa[0][ip2]);
        vh = fma(2.0, u2, vh);
        sa[1][i] = fma(dt, u2, wv);  // a1
      }
      if (s > 0) stage(s - 1, sb ^ 1, 2);
      __syncthreads();
      if (own) {
        const double* X = sTr + (size_t)s * n;
        const double u1 = l96_ad(X[im2], X[im1], X[ip1], X[ip2], sa[1][im1], sa[1][i], sa[1][ip1], sa[1][ip2]);
        g = vh + u1 + force(s);
        if (s > 0) sa[0][i] = c6 * g;
        else sg[i] = g;
      }
      sb ^= 1;
      __syncthreads();
    }
    // hp = p + U_B g
    const double hp = own ? sp_[i] + circ(sg) : 0.0;
    return hp;
  };
  // W = S^T r into sW (barrier after)
  auto lmp_w = [&](double r_i) {
    if (own) sg[i] = r_i;
    __syncthreads();
    for (int q = i; q < k; q += NT) {
      double s = 0.0;
      const double* Sq = sS + (size_t)q * n;
      for (int e = 0; e < n; ++e) s = fma(Sq[e], sg[e], s);
      sW[q] = s;
    }
    __syncthreads();
  };
  // z = r + S (coef o W)  (after lmp_w)
  auto lmp_apply = [&](double r_i) -> double {
    double z = r_i;
    if (own)
      for (int q = 0; q < k; ++q) z = fma(sS[(size_t)q * n + i], sC[q] * sW[q], z);
    return z;
  };

  // ---- init (krylov.py:63-73) ----------------------------------------------
  const double b_i = own ? A.b[(size_t)c * n + i] : 0.0;
  double x_i = 0.0, r_i = b_i, z_i = b_i;
  if (k) {
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
    double q = 0.0;
    if (k) {
      lmp_w(r_i);
      for (int j = i; j < k; j += NT) q += sC[j] * (sW[j] * sW[j]);
    }
    const double3 red = bsum3<NT>(own ? r_i * r_i : 0.0, q, (A.hist_J && own) ? x_i * (b_i + r_i) : 0.0, sh);
    const double rz_new = red.x + red.y;
    done_it = it;
    if (i == 0) {
      A.hist_rz[(size_t)c * L + it] = rz_new;
      if (A.hist_J) A.hist_J[(size_t)c * L + it] = J0 - 0.5 * red.z;
    }
    if (rz_new <= 0.0 || (A.rtol >= 0.0 && sqrt(rz_new) <= A.rtol * sqrt(rz0))) {
      status = 1;
      break;
    }
    const double beta = rz_new / rz;
    const double zr = k ? lmp_apply(r_i) : r_i;
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
  const size_t smem = small_smem_doubles(n, A.P.n_steps, A.P.G * A.P.T, A.P.ntaps, A.k) * sizeof(double);
  if (smem > PS_MAXDYN) {
    set_error("pcg_small: trajectory + observations + LMP exceed shared memory");
    return EDAK_EUNSUPPORTED;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_pcg_small<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, PS_MAXDYN);
    cudaFuncSetAttribute(k_pcg_small<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, PS_MAXDYN);
    cudaFuncSetAttribute(k_pcg_small<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, PS_MAXDYN);
    attr = true;
  }
  if (n <= 64)
    k_pcg_small<64><<<M, 64, smem, st>>>(A);
  else if (n <= 128)
    k_pcg_small<128><<<M, 128, smem, st>>>(A);
  else
    k_pcg_small<256><<<M, 256, smem, st>>>(A);
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
