// Hybrid-storage window sweeps (stage_mode 2): the trajectory keeps its
// stored RK4 stages (Trajectory.stages, model.py:95-97: stages[s] =
// (x1 = state, x2, x3, x4)).  The sweeps stream x1, x2, x3 and recompute only
// x4 = x1 + dt f(x3) (bit-exact, model.py:45), so
//   * per element-step each sweep reads 24 B instead of 8 (state only) or 32
//     (all four stages) -- still below the fp64 time at cfg4 sizes;
//   * the DP work drops by the two stage recomputes (12 of ~42/48 DP
//     instructions per element-step);
//   * no stage needs an exchange round: x1/x2/x3 windows come from the staged
//     tiles with +-4 halos, and x4's +-2 halo is recomputed from x3's +-4.
// The three arrays of step s+1 (TL) / s-1 (AD) are staged by coalesced
// cp.async into padded shared tiles while step s runs.  Results are
// bit-identical to the recompute-everything kernels (same arithmetic on the
// same stage values).
#include "sweep.cuh"

namespace edak {

struct SweepGeom3 {
  int W, HL, periodic, nact, pair;
};

// shared staging with a 4-element halo, padded 2 doubles per C (16-byte
// aligned runs): 16-byte cp.async pairs with immediate offsets when the
// window does not wrap and rows are 16-byte aligned (n even, even tile base),
// 8-byte copies otherwise; both fill the same layout, read with 16-byte loads
template <int C, int NT>
struct Stage4 {
  static_assert(C % 2 == 0, "pairs");
  static constexpr int H = 4;
  static constexpr int R = C * NT;
  static constexpr int NPAIR = (R + 2 * H) / 2;
  static constexpr int IT = (NPAIR + NT - 1) / NT;
  static constexpr int PLEN = (R + 2 * H) + 2 * ((R + 2 * H) / C) + 2;
  __device__ static __forceinline__ int pi(int q) { return (q + H) + 2 * ((q + H) / C); }
  // gm4 = ring index (unwrapped, may be < 0) of window element -4
  __device__ static __forceinline__ void stage(double* buf, const double* __restrict__ src, int gm4, int n,
                                               int used, bool pair) {
    const int t = threadIdx.x;
    if (pair) {
      const int np = (used + 2 * H) >> 1;
      double* d = buf + 2 * t + 2 * (t / (C / 2));
      constexpr int DSTEP = 2 * NT + 2 * (NT / (C / 2));
      if (gm4 >= 0 && gm4 + used + 2 * H <= n) {
        const double* p = src + gm4 + 2 * t;
#pragma unroll
        for (int it = 0; it < IT; ++it)
          if (t + it * NT < np) cp_async16(d + it * DSTEP, p + 2 * it * NT);
      } else {
#pragma unroll
        for (int it = 0; it < IT; ++it) {
          const int m = t + it * NT;
          if (m < np) {
            int g = gm4 + 2 * m;
            g = g < 0 ? g + n : (g >= n ? g - n : g);
            cp_async16(d + it * DSTEP, src + g);
          }
        }
      }
      return;
    }
    for (int q = t - H; q < used + H; q += NT) {
      int g = (gm4 + H + q) % n;
      if (g < 0) g += n;
      cp_async8(buf + pi(q), src + g);
    }
  }
  // window [-2, C + 2) of thread t
  __device__ static __forceinline__ void win2(const double* buf, int t, double (&a)[C + 4]) {
    const double* w = buf + (C + 2) * t;
#pragma unroll
    for (int k = 0; k < C + 4; k += 2) {
      const int off = (2 + k) + 2 * ((2 + k) / C);
      const double2 v = *reinterpret_cast<const double2*>(w + off);
      a[k] = v.x;
      a[k + 1] = v.y;
    }
  }
  // window [-4, C + 4) of thread t
  __device__ static __forceinline__ void win4(const double* buf, int t, double (&a)[C + 8]) {
    const double* w = buf + (C + 2) * t;
#pragma unroll
    for (int k = 0; k < C + 8; k += 2) {
      const int off = k + 2 * (k / C);
      const double2 v = *reinterpret_cast<const double2*>(w + off);
      a[k] = v.x;
      a[k + 1] = v.y;
    }
  }
};

// x4 on [-2, C + 2) (index m <-> element m - 2) from x3 on [-4, C + 4) and X
template <int C>
__device__ __forceinline__ void x4_from_x3(const double (&X)[C + 4], const double (&x3)[C + 8], double dt, double F,
                                           double (&x4)[C + 4]) {
#pragma unroll
  for (int m = 0; m < C + 4; ++m) {
    // element e = m - 2: x3[e+1], x3[e-2], x3[e-1], x3[e] at window index e + 4
    x4[m] = axpy_rn(X[m], dt, l96_f(x3[m + 3], x3[m], x3[m + 1], x3[m + 2], F));
  }
}

// ------------------------------------------------------------------- TL --
template <int C, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_tl3(edak_problem P, const double* __restrict__ vin,
                                                  double* __restrict__ obs, const int32_t* __restrict__ col_traj,
                                                  SweepGeom3 geo, int s0, int s1, double* __restrict__ vout) {
  using SS = Stage4<C, NT>;
  extern __shared__ __align__(16) double dsm_[];
  XBuf<NT>& xb = *reinterpret_cast<XBuf<NT>*>(dsm_);
  xb.init_pads();
  double* SB = dsm_ + sizeof(XBuf<NT>) / sizeof(double);  // [parity][3][PLEN]
  Ring<C, NT> R;
  const int n = P.n;
  const int i0 = blockIdx.x * geo.W;
  R.init(n, geo.periodic ? 0 : i0 - geo.HL, geo.nact, geo.periodic);
  const int col = blockIdx.y;
  const int wlo = geo.periodic ? 0 : geo.HL;
  const int whi = geo.periodic ? n : geo.HL + min(geo.W, n - i0);
  const int traj = col_traj ? col_traj[col] : 0;
  const double* sg = P.stages + (size_t)traj * P.traj_stride;  // [s][4][n]
  const int G = P.G;
  double* ob = obs + (size_t)col * G * P.T;
  const double dt = P.dt, h = 0.5 * dt, c6 = dt / 6.0, F = P.forcing;
  const int used = R.nact * C;
  const int gst = R.base - SS::H;
  const bool pair = geo.pair != 0;
  int buf = 0;

  int gw[C];
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const int e = R.t * C + j;
    gw[j] = (R.t < R.nact && e >= wlo && e < whi) ? __ldg(P.gpos + R.gidx(j)) : -1;
  }
  auto capture = [&](int level, const double (&v)[C + 4]) {
    const int tp = __ldg(P.tpos + level);
    if (tp < 0) return;
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (gw[j] >= 0) ob[(size_t)tp * G + gw[j]] = v[j + 2];
  };
  auto stage_step = [&](int s) {
    double* b = SB + (size_t)(s & 1) * 3 * SS::PLEN;
    const double* src = sg + (size_t)s * 4 * n;
    SS::stage(b, src, gst, n, used, pair);
    SS::stage(b + SS::PLEN, src + n, gst, n, used, pair);
    SS::stage(b + 2 * SS::PLEN, src + 2 * n, gst, n, used, pair);
    cp_commit();
  };

  double v[C + 4];
  R.load_own(vin + (size_t)col * n, v);
  if (s0 == 0) capture(0, v);
  stage_step(s0);
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    const double* b = SB + (size_t)(s & 1) * 3 * SS::PLEN;
    cp_wait_all();
    xchg1(R, xb, buf, v);  // barrier: step s tiles visible, step s-1 tiles free
    if (s + 1 < s1) stage_step(s + 1);
    double a[C], acc[C], u[C + 4], w[C + 4];
    SS::win2(b, R.t, w);  // x1 = X
#pragma unroll
    for (int j = 0; j < C; ++j) {
      a[j] = l96_tl(v[j + 3], v[j], v[j + 1], v[j + 2], w[j + 3], w[j], w[j + 1]);
      acc[j] = a[j];
      u[j + 2] = fma(h, a[j], v[j + 2]);
    }
    xchg1(R, xb, buf, u);
    SS::win2(b + SS::PLEN, R.t, w);  // x2
#pragma unroll
    for (int j = 0; j < C; ++j) {
      a[j] = l96_tl(u[j + 3], u[j], u[j + 1], u[j + 2], w[j + 3], w[j], w[j + 1]);
      acc[j] = fma(2.0, a[j], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < C; ++j) u[j + 2] = fma(h, a[j], v[j + 2]);
    xchg1(R, xb, buf, u);
    double x3[C + 8], x4[C + 4];
    SS::win4(b + 2 * SS::PLEN, R.t, x3);
#pragma unroll
    for (int j = 0; j < C; ++j) {
      a[j] = l96_tl(u[j + 3], u[j], u[j + 1], u[j + 2], x3[j + 5], x3[j + 2], x3[j + 3]);
      acc[j] = fma(2.0, a[j], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < C; ++j) u[j + 2] = fma(dt, a[j], v[j + 2]);
    SS::win2(b, R.t, w);  // X again, for x4 = X + dt f(x3)
    x4_from_x3<C>(w, x3, dt, F, x4);
    xchg1(R, xb, buf, u);
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const double a4 = l96_tl(u[j + 3], u[j], u[j + 1], u[j + 2], x4[j + 3], x4[j], x4[j + 1]);
      v[j + 2] = fma(c6, acc[j] + a4, v[j + 2]);
    }
    capture(s + 1, v);
  }
  if (vout && R.t < R.nact) {
    double* vo = vout + (size_t)col * n;
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int e = R.t * C + j;
      if (e >= wlo && e < whi) vo[R.gidx(j)] = v[j + 2];
    }
  }
}

// ------------------------------------------------------------------- AD --
template <int C>
__device__ __forceinline__ void ad_sub3(const double (&w)[C + 4], const double (&x)[C + 4], double (&u)[C]) {
#pragma unroll
  for (int j = 0; j < C; ++j)
    u[j] = l96_ad(x[j], x[j + 1], x[j + 3], x[j + 4], w[j + 1], w[j + 2], w[j + 3], w[j + 4]);
}

template <int C, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_ad3(edak_problem P, const double* __restrict__ forcing,
                                                  double* __restrict__ gout, const int32_t* __restrict__ col_traj,
                                                  SweepGeom3 geo, int s0, int s1, const double* __restrict__ gin) {
  using SS = Stage4<C, NT>;
  extern __shared__ __align__(16) double dsm_[];
  XBuf<NT>& xb = *reinterpret_cast<XBuf<NT>*>(dsm_);
  xb.init_pads();
  double* SB = dsm_ + sizeof(XBuf<NT>) / sizeof(double);
  Ring<C, NT> R;
  const int n = P.n, N = P.n_steps;
  const int i0 = blockIdx.x * geo.W;
  R.init(n, geo.periodic ? 0 : i0 - geo.HL, geo.nact, geo.periodic);
  const int col = blockIdx.y;
  const int wlo = geo.periodic ? 0 : geo.HL;
  const int whi = geo.periodic ? n : geo.HL + min(geo.W, n - i0);
  const int traj = col_traj ? col_traj[col] : 0;
  const double* sg = P.stages + (size_t)traj * P.traj_stride;
  const int G = P.G;
  const double* fc = forcing + (size_t)col * G * P.T;
  const double dt = P.dt, F = P.forcing, h = 0.5 * dt;
  const double c6 = dt / 6.0, c3 = 2.0 * dt / 6.0;
  const double inv_s2 = 1.0 / P.sigma2;
  const int used = R.nact * C;
  const int gst = R.base - SS::H;
  const bool pair = geo.pair != 0;
  int buf = 0;

  int gp[C];
#pragma unroll
  for (int j = 0; j < C; ++j) gp[j] = __ldg(P.gpos + R.gidx(j));
  auto add_force = [&](int level, double (&gg)[C + 4]) {
    const int tp = __ldg(P.tpos + level);
    if (tp < 0) return;
    const double* f = fc + (size_t)tp * G;
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (gp[j] >= 0) gg[j + 2] += __ldg(f + gp[j]) * inv_s2;
  };
  auto stage_step = [&](int s) {
    double* b = SB + (size_t)(s & 1) * 3 * SS::PLEN;
    const double* src = sg + (size_t)s * 4 * n;
    SS::stage(b, src, gst, n, used, pair);
    SS::stage(b + SS::PLEN, src + n, gst, n, used, pair);
    SS::stage(b + 2 * SS::PLEN, src + 2 * n, gst, n, used, pair);
    cp_commit();
  };

  double g[C + 4];
  if (gin) {
    R.load_own(gin + (size_t)col * n, g);
  } else {
#pragma unroll
    for (int j = 0; j < C; ++j) g[j + 2] = 0.0;
    add_force(N, g);
  }
  stage_step(s1 - 1);
  cp_wait_all();
  __syncthreads();

#pragma unroll 1
  for (int s = s1 - 1; s >= s0; --s) {
    const double* b = SB + (size_t)(s & 1) * 3 * SS::PLEN;
    xchg1(R, xb, buf, g);  // g halo; every thread is done with step s+1's tiles
    if (s > s0) stage_step(s - 1);
    double vh[C], u[C], a[C + 4];
    {
      double w[C + 4], x3[C + 8], x4[C + 4];
      SS::win2(b, R.t, w);
      SS::win4(b + 2 * SS::PLEN, R.t, x3);
      x4_from_x3<C>(w, x3, dt, F, x4);
#pragma unroll
      for (int k = 0; k < C + 4; ++k) a[k] = c6 * g[k];  // a4 = (dt/6) w
      ad_sub3<C>(a, x4, u);
    }
#pragma unroll
    for (int j = 0; j < C; ++j) {
      vh[j] = g[j + 2] + u[j];
      a[j + 2] = fma(dt, u[j], c3 * g[j + 2]);  // a3
    }
    xchg1(R, xb, buf, a);
    {
      double x3[C + 8], w[C + 4];
      SS::win4(b + 2 * SS::PLEN, R.t, x3);
#pragma unroll
      for (int k = 0; k < C + 4; ++k) w[k] = x3[k + 2];
      ad_sub3<C>(a, w, u);
    }
#pragma unroll
    for (int j = 0; j < C; ++j) {
      vh[j] += u[j];
      a[j + 2] = fma(h, u[j], c3 * g[j + 2]);  // a2
    }
    xchg1(R, xb, buf, a);
    {
      double w[C + 4];
      SS::win2(b + SS::PLEN, R.t, w);
      ad_sub3<C>(a, w, u);
    }
#pragma unroll
    for (int j = 0; j < C; ++j) {
      vh[j] += u[j];
      a[j + 2] = fma(h, u[j], c6 * g[j + 2]);  // a1
    }
    cp_wait_all();          // step s-1 tiles landed ...
    xchg1(R, xb, buf, a);   // ... and are visible after this barrier
    {
      double w[C + 4];
      SS::win2(b, R.t, w);
      ad_sub3<C>(a, w, u);
    }
#pragma unroll
    for (int j = 0; j < C; ++j) g[j + 2] = vh[j] + u[j];
    add_force(s, g);
  }
  if (R.t < R.nact) {
    double* go = gout + (size_t)col * n;
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int e = R.t * C + j;
      if (e >= wlo && e < whi) go[R.gidx(j)] = g[j + 2];
    }
  }
}

// ------------------------------------------------------------ launchers --
template <int C, int NT>
static size_t smem3() {
  return sizeof(XBuf<NT>) + 2 * 3 * Stage4<C, NT>::PLEN * sizeof(double);
}

template <typename K>
static void attr3(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

static int env3(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// C = 8, NT = 128 tiles (range 1024) or periodic rings n = 8 * nact,
// 64 <= nact <= 128.  Returns false when the family does not apply.
static bool plan3(int n, int hl, int hr, SweepGeom3& geo, int& nt) {
  constexpr int C = 8, NT = 128, RNG = C * NT;
  if (n % C == 0 && n / C <= NT && n / C >= 64) {
    geo = {n, 0, 1, n / C, n % 2 == 0};
    nt = 1;
    return true;
  }
  if (n < RNG + 64) return false;
  const int W = RNG - hl - hr;
  if (W < 256) return false;
  nt = (n + W - 1) / W;
  int Wt = ((n + nt - 1) / nt + 1) & ~1;  // even tile width (pair staging)
  if (Wt > W) Wt = W;
  geo = {Wt, hl, 0, NT, (n % 2 == 0 && Wt % 2 == 0 && hl % 2 == 0) ? 1 : 0};
  return true;
}

int sweep3_mode(const edak_problem* P, int K) {
  if (P->stage_mode != 2) return 0;
  SweepGeom3 geo;
  int nt;
  if (!plan3(P->n, 8 * K + 8, 8 * K + 8, geo, nt)) return 0;
  return geo.periodic ? 1 : 2;
}

int launch_tl3(const edak_problem* P, const double* vin, double* obs, int ncols, const int32_t* col_traj, int s0,
               int s1, double* vout, cudaStream_t st) {
  SweepGeom3 geo;
  int nt;
  const int K = s1 - s0;
  if (!plan3(P->n, 8 * K + 4, 4 * K + 4, geo, nt)) return EDAK_EUNSUPPORTED;
  if (((uintptr_t)P->stages & 15) || (P->traj_stride & 1) || getenv("EDAK_NO_PAIR")) geo.pair = 0;
  const size_t sm = smem3<8, 128>();
  if (env3("EDAK_TL3_MINB", 4) == 3) {
    attr3(k_tl3<8, 128, 3>, sm);
    k_tl3<8, 128, 3><<<dim3(nt, ncols), 128, sm, st>>>(*P, vin, obs, col_traj, geo, s0, s1, vout);
  } else {
    attr3(k_tl3<8, 128, 4>, sm);
    k_tl3<8, 128, 4><<<dim3(nt, ncols), 128, sm, st>>>(*P, vin, obs, col_traj, geo, s0, s1, vout);
  }
  count_launch();
  return check_launch("k_tl3");
}

int launch_ad3(const edak_problem* P, const double* forcing, double* gout, int ncols, const int32_t* col_traj,
               int s0, int s1, const double* gin, cudaStream_t st) {
  SweepGeom3 geo;
  int nt;
  const int K = s1 - s0;
  if (!plan3(P->n, 4 * K + 8, 8 * K + 8, geo, nt)) return EDAK_EUNSUPPORTED;
  if (((uintptr_t)P->stages & 15) || (P->traj_stride & 1) || getenv("EDAK_NO_PAIR")) geo.pair = 0;
  const size_t sm = smem3<8, 128>();
  if (env3("EDAK_AD3_MINB", 3) == 2) {
    attr3(k_ad3<8, 128, 2>, sm);
    k_ad3<8, 128, 2><<<dim3(nt, ncols), 128, sm, st>>>(*P, forcing, gout, col_traj, geo, s0, s1, gin);
  } else {
    attr3(k_ad3<8, 128, 3>, sm);
    k_ad3<8, 128, 3><<<dim3(nt, ncols), 128, sm, st>>>(*P, forcing, gout, col_traj, geo, s0, s1, gin);
  }
  count_launch();
  return check_launch("k_ad3");
}

}  // namespace edak
