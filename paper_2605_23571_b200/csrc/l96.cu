// Lorenz-96 window sweeps on sm_100a:
//   k_integrate : nonlinear RK4 producer, bit-exact with model.integrate
//                 (model.py:38-48,118-131)
//   k_tl        : tangent-linear sweep + time-major observation capture
//                 (model.tlm + ObsNetwork.observe_tlm, model.py:56-63,134-144,
//                 obs.py:47-50)
//   k_ad        : adjoint sweep with observation forcing
//                 (model.adjoint + ObsNetwork.observe_adj, model.py:66-84,
//                 147-157, obs.py:52-57)
// The sweeps recompute the RK4 stages from the stored states (16 B/elem-step
// of HBM instead of 64) with the contracted chain stg_* of common.cuh: within
// ~1 ulp of the reference's stored stages, restarted from the exact state at
// every step (EDAK_STAGE_FMA=0: the IEEE-ordered chain, bit for bit);
// STREAM=true reads stored stages instead.
#include <cstdio>
#include <cstdlib>

#include "sweep.cuh"
#include <type_traits>

namespace edak {


// ------------------------------------------------------------------ RK4 --

// One RK4 stage chain on own elements.  x (with halo) -> (k, x + c*k)
template <int C>
__device__ __forceinline__ void l96_stage(const double (&x)[C + 4], const double (&X)[C + 4], double c,
                                          double F, double (&kk)[C], double (&xn)[C + 4]) {
#pragma unroll
  for (int j = 0; j < C; ++j) {
    kk[j] = l96_f(x[j + 3], x[j], x[j + 1], x[j + 2], F);
    xn[j + 2] = axpy_rn(X[j + 2], c, kk[j]);
  }
}

template <int C, int NT>
__global__ void __launch_bounds__(NT) k_integrate(int n, int K, int s0, double dt, double F,
                                                  const double* __restrict__ xin, int64_t in_stride,
                                                  double* __restrict__ states, int64_t st_stride,
                                                  double* __restrict__ stages, int64_t sg_stride,
                                                  SweepGeom geo) {
  extern __shared__ __align__(16) double dsm_[];
  XBuf<NT>& xb = *reinterpret_cast<XBuf<NT>*>(dsm_);
  xb.init_pads();
  Ring<C, NT> R;
  const int i0 = blockIdx.x * geo.W;
  R.init(n, geo.periodic ? 0 : i0 - geo.HL, geo.nact, geo.periodic);
  const int col = blockIdx.y;
  const int wlo = geo.periodic ? 0 : geo.HL;
  const int whi = geo.periodic ? n : geo.HL + min(geo.W, n - i0);
  const double h = 0.5 * dt, c6 = dt / 6.0;
  double* st = states + (size_t)col * st_stride;
  double* sg = stages ? stages + (size_t)col * sg_stride : nullptr;
  int buf = 0;

  double x[C + 4];
  {
    // 16-byte pairs where the window does not wrap and the row is 16-byte
    // aligned (even C, ring bases and n: every tile base is even), else the
    // scalar loads
    const double* src = xin + (size_t)col * in_stride;
    const int g = R.g0 >= 2 ? R.g0 - 2 : R.g0 - 2 + n;
    if (C % 2 == 0 && g % 2 == 0 && g + C + 4 <= n && ((uintptr_t)src & 15) == 0) {
#pragma unroll
      for (int k = 0; k < (C + 4) / 2; ++k) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(src + g) + k);
        x[2 * k] = v.x;
        x[2 * k + 1] = v.y;
      }
    } else {
      R.load_halo(src, x);
    }
  }
  for (int s = 0; s < K; ++s) {
    double k1[C], k2[C], k3[C], k4[C], x2[C + 4], x3[C + 4], x4[C + 4];
    l96_stage<C>(x, x, h, F, k1, x2);
    xchg1(R, xb, buf, x2);
    l96_stage<C>(x2, x, h, F, k2, x3);
    xchg1(R, xb, buf, x3);
    l96_stage<C>(x3, x, dt, F, k3, x4);
    xchg1(R, xb, buf, x4);
    double xn[C + 4];
#pragma unroll
    for (int j = 0; j < C; ++j) {
      k4[j] = l96_f(x4[j + 3], x4[j], x4[j + 1], x4[j + 2], F);
      // x + (dt/6) * (((k1 + 2 k2) + 2 k3) + k4)   (model.py:47)
      double sum = __dadd_rn(__dadd_rn(__dadd_rn(k1[j], 2.0 * k2[j]), 2.0 * k3[j]), k4[j]);
      xn[j + 2] = __dadd_rn(x[j + 2], __dmul_rn(c6, sum));
    }
    // store own elements inside the output window (16-byte pairs when the
    // row, the thread's first element and the window bounds are even)
    double* srow = st + (size_t)(s0 + s + 1) * n;
    if (R.t < R.nact && !sg && C % 2 == 0 && n % 2 == 0 && R.g0 % 2 == 0 && wlo % 2 == 0 && whi % 2 == 0 &&
        ((uintptr_t)srow & 15) == 0) {
#pragma unroll
      for (int k = 0; k < C / 2; ++k) {
        const int e = R.t * C + 2 * k;
        const int g = R.gidx(2 * k);
        if (e >= wlo && e < whi && g + 1 < n)
          *reinterpret_cast<double2*>(srow + g) = make_double2(xn[2 * k + 2], xn[2 * k + 3]);
        else if (e >= wlo && e < whi) {
          srow[g] = xn[2 * k + 2];
          srow[R.gidx(2 * k + 1)] = xn[2 * k + 3];
        }
      }
    } else if (R.t < R.nact) {
#pragma unroll
      for (int j = 0; j < C; ++j) {
        const int e = R.t * C + j;
        if (e >= wlo && e < whi) {
          const int g = R.gidx(j);
          st[(size_t)(s0 + s + 1) * n + g] = xn[j + 2];
          if (sg) {
            double* o = sg + (size_t)(s0 + s) * 4 * n + g;
            o[0] = x[j + 2];
            o[n] = x2[j + 2];
            o[2 * n] = x3[j + 2];
            o[3 * n] = x4[j + 2];
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < C; ++j) x[j + 2] = xn[j + 2];
    if (s + 1 < K) xchg1(R, xb, buf, x);
  }
}

// ------------------------------------------------------------------- TL --

template <int C>
__device__ __forceinline__ void tl_sub(const double (&u)[C + 4], const double (&x)[C + 4], double (&a)[C]) {
#pragma unroll
  for (int j = 0; j < C; ++j)
    a[j] = l96_tl(u[j + 3], u[j], u[j + 1], u[j + 2], x[j + 3], x[j], x[j + 1]);
}
// the same with the stage's differences d[j] = x[j+3] - x[j] precomputed
template <int C>
__device__ __forceinline__ void tl_sub_d(const double (&u)[C + 4], const double (&x)[C + 4], const double (&d)[C],
                                         double (&a)[C]) {
#pragma unroll
  for (int j = 0; j < C; ++j) a[j] = l96_tl_d(u[j + 3], u[j], u[j + 1], u[j + 2], d[j], x[j + 1]);
}

// WT: warp tile (NT == 32): halos by shuffles, no CTA barrier (sweep.cuh)
template <int C, int NT, bool STREAM, int MINB = 1, bool PAIR = false, int DEPTH = 1, bool WT = false>
__global__ void __launch_bounds__(NT, MINB) k_tl(edak_problem P, const double* __restrict__ vin,
                                           double* __restrict__ obs, const int32_t* __restrict__ col_traj,
                                           SweepGeom geo, int s0, int s1, double* __restrict__ vout) {
  static_assert(!WT || (NT == 32 && PAIR && !STREAM), "warp tiles: one warp, pair staging");
  extern __shared__ __align__(16) double dsm_[];
  XBuf<NT>& xb = *reinterpret_cast<XBuf<NT>*>(dsm_);
  if (!WT) xb.init_pads();
  Ring<C, NT> R;
  const int n = P.n;
  const int i0 = blockIdx.x * geo.W;
  R.init(n, geo.periodic ? 0 : i0 - geo.HL, geo.nact, geo.periodic);
  const int col = blockIdx.y;
  const int wlo = geo.periodic ? 0 : geo.HL;
  const int whi = geo.periodic ? n : geo.HL + min(geo.W, n - i0);
  const int traj = col_traj ? col_traj[col] : 0;
  const double* tr = (STREAM ? P.stages : P.states) + (size_t)traj * P.traj_stride;
  const int G = P.G;
  double* ob = obs + (size_t)col * G * P.T;
  const double dt = P.dt, h = 0.5 * dt, c6 = dt / 6.0, F = P.forcing;
  int buf = 0;

  // window chunk [s0, s1): v enters at level s0 and leaves at level s1
  double v[C + 4];
  R.load_own2(vin + (size_t)col * n, v);

  // observed own elements inside the output window: grid position or -1
  int gw[C];
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const int e = R.t * C + j;
    gw[j] = (R.t < R.nact && e >= wlo && e < whi) ? __ldg(P.gpos + R.gidx(j)) : -1;
  }
  auto capture_tp = [&](int tp) {
#ifdef EDAK_EXP_NOCAPTURE  // timing ablation (wrong results): no observation capture / forcing
    return;
#endif
    if (tp < 0) return;
    double* ot = ob + (size_t)tp * G;  // one base per level, 32-bit grid offsets
    asm("" : "+l"(ot));  // opaque: keeps ptxas from re-expanding a 64-bit index per element
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (gw[j] >= 0) ot[gw[j]] = v[j + 2];
  };
  auto capture = [&](int level) {
    const int tp = __ldg(P.tpos + level);
    if (tp < 0) return;
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (gw[j] >= 0) ob[(size_t)tp * G + gw[j]] = v[j + 2];
  };
  if (s0 == 0) capture(0);

  // software pipeline: the state of step s+1 is staged (cp.async, coalesced)
  // into the other shared buffer while step s runs; STREAM reads stored
  // stages straight from memory
  // DEPTH = 1: X_{s+1} is staged during step s (two buffers); DEPTH = 2: X_{s+2}
  // (three buffers, one empty commit group past the window end so that
  // wait_group DEPTH - 1 always means "X_s has landed")
  using SS = std::conditional_t<PAIR, Stage2<C, NT>, Stage<C, NT>>;
  constexpr int NB = DEPTH + 1;
  double* XB0 = dsm_ + (WT ? 0 : sizeof(XBuf<NT>) / sizeof(double));
  const int used = R.nact * C;
  const int gst = PAIR ? R.base - 2 : wrap(R.base - 2 + (int)threadIdx.x, n);
  const size_t sstride = STREAM ? (size_t)4 * n : (size_t)n;
  auto sbuf = [&](int level) { return XB0 + (size_t)(level % NB) * SS::PLEN; };
  auto X1 = [&](double (&a)[C + 4]) {
    if constexpr (WT) wxchg1<C>(a); else xchg1(R, xb, buf, a);
  };
  auto X2 = [&](double (&a)[C + 4], double (&b)[C + 4]) {
    if constexpr (WT) { wxchg1<C>(a); wxchg1<C>(b); } else xchg2(R, xb, buf, a, b);
  };
  if (!STREAM) {
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      if (s0 + d < s1) SS::stage(sbuf(s0 + d), tr + (size_t)(s0 + d) * n, gst, n, used);
      else cp_commit();
    }
  }
  // running pointers / buffer indices (no per-step 64-bit index math or
  // modulo; the asm keeps ptxas from re-deriving them from s)
  const double* nsrc = tr + (size_t)(s0 + DEPTH) * n;
  const int32_t* tpp = P.tpos + s0 + 1;
  int bcur = s0 % NB, bnext = (s0 + DEPTH) % NB;
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    const double* Xs = tr + (size_t)s * sstride;
    asm("" : "+l"(nsrc), "+l"(tpp));
    const int tp_next = __ldg(tpp);  // consumed at the end of the step
    double X[C + 4];
    if (!STREAM) cp_wait_group<DEPTH - 1>();
    if constexpr (WT) __syncwarp();  // staged X_s visible, X_{s-1}'s buffer free
    X1(v);  // (CTA tiles: its barrier does the same)
    if (STREAM) {
      R.load_halo(Xs, X);
    } else {
      if (s + DEPTH < s1) SS::stage(XB0 + (size_t)bnext * SS::PLEN, nsrc, gst, n, used);
      else if (DEPTH > 1) cp_commit();
      SS::win(XB0 + (size_t)bcur * SS::PLEN, R.t, X);
    }
    nsrc += n;
    ++tpp;
    bcur = bcur + 1 == NB ? 0 : bcur + 1;
    bnext = bnext + 1 == NB ? 0 : bnext + 1;
    double acc[C], a[C], kk[C], dd[C];
    double x2[C + 4], u2[C + 4];
#pragma unroll
    for (int j = 0; j < C; ++j) dd[j] = __dsub_rn(X[j + 3], X[j]);
    tl_sub_d<C>(v, X, dd, a);
    if (STREAM) {
      R.load_halo(Xs + n, x2);
    } else {
#pragma unroll
      for (int j = 0; j < C; ++j) {
        kk[j] = stg_f_d(dd[j], X[j + 1], X[j + 2], F);
        x2[j + 2] = stg_axpy(X[j + 2], h, kk[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < C; ++j) {
      acc[j] = a[j];
      u2[j + 2] = fma(h, a[j], v[j + 2]);
    }
    if (STREAM) X1(u2); else X2(x2, u2);

    double x3[C + 4], u3[C + 4];
#pragma unroll
    for (int j = 0; j < C; ++j) dd[j] = __dsub_rn(x2[j + 3], x2[j]);
    tl_sub_d<C>(u2, x2, dd, a);
    if (STREAM) {
      R.load_halo(Xs + 2 * n, x3);
    } else {
#pragma unroll
      for (int j = 0; j < C; ++j) {
        kk[j] = stg_f_d(dd[j], x2[j + 1], x2[j + 2], F);
        x3[j + 2] = stg_axpy(X[j + 2], h, kk[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < C; ++j) {
      acc[j] = fma(2.0, a[j], acc[j]);
      u3[j + 2] = fma(h, a[j], v[j + 2]);
    }
    if (STREAM) X1(u3); else X2(x3, u3);

    double x4[C + 4], u4[C + 4];
#pragma unroll
    for (int j = 0; j < C; ++j) dd[j] = __dsub_rn(x3[j + 3], x3[j]);
    tl_sub_d<C>(u3, x3, dd, a);
    if (STREAM) {
      R.load_halo(Xs + 3 * n, x4);
    } else {
#pragma unroll
      for (int j = 0; j < C; ++j) {
        kk[j] = stg_f_d(dd[j], x3[j + 1], x3[j + 2], F);
        x4[j + 2] = stg_axpy(X[j + 2], dt, kk[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < C; ++j) {
      acc[j] = fma(2.0, a[j], acc[j]);
      u4[j + 2] = fma(dt, a[j], v[j + 2]);
    }
    if (STREAM) X1(u4); else X2(x4, u4);

    tl_sub<C>(u4, x4, a);
#pragma unroll
    for (int j = 0; j < C; ++j) v[j + 2] = fma(c6, acc[j] + a[j], v[j + 2]);
    capture_tp(tp_next);
  }
  if (vout && R.t < R.nact) R.store_own(vout + (size_t)col * n, v, wlo, whi);
}

// ------------------------------------------------------------------- AD --

template <int C>
__device__ __forceinline__ void ad_sub(const double (&w)[C + 4], const double (&x)[C + 4], double (&u)[C]) {
#pragma unroll
  for (int j = 0; j < C; ++j)
    u[j] = l96_ad(x[j], x[j + 1], x[j + 3], x[j + 4], w[j + 1], w[j + 2], w[j + 3], w[j + 4]);
}

template <int C, int NT, bool STREAM, int MINB = 1, bool PAIR = false, int DEPTH = 1, bool WT = false>
__global__ void __launch_bounds__(NT, MINB) k_ad(edak_problem P, const double* __restrict__ forcing,
                                           double* __restrict__ gout, const int32_t* __restrict__ col_traj,
                                           SweepGeom geo, int s0, int s1, const double* __restrict__ gin) {
  static_assert(!WT || (NT == 32 && PAIR && !STREAM), "warp tiles: one warp, pair staging");
  extern __shared__ __align__(16) double dsm_[];
  XBuf<NT>& xb = *reinterpret_cast<XBuf<NT>*>(dsm_);
  if (!WT) xb.init_pads();
  Ring<C, NT> R;
  const int n = P.n, N = P.n_steps;
  const int i0 = blockIdx.x * geo.W;
  R.init(n, geo.periodic ? 0 : i0 - geo.HL, geo.nact, geo.periodic);
  const int col = blockIdx.y;
  const int wlo = geo.periodic ? 0 : geo.HL;
  const int whi = geo.periodic ? n : geo.HL + min(geo.W, n - i0);
  const int traj = col_traj ? col_traj[col] : 0;
  const double* tr = (STREAM ? P.stages : P.states) + (size_t)traj * P.traj_stride;
  const int G = P.G;
  const double* fc = forcing + (size_t)col * G * P.T;
  const double dt = P.dt, h = 0.5 * dt, F = P.forcing;
  const double c6 = dt / 6.0, s2 = P.sigma2;
  int buf = 0;

  // forcing w_all[level] at own elements: R^-1 d at observed points
  // (obs.py:54-56 with covariance.py:71: w / sigma**2), 0 elsewhere
  double* FS = dsm_ + (WT ? 0 : sizeof(XBuf<NT>) / sizeof(double)) + (DEPTH + 1) * Stage2<C, NT>::PLEN;
  int gp[C];
#pragma unroll
  for (int j = 0; j < C; ++j) gp[j] = __ldg(P.gpos + R.gidx(j));
  auto is_obs = [&](int j) { return gp[j] >= 0; };
  auto gpos_of = [&](int j) { return gp[j]; };
  // (the reference divides by sigma**2; we multiply by its reciprocal, a
  // 0.5-ulp difference inside the 1e-12 parity budget, and hoist the level
  // lookup: an IEEE division per observed element cost ~12 DP instructions)
  const double inv_s2 = 1.0 / s2;
  auto add_force = [&](int level, double (&gg)[C + 4]) {
    const int tp = __ldg(P.tpos + level);
    if (tp < 0) return;
    const double* f = fc + (size_t)tp * G;
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (is_obs(j)) gg[j + 2] += __ldg(f + gpos_of(j)) * inv_s2;
  };
  // PAIR path: the forcing of level s is fetched by cp.async into per-thread
  // smem slots at the start of step s (with the next state tile) and added at
  // its end, so its global latency hides behind the step instead of stalling
  // every warp of the CTA at once (long_scoreboard in the ncu profile)
  auto fetch_force = [&](int tp, int sbuf) {
#ifdef EDAK_EXP_NOCAPTURE
    return;
#endif
    if (tp < 0) return;
    const double* f = fc + (size_t)tp * G;
    asm("" : "+l"(f));  // opaque base: 32-bit grid offsets per element (see k_tl capture)
    double* d = FS + (size_t)sbuf * C * NT + threadIdx.x;
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (is_obs(j)) cp_async8(d + j * NT, f + gpos_of(j));
  };
  auto add_fetched = [&](int tp, int sbuf, double (&gg)[C + 4]) {
#ifdef EDAK_EXP_NOCAPTURE
    return;
#endif
    if (tp < 0) return;
    const double* d = FS + (size_t)sbuf * C * NT + threadIdx.x;
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (is_obs(j)) gg[j + 2] += d[j * NT] * inv_s2;
  };

  // window chunk [s0, s1), swept backward: g enters at level s1 (w_all[N]
  // when s1 == N, model.py:154) and leaves at level s0
  double g[C + 4];
  if (gin) {
    R.load_own2(gin + (size_t)col * n, g);
  } else {
#pragma unroll
    for (int j = 0; j < C; ++j) g[j + 2] = 0.0;
    add_force(N, g);
  }

  // DEPTH = 1: X_{s-1} (and the forcing of level s-1) is staged during step s
  // into the buffer X_{s+1} used.  DEPTH = 2: X_{s-2} is staged during step s
  // (three buffers); the forcing of level s is fetched at the start of step s
  // into per-thread slots, in its own commit group ahead of X_{s-2}'s, so the
  // end-of-step wait_group 1 covers both it and X_{s-1}
  using SS = std::conditional_t<PAIR, Stage2<C, NT>, Stage<C, NT>>;
  constexpr int NB = DEPTH + 1;
  double* XB0 = dsm_ + (WT ? 0 : sizeof(XBuf<NT>) / sizeof(double));
  const int used = R.nact * C;
  const int gst = PAIR ? R.base - 2 : wrap(R.base - 2 + (int)threadIdx.x, n);
  const size_t sstride = STREAM ? (size_t)4 * n : (size_t)n;
  auto sbuf = [&](int level) { return XB0 + (size_t)(level % NB) * SS::PLEN; };
  auto X1 = [&](double (&a)[C + 4]) {
    if constexpr (WT) wxchg1<C>(a); else xchg1(R, xb, buf, a);
  };
  int tp_cur = PAIR ? __ldg(P.tpos + s1 - 1) : -1;
  if (!STREAM) {
    if (DEPTH == 1) {
      if (PAIR) fetch_force(tp_cur, (s1 - 1) & 1);
      SS::stage(sbuf(s1 - 1), tr + (size_t)(s1 - 1) * n, gst, n, used);
      cp_wait_all();
    } else {
      SS::stage(sbuf(s1 - 1), tr + (size_t)(s1 - 1) * n, gst, n, used);
      if (s1 - 2 >= s0) SS::stage(sbuf(s1 - 2), tr + (size_t)(s1 - 2) * n, gst, n, used);
      else cp_commit();
      cp_wait_group<1>();
    }
    if constexpr (WT) __syncwarp(); else __syncthreads();
  }
  const double* psrc = tr + (size_t)(s1 - 2) * n;  // X_{s-1}: running pointer (see k_tl)
  const int32_t* tpp = P.tpos + s1 - 2;
#pragma unroll 1
  for (int s = s1 - 1; s >= s0; --s) {
    const double* Xs = tr + (size_t)s * sstride;
    asm("" : "+l"(psrc), "+l"(tpp));
    const int tp_next = (PAIR && s > s0) ? __ldg(tpp) : -1;
    double X[C + 4], x2[C + 4], x3[C + 4], x4[C + 4];
    if (STREAM) R.load_halo(Xs, X);
    else SS::win(sbuf(s), R.t, X);  // staged, published by the last barrier
    if (STREAM) {
      R.load_halo(Xs + n, x2);
      R.load_halo(Xs + 2 * n, x3);
      R.load_halo(Xs + 3 * n, x4);
      X1(g);
    } else {
#pragma unroll
      for (int j = 0; j < C; ++j) x2[j + 2] = stg_axpy(X[j + 2], h, stg_f(X[j + 3], X[j], X[j + 1], X[j + 2], F));
      if constexpr (WT) {
        wxchg1<C>(x2);
        wxchg1<C>(g);
        __syncwarp();  // every lane is done reading step s + 1's buffer
      } else {
        xchg2(R, xb, buf, x2, g);
      }
      if (DEPTH == 1) {
        // X_{s-1} goes to the buffer X_{s+1} used: every thread read it last step
        if (s > s0) {
          if (PAIR) fetch_force(tp_next, (s - 1) & 1);  // same commit group as X_{s-1}
          SS::stage(sbuf(s - 1), STREAM ? Xs - n : psrc, gst, n, used);
        }
      } else {
        // X_{s-2} goes to the buffer X_{s+1} used (every thread is past this
        // step's first barrier, so done with step s + 1)
        if (PAIR) fetch_force(tp_cur, 0);
        cp_commit();
        if (s - 2 >= s0) SS::stage(sbuf(s - 2), Xs - 2 * n, gst, n, used);
        else cp_commit();
      }
#pragma unroll
      for (int j = 0; j < C; ++j)
        x3[j + 2] = stg_axpy(X[j + 2], h, stg_f(x2[j + 3], x2[j], x2[j + 1], x2[j + 2], F));
      X1(x3);
#pragma unroll
      for (int j = 0; j < C; ++j)
        x4[j + 2] = stg_axpy(X[j + 2], dt, stg_f(x3[j + 3], x3[j], x3[j + 1], x3[j + 2], F));
      X1(x4);
    }
    // step_adj (model.py:66-84): with w = (dt/6) g and c3 = 2 c6, dt = 2h,
    //   a3 = dt u4 + c3 g = 2 b3,  b3 = h u4 + w   (u3 = 2 J3^T b3)
    //   a2 = h u3 + c3 g  = 2 b2,  b2 = h u3' + w  (u2 = 2 J2^T b2)
    //   a1 = h u2 + c6 g  = dt u2' + w
    // so the powers of two fold into the vh accumulation (exact scalings) and
    // only w, not g, stays live through the stages
    double vh[C], u[C], a[C + 4], w[C];
#pragma unroll
    for (int k = 0; k < C + 4; ++k) a[k] = c6 * g[k];  // a4 = (dt/6) g, halo included
#pragma unroll
    for (int j = 0; j < C; ++j) w[j] = a[j + 2];
    ad_sub<C>(a, x4, u);
#pragma unroll
    for (int j = 0; j < C; ++j) {
      vh[j] = g[j + 2] + u[j];
      a[j + 2] = fma(h, u[j], w[j]);  // b3
    }
    X1(a);
    ad_sub<C>(a, x3, u);  // u3'
#pragma unroll
    for (int j = 0; j < C; ++j) {
      vh[j] = fma(2.0, u[j], vh[j]);
      a[j + 2] = fma(h, u[j], w[j]);  // b2
    }
    X1(a);
    ad_sub<C>(a, x2, u);  // u2'
#pragma unroll
    for (int j = 0; j < C; ++j) {
      vh[j] = fma(2.0, u[j], vh[j]);
      a[j + 2] = fma(dt, u[j], w[j]);  // a1
    }
    if (!STREAM) {  // X_{s-1} landed; published by this barrier
      if (DEPTH == 1) cp_wait_all();
      else cp_wait_group<1>();
      if constexpr (WT) __syncwarp();
    }
    X1(a);
    ad_sub<C>(a, X, u);
#pragma unroll
    for (int j = 0; j < C; ++j) g[j + 2] = vh[j] + u[j];
    if (PAIR) {
      add_fetched(tp_cur, DEPTH == 1 ? (s & 1) : 0, g);
      tp_cur = tp_next;
    } else {
      add_force(s, g);
    }
    psrc -= n;
    --tpp;
  }
  if (R.t < R.nact) R.store_own(gout + (size_t)col * n, g, wlo, whi);
}

// ------------------------------------------------------------ launchers --

// opt a kernel into > 48 KB of dynamic shared memory (idempotent)
template <int NT, int C = 0, int EXTRA = 0, int NSB = 2, bool XB = true, typename K, typename... Args>
static void go(K kernel, dim3 grid, cudaStream_t st, Args... args) {
  const size_t bytes = (XB ? sizeof(XBuf<NT>) : 0) +
                       (C ? NSB * (size_t)Stage2<C ? (C + 1) / 2 * 2 : 2, NT>::PLEN * sizeof(double) : 0) +
                       (size_t)EXTRA * sizeof(double);
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  kernel<<<grid, NT, bytes, st>>>(args...);
}

// pick (C, NT) and tile geometry for a sweep with halos (hl, hr) per step
static int env_int(const char* name, int dflt);

static bool plan(int n, int hl_total, int hr_total, int& C, int& NT, SweepGeom& geo, int& ntiles,
                 bool sweep = true, int force_c = 0, int force_nt = 0) {
  // periodic single tile: the whole ring in one CTA (no halo redundancy)
  const int cand_p[][2] = {{8, 128}, {4, 64}, {4, 128}, {4, 256}, {4, 512},
                           {2, 64}, {2, 128}, {2, 256}, {2, 512}};
  for (auto& f : cand_p) {
    if (n % f[0] == 0 && n / f[0] <= f[1] && n / f[0] >= 2 && (f[0] < 8 || n / f[0] >= 64)) {
      C = f[0];
      NT = f[1];
      geo.W = n;
      geo.HL = 0;
      geo.periodic = 1;
      geo.nact = n / C;
      ntiles = 1;
      return true;
    }
  }
  // tile mode: C = 8 elements per thread, 128 threads (range 1024) measured
  // fastest on B200 for the cfg4 sweeps (tools/ab_sweeps.py, profiles/)
  C = 8;
  NT = 128;
  const char* f = sweep && !force_c ? getenv("EDAK_SWEEP_FAMILY") : nullptr;
  if (force_c) {
    C = force_c;
    NT = force_nt;
  } else if (f) {  // A/B testing of the TL/AD sweeps: "C,NT"
    int c2 = 0, t2 = 0;
    if (sscanf(f, "%d,%d", &c2, &t2) == 2) {
      C = c2;
      NT = t2;
    }
  }
  int range = C * NT;
  if (range - hl_total - hr_total < 256) {  // long windows: widen the range
    C = 4;
    NT = 512;
    range = C * NT;
  }
  const int W = range - hl_total - hr_total;
  if (W < 64) return false;
  ntiles = (n + W - 1) / W;
  if (sweep) {  // A/B: more, narrower tiles per column (wave quantisation of a member group's launch)
    const int tmin = env_int("EDAK_SWEEP_TILES", 0);
    if (tmin > ntiles && n / tmin >= 64) ntiles = tmin;
  }
  geo.W = ((n + ntiles - 1) / ntiles + 1) & ~1;  // balanced tiles, even width (W budget is even)
  if (geo.W > W) geo.W = W;
  geo.HL = hl_total;
  geo.periodic = 0;
  geo.nact = NT;
  return true;
}

#define EDAK_DISPATCH(C_, NT_, ...)                                   \
  if (C_ == 4 && NT_ == 64) { constexpr int CC = 4, TT = 64; __VA_ARGS__; }   \
  else if (C_ == 4 && NT_ == 128) { constexpr int CC = 4, TT = 128; __VA_ARGS__; } \
  else if (C_ == 4 && NT_ == 256) { constexpr int CC = 4, TT = 256; __VA_ARGS__; } \
  else if (C_ == 4 && NT_ == 512) { constexpr int CC = 4, TT = 512; __VA_ARGS__; } \
  else if (C_ == 2 && NT_ == 64) { constexpr int CC = 2, TT = 64; __VA_ARGS__; }   \
  else if (C_ == 2 && NT_ == 128) { constexpr int CC = 2, TT = 128; __VA_ARGS__; } \
  else if (C_ == 2 && NT_ == 256) { constexpr int CC = 2, TT = 256; __VA_ARGS__; } \
  else if (C_ == 2 && NT_ == 512) { constexpr int CC = 2, TT = 512; __VA_ARGS__; } \
  else if (C_ == 8 && NT_ == 128) { constexpr int CC = 8, TT = 128; __VA_ARGS__; } \
  else if (C_ == 8 && NT_ == 256) { constexpr int CC = 8, TT = 256; __VA_ARGS__; } \
  else { set_error("no kernel family"); return EDAK_EUNSUPPORTED; }

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// window chunking: a tile sweep of K steps needs redundant halos ~12K wide;
// splitting the window into chunks of <= SWEEP_CHUNK steps (ring state
// handed over through HBM between chunks: 16 B/element per boundary) keeps
// the halo small.  work2 = 2 * ncols * n doubles (NULL: one chunk).
constexpr int SWEEP_CHUNK = 12;  // measured best at cfg4/cfg5 (tools/ab_tiles.py)

static int sweep_chunk() {
  const char* e = getenv("EDAK_SWEEP_CHUNK");  // A/B knob
  const int v = e ? atoi(e) : SWEEP_CHUNK;
  return v >= 1 ? v : SWEEP_CHUNK;
}

// state-staging prefetch distance (1 or 2 steps ahead) of the pair-staged
// sweeps.  Measured on B200 (tools/ab_knobs.py): TL 2 (cfg4 0.341 -> 0.334 ms
// per sweep), AD 1 (2 is no faster at cfg4 and 2% slower at cfg5)
static int sweep_depth(const char* knob, int dflt) {
  const char* e = getenv(knob);
  const int v = e ? atoi(e) : dflt;
  return v == 2 ? 2 : 1;
}

// The TMA tile sweeps on long rings (sweep_tile.cu tile_family_nt) with a
// window of at most one 12-step chunk: 16 x 128 element tiles (half the
// halo share, 2 CTAs per SM) -- cfg5: Hessian block 3.85 -> 3.73 ms, pass
// 231 -> 225 ms.  Longer windows keep 16 x 64 tiles and 12-step chunks: the
// 16 x 128 family as ONE 24-step chunk is faster alone (cfg4 Hessian block
// 0.758 -> 0.750 ms) but slows the two-stream PCG pass (72.4 -> 73.4 ms),
// and as two chunks it gains nothing (profiles/r2_sweep_family_ab.txt).
// EDAK_SWEEP_FAMILY / EDAK_SWEEP_CHUNK override.
int tile_family_nt(const edak_problem* P);
static int big_tiles(const edak_problem* P) {
  if (getenv("EDAK_SWEEP_FAMILY") || P->stage_mode != 0 || env_int("EDAK_SWEEP_LEGACY", 0)) return 0;
  // the pair-staged layout the TMA kernels need (pair_ok's problem-level part)
  if (getenv("EDAK_NO_PAIR") || P->n % 2 || P->traj_stride % 2 || ((uintptr_t)P->states & 15)) return 0;
  return tile_family_nt(P) == 128;
}

static int plan_chunks(int N, bool periodic, const double* work2) {
  const int K = sweep_chunk();
  if (periodic || !work2 || N <= K) return 1;
  if (const char* e = getenv("EDAK_SWEEP_NOCHUNK")) return 1;
  return (N + K - 1) / K;
}

// 16-byte pair staging: every row start and tile base even, rows 16-B aligned
static bool pair_ok(const edak_problem* P, const SweepGeom& geo) {
  if (getenv("EDAK_NO_PAIR")) return false;
  return P->n % 2 == 0 && P->traj_stride % 2 == 0 && ((uintptr_t)P->states & 15) == 0 &&
         (geo.periodic || (geo.W % 2 == 0 && geo.HL % 2 == 0));
}

// the tile family the pair-staged sweeps run: same 1024-element range as
// (8, 128) but 16 elements per thread on 64 threads -- twice the independent
// DP chains per thread and half the exchange traffic per element (cfg4: TL
// 0.354 -> 0.341, AD 0.412 -> 0.398 ms per sweep, tools/ab_tiles.py)
static void widen_pairs(const edak_problem* P, bool stream, int& C, int& NT, SweepGeom& geo) {
  const char* fam = getenv("EDAK_SWEEP_FAMILY");  // explicit A/B family wins
  if (C != 8 || NT != 128 || stream || geo.periodic || !pair_ok(P, geo) || (fam && *fam)) return;
  C = 16;
  NT = 64;
  geo.nact = NT;
}

int launch_tl_tile(const edak_problem* P, const double* vin, double* obs, int ncols, const int32_t* col_traj,
                   const SweepGeom& geo, int nt, int NT, int s0, int s1, double* vout, cudaStream_t st);
int launch_ad_tile(const edak_problem* P, const double* forcing, double* gout, int ncols, const int32_t* col_traj,
                   const SweepGeom& geo, int nt, int NT, int s0, int s1, const double* gin, cudaStream_t st);

// warp-tile sweeps (EDAK_SWEEP_WARP): one warp per tile of 16 x 32 = 512
// ring elements, halos by shuffles, no CTA barrier.  Window chunks of K steps
// (EDAK_WARP_CHUNK) keep the redundant halo (12K + 8) a small share of the
// 512-element range.  Returns false when the problem does not qualify
// (periodic single-tile rings, odd n / unaligned rows, streamed stages).
static int warp_chunk() { return env_int("EDAK_WARP_CHUNK", 6); }
static bool warp_plan(const edak_problem* P, int hl, int hr, SweepGeom& geo, int& nt) {
  constexpr int RANGE = 16 * 32;
  const int W = RANGE - hl - hr;
  if (W < 64 || P->n < 2 * RANGE) return false;
  nt = (P->n + W - 1) / W;
  geo.W = ((P->n + nt - 1) / nt + 1) & ~1;
  if (geo.W > W) geo.W = W;
  geo.HL = hl;
  geo.periodic = 0;
  geo.nact = 32;
  return pair_ok(P, geo);
}
static bool warp_mode(const edak_problem* P, const double* work2) {
  return env_int("EDAK_SWEEP_WARP", 0) != 0 && P->stage_mode == 0 && (work2 || P->n_steps <= warp_chunk());
}

int launch_tl(const edak_problem* P, const double* v0, double* obs, int ncols, const int32_t* col_traj,
              cudaStream_t st, double* work2) {
  int C, NT, nt;
  SweepGeom geo;
  const int N = P->n_steps;
  if (warp_mode(P, work2)) {
    const int K = warp_chunk();
    const int nch = (N + K - 1) / K;
    const size_t blk = (size_t)ncols * P->n;
    bool ok = true;
    for (int c = 0; c < nch && ok; ++c) {
      const int s0 = (int)((long)N * c / nch), s1 = (int)((long)N * (c + 1) / nch), Kc = s1 - s0;
      ok = warp_plan(P, 8 * Kc + 4, 4 * Kc + 4, geo, nt);
    }
    for (int c = 0; c < nch && ok; ++c) {
      const int s0 = (int)((long)N * c / nch), s1 = (int)((long)N * (c + 1) / nch), Kc = s1 - s0;
      warp_plan(P, 8 * Kc + 4, 4 * Kc + 4, geo, nt);
      const double* vin = c == 0 ? v0 : work2 + (size_t)((c - 1) & 1) * blk;
      double* vout = c + 1 < nch ? work2 + (size_t)(c & 1) * blk : nullptr;
      go<32, 16, 0, 3, false>(k_tl<16, 32, false, 8, true, 2, true>, dim3(nt, ncols), st, *P,
                                                 vin, obs, col_traj, geo, s0, s1, vout);
      count_launch();
      int rc = check_launch("k_tl (warp tiles)");
      if (rc) return rc;
    }
    if (ok) return EDAK_OK;
  }
  // probe geometry with the full window to learn the mode
  if (!plan(P->n, 8 * N + 4, 4 * N + 4, C, NT, geo, nt) && !work2) {
    set_error("window too long for the tile family");
    return EDAK_EUNSUPPORTED;
  }
  const bool big = !geo.periodic && N <= sweep_chunk() && big_tiles(P);
  const int nch = plan_chunks(N, geo.periodic && nt == 1, work2);
  const bool stream = P->stage_mode != 0;  // 1 stream, 2 hybrid (small rings)
  const size_t blk = (size_t)ncols * P->n;
  for (int c = 0; c < nch; ++c) {
    const int s0 = (int)((long)N * c / nch), s1 = (int)((long)N * (c + 1) / nch), K = s1 - s0;
    // halos: stencil reach per step (TL 8 left / 4 right) plus the edge
    // garbage of the exchanged stage recompute
    if (!plan(P->n, 8 * K + 4, 4 * K + 4, C, NT, geo, nt, true, big ? 16 : 0, big ? 128 : 0)) {
      set_error("window chunk too long for the tile family");
      return EDAK_EUNSUPPORTED;
    }
    widen_pairs(P, stream, C, NT, geo);
    const double* vin = c == 0 ? v0 : work2 + (size_t)((c - 1) & 1) * blk;
    double* vout = c + 1 < nch ? work2 + (size_t)(c & 1) * blk : nullptr;
    dim3 grid(nt, ncols);
    if (C == 16 && (NT == 64 || NT == 128) && !stream && pair_ok(P, geo) && !env_int("EDAK_SWEEP_LEGACY", 0)) {
      const int rc = launch_tl_tile(P, vin, obs, ncols, col_traj, geo, nt, NT, s0, s1, vout, st);
      if (rc != EDAK_EUNSUPPORTED) {
        if (rc) return rc;
        continue;
      }
    }
    // measured best on B200: 4 resident CTAs (126 regs, no spills)
    const int mb = env_int("EDAK_TL_MINB", 4);
    if (C == 8 && NT == 128 && !stream && mb == 4 && pair_ok(P, geo)) {
      go<128, 8>(k_tl<8, 128, false, 4, true>, grid, st, *P, vin, obs, col_traj, geo, s0, s1, vout);
    } else if (C == 16 && NT == 64 && !stream && pair_ok(P, geo)) {  // the pair-staged default
      if (sweep_depth("EDAK_TL_DEPTH", 2) == 2)
        go<64, 16, 0, 3>(k_tl<16, 64, false, 4, true, 2>, grid, st, *P, vin, obs, col_traj, geo, s0, s1, vout);
      else
        go<64, 16>(k_tl<16, 64, false, 4, true>, grid, st, *P, vin, obs, col_traj, geo, s0, s1, vout);
    } else if (C == 16 && NT == 128 && !stream && pair_ok(P, geo)) {
      go<128, 16, 0, 3>(k_tl<16, 128, false, 2, true, 2>, grid, st, *P, vin, obs, col_traj, geo, s0, s1, vout);
    } else if (C == 12 && NT == 96 && !stream && pair_ok(P, geo)) {
      go<96, 12>(k_tl<12, 96, false, 4, true>, grid, st, *P, vin, obs, col_traj, geo, s0, s1, vout);
    } else if (C == 8 && NT == 256 && !stream && pair_ok(P, geo)) {
      go<256, 8>(k_tl<8, 256, false, 2, true>, grid, st, *P, vin, obs, col_traj, geo, s0, s1, vout);
    } else if (C == 8 && NT == 128 && !stream && mb == 3) {
      go<128, 8>(k_tl<8, 128, false, 3>, grid, st, *P, vin, obs, col_traj, geo, s0, s1, vout);
    } else if (C == 8 && NT == 128 && !stream && mb == 4) {
      go<128, 8>(k_tl<8, 128, false, 4>, grid, st, *P, vin, obs, col_traj, geo, s0, s1, vout);
    } else {
      EDAK_DISPATCH(C, NT, {
        if (stream) go<TT, CC>(k_tl<CC, TT, true>, grid, st, *P, vin, obs, col_traj, geo, s0, s1, vout);
        else go<TT, CC>(k_tl<CC, TT, false>, grid, st, *P, vin, obs, col_traj, geo, s0, s1, vout);
      });
    }
    count_launch();
    int rc = check_launch("k_tl");
    if (rc) return rc;
  }
  return EDAK_OK;
}

int launch_ad(const edak_problem* P, const double* forcing, double* g, int ncols, const int32_t* col_traj,
              cudaStream_t st, double* work2) {
  int C, NT, nt;
  SweepGeom geo;
  const int N = P->n_steps;
  if (warp_mode(P, work2)) {
    const int K = warp_chunk();
    const int nch = (N + K - 1) / K;
    const size_t blk = (size_t)ncols * P->n;
    bool ok = true;
    for (int c = 0; c < nch && ok; ++c) {
      const int s0 = (int)((long)N * c / nch), s1 = (int)((long)N * (c + 1) / nch), Kc = s1 - s0;
      ok = warp_plan(P, 4 * Kc + 8, 8 * Kc + 8, geo, nt);
    }
    for (int c = nch - 1, k = 0; c >= 0 && ok; --c, ++k) {
      const int s0 = (int)((long)N * c / nch), s1 = (int)((long)N * (c + 1) / nch), Kc = s1 - s0;
      warp_plan(P, 4 * Kc + 8, 8 * Kc + 8, geo, nt);
      const double* gin = k == 0 ? nullptr : work2 + (size_t)((k - 1) & 1) * blk;
      double* gout = c == 0 ? g : work2 + (size_t)(k & 1) * blk;
      go<32, 16, 2 * 16 * 32, 2, false>(k_ad<16, 32, false, 8, true, 1, true>, dim3(nt, ncols),
                                                           st, *P, forcing, gout, col_traj, geo, s0, s1, gin);
      count_launch();
      int rc = check_launch("k_ad (warp tiles)");
      if (rc) return rc;
    }
    if (ok) return EDAK_OK;
  }
  if (!plan(P->n, 4 * N + 8, 8 * N + 8, C, NT, geo, nt) && !work2) {
    set_error("window too long for the tile family");
    return EDAK_EUNSUPPORTED;
  }
  const bool big = !geo.periodic && N <= sweep_chunk() && big_tiles(P);
  const int nch = plan_chunks(N, geo.periodic && nt == 1, work2);
  const bool stream = P->stage_mode != 0;  // 1 stream, 2 hybrid (small rings)
  const size_t blk = (size_t)ncols * P->n;
  for (int c = nch - 1, k = 0; c >= 0; --c, ++k) {
    const int s0 = (int)((long)N * c / nch), s1 = (int)((long)N * (c + 1) / nch), K = s1 - s0;
    if (!plan(P->n, 4 * K + 8, 8 * K + 8, C, NT, geo, nt, true, big ? 16 : 0, big ? 128 : 0)) {
      set_error("window chunk too long for the tile family");
      return EDAK_EUNSUPPORTED;
    }
    widen_pairs(P, stream, C, NT, geo);
    const double* gin = k == 0 ? nullptr : work2 + (size_t)((k - 1) & 1) * blk;
    double* gout = c == 0 ? g : work2 + (size_t)(k & 1) * blk;
    dim3 grid(nt, ncols);
    if (C == 16 && (NT == 64 || NT == 128) && !stream && pair_ok(P, geo) && !env_int("EDAK_SWEEP_LEGACY", 0)) {
      const int rc = launch_ad_tile(P, forcing, gout, ncols, col_traj, geo, nt, NT, s0, s1, gin, st);
      if (rc != EDAK_EUNSUPPORTED) {
        if (rc) return rc;
        continue;
      }
    }
    // measured best on B200: 3 resident CTAs (168 regs, no spills)
    const int mb = env_int("EDAK_AD_MINB", 3);
    if (C == 8 && NT == 128 && !stream && mb == 3 && pair_ok(P, geo)) {
      go<128, 8, 2 * 8 * 128>(k_ad<8, 128, false, 3, true>, grid, st, *P, forcing, gout, col_traj, geo, s0, s1,
                              gin);
    } else if (C == 16 && NT == 64 && !stream && pair_ok(P, geo)) {  // the pair-staged default
      if (sweep_depth("EDAK_AD_DEPTH", 1) == 2)
        go<64, 16, 16 * 64, 3>(k_ad<16, 64, false, 3, true, 2>, grid, st, *P, forcing, gout, col_traj, geo, s0,
                                s1, gin);
      else
        go<64, 16, 2 * 16 * 64>(k_ad<16, 64, false, 3, true>, grid, st, *P, forcing, gout, col_traj, geo, s0, s1,
                                gin);
    } else if (C == 16 && NT == 128 && !stream && pair_ok(P, geo)) {
      go<128, 16, 2 * 16 * 128>(k_ad<16, 128, false, 2, true>, grid, st, *P, forcing, gout, col_traj, geo, s0,
                                s1, gin);
    } else if (C == 12 && NT == 96 && !stream && pair_ok(P, geo)) {
      go<96, 12, 2 * 12 * 96>(k_ad<12, 96, false, 2, true>, grid, st, *P, forcing, gout, col_traj, geo, s0, s1,
                              gin);
    } else if (C == 8 && NT == 256 && !stream && pair_ok(P, geo)) {
      go<256, 8, 2 * 8 * 256>(k_ad<8, 256, false, 1, true>, grid, st, *P, forcing, gout, col_traj, geo, s0, s1,
                              gin);
    } else if (C == 8 && NT == 128 && !stream && mb == 3) {
      go<128, 8>(k_ad<8, 128, false, 3>, grid, st, *P, forcing, gout, col_traj, geo, s0, s1, gin);
    } else if (C == 8 && NT == 128 && !stream && mb == 2) {
      go<128, 8>(k_ad<8, 128, false, 2>, grid, st, *P, forcing, gout, col_traj, geo, s0, s1, gin);
    } else {
      EDAK_DISPATCH(C, NT, {
        if (stream) go<TT, CC>(k_ad<CC, TT, true>, grid, st, *P, forcing, gout, col_traj, geo, s0, s1, gin);
        else go<TT, CC>(k_ad<CC, TT, false>, grid, st, *P, forcing, gout, col_traj, geo, s0, s1, gin);
      });
    }
    count_launch();
    int rc = check_launch("k_ad");
    if (rc) return rc;
  }
  return EDAK_OK;
}

int launch_integrate(int n, int n_steps, double dt, double F, const double* x0, int ncols, double* states,
                     int64_t st_stride, double* stages, int64_t sg_stride, cudaStream_t st) {
  // chunks of K steps per launch (tile mode halo 8K left, 4K right)
  int C, NT, nt;
  SweepGeom geo;
  const int Kmax = 16;
  int s0 = 0;
  // level 0 = x0
  cudaError_t e = cudaMemcpy2DAsync(states, st_stride * sizeof(double), x0, (size_t)n * sizeof(double),
                                    (size_t)n * sizeof(double), ncols, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return EDAK_ECUDA;
  }
  while (s0 < n_steps) {
    int K = n_steps - s0;
    if (!plan(n, 8 * K + 4, 4 * K + 4, C, NT, geo, nt, false) || (!geo.periodic && K > Kmax)) {
      K = K < Kmax ? K : Kmax;
      if (!plan(n, 8 * K + 4, 4 * K + 4, C, NT, geo, nt, false)) {
        set_error("integrate: no tile plan");
        return EDAK_EUNSUPPORTED;
      }
    }
    dim3 grid(nt, ncols);
    const double* xin = states + (size_t)s0 * n;
    EDAK_DISPATCH(C, NT, {
      go<TT>(k_integrate<CC, TT>, grid, st, n, K, s0, dt, F, xin, st_stride, states, st_stride, stages,
                                               sg_stride, geo);
    });
    count_launch();
    int rc = check_launch("k_integrate");
    if (rc) return rc;
    s0 += K;
  }
  return EDAK_OK;
}

// nonlinear observation G(x) (obs.py:43-45)
__global__ void k_observe(const double* __restrict__ states, int64_t stride, int n,
                          const int32_t* __restrict__ grid, int G, const int32_t* __restrict__ times, int T,
                          double* __restrict__ y) {
  const int col = blockIdx.y;
  const int p = G * T;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < p; q += gridDim.x * blockDim.x) {
    const int tp = q / G, g = q - tp * G;
    y[(size_t)col * p + q] = states[(size_t)col * stride + (size_t)times[tp] * n + grid[g]];
  }
}

int launch_observe(const double* states, int64_t stride, int n, const int32_t* grid, int G,
                   const int32_t* times, int T, int ncols, double* y, cudaStream_t st) {
  const int p = G * T;
  dim3 gridd((p + 255) / 256 < 1024 ? (p + 255) / 256 : 1024, ncols);
  k_observe<<<gridd, 256, 0, st>>>(states, stride, n, grid, G, times, T, y);
  count_launch();
  return check_launch("k_observe");
}

}  // namespace edak
