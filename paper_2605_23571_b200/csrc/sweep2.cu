// Second-generation window sweeps (recompute mode): RK4 stage states live in
// padded shared memory instead of registers.
//
// k_tl2 / k_ad2 compute exactly what k_tl / k_ad compute (same operations in
// the same order, bit-identical results) but
//   * the state tile of the next step is staged by cp.async (LDGSTS) into a
//     shared buffer while the current step runs (no register prefetch);
//   * each recomputed stage x2/x3/x4 is written once to shared memory and read
//     back with its +-2 halo, so the x-stage exchange rounds disappear and no
//     thread keeps four stage arrays live (TL ~100, AD ~120 registers instead
//     of 208 / 254 -> 2x the resident warps per SM);
//   * the shared layout pads one double per 8 (thread t's window starts at
//     9t): every 64-bit access pattern is bank-conflict free.
// Register exchanges (Ring/XBuf) remain for the perturbation / adjoint arrays.
#include <cstdio>
#include <cstdlib>

#include "sweep.cuh"

namespace edak {

struct SweepGeom2 {
  int W, HL, periodic, nact;
};

template <int C, int NT>
struct Tile2 {
  static constexpr int R = C * NT;              // range elements
  static constexpr int LEN = R + 4;             // q in [-2, R + 2)
  static constexpr int PLEN = LEN + LEN / 8 + 2;
  __device__ static __forceinline__ int pi(int q) {
    const int u = q + 2;
    return u + (u >> 3);
  }
};


// stage the ring window [base-2, base+R+2) of one state level into buf.
// Thread i copies q = i - 2 + k NT: consecutive threads read consecutive ring
// positions (coalesced), the padded smem index advances by a constant stride,
// and the ring index wraps with a conditional subtract (NT < n).
template <int C, int NT>
__device__ __forceinline__ void stage_state(double* buf, const double* __restrict__ src, int g0, int n) {
  using T = Tile2<C, NT>;
  static_assert(NT % 8 == 0, "padded stride");
  int g = g0;
  double* d = buf + T::pi((int)threadIdx.x - 2);
  for (int q = (int)threadIdx.x - 2; q < T::R + 2; q += NT) {
    cp_async8(d, src + g);
    d += NT + NT / 8;
    g += NT;
    if (g >= n) g -= n;
  }
  cp_commit();
}

// thread window (own + 2 halo each side): constant offsets from 9t (C = 8)
template <int C, int NT>
__device__ __forceinline__ void read_win(const double* buf, int t, double (&a)[C + 4]) {
  static_assert(C == 8, "padded layout assumes 8 elements per thread");
  const double* w = buf + 9 * t;
#pragma unroll
  for (int k = 0; k < C + 4; ++k) a[k] = w[k + (k >> 3)];
}

template <int C, int NT>
__device__ __forceinline__ double own_at(const double* buf, int t, int j) {
  return buf[9 * t + (j + 2) + ((j + 2) >> 3)];
}

// write own elements; for a periodic ring the first two / last two elements
// are also copied into the wrapped halo slots
template <int C, int NT>
__device__ __forceinline__ void write_own(double* buf, int t, const double (&x)[C], bool periodic, int n,
                                          int nact) {
  using T = Tile2<C, NT>;
  if (periodic && t >= nact) return;  // idle threads of a periodic ring
  double* w = buf + 9 * t;
#pragma unroll
  for (int j = 0; j < C; ++j) w[(j + 2) + ((j + 2) >> 3)] = x[j];
  if (periodic) {
    if (t == 0) {
      buf[T::pi(n)] = x[0];
      buf[T::pi(n + 1)] = x[1];
    }
    if (t == nact - 1) {
      buf[T::pi(-2)] = x[C - 2];
      buf[T::pi(-1)] = x[C - 1];
    }
  }
}

template <int C, int NT>
__device__ __forceinline__ void zero_halo(double* buf) {
  using T = Tile2<C, NT>;
  if (threadIdx.x < 4) {
    const int q = threadIdx.x < 2 ? (int)threadIdx.x - 2 : T::R + (int)threadIdx.x - 2;
    buf[T::pi(q)] = 0.0;
  }
}

// ------------------------------------------------------------------- TL --
template <int C, int NT>
__global__ void __launch_bounds__(NT, 4) k_tl2(edak_problem P, const double* __restrict__ vin,
                                            double* __restrict__ obs, const int32_t* __restrict__ col_traj,
                                            SweepGeom2 geo, int s0, int s1, double* __restrict__ vout) {
  using T = Tile2<C, NT>;
  extern __shared__ __align__(16) double dsm_[];
  XBuf<NT>& xb = *reinterpret_cast<XBuf<NT>*>(dsm_);
  xb.init_pads();
  double* XB0 = dsm_ + sizeof(XBuf<NT>) / sizeof(double);
  double* XB1 = XB0 + T::PLEN;
  double* SA = XB1 + T::PLEN;
  double* SB = SA + T::PLEN;
  Ring<C, NT> R;
  const int n = P.n;
  const int i0 = blockIdx.x * geo.W;
  const int base = geo.periodic ? 0 : i0 - geo.HL;
  R.init(n, base, geo.nact, geo.periodic);
  const int t = threadIdx.x;
  const int g0 = wrap(base - 2 + t, n);
  const int col = blockIdx.y;
  const int wlo = geo.periodic ? 0 : geo.HL;
  const int whi = geo.periodic ? n : geo.HL + min(geo.W, n - i0);
  const bool per = geo.periodic;
  const int traj = col_traj ? col_traj[col] : 0;
  const double* tr = P.states + (size_t)traj * P.traj_stride;
  const int G = P.G;
  double* ob = obs + (size_t)col * G * P.T;
  const double dt = P.dt, h = 0.5 * dt, c6 = dt / 6.0, F = P.forcing;
  int buf = 0;

  stage_state<C, NT>((s0 & 1) ? XB1 : XB0, tr + (size_t)s0 * n, g0, n);
  zero_halo<C, NT>(SA);
  zero_halo<C, NT>(SB);
  double v[C + 4];
  R.load_own(vin + (size_t)col * n, v);

  int gw[C];
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const int e = t * C + j;
    gw[j] = (t < R.nact && e >= wlo && e < whi) ? __ldg(P.gpos + R.gidx(j)) : -1;
  }
  auto capture = [&](int level) {
    const int tp = __ldg(P.tpos + level);
    if (tp < 0) return;
#pragma unroll
    for (int j = 0; j < C; ++j)
      if (gw[j] >= 0) ob[(size_t)tp * G + gw[j]] = v[j + 2];
  };
  if (s0 == 0) capture(0);

#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    const double* Xb = (s & 1) ? XB1 : XB0;
    cp_wait_all();
    xchg1(R, xb, buf, v);  // barrier also publishes the staged X_s
    // the other buffer held X_{s-1}, last read before this barrier
    if (s + 1 < s1) stage_state<C, NT>(((s + 1) & 1) ? XB1 : XB0, tr + (size_t)(s + 1) * n, g0, n);
    double a[C], acc[C], xn[C], u[C + 4], xw[C + 4];
    read_win<C, NT>(Xb, t, xw);
    // sub-stage 1: a1 = TL(X, v); x2 = X + h f(X); u2 = v + h a1
#pragma unroll
    for (int j = 0; j < C; ++j) {
      a[j] = l96_tl(v[j + 3], v[j], v[j + 1], v[j + 2], xw[j + 3], xw[j], xw[j + 1]);
      xn[j] = axpy_rn(xw[j + 2], h, l96_f(xw[j + 3], xw[j], xw[j + 1], xw[j + 2], F));
      acc[j] = a[j];
      u[j + 2] = fma(h, a[j], v[j + 2]);
    }
    write_own<C, NT>(SA, t, xn, per, n, R.nact);
    xchg1(R, xb, buf, u);  // barrier also publishes x2
    // sub-stage 2: a2 = TL(x2, u2); x3 = X + h f(x2); u3 = v + h a2
    read_win<C, NT>(SA, t, xw);
#pragma unroll
    for (int j = 0; j < C; ++j) {
      a[j] = l96_tl(u[j + 3], u[j], u[j + 1], u[j + 2], xw[j + 3], xw[j], xw[j + 1]);
      xn[j] = axpy_rn(own_at<C, NT>(Xb, t, j), h, l96_f(xw[j + 3], xw[j], xw[j + 1], xw[j + 2], F));
      acc[j] = fma(2.0, a[j], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < C; ++j) u[j + 2] = fma(h, a[j], v[j + 2]);
    write_own<C, NT>(SB, t, xn, per, n, R.nact);
    xchg1(R, xb, buf, u);
    // sub-stage 3: a3 = TL(x3, u3); x4 = X + dt f(x3); u4 = v + dt a3
    read_win<C, NT>(SB, t, xw);
#pragma unroll
    for (int j = 0; j < C; ++j) {
      a[j] = l96_tl(u[j + 3], u[j], u[j + 1], u[j + 2], xw[j + 3], xw[j], xw[j + 1]);
      xn[j] = axpy_rn(own_at<C, NT>(Xb, t, j), dt, l96_f(xw[j + 3], xw[j], xw[j + 1], xw[j + 2], F));
      acc[j] = fma(2.0, a[j], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < C; ++j) u[j + 2] = fma(dt, a[j], v[j + 2]);
    write_own<C, NT>(SA, t, xn, per, n, R.nact);
    xchg1(R, xb, buf, u);
    // sub-stage 4: a4 = TL(x4, u4); v += dt/6 (a1 + 2a2 + 2a3 + a4)
    read_win<C, NT>(SA, t, xw);
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const double a4 = l96_tl(u[j + 3], u[j], u[j + 1], u[j + 2], xw[j + 3], xw[j], xw[j + 1]);
      v[j + 2] = fma(c6, acc[j] + a4, v[j + 2]);
    }
    capture(s + 1);
  }
  if (vout && t < R.nact) {
    double* vo = vout + (size_t)col * n;
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int e = t * C + j;
      if (e >= wlo && e < whi) vo[R.gidx(j)] = v[j + 2];
    }
  }
}

// ------------------------------------------------------------------- AD --
template <int C, int NT>
__global__ void __launch_bounds__(NT, 4) k_ad2(edak_problem P, const double* __restrict__ forcing,
                                            double* __restrict__ gout, const int32_t* __restrict__ col_traj,
                                            SweepGeom2 geo, int s0, int s1, const double* __restrict__ gin) {
  using T = Tile2<C, NT>;
  extern __shared__ __align__(16) double dsm_[];
  XBuf<NT>& xb = *reinterpret_cast<XBuf<NT>*>(dsm_);
  xb.init_pads();
  double* XB0 = dsm_ + sizeof(XBuf<NT>) / sizeof(double);
  double* XB1 = XB0 + T::PLEN;
  double* S2 = XB1 + T::PLEN;
  double* S3 = S2 + T::PLEN;
  double* S4 = S3 + T::PLEN;
  Ring<C, NT> R;
  const int n = P.n;
  const int i0 = blockIdx.x * geo.W;
  const int base = geo.periodic ? 0 : i0 - geo.HL;
  R.init(n, base, geo.nact, geo.periodic);
  const int t = threadIdx.x;
  const int g0 = wrap(base - 2 + t, n);
  const int col = blockIdx.y;
  const int wlo = geo.periodic ? 0 : geo.HL;
  const int whi = geo.periodic ? n : geo.HL + min(geo.W, n - i0);
  const bool per = geo.periodic;
  const int traj = col_traj ? col_traj[col] : 0;
  const double* tr = P.states + (size_t)traj * P.traj_stride;
  const int G = P.G;
  const double* fc = forcing + (size_t)col * G * P.T;
  const double dt = P.dt, h = 0.5 * dt, F = P.forcing;
  const double c6 = dt / 6.0, c3 = 2.0 * dt / 6.0, s2 = P.sigma2;
  int buf = 0;

  int gp[C];
#pragma unroll
  for (int j = 0; j < C; ++j) gp[j] = __ldg(P.gpos + R.gidx(j));
  // w_all[level] at own elements: R^-1 d at observed points, 0 elsewhere
  const double inv_s2 = 1.0 / s2;  // as k_ad: reciprocal, hoisted level lookup
  auto force = [&](int level, double (&f)[C]) {
    const int tp = __ldg(P.tpos + level);
#pragma unroll
    for (int j = 0; j < C; ++j)
      f[j] = (tp < 0 || gp[j] < 0) ? 0.0 : __ldg(fc + (size_t)tp * G + gp[j]) * inv_s2;
  };

  stage_state<C, NT>((s1 - 1) & 1 ? XB1 : XB0, tr + (size_t)(s1 - 1) * n, g0, n);
  zero_halo<C, NT>(S2);
  zero_halo<C, NT>(S3);
  zero_halo<C, NT>(S4);
  double g[C + 4];
  if (gin) {
    R.load_own(gin + (size_t)col * n, g);
  } else {
    double f[C];
    force(P.n_steps, f);
#pragma unroll
    for (int j = 0; j < C; ++j) g[j + 2] = f[j];
  }
  cp_wait_all();
  __syncthreads();

#pragma unroll 1
  for (int s = s1 - 1; s >= s0; --s) {
    double* Xb = (s & 1) ? XB1 : XB0;
    double fs[C];
    force(s, fs);  // consumed at the end of the step: latency hidden
    double xn[C], xw[C + 4];
    read_win<C, NT>(Xb, t, xw);
#pragma unroll
    for (int j = 0; j < C; ++j) xn[j] = axpy_rn(xw[j + 2], h, l96_f(xw[j + 3], xw[j], xw[j + 1], xw[j + 2], F));
    write_own<C, NT>(S2, t, xn, per, n, R.nact);
    xchg1(R, xb, buf, g);  // barrier: x2 visible, g halo exchanged
    if (s > s0) stage_state<C, NT>((s - 1) & 1 ? XB1 : XB0, tr + (size_t)(s - 1) * n, g0, n);
    read_win<C, NT>(S2, t, xw);
#pragma unroll
    for (int j = 0; j < C; ++j)
      xn[j] = axpy_rn(own_at<C, NT>(Xb, t, j), h, l96_f(xw[j + 3], xw[j], xw[j + 1], xw[j + 2], F));
    write_own<C, NT>(S3, t, xn, per, n, R.nact);
    __syncthreads();
    read_win<C, NT>(S3, t, xw);
#pragma unroll
    for (int j = 0; j < C; ++j)
      xn[j] = axpy_rn(own_at<C, NT>(Xb, t, j), dt, l96_f(xw[j + 3], xw[j], xw[j + 1], xw[j + 2], F));
    write_own<C, NT>(S4, t, xn, per, n, R.nact);
    __syncthreads();
    // step_adj (model.py:66-84)
    double vh[C], u[C], a[C + 4];
#pragma unroll
    for (int k = 0; k < C + 4; ++k) a[k] = c6 * g[k];  // a4 = (dt/6) w, halo included
    read_win<C, NT>(S4, t, xw);
#pragma unroll
    for (int j = 0; j < C; ++j)
      u[j] = l96_ad(xw[j], xw[j + 1], xw[j + 3], xw[j + 4], a[j + 1], a[j + 2], a[j + 3], a[j + 4]);
#pragma unroll
    for (int j = 0; j < C; ++j) {
      vh[j] = g[j + 2] + u[j];
      a[j + 2] = fma(dt, u[j], c3 * g[j + 2]);  // a3
    }
    xchg1(R, xb, buf, a);
    read_win<C, NT>(S3, t, xw);
#pragma unroll
    for (int j = 0; j < C; ++j)
      u[j] = l96_ad(xw[j], xw[j + 1], xw[j + 3], xw[j + 4], a[j + 1], a[j + 2], a[j + 3], a[j + 4]);
#pragma unroll
    for (int j = 0; j < C; ++j) {
      vh[j] += u[j];
      a[j + 2] = fma(h, u[j], c3 * g[j + 2]);  // a2
    }
    xchg1(R, xb, buf, a);
    read_win<C, NT>(S2, t, xw);
#pragma unroll
    for (int j = 0; j < C; ++j)
      u[j] = l96_ad(xw[j], xw[j + 1], xw[j + 3], xw[j + 4], a[j + 1], a[j + 2], a[j + 3], a[j + 4]);
#pragma unroll
    for (int j = 0; j < C; ++j) {
      vh[j] += u[j];
      a[j + 2] = fma(h, u[j], c6 * g[j + 2]);  // a1
    }
    cp_wait_all();                 // X_{s-1} landed ...
    xchg1(R, xb, buf, a);          // ... and is visible after this barrier
    read_win<C, NT>(Xb, t, xw);    // X_s is only overwritten two steps later
#pragma unroll
    for (int j = 0; j < C; ++j)
      u[j] = l96_ad(xw[j], xw[j + 1], xw[j + 3], xw[j + 4], a[j + 1], a[j + 2], a[j + 3], a[j + 4]);
#pragma unroll
    for (int j = 0; j < C; ++j) g[j + 2] = (vh[j] + u[j]) + fs[j];
  }
  if (t < R.nact) {
    double* go = gout + (size_t)col * n;
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int e = t * C + j;
      if (e >= wlo && e < whi) go[R.gidx(j)] = g[j + 2];
    }
  }
}

// ------------------------------------------------------------ launchers --
template <int C, int NT>
size_t tl2_smem() {
  return sizeof(XBuf<NT>) + 4 * Tile2<C, NT>::PLEN * sizeof(double);
}
template <int C, int NT>
size_t ad2_smem() {
  return sizeof(XBuf<NT>) + 5 * Tile2<C, NT>::PLEN * sizeof(double);
}

template <typename K>
static void attr(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int C, int NT>
int launch_tl2_t(const edak_problem* P, const double* vin, double* obs, int ncols, const int32_t* col_traj,
                 SweepGeom2 geo, int nt, int s0, int s1, double* vout, cudaStream_t st) {
  const size_t sm = tl2_smem<C, NT>();
  attr(k_tl2<C, NT>, sm);
  k_tl2<C, NT><<<dim3(nt, ncols), NT, sm, st>>>(*P, vin, obs, col_traj, geo, s0, s1, vout);
  return check_launch("k_tl2");
}

template <int C, int NT>
int launch_ad2_t(const edak_problem* P, const double* forcing, double* gout, int ncols, const int32_t* col_traj,
                 SweepGeom2 geo, int nt, int s0, int s1, const double* gin, cudaStream_t st) {
  const size_t sm = ad2_smem<C, NT>();
  attr(k_ad2<C, NT>, sm);
  k_ad2<C, NT><<<dim3(nt, ncols), NT, sm, st>>>(*P, forcing, gout, col_traj, geo, s0, s1, gin);
  return check_launch("k_ad2");
}

// C = 8, NT = 128 (range 1024) tiles; periodic rings of n = 8 * nact with
// 64 <= nact <= 128 also use this family.
bool plan2(int n, int hl, int hr, SweepGeom2& geo, int& nt) {
  constexpr int C = 8, NT = 128, RNG = C * NT;
  if (n % C == 0 && n / C <= NT && n / C >= 64) {
    geo = {n, 0, 1, n / C};
    nt = 1;
    return true;
  }
  if (n < RNG + 64) return false;  // small rings: first-generation kernels
  const int W = RNG - hl - hr;
  if (W < 256) return false;
  nt = (n + W - 1) / W;
  geo = {(n + nt - 1) / nt, hl, 0, NT};
  return true;
}

int launch_tl2(const edak_problem* P, const double* vin, double* obs, int ncols, const int32_t* col_traj,
               int s0, int s1, double* vout, cudaStream_t st) {
  SweepGeom2 geo;
  int nt;
  const int K = s1 - s0;
  if (!plan2(P->n, 8 * K + 4, 4 * K + 4, geo, nt)) return EDAK_EUNSUPPORTED;
  count_launch();
  return launch_tl2_t<8, 128>(P, vin, obs, ncols, col_traj, geo, nt, s0, s1, vout, st);
}

int launch_ad2(const edak_problem* P, const double* forcing, double* gout, int ncols, const int32_t* col_traj,
               int s0, int s1, const double* gin, cudaStream_t st) {
  SweepGeom2 geo;
  int nt;
  const int K = s1 - s0;
  if (!plan2(P->n, 4 * K + 8, 8 * K + 8, geo, nt)) return EDAK_EUNSUPPORTED;
  count_launch();
  return launch_ad2_t<8, 128>(P, forcing, gout, ncols, col_traj, geo, nt, s0, s1, gin, st);
}

// 0: not applicable (stream mode, small ring, EDAK_SWEEP_V2 unset);
// 1: periodic single tile (whole window in one launch); 2: tiles (chunked)
int sweep2_mode(const edak_problem* P, int K) {
  // opt-in: measured slower than the register kernels on B200 (profiles/)
  if (P->stage_mode != 0 || !getenv("EDAK_SWEEP_V2")) return 0;
  SweepGeom2 geo;
  int nt;
  if (!plan2(P->n, 8 * K + 8, 8 * K + 8, geo, nt)) return 0;
  return geo.periodic ? 1 : 2;
}

}  // namespace edak
