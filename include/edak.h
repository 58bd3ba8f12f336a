/*
 * edak.h -- C ABI of the B200 (sm_100a) Hessian-block / LMP-PCG engine.
 *
 * Plain C: raw device pointers, sizes and a cudaStream_t (passed as void*).
 * No torch types.  Every entry point is stream-ordered, allocates nothing,
 * keeps no pointer after it returns, and returns 0 on success or a negative
 * EDAK_E* code (the last CUDA error string is available from
 * edak_last_error()).
 *
 * Layout: a block of vectors is stored column by column -- column c of an
 * (n x ncols) block starts at ptr + c * n -- i.e. the TRANSPOSE of the
 * reference's numpy (n, ell) arrays.  Observation vectors are time-major
 * (obs.py:45,50): entry t_pos * G + g_pos, p = G * T per column.
 *
 * Each function names the reference interface it replaces
 * (/root/reference/pkg/src/edasketch/<file>:<lines>).  The Python host
 * layer (paper_2605_23571_b200/) binds these through ctypes; see
 * INTEGRATION.md for the binding a reference maintainer would add.
 */
#ifndef EDAK_H
#define EDAK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EDAK_OK 0
#define EDAK_EINVAL -1      /* bad sizes / null pointers */
#define EDAK_ECUDA -2       /* CUDA launch/runtime error */
#define EDAK_EUNSUPPORTED -3 /* shape outside the compiled kernel family */

/* One linearization set: the 4D-Var window operator pieces shared by every
 * column of a block (model.py, obs.py, covariance.py).  The struct is
 * plain-old-data; all pointers are device pointers. */
typedef struct edak_problem {
  int32_t n;             /* ring size (Trajectory.n, model.py:113-115)          */
  int32_t n_steps;       /* window steps N (Trajectory.n_steps, model.py:109)  */
  double dt;             /* RK4 step (Trajectory.dt)                            */
  double forcing;        /* F (Trajectory.forcing)                              */
  /* linearization trajectories: states[traj][s][i], s = 0..N-1 (the RK4
   * stages are recomputed from states[s], model.py:38-48, to within ~1 ulp:
   * FMA-contracted, restarted from the exact state every step), or,
   * when stage_mode == 1, stages[traj][s][k][i] streamed as stored
   * (Trajectory.stages, model.py:95-97). */
  const double* states;
  const double* stages;
  int64_t traj_stride;   /* doubles between consecutive trajectories        */
  int32_t stage_mode;    /* 0 = recompute stages from states, 1 = stream all
                          * four stored stages                              */
  int32_t pad0;
  /* observation network (ObsNetwork, obs.py:23-41) as position maps */
  const int32_t* gpos;   /* [n]: position of grid point i in net.grid, or -1 */
  const int32_t* tpos;   /* [N+1]: position of level t in net.times, or -1   */
  int32_t G;             /* net.grid.size                                    */
  int32_t T;             /* net.times.size                                   */
  double sigma2;         /* DiagonalNoise.sigma ** 2 (covariance.py:69-71)   */
  /* circulant U_B (GridCovFactor.apply, covariance.py:41-47) as taps:
   * (U_B v)_i = sum_k taps[k] * v[(i + tap_w - k) mod n], k < ntaps */
  const double* taps;
  int32_t ntaps;
  int32_t tap_w;
  /* optional overlap-save form of the same factor (circ_os.cu): with
   * M = 2^os_logm (10 or 11) and K = ntaps <= M/2 + 1, os_spec holds the M
   * complex values fft(h)/M of the block kernel h[m mod M] = taps[m + tap_w]
   * in bit-reversed order and os_tw = exp(-2 pi i m / (2M)), m < M, both
   * as interleaved (re, im) doubles.  NULL: U_B is the tap convolution. */
  const double* os_spec;
  const double* os_tw;
  int32_t os_logm;
  int32_t pad1;
} edak_problem;

/* ---- library --------------------------------------------------------- */
const char* edak_version(void);
const char* edak_last_error(void);
/* number of kernels this library has launched since load (for bench.py's
 * gpu_launches claim) */
int64_t edak_launch_count(void);

/* ---- model: nonlinear producer (model.integrate, model.py:118-131) ---- */
/* states_out[c][s][i] for s = 0..n_steps (n_steps+1 levels), bit-exact with
 * the reference RK4 (model.py:38-48).  x0 is (ncols x n).  out_stride =
 * doubles between columns of states_out (>= (n_steps+1)*n).  stages_out may
 * be NULL; else (ncols x n_steps x 4 x n) with stride stg_stride. */
int edak_integrate(int n, int n_steps, double dt, double forcing,
                   const double* x0, int ncols, double* states_out,
                   int64_t out_stride, double* stages_out, int64_t stg_stride,
                   void* stream);

/* ---- model: per-vector operators (model.py:20-84) --------------------- */
/* Blocks of ncols vectors of length n (column c at c * n), each operation
 * IEEE-rounded in the reference's numpy order (bit-identical results).
 * out = tendency(x, forcing)                     (model.py:20-22) */
int edak_tendency(int n, int ncols, const double* x, double forcing, double* out,
                  void* stream);
/* out = tendency_tlm(x, v) = J(x) v              (model.py:25-28) */
int edak_tendency_tlm(int n, int ncols, const double* x, const double* v,
                      double* out, void* stream);
/* out = tendency_adj(x, w) = J(x)^T w            (model.py:31-35) */
int edak_tendency_adj(int n, int ncols, const double* x, const double* w,
                      double* out, void* stream);
/* out = y + c * z (product rounded, then the sum): the stage updates of
 * _rk4_stages / step_tlm / step_adj (model.py:41-45, 58-61, 71-83); with
 * y == NULL, out = c * z (the scalings of step_adj, model.py:71-74) */
int edak_axpy_rn(int64_t len, const double* y, double c, const double* z,
                 double* out, void* stream);
/* out = y + c * (((a1 + 2 a2) + 2 a3) + a4)  (model.py:47, 63) */
int edak_rk4_combine(int64_t len, const double* y, double c, const double* a1,
                     const double* a2, const double* a3, const double* a4,
                     double* out, void* stream);

/* nonlinear observation G(x) (ObsNetwork.observe, obs.py:43-45):
 * y[c][t_pos*G+g_pos] = states[c][times[t_pos]][grid[g_pos]] */
int edak_observe(const double* states, int64_t traj_stride, int n,
                 const int32_t* grid, int G, const int32_t* times, int T,
                 int ncols, double* y, void* stream);

/* ---- covariance ------------------------------------------------------ */
/* out = U_B in, column-wise (GridCovFactor.apply/apply_t, covariance.py:41-47) */
int edak_circ_apply(const edak_problem* P, const double* in, double* out,
                    int ncols, void* stream);

/* ---- window operator halves (obs.py:47-57 over model.py:134-157) ------ */
/* Sweep workspace: edak_sweep_work_doubles doubles lets long windows run
 * as chunks of <= 8 steps (smaller redundant halos); NULL = one chunk. */
int64_t edak_sweep_work_doubles(const edak_problem* P, int ncols);
/* obs[c] = G_traj(c) v0[c]  (observe_tlm, obs.py:47-50): raw, not R^-1-scaled */
int edak_tl_sweep(const edak_problem* P, const double* v0, double* obs,
                  int ncols, const int32_t* col_traj, double* work, void* stream);
/* g[c] = G_traj(c)^T (forcing[c] / sigma2)  (observe_adj(rn.solve(.)),
 * obs.py:52-57 with covariance.py:69-71) */
int edak_ad_sweep(const edak_problem* P, const double* forcing, double* g,
                  int ncols, const int32_t* col_traj, double* work, void* stream);

/* ---- member problem (assim.py) -------------------------------------- */
/* Empty blocks (ncols == 0, or a zero GEMM dimension) are no-ops that return
 * EDAK_OK without touching any pointer, like the reference's loops over zero
 * columns. */
/* workspace (doubles) needed by edak_hessian_block / edak_rhs / edak_cost */
int64_t edak_work_doubles(const edak_problem* P, int ncols);
/* az[c] = ident * z[c] + A_traj(c) z[c],  A = U_B^T G^T R^-1 G U_B
 * (MemberProblem.a_apply / hessian_apply, assim.py:55-72).  obs_out, if not
 * NULL, receives the raw TL observations G U_B z (ncols x p). */
int edak_hessian_block(const edak_problem* P, const double* z, double* az,
                       int ncols, const int32_t* col_traj, double ident,
                       double* work, double* obs_out, double* dot_part,
                       void* stream);
/* when ident != 0 and dot_part != NULL the final U_B pass also writes tile
 * partials of z[c] . az[c] (PCG p . Hp): dot_part[c * tiles + t],
 * tiles = edak_hessian_dot_tiles(n) */
int64_t edak_hessian_dot_tiles(int n);
/* b[c] = U_B^T G^T R^-1 d[c]  (MemberProblem.rhs, assim.py:74-77) */
int edak_rhs(const edak_problem* P, const double* innov, double* b, int ncols,
             const int32_t* col_traj, double* work, void* stream);
/* J[c] = 1/2 z.z + 1/2 |G U_B z - d|^2 / sigma2 (quadratic_cost,
 * assim.py:79-82) */
int edak_cost(const edak_problem* P, const double* z, const double* innov,
              double* J, int ncols, const int32_t* col_traj, double* work,
              void* stream);

/* ---- dense fp64 tensor-core (DMMA) kernels -------------------------- */
/* C[a + b*ldc] = sum_i A[i + a*lda] * B[i + b*ldb] for a < m, b < nb
 * (A^T B with the long dimension K contiguous; Gram Y^T Y, Phi^T Y,
 * S^T R -- nystrom.py:118-125, lmp.py:62-65).  Deterministic split-K:
 * partial[] needs edak_gemm_tn_partials(m, nb, K) doubles. */
int64_t edak_gemm_tn_partials(int m, int nb, int64_t K);
int edak_gemm_tn(const double* A, int64_t lda, const double* B, int64_t ldb,
                 double* C, int ldc, int m, int nb, int64_t K, double* partial,
                 void* stream);
/* D[i + j*ldd] = beta * Cin[i + j*ldc] + sum_l A[i + l*lda] * s_l * B[l + j*ldb]
 * (s_l = bscale[l], or 1 when bscale is NULL)
 * (A is M x kk column-major, B kk x N) -- Q_Y U_T (nystrom.py:131),
 * S (c o S^T v) (lmp.py:65); Cin may alias D. */
int edak_gemm_nn(const double* A, int64_t lda, const double* B, int ldb,
                 const double* bscale, const double* Cin, int64_t ldc,
                 double beta, double* D, int64_t ldd, int64_t M, int N, int kk,
                 void* stream);

/* ---- small dense (l x l, l <= 256) single-CTA solvers ---------------- */
/* Upper Cholesky W = C^T C reading W's upper triangle, with the reference
 * shift schedule (nystrom.py:67-93): try nu = 0, then nu = eps*scale*10^r,
 * r = 0..4 (mode != 0).  info[0] = attempts made (0 = plain succeeded),
 * info[1] = 0 ok / 1 breakdown; nu_out[0] = shift used. */
int edak_potrf_shifted(const double* W, int l, double* C, int mode,
                       double scale, double* nu_out, int32_t* info,
                       void* stream);
/* Rinv = R^-1 for upper-triangular R (l x l) */
int edak_trinv_upper(const double* R, int l, double* Rinv, void* stream);
/* Fused blocked Cholesky (same shift schedule / breakdown test / info as
 * edak_potrf_shifted) and inverse: C upper with W = C^T C and, if Cinv !=
 * NULL, Cinv = C^-1 (nystrom.py:67-93,129).  work: NULL for l <= 128, else
 * edak_chol_inv_work_doubles(l) doubles. */
int64_t edak_chol_inv_work_doubles(int l);
int edak_chol_inv(const double* W, int l, double* C, double* Cinv, int mode,
                  double scale, double* nu_out, int32_t* info, double* work,
                  void* stream);
/* one-sided (Hestenes) Jacobi SVD of M (rows x cols, rows >= cols,
 * column-major): M V = U diag(sig), sig descending (np.linalg.svd,
 * nystrom.py:130).  U (rows x cols), sig (cols), V (cols x cols) or NULL.
 * work >= edak_svd_work_doubles(rows, cols). */
int64_t edak_svd_work_doubles(int rows, int cols);
int edak_svd_jacobi(const double* M, int rows, int cols, double* U, double* sig,
                    double* V, double* work, void* stream);

/* ---- batched PCG (krylov.pcg, krylov.py:49-97) ---------------------- */
/* One column per ensemble member (n x ncols blocks).  Per-member device
 * status: 0 running, 1 stopped (converged), 2 p.Hp <= 0 at iters[c]
 * (krylov.py:82-84), 3 r.Pr < 0 at start (krylov.py:73-74).  hist_* are
 * (ncols x hist_ld) row-major histories indexed by iteration. */
/* workspace (doubles) of the batched PCG: per-member tile partials of the
 * fixed-order dot products and the double-buffered r.z */
int64_t edak_pcg_work_doubles(int n, int ncols);
/* x = 0, r = b, p = z (= P b), rz = r.z, hist_rz[.,0] = rz (krylov.py:68-78) */
int edak_pcg_init(int n, int ncols, const double* b, const double* z, double* x,
                  double* r, double* p, double* work, double* hist_rz, int hist_ld,
                  int32_t* status, int32_t* iters, void* stream);
/* hist_J[., 0] = J(0) = 1/2 d.R^-1 d (assim.py:79-82 at z = 0) */
int edak_pcg_cost0(int p_obs, int ncols, const double* d, double sigma2,
                   double* hist_J, int hist_ld, void* stream);
/* php = p.hp, breakdown test, alpha = rz/php, x += alpha p, r -= alpha hp;
 * if b (the rhs block) is not NULL, the partials of x.(b + r) that give
 * J(x_it) = J(0) - 1/2 x.(b + r) (J identity, (I+A)x = b - r;
 * krylov.py:79-89,108-113) */
int edak_pcg_alpha(int n, int ncols, const double* p, const double* hp,
                   double* x, double* r, double* work, int32_t* status,
                   int32_t* iters, int it, const double* b,
                   const double* php_part, int php_tiles, void* stream);
/* Fused single-pass-LMP step: W = S^T r; rz_new = |r|^2 + W^T diag(coef) W
 * (= r.Pr exactly); record / stop test / beta; p = r + beta p + S(coef o W)
 * (= Pr + beta p, krylov.py:86-96) in the GEMM epilogue.  lmpwork >=
 * edak_lmp_work_doubles(n, k, ncols). */
int edak_pcg_lmp_beta(int n, int k, int ncols, const double* S, const double* coef,
                      const double* r, double* p, double* work, double* lmpwork,
                      double rtol, double* hist_rz, double* hist_J, int hist_ld,
                      int32_t* status, int32_t* iters, int it, void* stream);
/* rz_new = r.z, hist_rz[., it] (+ hist_J[., it] when not NULL), stop test
 * (rtol < 0 = None), p = z + beta p (krylov.py:86-96) */
int edak_pcg_beta(int n, int ncols, const double* z, const double* r, double* p,
                  double* work, double rtol, double* hist_rz, double* hist_J,
                  int hist_ld, int32_t* status, int32_t* iters, int it,
                  void* stream);
/* z = r + S diag(coef) S^T r -- one symmetric factor of the spectral LMP
 * (SpectralLmp._project / apply_sqrt, lmp.py:62-70); with coef =
 * theta/(lam+1) - 1 and orthonormal S it is P itself (lmp.py:72-74). */
int64_t edak_lmp_work_doubles(int n, int k, int ncols);
/* Whole batched LMP-PCG solve for small rings (8 <= n <= 256; G*T <= 8192
 * observations): one CTA per member runs every iteration -- U_B, TL sweep,
 * AD sweep, U_B + I, the recurrence with the J identity, the single-pass LMP
 * (S, coef; S == NULL: no preconditioner) -- in one launch (krylov.py:49-97
 * for each member; cfg1/cfg2 are latency-bound).  b (M, n),
 * d (M, G*T) innovations for the J trace (NULL: no trace), outputs x (M, n),
 * hist_rz / hist_J (M, hist_ld >= max_iters + 1), status (0 running/max,
 * 1 converged, 2 A not PD at iters, 3 P not PD), iters. */
int edak_pcg_small(const edak_problem* P, const int32_t* col_traj, int ncols,
                   const double* b, const double* d, const double* S,
                   const double* coef, int k, int max_iters, double rtol,
                   double* x, double* hist_rz, double* hist_J, int hist_ld,
                   int32_t* status, int32_t* iters, void* stream);
int edak_lmp_apply(int n, int k, int ncols, const double* S, const double* coef,
                   const double* r, double* z, double* work, void* stream);
/* column dots out[c] = a[c] . b[c], fixed order (deterministic) */
int edak_col_dots(int n, int ncols, const double* a, const double* b,
                  double* out, void* stream);

/* ---- measurement ---------------------------------------------------- */
/* fp64 roofline denominators (bench.py): an FMA-pipe loop, 2*8*iters*256*
 * blocks flop per launch, and a DMMA.8x8x4 loop, 512*8*iters*8*blocks flop */
int edak_peak_dfma(double* sink, int iters, int blocks, void* stream);
int edak_peak_dmma(double* sink, int iters, int blocks, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EDAK_H */
