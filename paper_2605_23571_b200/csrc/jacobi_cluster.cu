// One-sided (Hestenes) Jacobi SVD of the (l x l) Nystrom matrix T on a
// thread-block cluster of 8 CTAs (8 SMs) instead of one CTA
// (nystrom.py:130 np.linalg.svd; the single-CTA k_svd_jacobi is bound by one
// SM's issue rate and shared-memory bandwidth: ~2.4 us per round at l = 128).
//
// Column pairs follow the same round-robin tournament as k_svd_jacobi.  Pair
// k lives in registers of a half-warp (16 lanes x RPL rows per lane); pairs
// are spread over the cluster's CTAs.  A round is: one dot (+ 4 shuffles),
// the rotation from lane 0's sums (tracked column norms), the rotation in
// registers, then each pair publishes its two columns in its own CTA's
// double-buffered slot, ONE cluster barrier, and each pair pulls its next
// columns from the neighbouring pairs' slots -- through distributed shared
// memory when the neighbour sits on another SM.  Outputs as k_svd_jacobi:
// U (unit columns, descending sigma), sig, and with Vout the right singular
// vectors: each column then travels as [a; v] (rows + cols entries, v
// starting as e_id), rotated as one, with the dots over the a part only.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace edak {

constexpr int JC_CL = 8;           // CTAs per cluster (portable size)
constexpr int JC_MAXROWS = 256;    // rows <= 256 -> <= 16 rows per lane

__device__ __forceinline__ double jc_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

template <int CL>
__device__ __forceinline__ void jc_sync(cg::cluster_group& cluster) {
  if constexpr (CL == 1)
    __syncthreads();
  else
    cluster.sync();
}
template <int CL, typename T>
__device__ __forceinline__ T* jc_map(cg::cluster_group& cluster, T* p, int r) {
  if constexpr (CL == 1)
    return p;
  else
    return cluster.map_shared_rank(p, r);
}

// smem per CTA: slots [2 buf][ppc][2 (p, q)][E] + meta [2][ppc][4].
// CL = 1: every pair in one CTA (16 lanes per pair, up to 32 pairs), one
// __syncthreads per round instead of a cluster barrier (small l).
template <int CL, int RPL>
__device__ __forceinline__ void jc_body(const double* __restrict__ M, int rows, int cols, int ppc,
                                        double* __restrict__ U, double* __restrict__ sig,
                                        double* __restrict__ Vout, double* __restrict__ work, double* jcs,
                                        int& rot_flag, int& stop_all) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = CL == 1 ? 0 : (int)cluster.block_rank();
  const int t = threadIdx.x, hl = t & 15, lp = t >> 4;  // local pair
  const int m = cols + (cols & 1), np = m / 2;
  const int k = rank * ppc + lp;                        // global pair index
  const bool act = lp < ppc && k < np;
  const int E = rows + (Vout ? cols : 0);               // extended column length
  const size_t slot_sz = (size_t)E;
  double* slots = jcs;                                  // [2][ppc][2][rows]
  double* meta = jcs + 2 * (size_t)ppc * 2 * E;         // [2][ppc][4]: idp, nrm_p, idq, nrm_q
  const double tol2 = (double)rows * 2.220446049250313e-16 * 2.220446049250313e-16;
  const int src = (t & 31) & 16;                        // lane 0 of this half-warp
  auto hsum = [&](double v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return __shfl_sync(0xffffffffu, v, src);
  };
  int idp = k, idq = m - 1 - k;
  double xp[RPL], xq[RPL];
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = hl + 16 * r;
    if (i < rows) {
      xp[r] = (act && idp < cols) ? M[i + (size_t)idp * rows] : 0.0;
      xq[r] = (act && idq < cols) ? M[i + (size_t)idq * rows] : 0.0;
    } else {
      xp[r] = (act && i < E && i - rows == idp) ? 1.0 : 0.0;
      xq[r] = (act && i < E && i - rows == idq) ? 1.0 : 0.0;
    }
  }
  // where pair kk's slot lives: CTA kk / ppc, local kk % ppc
  auto slot_of = [&](int buf, int kk, int which) -> double* {
    double* local = slots + (((size_t)buf * ppc + (kk % ppc)) * 2 + which) * slot_sz;
    return jc_map<CL>(cluster, local, kk / ppc);
  };
  auto meta_of = [&](int buf, int kk) -> double* {
    double* local = meta + ((size_t)buf * ppc + (kk % ppc)) * 4;
    return jc_map<CL>(cluster, local, kk / ppc);
  };
  int buf = 0, sweep = 0;
  for (; sweep < 40; ++sweep) {
    double al = 0.0, be = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const bool in = hl + 16 * r < rows;
      al = fma(in ? xp[r] : 0.0, xp[r], al);
      be = fma(in ? xq[r] : 0.0, xq[r], be);
    }
    al = hsum(al);
    be = hsum(be);
    if (t == 0) rot_flag = 0;
    __syncthreads();
    for (int rd = 0; rd < m - 1; ++rd) {
      double ga = 0.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) ga = fma(hl + 16 * r < rows ? xp[r] : 0.0, xq[r], ga);
      ga = hsum(ga);
      if (act && al > 0.0 && be > 0.0 && ga * ga > tol2 * (al * be)) {
        const double zeta = (be - al) * jc_rcp(2.0 * ga);
        const double z2 = fma(zeta, zeta, 1.0);
        const double tt = copysign(jc_rcp(fabs(zeta) + z2 * rsqrt(z2)), zeta);
        const double c = rsqrt(fma(tt, tt, 1.0)), sn = c * tt;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const double x = xp[r], y = xq[r];
          xp[r] = c * x - sn * y;
          xq[r] = sn * x + c * y;
        }
        al = fma(-tt, ga, al);
        be = fma(tt, ga, be);
        if (hl == 0) rot_flag = 1;
      }
      // publish own columns (local slots), one cluster barrier, pull the next
      if (act) {
        double* sp = slots + (((size_t)buf * ppc + lp) * 2 + 0) * slot_sz;
        double* sq = slots + (((size_t)buf * ppc + lp) * 2 + 1) * slot_sz;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int i = hl + 16 * r;
          if (i < E) {
            sp[i] = xp[r];
            sq[i] = xq[r];
          }
        }
        if (hl == 0) {
          double* mt = meta + ((size_t)buf * ppc + lp) * 4;
          mt[0] = (double)idp;
          mt[1] = al;
          mt[2] = (double)idq;
          mt[3] = be;
        }
      }
      jc_sync<CL>(cluster);
      if (act) {
        // new p(k) = p(k+1) (1 <= k < np-1); new p(np-1) = q(np-1); p(0) stays
        // new q(k) = q(k-1) (k >= 1);        new q(0) = p(1)
        const bool last = k == np - 1;
        if (k >= 1) {
          if (last) {
#pragma unroll
            for (int r = 0; r < RPL; ++r) xp[r] = xq[r];
            idp = idq;
            al = be;
          } else {
            const double* rp = slot_of(buf, k + 1, 0);
            const double* mt = meta_of(buf, k + 1);
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
              const int i = hl + 16 * r;
              xp[r] = i < E ? rp[i] : 0.0;
            }
            idp = (int)mt[0];
            al = mt[1];
          }
          const double* rq = slot_of(buf, k - 1, 1);
          const double* mq = meta_of(buf, k - 1);
#pragma unroll
          for (int r = 0; r < RPL; ++r) {
            const int i = hl + 16 * r;
            xq[r] = i < E ? rq[i] : 0.0;
          }
          idq = (int)mq[2];
          be = mq[3];
        } else if (np > 1) {
          const double* rp = slot_of(buf, 1, 0);
          const double* mt = meta_of(buf, 1);
#pragma unroll
          for (int r = 0; r < RPL; ++r) {
            const int i = hl + 16 * r;
            xq[r] = i < E ? rp[i] : 0.0;
          }
          idq = (int)mt[0];
          be = mt[1];
        }
      }
      buf ^= 1;
    }
    // any rotation anywhere in the cluster this sweep?
    jc_sync<CL>(cluster);
    if (t == 0) {
      int any = 0;
      for (int c = 0; c < CL; ++c) any |= *jc_map<CL>(cluster, &rot_flag, c);
      stop_all = !any;
    }
    jc_sync<CL>(cluster);  // every CTA has read every flag before they are reset
    if (stop_all) break;
  }
  // columns back to the workspace by id; CTA 0 ranks and scatters
  double* A = work;
  double* Vw = work + (size_t)rows * cols;
  double* nrm = Vw + (size_t)cols * cols;
  if (act) {
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = hl + 16 * r;
      if (i < rows) {
        if (idp < cols) A[i + (size_t)idp * rows] = xp[r];
        if (idq < cols) A[i + (size_t)idq * rows] = xq[r];
      } else if (i < E) {
        if (idp < cols) Vw[(i - rows) + (size_t)idp * cols] = xp[r];
        if (idq < cols) Vw[(i - rows) + (size_t)idq * cols] = xq[r];
      }
    }
  }
  if (rank == 0 && t == 0) nrm[cols] = (double)(sweep + 1);
  __threadfence();
  jc_sync<CL>(cluster);
  if (rank != 0) return;
  const int lane = t & 31, warp = t >> 5, nw = blockDim.x / 32;
  for (int j = warp; j < cols; j += nw) {
    double s = 0.0;
    const double* a = A + (size_t)j * rows;
    for (int i = lane; i < rows; i += 32) s += a[i] * a[i];
    s = warp_sum(s);
    if (lane == 0) nrm[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = warp; j < cols; j += nw) {
    const double sj = nrm[j];
    int rk = 0;
    for (int i = lane; i < cols; i += 32) {
      const double si = nrm[i];
      rk += (si > sj || (si == sj && i < j)) ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) rk += __shfl_xor_sync(0xffffffffu, rk, o);
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    const double* a = A + (size_t)j * rows;
    double* u = U + (size_t)rk * rows;
    for (int i = lane; i < rows; i += 32) u[i] = a[i] * inv;
    if (Vout) {
      const double* v = Vw + (size_t)j * cols;
      double* vo = Vout + (size_t)rk * cols;
      for (int i = lane; i < cols; i += 32) vo[i] = v[i];
    }
    if (lane == 0) sig[rk] = sj;
  }
}

__global__ void __cluster_dims__(JC_CL, 1, 1) __launch_bounds__(256)
    k_svd_jacobi_cluster(const double* __restrict__ M, int rows, int cols, int ppc, double* __restrict__ U,
                         double* __restrict__ sig, double* __restrict__ Vout, double* __restrict__ work) {
  extern __shared__ __align__(16) double jcs[];
  __shared__ int rot_flag, stop_all;
  jc_body<JC_CL, JC_MAXROWS / 16>(M, rows, cols, ppc, U, sig, Vout, work, jcs, rot_flag, stop_all);
}

constexpr int JT_MAXE = 128;  // one-CTA variant: extended column length <= 128 (8 rows per lane)
// measured (tools/jacobi_probe.py): one CTA wins up to ~20 pairs (50x40 with
// V: 0.30 vs 0.33 ms), the 8-CTA cluster from 32 pairs (64x64: 0.67 vs 0.74)
constexpr int JT_MAXPAIRS = 24;

__global__ void __launch_bounds__(512)
    k_svd_jacobi_cta(const double* __restrict__ M, int rows, int cols, int ppc, double* __restrict__ U,
                     double* __restrict__ sig, double* __restrict__ Vout, double* __restrict__ work) {
  extern __shared__ __align__(16) double jcs[];
  __shared__ int rot_flag, stop_all;
  jc_body<1, JT_MAXE / 16>(M, rows, cols, ppc, U, sig, Vout, work, jcs, rot_flag, stop_all);
}

// ---------------------------------------------------------------------
// Block variant (k_svd_bjacobi_cluster, the default for 32 <= cols <= 256):
// the same one-sided Jacobi, but the tournament runs over 16 BLOCKS of b =
// cols / 16 columns (rounded up to even, zero-padded) instead of over single
// columns.  CTA c of the cluster
// holds the block pair (P_c, Q_c) in shared memory; one outer round
// orthogonalises every column of P_c against every column of Q_c in b inner
// rounds of b disjoint pairs (pair i: P_i with Q_(i+s) mod b), each closed by
// one __syncthreads; the blocks then move to the neighbouring CTAs through
// distributed shared memory behind ONE cluster barrier (the same block
// round-robin as the column tournament above).  The first outer round of
// every sweep also sweeps the pairs inside P_c and inside Q_c (2b - 1 inner
// rounds of the round-robin over the CTA's 2b columns).  Per sweep: the
// same number of pair rounds as the column tournament, but 15 cluster
// barriers instead of cols - 1 (the column kernel spends ~1.3 us per round on
// its barrier and DSMEM round trip).  Rotation, threshold (dgesvj's
// sqrt(m) eps), tracked norms and the final ranking as in jc_body.
constexpr int BJ_NB = 16;  // blocks (8 CTAs x 2)

template <int RPL>
__global__ void __cluster_dims__(JC_CL, 1, 1) __launch_bounds__(256)
    k_svd_bjacobi_cluster(const double* __restrict__ M, int rows, int cols, int b, double* __restrict__ U,
                          double* __restrict__ sig, double* __restrict__ Vout, double* __restrict__ work) {
  extern __shared__ __align__(16) double bjs[];
  __shared__ int rot_flag, stop_all;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int t = threadIdx.x, hl = t & 15, hw = t >> 4;  // half-warp = pair slot
  const int E = rows + (Vout ? cols : 0);
  const int np = BJ_NB / 2;                              // = JC_CL block pairs
  const int nb2 = 2 * b;
  // smem: cols [2 buf][2b][E], norms [2 buf][2b], ids [2 buf][2b] (as double)
  double* colsm = bjs;
  double* nrm = colsm + 2 * (size_t)nb2 * E;
  double* ids = nrm + 2 * nb2;
  auto col = [&](int buf, int j) { return colsm + ((size_t)buf * nb2 + j) * E; };
  const double tol2 = (double)rows * 2.220446049250313e-16 * 2.220446049250313e-16;
  const int src = (t & 31) & 16;
  auto hsum = [&](double v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return __shfl_sync(0xffffffffu, v, src);
  };
  // block ids of this CTA at the start: P = rank, Q = 2 np - 1 - rank
  // (global column id = block * b + local), columns >= cols are zero
  {
    const int bp = rank, bq = BJ_NB - 1 - rank;
    for (int e = t; e < nb2 * E; e += blockDim.x) {
      const int j = e / E, i = e % E;
      const int gid = (j < b ? bp * b + j : bq * b + (j - b));
      double v = 0.0;
      if (gid < cols) v = i < rows ? M[i + (size_t)gid * rows] : (i - rows == gid ? 1.0 : 0.0);
      col(0, j)[i] = v;
    }
    for (int j = t; j < nb2; j += blockDim.x) ids[j] = (double)(j < b ? bp * b + j : bq * b + (j - b));
  }
  __syncthreads();
  int buf = 0, sweep = 0;
  // one Jacobi rotation of columns (jp, jq) of buffer buf by half-warp hw
  // one Jacobi rotation of the column pair (xp, xq) held in this half-warp's
  // registers with squared norms (al, be); true when it rotated
  auto rot_regs = [&](double (&xp)[RPL], double (&xq)[RPL], double& al, double& be) {
    double g0 = 0.0, g1 = 0.0;  // two chains: the dot is on the round's critical path
#pragma unroll
    for (int r = 0; r < RPL; r += 2) {
      g0 = fma(hl + 16 * r < rows ? xp[r] : 0.0, xq[r], g0);
      if (r + 1 < RPL) g1 = fma(hl + 16 * (r + 1) < rows ? xp[r + 1] : 0.0, xq[r + 1], g1);
    }
    const double ga = hsum(g0 + g1);
    if (!(al > 0.0 && be > 0.0 && ga * ga > tol2 * (al * be))) return false;
    // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (be - al) / (2 ga),
    // as t = 2 ga sign(d) / (|d| + sqrt(d^2 + 4 ga^2)) with d = be - al:
    // one reciprocal on the chain instead of two
    const double d = be - al, g2 = 2.0 * ga;
    const double h = sqrt(fma(d, d, g2 * g2));
    const double tt = g2 * copysign(jc_rcp(fabs(d) + h), d);
    const double c = rsqrt(fma(tt, tt, 1.0)), sn = c * tt;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const double x = xp[r], y = xq[r];
      xp[r] = c * x - sn * y;
      xq[r] = sn * x + c * y;
    }
    al = fma(-tt, ga, al);
    be = fma(tt, ga, be);
    return true;
  };
  auto ld_col = [&](const double* c, double (&x)[RPL]) {
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = hl + 16 * r;
      x[r] = i < E ? c[i] : 0.0;
    }
  };
  auto st_col = [&](double* c, const double (&x)[RPL]) {
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = hl + 16 * r;
      if (i < E) c[i] = x[r];
    }
  };
  // columns (jp, jq) of buffer buf, through shared memory (round-robin phase)
  auto rotate = [&](int jp, int jq) {
    double xp[RPL], xq[RPL];
    double* np_ = nrm + (size_t)buf * nb2;
    ld_col(col(buf, jp), xp);
    ld_col(col(buf, jq), xq);
    double al = np_[jp], be = np_[jq];
    if (rot_regs(xp, xq, al, be)) {
      st_col(col(buf, jp), xp);
      st_col(col(buf, jq), xq);
      if (hl == 0) {
        np_[jp] = al;
        np_[jq] = be;
        rot_flag = 1;
      }
    }
  };
  for (; sweep < 40; ++sweep) {
    // exact norms at the start of every sweep (tracked through the rotations)
    for (int j = hw; j < nb2; j += blockDim.x / 16) {
      const double* c = col(buf, j);
      double a = 0.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = hl + 16 * r;
        a = fma(i < rows ? c[i] : 0.0, i < rows ? c[i] : 0.0, a);
      }
      a = hsum(a);
      if (hl == 0) nrm[(size_t)buf * nb2 + j] = a;
    }
    if (t == 0) rot_flag = 0;
    __syncthreads();
    for (int rd = 0; rd < 2 * np - 1; ++rd) {
      if (rd == 0) {  // every pair among the CTA's 2b columns: round-robin, 2b - 1 rounds
        for (int s = 0; s < nb2 - 1; ++s) {
          if (hw < b) {
            const int k = hw;
            const int a0 = k == 0 ? 0 : (k - 1 + s) % (nb2 - 1) + 1;
            const int a1 = (nb2 - 2 - k + s) % (nb2 - 1) + 1;
            rotate(a0, a1);
          }
          __syncthreads();
        }
      } else {  // P x Q cross pairs: b rounds of b disjoint pairs; P_hw stays
        // in registers, only the Q columns go through shared memory
        double xp[RPL], al = 0.0;
        bool rp = false;
        double* np_ = nrm + (size_t)buf * nb2;
        if (hw < b) {
          ld_col(col(buf, hw), xp);
          al = np_[hw];
        }
        for (int s = 0; s < b; ++s) {
          if (hw < b) {
            const int jq = b + (hw + s) % b;
            double xq[RPL];
            ld_col(col(buf, jq), xq);
            double be = np_[jq];
            if (rot_regs(xp, xq, al, be)) {
              rp = true;
              st_col(col(buf, jq), xq);
              if (hl == 0) np_[jq] = be;
            }
          }
          __syncthreads();
        }
        if (hw < b && rp) {
          st_col(col(buf, hw), xp);
          if (hl == 0) {
            np_[hw] = al;
            rot_flag = 1;
          }
        }
        __syncthreads();
      }
      // block round-robin across the cluster: P(k) <- P(k+1) (1 <= k < np-1),
      // P(np-1) <- Q(np-1), P(0) stays; Q(k) <- Q(k-1) (k >= 1), Q(0) <- P(1)
      cluster.sync();
      const int k = rank;
      int srcP, whichP, srcQ, whichQ;  // (CTA, 0 = its P / 1 = its Q)
      if (k == 0) {
        srcP = 0, whichP = 0;
        srcQ = 1, whichQ = 0;
      } else {
        if (k == np - 1) srcP = k, whichP = 1;
        else srcP = k + 1, whichP = 0;
        srcQ = k - 1, whichQ = 1;
      }
      const double* rP = cluster.map_shared_rank(col(buf, whichP * b), srcP);
      const double* rQ = cluster.map_shared_rank(col(buf, whichQ * b), srcQ);
      const double* nP = cluster.map_shared_rank(nrm + (size_t)buf * nb2 + whichP * b, srcP);
      const double* nQ = cluster.map_shared_rank(nrm + (size_t)buf * nb2 + whichQ * b, srcQ);
      const double* iP = cluster.map_shared_rank(ids + (size_t)buf * nb2 + whichP * b, srcP);
      const double* iQ = cluster.map_shared_rank(ids + (size_t)buf * nb2 + whichQ * b, srcQ);
      const int nb = buf ^ 1;
      const size_t blk = (size_t)b * E;  // a block's columns are contiguous
      {
        const double2* sp = reinterpret_cast<const double2*>(rP);
        const double2* sq = reinterpret_cast<const double2*>(rQ);
        double2* dp = reinterpret_cast<double2*>(col(nb, 0));
        double2* dq = reinterpret_cast<double2*>(col(nb, b));
        for (size_t e = t; e < blk / 2; e += blockDim.x) {
          dp[e] = sp[e];
          dq[e] = sq[e];
        }
      }
      for (int j = t; j < b; j += blockDim.x) {
        nrm[(size_t)nb * nb2 + j] = nP[j];
        nrm[(size_t)nb * nb2 + b + j] = nQ[j];
        ids[(size_t)nb * nb2 + j] = iP[j];
        ids[(size_t)nb * nb2 + b + j] = iQ[j];
      }
      buf = nb;
      __syncthreads();
    }
    // any rotation anywhere in the cluster this sweep?
    cluster.sync();
    if (t == 0) {
      int any = 0;
      for (int c = 0; c < JC_CL; ++c) any |= *cluster.map_shared_rank(&rot_flag, c);
      stop_all = !any;
    }
    cluster.sync();
    if (stop_all) break;
  }
  // columns back to the workspace by id; CTA 0 ranks and scatters (as jc_body)
  double* A = work;
  double* Vw = work + (size_t)rows * cols;
  double* nrmw = Vw + (size_t)cols * cols;
  for (int e = t; e < nb2 * E; e += blockDim.x) {
    const int j = e / E, i = e % E;
    const int gid = (int)ids[(size_t)buf * nb2 + j];
    if (gid >= cols) continue;
    const double v = col(buf, j)[i];
    if (i < rows) A[i + (size_t)gid * rows] = v;
    else Vw[(i - rows) + (size_t)gid * cols] = v;
  }
  if (rank == 0 && t == 0) nrmw[cols] = (double)(sweep + 1);
  __threadfence();
  cluster.sync();
  if (rank != 0) return;
  const int lane = t & 31, warp = t >> 5, nw = blockDim.x / 32;
  for (int j = warp; j < cols; j += nw) {
    double s2 = 0.0;
    const double* a = A + (size_t)j * rows;
    for (int i = lane; i < rows; i += 32) s2 += a[i] * a[i];
    s2 = warp_sum(s2);
    if (lane == 0) nrmw[j] = sqrt(s2);
  }
  __syncthreads();
  for (int j = warp; j < cols; j += nw) {
    const double sj = nrmw[j];
    int rk = 0;
    for (int i = lane; i < cols; i += 32) {
      const double si = nrmw[i];
      rk += (si > sj || (si == sj && i < j)) ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) rk += __shfl_xor_sync(0xffffffffu, rk, o);
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    const double* a = A + (size_t)j * rows;
    double* u = U + (size_t)rk * rows;
    for (int i = lane; i < rows; i += 32) u[i] = a[i] * inv;
    if (Vout) {
      const double* v = Vw + (size_t)j * cols;
      double* vo = Vout + (size_t)rk * cols;
      for (int i = lane; i < cols; i += 32) vo[i] = v[i];
    }
    if (lane == 0) sig[rk] = sj;
  }
}

// returns -1 when the shape is not handled by the register kernels
int launch_svd_jacobi_cluster(const double* M, int rows, int cols, double* U, double* sig, double* V,
                              double* work, cudaStream_t st) {
  const int E = rows + (V ? cols : 0);
  if (E > JC_MAXROWS || cols > rows || cols < 2) return -1;
  const int m = cols + (cols & 1), np = m / 2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_svd_jacobi_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_svd_jacobi_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const char* force = getenv("EDAK_JACOBI_CLUSTER");
  if (E <= JT_MAXE && np <= JT_MAXPAIRS && !(force && force[0] == '1')) {
    const size_t smem = (2 * (size_t)np * 2 * E + 2 * (size_t)np * 4) * sizeof(double);
    k_svd_jacobi_cta<<<1, ((16 * np + 31) / 32) * 32, smem, st>>>(M, rows, cols, np, U, sig, V, work);
    count_launch();
    return check_launch("k_svd_jacobi_cta");
  }
  // block Jacobi (k_svd_bjacobi_cluster) from 32 columns: b = cols / 16
  // columns per block (zero-padded), 2b half-warps' worth of pairs per CTA
  const char* eb = getenv("EDAK_JACOBI_BLOCK");
  // (b even: the 2b or b active half-warps then fill whole warps, which the
  // full-mask shuffles need)
  const int bsz = (((cols + BJ_NB - 1) / BJ_NB) + 1) & ~1;
  if (!(eb && eb[0] == '0') && cols >= 32 && bsz <= 16 && E % 2 == 0) {
    static bool battr = false;
    if (!battr) {
      cudaFuncSetAttribute(k_svd_bjacobi_cluster<JC_MAXROWS / 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
      cudaFuncSetAttribute(k_svd_bjacobi_cluster<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      battr = true;
    }
    const size_t smem = (2 * (size_t)(2 * bsz) * E + 4 * (size_t)(2 * bsz)) * sizeof(double);
    if (E <= 128)  // 8 rows per lane: half the loads and dot chain of the 256-row build
      k_svd_bjacobi_cluster<8><<<JC_CL, 256, smem, st>>>(M, rows, cols, bsz, U, sig, V, work);
    else
      k_svd_bjacobi_cluster<JC_MAXROWS / 16><<<JC_CL, 256, smem, st>>>(M, rows, cols, bsz, U, sig, V, work);
    count_launch();
    return check_launch("k_svd_bjacobi_cluster");
  }
  const int ppc = (np + JC_CL - 1) / JC_CL;
  if (ppc * 16 > 256) return -1;
  const size_t smem = (2 * (size_t)ppc * 2 * E + 2 * (size_t)ppc * 4) * sizeof(double);
  k_svd_jacobi_cluster<<<JC_CL, 256, smem, st>>>(M, rows, cols, ppc, U, sig, V, work);
  count_launch();
  return check_launch("k_svd_jacobi_cluster");
}

}  // namespace edak
