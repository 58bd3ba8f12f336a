// Register-chunk / shared-memory halo machinery for periodic 1-D stencil
// sweeps over the Lorenz-96 ring.
//
// A CTA owns a contiguous "range" of NT*C ring elements; thread t holds
// elements [t*C, t*C + C) in registers, in arrays laid out with a 2-element
// halo on each side: a[0..1] = elements -2,-1; a[2..C+1] = own; a[C+2..C+3] =
// elements C, C+1.  One exchange round publishes every thread's first two and
// last two own values to shared memory and fills the neighbours' halos, with a
// single __syncthreads (double-buffered slots, so round k+1 can start before a
// slow thread has finished reading round k).
//
// Tile mode: the range is a window of the ring [base, base + NT*C) with
// redundant halos; values near the range edges go stale one stencil reach per
// sub-stage, and the host sizes the halos so the output window stays exact.
// Periodic mode: nact = n / C threads cover the whole ring and the halo of
// thread 0 / nact-1 wraps.
#pragma once
#include "common.cuh"

namespace edak {

struct SweepGeom {
  int W;         // output window per tile (ring elements)
  int HL;        // left halo
  int periodic;  // 1: one tile covers the ring, nact = n / C
  int nact;
};

template <int C, int NT>
struct Ring {
  int t, prev, next, nact;
  bool hp, hn;
  int base;  // ring index of range element 0 (before wrap)
  int n;
  int g0;    // ring index of own element 0 (wrapped)

  __device__ __forceinline__ void init(int n_, int base_, int nact_, bool periodic) {
    n = n_;
    t = threadIdx.x;
    nact = nact_;
    base = base_;
    g0 = wrap(base + t * C, n);
    if (periodic) {
      prev = t == 0 ? nact - 1 : t - 1;
      next = t + 1 >= nact ? 0 : t + 1;
      hp = hn = true;
    } else {
      prev = t - 1;
      next = t + 1;
      hp = t > 0;
      hn = t + 1 < nact;
    }
  }
  // ring index of own element j (0 <= j < C; C <= n)
  __device__ __forceinline__ int gidx(int j) const {
    const int g = g0 + j;
    return g >= n ? g - n : g;
  }

  // load own elements and 2+2 halo of a ring vector straight from memory
  __device__ __forceinline__ void load_halo(const double* __restrict__ src, double (&a)[C + 4]) const {
#ifdef EDAK_EXP_NOLOAD
#pragma unroll
    for (int k = 0; k < C + 4; ++k) a[k] = 8.0 + 0.001 * k * (double)(size_t)(src - (const double*)0) * 1e-12;
    return;
#endif
    const int g = g0 >= 2 ? g0 - 2 : g0 - 2 + n;
    if (g + C + 4 <= n) {  // window does not wrap: straight loads
#pragma unroll
      for (int k = 0; k < C + 4; ++k) a[k] = __ldg(src + g + k);
    } else {
#pragma unroll
      for (int k = 0; k < C + 4; ++k) a[k] = __ldg(src + wrap(g + k, n));
    }
  }
  // the same as 16-byte pairs where the row is 16-byte aligned and the
  // thread's range starts even and does not wrap (every pair-layout tile)
  __device__ __forceinline__ void load_own2(const double* __restrict__ src, double (&a)[C + 4]) const {
    if (C % 2 == 0 && g0 % 2 == 0 && g0 + C <= n && ((uintptr_t)src & 15) == 0) {
#pragma unroll
      for (int k = 0; k < C / 2; ++k) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(src + g0) + k);
        a[2 * k + 2] = v.x;
        a[2 * k + 3] = v.y;
      }
    } else {
      load_own(src, a);
    }
  }
  // own elements inside the output window [wlo, whi) of the range: 16-byte
  // pair stores when the column base is 16-byte aligned and the ring, the
  // thread's first element and the window bounds are even (a pair is then
  // aligned, never wraps and is inside or outside as a whole), else scalar
  // (16 stores C * 8 B apart per thread: their issue ended every CTA)
  __device__ __forceinline__ void store_own(double* __restrict__ out, const double (&a)[C + 4], int wlo,
                                            int whi) const {
    if (C % 2 == 0 && n % 2 == 0 && g0 % 2 == 0 && wlo % 2 == 0 && whi % 2 == 0 && ((uintptr_t)out & 15) == 0) {
#pragma unroll
      for (int k = 0; k < C / 2; ++k) {
        const int e = t * C + 2 * k;
        if (e >= wlo && e < whi)
          *reinterpret_cast<double2*>(out + gidx(2 * k)) = make_double2(a[2 * k + 2], a[2 * k + 3]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < C; ++j) {
        const int e = t * C + j;
        if (e >= wlo && e < whi) out[gidx(j)] = a[j + 2];
      }
    }
  }
  __device__ __forceinline__ void load_own(const double* __restrict__ src, double (&a)[C + 4]) const {
    if (g0 + C <= n) {
#pragma unroll
      for (int k = 0; k < C; ++k) a[k + 2] = __ldg(src + g0 + k);
    } else {
#pragma unroll
      for (int k = 0; k < C; ++k) a[k + 2] = __ldg(src + wrap(g0 + k, n));
    }
  }

  // publish the first two / last two own values as two 16-byte pairs into
  // the planes sh2[0][NT + 2] (first pair) and sh2[1][NT + 2] (last pair),
  // slot t + 1: one STS.128 / LDS.128 per pair instead of two 8-byte
  // accesses (the halo traffic was ~28% of the TL sweep, ablation in
  // profiles/r1_sweep_knobs_ab.txt).  Slots 0 and NT + 1 are zero pads, so a
  // tile's edge threads read zeros without a branch (their halo is in the
  // budgeted garbage zone anyway).
  static constexpr int S = NT + 2;
  __device__ __forceinline__ void put(double* sh, const double (&a)[C + 4]) const {
    double2* p = reinterpret_cast<double2*>(sh);
    p[t + 1] = make_double2(a[2], a[3]);
    p[S + t + 1] = make_double2(a[C], a[C + 1]);
  }
  __device__ __forceinline__ void get(const double* sh, double (&a)[C + 4]) const {
    const double2* p = reinterpret_cast<const double2*>(sh);
    const double2 l = p[S + prev + 1], r = p[next + 1];
    a[0] = l.x;
    a[1] = l.y;
    a[C + 2] = r.x;
    a[C + 3] = r.y;
  }
};

// shared-memory exchange buffers: [2 bufs][2 arrays][2 planes of NT + 2
// 16-byte pairs] (stored as [4][NT + 2] doubles: the same bytes)
template <int NT>
struct XBuf {
  double v[2][2][4][NT + 2];
  // zero the pad slots (call once before the first exchange's barrier)
  __device__ __forceinline__ void init_pads() {
    const int i = threadIdx.x;
    if (i < 16) {
      const int b = i >> 3, a = (i >> 2) & 1, plane = (i >> 1) & 1, side = i & 1;
      double2* p = reinterpret_cast<double2*>(&v[b][a][0][0]);
      p[plane * (NT + 2) + (side ? NT + 1 : 0)] = make_double2(0.0, 0.0);
    }
  }
};

// EDAK_EXP_NOSYNC: timing experiments only (results are wrong without it)
#ifdef EDAK_EXP_NOSYNC
#define EDAK_XSYNC() __syncwarp()
#else
#define EDAK_XSYNC() __syncthreads()
#endif

// EDAK_EXP_NOXCHG: timing ablation (wrong results): barriers without the halo traffic
template <int C, int NT>
__device__ __forceinline__ void xchg1(const Ring<C, NT>& R, XBuf<NT>& X, int& buf, double (&a)[C + 4]) {
#ifdef EDAK_EXP_NOXCHG
  EDAK_XSYNC();
  return;
#endif
  R.put(&X.v[buf][0][0][0], a);
  EDAK_XSYNC();
  R.get(&X.v[buf][0][0][0], a);
  buf ^= 1;
}

template <int C, int NT>
__device__ __forceinline__ void xchg2(const Ring<C, NT>& R, XBuf<NT>& X, int& buf, double (&a)[C + 4],
                                      double (&b)[C + 4]) {
#ifdef EDAK_EXP_NOXCHG
  EDAK_XSYNC();
  return;
#endif
  R.put(&X.v[buf][0][0][0], a);
  R.put(&X.v[buf][1][0][0], b);
  EDAK_XSYNC();
  R.get(&X.v[buf][0][0][0], a);
  R.get(&X.v[buf][1][0][0], b);
  buf ^= 1;
}

// ---- warp tiles: the range is one warp's, halos move by shuffles ----------
// Lane t's left halo is lane t-1's last two own values, its right halo lane
// t+1's first two.  Lane 0 / 31 receive their own values instead: finite
// garbage inside the budgeted halo zone, like the zero pads of the CTA
// exchange.  No barrier and no shared memory, so ptxas can schedule the next
// sub-stage's interior elements across the exchange.
template <int C>
__device__ __forceinline__ void wxchg1(double (&a)[C + 4]) {
  a[0] = __shfl_up_sync(0xffffffffu, a[C], 1);
  a[1] = __shfl_up_sync(0xffffffffu, a[C + 1], 1);
  a[C + 2] = __shfl_down_sync(0xffffffffu, a[2], 1);
  a[C + 3] = __shfl_down_sync(0xffffffffu, a[3], 1);
}

// ---- coalesced staging of state tiles through shared memory -------------
// Loading each thread's (C + 4)-element window straight from global memory
// costs C + 4 loads whose lanes are C*8 bytes apart (one L1 wavefront per
// lane-sector): ~30% of the TL sweep's time.  Instead the CTA copies the
// window [base - 2, base + used + 2) with cp.async (consecutive threads ->
// consecutive addresses), into a layout padded by one double per C so that
// thread t's window starts at (C + 1) t: both the copy and the window reads
// are bank-conflict free.
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}
// zero-filling variant: src_bytes = 0 writes 0.0 without touching src
__device__ __forceinline__ void cp_async8z(double* dst, const double* src, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int C, int NT>
struct Stage {
  static constexpr int R = C * NT;
  static constexpr int PLEN = (R + 4) + (R + 4) / C + 2;
  __device__ static __forceinline__ int pi(int q) { return (q + 2) + (q + 2) / C; }
  // g0 = ring index of window element -2 for THIS thread's first copy (base - 2 + t)
  __device__ static __forceinline__ void stage(double* buf, const double* __restrict__ src, int g0, int n,
                                               int used) {
    static_assert(NT % C == 0, "padded stride");
    int g = g0;
    double* d = buf + pi((int)threadIdx.x - 2);
    for (int q = (int)threadIdx.x - 2; q < used + 2; q += NT) {
      cp_async8(d, src + g);
      d += NT + NT / C;
      g += NT;
      while (g >= n) g -= n;
    }
    cp_commit();
  }
  __device__ static __forceinline__ void win(const double* buf, int t, double (&a)[C + 4]) {
    const double* w = buf + (C + 1) * t;
#pragma unroll
    for (int k = 0; k < C + 4; ++k) a[k] = w[k + k / C];
  }
};

// Pair-staged variant (even n, even tile base, 16-byte aligned rows): the
// window is copied as 16-byte pairs by a fully unrolled, compile-time trip
// count of cp.async.cg (ceil((R + 4) / 2 / NT) per thread, ~7 instructions
// each) instead of the generic 8-byte loop (~30 instructions per copy,
// R / NT + 1 copies: ~12 issue slots per element-step, the largest non-DP
// cost of the sweeps).  Layout pads 2 doubles per C elements so that pairs
// stay 16-byte aligned; thread t's window then starts at (C + 2) t and is read
// with 16-byte loads, conflict-free (5t mod 8 distinct per quarter-warp).
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}

template <int C, int NT>
struct Stage2 {
  static_assert(C % 2 == 0, "pairs");
  static constexpr int R = C * NT;
  static constexpr int NPAIR = (R + 4) / 2;
  static constexpr int IT = (NPAIR + NT - 1) / NT;
  static constexpr int PLEN = (R + 4) + 2 * ((R + 4) / C) + 2;
  // gm2 = ring index (unwrapped, may be < 0) of window element -2;
  // pairs m < (used + 4) / 2 are copied
  __device__ static __forceinline__ void stage(double* buf, const double* __restrict__ src, int gm2, int n,
                                               int used) {
#ifdef EDAK_EXP_NOSTAGE  // timing ablation (wrong results): no state staging
    cp_commit();
    return;
#endif
    const int t = threadIdx.x;
    const int np = (used + 4) >> 1;
    double* d = buf + 2 * t + 2 * (t / (C / 2));
    constexpr int DSTEP = 2 * NT + 2 * (NT / (C / 2));  // smem doubles per NT pairs
    constexpr int NFULL = (R + 4) / 2;  // pairs of a full tile (tile mode: used == R)
    if (gm2 >= 0 && gm2 + used + 4 <= n && np == NFULL) {
      // full tile inside [0, n): only the last copy is predicated, on a
      // compile-time bound (the loop-invariant test hoists out of the sweep)
      const double* p = src + gm2 + 2 * t;
#pragma unroll
      for (int it = 0; it < IT; ++it)
        if (it + 1 < IT || t + it * NT < NFULL) cp_async16(d + it * DSTEP, p + 2 * it * NT);
    } else if (gm2 >= 0 && gm2 + used + 4 <= n) {
      // window inside [0, n): immediate offsets, ~2 instructions per copy
      const double* p = src + gm2 + 2 * t;
#pragma unroll
      for (int it = 0; it < IT; ++it)
        if (t + it * NT < np) cp_async16(d + it * DSTEP, p + 2 * it * NT);
    } else {
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const int m = t + it * NT;
        if (m < np) {
          int g = gm2 + 2 * m;
          g = g < 0 ? g + n : (g >= n ? g - n : g);
          cp_async16(d + it * DSTEP, src + g);
        }
      }
    }
    cp_commit();
  }
  __device__ static __forceinline__ void win(const double* buf, int t, double (&a)[C + 4]) {
    const double2* w = reinterpret_cast<const double2*>(buf + (C + 2) * t);
#pragma unroll
    for (int k = 0; k < C / 2; ++k) {
      const double2 v = w[k];
      a[2 * k] = v.x;
      a[2 * k + 1] = v.y;
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double2 v = w[C / 2 + 1 + k];
      a[C + 2 * k] = v.x;
      a[C + 2 * k + 1] = v.y;
    }
  }
};

}  // namespace edak
