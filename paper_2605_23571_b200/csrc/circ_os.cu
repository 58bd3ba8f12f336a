// Circulant U_B (GridCovFactor.apply, covariance.py:41-47) by overlap-save
// block FFTs: out = u (*) v with the banded generator u (taps, circ.cu).
//
// One CTA = one block of V = M - K + 1 consecutive outputs of TWO columns,
// packed as one complex vector z_q = a_q + i b_q (q < M) over the block's
// input window.  Because u is real, the circular convolution of the block
// with u is (u * a) + i (u * b): no real-FFT split or merge.  z is
// transformed in shared memory by a radix-2/radix-8 decimation-in-frequency
// FFT (natural -> bit-reversed order), multiplied by the block kernel's
// spectrum H (host-computed, stored in the same bit-reversed order, 1/M
// folded in), and brought back by the mirrored decimation-in-time inverse
// (bit-reversed -> natural): no permutation pass.  Outputs q in [L, L + V)
// of the block are exact linear-convolution values (L = left reach of u).
//
// Work per output: ~2 log2(M) complex butterflies for two columns at
// (M / V) redundancy, against K FMAs per column for the tap convolution
// (cfg4: M = 1024, K = 189, V = 836).
#include "common.cuh"
#include <cstdlib>

namespace edak {

namespace os {

__device__ __forceinline__ int pz(int j) { return j + (j >> 3); }  // 1 pad per 8 (16-byte banks)

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cmul_mi(double2 a) { return make_double2(a.y, -a.x); }
__device__ __forceinline__ double2 cmul_pi(double2 a) { return make_double2(-a.y, a.x); }

// W_M^e = exp(-2 pi i e / M) from T[m] = exp(-2 pi i m / (2M)), m < M
template <int M>
__device__ __forceinline__ double2 tw(const double2* __restrict__ T, int e) {
  const int m = 2 * e;
  if (m < M) return __ldg(T + m);
  const double2 v = __ldg(T + (m - M));
  return make_double2(-v.x, -v.y);
}

// multiply by the eighth roots exp(-+2 pi i m / 8), m = 0..3
template <bool INV>
__device__ __forceinline__ double2 w8(double2 a, int m) {
  const double r = 0.70710678118654752440;
  if (m == 0) return a;
  if (m == 2) return INV ? cmul_pi(a) : cmul_mi(a);
  if (m == 1) return INV ? make_double2(r * (a.x - a.y), r * (a.x + a.y)) : make_double2(r * (a.x + a.y), r * (a.y - a.x));
  return INV ? make_double2(-r * (a.x + a.y), r * (a.x - a.y)) : make_double2(r * (a.y - a.x), -r * (a.x + a.y));
}

// Twiddles of every pass, fetched once per thread at kernel start (their
// loads then overlap the input loads instead of stalling each pass): the
// DIF pass of radix-8 group stride q and the DIT pass of span q use the same
// W_M^e (conjugated), and so do the radix-2 stages of equal span.
template <int LOGM, int NT>
struct Tw {
  static constexpr int M = 1 << LOGM, R2 = LOGM % 3, R8 = LOGM / 3, P2 = M / 2 / NT;
  static_assert(M / 8 == NT, "one radix-8 group per thread and pass");
  double2 w2[R2 > 0 ? R2 : 1][P2];
  double2 w8[R8];
  __device__ __forceinline__ void load(const double2* __restrict__ T) {
    const int t = threadIdx.x;
    int h = M >> 1;
#pragma unroll
    for (int r = 0; r < R2; ++r, h >>= 1)
#pragma unroll
      for (int k = 0; k < P2; ++k) w2[r][k] = tw<M>(T, ((t + k * NT) % h) * (M / (2 * h)));
#pragma unroll
    for (int pass = 0; pass < R8; ++pass, h >>= 3) {
      const int q = h >> 2;
      w8[pass] = q > 1 ? tw<M>(T, (t % q) * (M / (2 * h))) : make_double2(1.0, 0.0);
    }
  }
};

// forward DIF over Z[pz(.)], M = 2^LOGM points: LOGM % 3 radix-2 stages,
// then radix-8 passes; output in bit-reversed order
template <int LOGM, int NT>
__device__ __forceinline__ void dif(double2* Z, const Tw<LOGM, NT>& W) {
  constexpr int M = 1 << LOGM;
  const int t = threadIdx.x;
  int h = M >> 1;
#pragma unroll
  for (int r = 0; r < LOGM % 3; ++r, h >>= 1) {
#pragma unroll
    for (int k = 0; k < M / 2 / NT; ++k) {
      const int p = t + k * NT;
      const int j = (p / h) * 2 * h + p % h;
      const double2 x = Z[pz(j)], y = Z[pz(j + h)];
      Z[pz(j)] = cadd(x, y);
      Z[pz(j + h)] = cmul(csub(x, y), W.w2[r][k]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int pass = 0; pass < LOGM / 3; ++pass, h >>= 3) {
    const int q = h >> 2;
    const int g = t;
    const int r0 = g % q, j0 = (g / q) * 2 * h + r0;
    double2 a[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) a[m] = Z[pz(j0 + m * q)];
    const double2 b1 = W.w8[pass];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const double2 x = a[m], y = a[m + 4];
      a[m] = cadd(x, y);
      a[m + 4] = cmul(w8<false>(csub(x, y), m), b1);
    }
    const double2 b2 = cmul(b1, b1);
#pragma unroll
    for (int mm = 0; mm < 4; ++mm) {
      const int m = (mm & 1) + 4 * (mm >> 1);  // 0, 1, 4, 5
      const double2 x = a[m], y = a[m + 2];
      a[m] = cadd(x, y);
      const double2 d = cmul(csub(x, y), b2);
      a[m + 2] = (m & 1) ? cmul_mi(d) : d;
    }
    const double2 b4 = cmul(b2, b2);
#pragma unroll
    for (int m = 0; m < 8; m += 2) {
      const double2 x = a[m], y = a[m + 1];
      a[m] = cadd(x, y);
      a[m + 1] = cmul(csub(x, y), b4);
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) Z[pz(j0 + m * q)] = a[m];
    __syncthreads();
  }
}

// inverse DIT (unscaled), bit-reversed -> natural: radix-8 passes from span
// 1, then LOGM % 3 radix-2 stages (the exact mirror of dif)
template <int LOGM, int NT>
__device__ __forceinline__ void dit(double2* Z, const Tw<LOGM, NT>& W) {
  constexpr int M = 1 << LOGM;
  const int t = threadIdx.x;
  int h = 1;
#pragma unroll
  for (int pass = LOGM / 3 - 1; pass >= 0; --pass, h <<= 3) {
    const int g = t;
    const int r0 = g % h, j0 = (g / h) * 8 * h + r0;
    double2 a[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) a[m] = Z[pz(j0 + m * h)];
    const double2 c1 = cconj(W.w8[pass]);
    const double2 c2 = cmul(c1, c1), c4 = cmul(c2, c2);
#pragma unroll
    for (int m = 0; m < 8; m += 2) {
      const double2 x = a[m], y = cmul(a[m + 1], c4);
      a[m] = cadd(x, y);
      a[m + 1] = csub(x, y);
    }
#pragma unroll
    for (int mm = 0; mm < 4; ++mm) {
      const int m = (mm & 1) + 4 * (mm >> 1);
      const double2 d = cmul(a[m + 2], c2);
      const double2 x = a[m], y = (m & 1) ? cmul_pi(d) : d;
      a[m] = cadd(x, y);
      a[m + 2] = csub(x, y);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const double2 x = a[m], y = w8<true>(cmul(a[m + 4], c1), m);
      a[m] = cadd(x, y);
      a[m + 4] = csub(x, y);
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) Z[pz(j0 + m * h)] = a[m];
    __syncthreads();
  }
#pragma unroll
  for (int r = LOGM % 3 - 1; r >= 0; --r, h <<= 1) {
#pragma unroll
    for (int k = 0; k < M / 2 / NT; ++k) {
      const int p = t + k * NT;
      const int j = (p / h) * 2 * h + p % h;
      const double2 x = Z[pz(j)], y = cmul(Z[pz(j + h)], cconj(W.w2[r][k]));
      Z[pz(j)] = cadd(x, y);
      Z[pz(j + h)] = csub(x, y);
    }
    __syncthreads();
  }
}

}  // namespace os

// transform + epilogue of one item (block blk of the column pair (ca, ca+1))
// whose input window already sits in Z
template <int LOGM, int NT>
__device__ __forceinline__ void os_item(double2* Z, double (*red)[NT / 32], const os::Tw<LOGM, NT>& W,
                                        const double2* __restrict__ H, int n, int L, int V, int ncols, int blk,
                                        int ca, double* __restrict__ out, double ident,
                                        const double* __restrict__ zadd, double* __restrict__ dotp, int dtiles,
                                        const double2* hpre = nullptr) {
  using namespace os;
  constexpr int M = 1 << LOGM;
  const int t = threadIdx.x, cb = ca + 1;
  const bool hb = cb < ncols;
  const int i0 = blk * V;
  dif<LOGM, NT>(Z, W);
  if (hpre) {  // block spectrum fetched at kernel start (its L2 latency hidden)
#pragma unroll
    for (int k = 0; k < M / NT; ++k) Z[pz(t + k * NT)] = cmul(Z[pz(t + k * NT)], hpre[k]);
  } else {
#pragma unroll
    for (int j = t; j < M; j += NT) Z[pz(j)] = cmul(Z[pz(j)], __ldg(H + j));
  }
  __syncthreads();
  dit<LOGM, NT>(Z, W);
  // epilogue: outputs i0 + j, j < V, at block position L + j
  double da = 0.0, db = 0.0;
  const int nv = min(V, n - i0);
  double* oa = out + (size_t)ca * n;
  double* ob = out + (size_t)cb * n;
  const double* za = zadd ? zadd + (size_t)ca * n : nullptr;
  const double* zb = zadd ? zadd + (size_t)cb * n : nullptr;
  for (int j = t; j < nv; j += NT) {
    const double2 y = Z[pz(L + j)];
    double va = y.x, vb = y.y;
    const int i = i0 + j;
    if (za) {
      const double z1 = za[i];
      va = fma(ident, z1, va);
      da = fma(z1, va, da);
      if (hb) {
        const double z2 = zb[i];
        vb = fma(ident, z2, vb);
        db = fma(z2, vb, db);
      }
    }
    oa[i] = va;
    if (hb) ob[i] = vb;
  }
  if (dotp) {  // fixed-order CTA reduction -> dotp[col][blk]; slots past the last block get 0
    da = warp_sum(da);
    db = warp_sum(db);
    if ((t & 31) == 0) {
      red[0][t >> 5] = da;
      red[1][t >> 5] = db;
    }
    __syncthreads();
    if (t < 2 && (t == 0 || hb)) {
      double s = 0.0;
      for (int w = 0; w < NT / 32; ++w) s += red[t][w];
      dotp[(size_t)(ca + t) * dtiles + blk] = s;
    }
    if (blk == 0) {
      for (int q = (int)gridDim.x + t; q < dtiles; q += NT) {
        dotp[(size_t)ca * dtiles + q] = 0.0;
        if (hb) dotp[(size_t)cb * dtiles + q] = 0.0;
      }
    }
    __syncthreads();  // red is reused by the next item
  }
}

// grid (blocks of V outputs, column pairs); L = left reach of u (taps k <
// K act on in[i + tap_w - k]: reach K - 1 - tap_w to the left, tap_w right)
template <int LOGM, int NT, int MINB = 1, bool PREH = false>
__global__ void __launch_bounds__(NT, MINB) k_circ_os(int n, int L, int V, int ncols, const double2* __restrict__ T,
                                                const double2* __restrict__ H, const double* __restrict__ in,
                                                double* __restrict__ out, double ident,
                                                const double* __restrict__ zadd, double* __restrict__ dotp,
                                                int dtiles) {
  using namespace os;
  constexpr int M = 1 << LOGM;
  __shared__ __align__(16) double2 Z[M + M / 8];
  __shared__ double red[2][NT / 32];
  const int t = threadIdx.x, blk = blockIdx.x;
  const int ca = 2 * blockIdx.y, cb = ca + 1;
  const bool hb = cb < ncols;
  const int i0 = blk * V;
  const double* A = in + (size_t)ca * n;
  const double* B = in + (size_t)(hb ? cb : ca) * n;
  // window [i0 - L, i0 - L + M) of the ring: n > M (os_logm_for), so one
  // conditional wrap per index; every load is issued before the first store
  double ra[M / NT], rb[M / NT];
#pragma unroll
  for (int k = 0; k < M / NT; ++k) {
    int g = i0 - L + t + k * NT;
    g = g < 0 ? g + n : (g >= n ? g - n : g);
    ra[k] = __ldg(A + g);
    rb[k] = hb ? __ldg(B + g) : 0.0;
  }
  Tw<LOGM, NT> W;
  W.load(T);
  double2 hv[PREH ? M / NT : 1];
  if (PREH) {
#pragma unroll
    for (int k = 0; k < M / NT; ++k) hv[k] = __ldg(H + t + k * NT);
  }
#pragma unroll
  for (int k = 0; k < M / NT; ++k) Z[pz(t + k * NT)] = make_double2(ra[k], rb[k]);
  __syncthreads();
  os_item<LOGM, NT>(Z, red, W, H, n, L, V, ncols, blk, ca, out, ident, zadd, dotp, dtiles,
                    PREH ? hv : nullptr);
}

// ---------------------------------------------------------------------
// Register-pass variant (k_circ_os16): the same overlap-save block FFT --
// the same in-place radix-2 DIF network, so the same bit-reversed output
// order and the same host spectrum H -- with its stages grouped into three
// register passes per direction instead of two radix-2 stages plus three
// radix-8 passes, each a shared-memory round trip:
//
//   M = 2048 (cfg5): radix-16 over bits [7, 11) straight from the global
//   window, radix-16 over bits [3, 7), then radix-8 over bits [0, 3) with
//   the spectrum product and the first inverse radix-8 on the same
//   registers; the inverse radix-16 over bits [3, 7) and over bits [7, 11),
//   whose registers are the natural-order outputs, stored straight to the
//   output column.  Shared memory carries 4 round trips of the block
//   instead of ~11: the 2048-point kernel was shared-memory-bandwidth bound
//   (~770 KB of LDS/STS traffic per block).
//
// A radix-2^K pass at bit offset b holds the elements base + m 2^b (m <
// 2^K; base has zero bits in [b, b + K)); local stage j (span 2^j in m)
// multiplies the difference of pair (m, m + 2^j) by W_{2^(j+1)}^(m mod 2^j)
// (compile-time roots) and by W_M^(r 2^(LOGM-1-b-j)), r = base mod 2^b.
namespace os16 {

using os::cadd;
using os::cconj;
using os::cmul;
using os::csub;

// a * W_{2^(J+1)}^p (forward) or its conjugate (INV), p < 2^J, J <= 3
template <int J, bool INV>
__device__ __forceinline__ double2 root(double2 a, int p) {
  if (p == 0) return a;
  constexpr int S = 3 - J;  // W_{2^(J+1)}^p = W_16^(p 2^S)
  const int q = p << S;     // 1..7 eighths of pi
  if (q == 4) return INV ? os::cmul_pi(a) : os::cmul_mi(a);
  if (q == 2 || q == 6) return os::w8<INV>(a, q >> 1);
  // odd sixteenths: cos / sin of pi q / 8
  const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
  double c, sn;
  if (q == 1) c = c1, sn = s1;
  else if (q == 3) c = s1, sn = c1;
  else if (q == 5) c = -s1, sn = c1;
  else c = -c1, sn = s1;  // q == 7
  const double w_im = INV ? sn : -sn;
  return make_double2(fma(a.x, c, -a.y * w_im), fma(a.x, w_im, a.y * c));
}

// forward DIF of 2^K registers; tw[j] = W_M^(r 2^(LOGM-1-b-j)) (TW: apply)
template <int K, bool TW>
__device__ __forceinline__ void dif(double2 (&a)[1 << K], const double2 (&tw)[K]) {
#pragma unroll
  for (int j = K - 1; j >= 0; --j) {
    const int hl = 1 << j;
#pragma unroll
    for (int m = 0; m < (1 << K); ++m) {
      if (m & hl) continue;
      const double2 x = a[m], y = a[m + hl];
      a[m] = cadd(x, y);
      double2 d = csub(x, y);
      switch (j) {
        case 0: break;
        case 1: d = root<1, false>(d, m & 1); break;
        case 2: d = root<2, false>(d, m & 3); break;
        default: d = root<3, false>(d, m & 7); break;
      }
      a[m + hl] = TW ? cmul(d, tw[j]) : d;
    }
  }
}

// inverse DIT (unscaled), the exact mirror of dif
template <int K, bool TW>
__device__ __forceinline__ void dit(double2 (&a)[1 << K], const double2 (&tw)[K]) {
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int hl = 1 << j;
#pragma unroll
    for (int m = 0; m < (1 << K); ++m) {
      if (m & hl) continue;
      double2 y = a[m + hl];
      if (TW) y = cmul(y, cconj(tw[j]));
      switch (j) {
        case 0: break;
        case 1: y = root<1, true>(y, m & 1); break;
        case 2: y = root<2, true>(y, m & 3); break;
        default: y = root<3, true>(y, m & 7); break;
      }
      const double2 x = a[m];
      a[m] = cadd(x, y);
      a[m + hl] = csub(x, y);
    }
  }
}

template <int M, int K>
__device__ __forceinline__ void load_tw(double2 (&tw)[K], const double2* __restrict__ T, int r, int sh) {
  // tw[j] = W_M^(r 2^(sh - j)), sh = LOGM - 1 - b
#pragma unroll
  for (int j = 0; j < K; ++j) tw[j] = os::tw<M>(T, (r << (sh - j)) & (M - 1));
}

}  // namespace os16

// M = 2^LOGM points, M / 16 threads: pass A = radix-16 over bits
// [LOGM - 4, LOGM) (one group per thread), pass B = radix-2^KB over bits
// [3, LOGM - 4) (KB = 4 at M = 2048: one group per thread; KB = 3 at M =
// 1024: two), pass C = radix-8 over bits [0, 3) (two groups per thread).
// The transform and epilogue of one item (block blk of the column pair
// (ca, ca + 1)) whose pass-A input a[m] = window element t + NT m is in
// registers; nb = blocks per column (the dot-partial slots past it get 0).
template <int LOGM>
__device__ __forceinline__ void os16_item(double2 (&a)[16], double2* Z, double (*red)[(1 << LOGM) / 16 / 32 > 0
                                                                                   ? (1 << LOGM) / 16 / 32
                                                                                   : 1],
                                          const double2* __restrict__ T, const double2* __restrict__ H, int n,
                                          int L, int V, int ncols, int blk, int ca, int nb,
                                          double* __restrict__ out, double ident, const double* __restrict__ zadd,
                                          double* __restrict__ dotp, int dtiles) {
  using namespace os16;
  static_assert(LOGM == 10 || LOGM == 11, "passes: [LOGM-4, LOGM) [3, LOGM-4) [0, 3)");
  constexpr int M = 1 << LOGM, NT = M / 16;
  constexpr int BA = LOGM - 4, BB = 3, KB = LOGM - 7;  // pass A / B bit offsets, pass B radix log2
  constexpr int GB = 16 >> KB;                         // pass-B groups per thread
  const int t = threadIdx.x, cb = ca + 1;
  const bool hb = cb < ncols;
  const int i0 = blk * V;
  double2 tw[4], twb[KB];
  load_tw<M, 4>(tw, T, t, LOGM - 1 - BA);
  dif<4, true>(a, tw);
#pragma unroll
  for (int m = 0; m < 16; ++m) Z[os::pz(t + NT * m)] = a[m];
  __syncthreads();
  // pass B: group q = t + NT h: base = (q mod 8) + 2^(LOGM-4) (q / 8),
  // elements base + 8 m; r = q mod 8 = t mod 8 for every h
  load_tw<M, KB>(twb, T, t & 7, LOGM - 1 - BB);
  auto baseB = [&](int h) {
    const int q = t + NT * h;
    return (q & 7) + ((q >> 3) << BA);
  };
#pragma unroll
  for (int h = 0; h < GB; ++h) {
    double2 b[1 << KB];
    const int bb = baseB(h);
#pragma unroll
    for (int m = 0; m < (1 << KB); ++m) b[m] = Z[os::pz(bb + (m << BB))];
    dif<KB, true>(b, twb);
#pragma unroll
    for (int m = 0; m < (1 << KB); ++m) Z[os::pz(bb + (m << BB))] = b[m];
  }
  __syncthreads();
  // pass C: bits [0, 3), groups g = t and t + NT (elements 8 g + m): the
  // last forward radix-8, the spectrum product, the first inverse radix-8
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int g8 = 8 * (t + NT * h);
    double2 c[8], hv[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) hv[m] = __ldg(H + g8 + m);
#pragma unroll
    for (int m = 0; m < 8; ++m) c[m] = Z[os::pz(g8 + m)];
    const double2 none[3] = {};
    dif<3, false>(c, none);
#pragma unroll
    for (int m = 0; m < 8; ++m) c[m] = cmul(c[m], hv[m]);
    dit<3, false>(c, none);
#pragma unroll
    for (int m = 0; m < 8; ++m) Z[os::pz(g8 + m)] = c[m];
  }
  __syncthreads();
  // inverse pass B
#pragma unroll
  for (int h = 0; h < GB; ++h) {
    double2 b[1 << KB];
    const int bb = baseB(h);
#pragma unroll
    for (int m = 0; m < (1 << KB); ++m) b[m] = Z[os::pz(bb + (m << BB))];
    dit<KB, true>(b, twb);
#pragma unroll
    for (int m = 0; m < (1 << KB); ++m) Z[os::pz(bb + (m << BB))] = b[m];
  }
  __syncthreads();
  // inverse pass A: natural-order outputs q = t + NT m, straight to HBM
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = Z[os::pz(t + NT * m)];
  dit<4, true>(a, tw);
  const int nv = min(V, n - i0);
  double* oa = out + (size_t)ca * n;
  double* ob = out + (size_t)cb * n;
  const double* za = zadd ? zadd + (size_t)ca * n : nullptr;
  const double* zb = zadd ? zadd + (size_t)cb * n : nullptr;
  double da = 0.0, db = 0.0;
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int j = t + NT * m - L;  // output i0 + j
    if (j < 0 || j >= nv) continue;
    double va = a[m].x, vb = a[m].y;
    const int i = i0 + j;
    if (za) {
      const double z1 = za[i];
      va = fma(ident, z1, va);
      da = fma(z1, va, da);
      if (hb) {
        const double z2 = zb[i];
        vb = fma(ident, z2, vb);
        db = fma(z2, vb, db);
      }
    }
    oa[i] = va;
    if (hb) ob[i] = vb;
  }
  if (dotp) {  // fixed-order CTA reduction -> dotp[col][blk]; slots past the last block get 0
    da = warp_sum(da);
    db = warp_sum(db);
    if ((t & 31) == 0) {
      red[0][t >> 5] = da;
      red[1][t >> 5] = db;
    }
    __syncthreads();
    if (t < 2 && (t == 0 || hb)) {
      double s = 0.0;
      for (int w = 0; w < NT / 32; ++w) s += red[t][w];
      dotp[(size_t)(ca + t) * dtiles + blk] = s;
    }
    if (blk == 0) {
      for (int q = nb + t; q < dtiles; q += NT) {
        dotp[(size_t)ca * dtiles + q] = 0.0;
        if (hb) dotp[(size_t)cb * dtiles + q] = 0.0;
      }
    }
  }
}


// one item per CTA, the window straight from HBM into registers
template <int LOGM, int MINB>
__global__ void __launch_bounds__((1 << LOGM) / 16, MINB)
    k_circ_os16(int n, int L, int V, int ncols, const double2* __restrict__ T, const double2* __restrict__ H,
                const double* __restrict__ in, double* __restrict__ out, double ident,
                const double* __restrict__ zadd, double* __restrict__ dotp, int dtiles) {
  constexpr int M = 1 << LOGM, NT = M / 16;
  __shared__ __align__(16) double2 Z[M + M / 8];
  __shared__ double red[2][NT / 32 > 0 ? NT / 32 : 1];
  const int t = threadIdx.x, blk = blockIdx.x;
  const int ca = 2 * blockIdx.y, cb = ca + 1;
  const bool hb = cb < ncols;
  const int i0 = blk * V;
  const double* A = in + (size_t)ca * n;
  const double* B = in + (size_t)(hb ? cb : ca) * n;
  // pass A: elements t + NT m of the window [i0 - L, i0 - L + M), from HBM
  double2 a[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    int g = i0 - L + t + NT * m;
    g = g < 0 ? g + n : (g >= n ? g - n : g);
    a[m] = make_double2(__ldg(A + g), hb ? __ldg(B + g) : 0.0);
  }
  if (zadd) {
    // the epilogue adds ident * z and reduces z . out over this block's
    // outputs [i0, i0 + nv): pull those lines of z towards L2 now, so the
    // epilogue's loads do not pay the DRAM latency at the end of every CTA
    // (ncu: long_scoreboard 62% of the z-adding call's samples, 649 against
    // 471 us per 256 cfg5 columns for the plain call)
    const int nv = min(V, n - i0);
    const double* za = zadd + (size_t)ca * n + i0;
    const double* zb = zadd + (size_t)(hb ? cb : ca) * n + i0;
    for (int q = 16 * t; q < nv + 15; q += 16 * NT) {
      const int qq = min(q, nv - 1);
      asm volatile("prefetch.global.L2 [%0];\n" ::"l"(za + qq));
      asm volatile("prefetch.global.L2 [%0];\n" ::"l"(zb + qq));
    }
  }
  os16_item<LOGM>(a, Z, red, T, H, n, L, V, ncols, blk, ca, (int)gridDim.x, out, ident, zadd, dotp, dtiles);
}

// U_B by overlap-save when the problem carries the block spectrum
// (edak_problem.os_logm/os_spec/os_tw, covariance.py DeviceFactor); returns
// EDAK_EUNSUPPORTED when it does not apply (the caller then convolves)
int launch_circ_os(const edak_problem* P, const double* in, double* out, int ncols, double ident,
                   const double* zadd, cudaStream_t st, double* dotp, int dtiles) {
  const int logm = P->os_logm, K = P->ntaps, n = P->n;
  if (!P->os_spec || !P->os_tw || (logm != 10 && logm != 11)) return EDAK_EUNSUPPORTED;
  const int M = 1 << logm, V = M - K + 1, L = K - 1 - P->tap_w;
  if (V < M / 2 || L < 0 || P->tap_w < 0 || n <= M) return EDAK_EUNSUPPORTED;
  const int nb = (n + V - 1) / V;
  if (dotp && nb > dtiles) return EDAK_EUNSUPPORTED;
  dim3 grid(nb, (ncols + 1) / 2);
  const double2* T = reinterpret_cast<const double2*>(P->os_tw);
  const double2* H = reinterpret_cast<const double2*>(P->os_spec);
  // resident CTAs per SM the M = 1024 kernel is built for (A/B knob; 6 =
  // 80 registers measured best: cfg4 U_B pair 3% faster than 1 (126 regs))
  // M = 1024 (cfg4): the block spectrum fetched at kernel start into 4
  // resident CTAs' registers (122, no spills): 19.2 -> 17.3 us per 100
  // columns (profiles/r2_circ_os_ab.txt); EDAK_CIRC_OS_PREH=0 / _MINB = A/B
  const char* e16 = getenv("EDAK_CIRC_OS16");
  const int os16 = e16 ? atoi(e16) : 1;  // register-pass kernels (0: the shared-memory radix-2/8 passes)
  if (logm == 10 && os16) {
    const char* e1 = getenv("EDAK_CIRC_OS16_MINB10");
    const int m1 = e1 ? atoi(e1) : 6;
    if (m1 == 8)
      k_circ_os16<10, 8><<<grid, 64, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
    else if (m1 == 4)
      k_circ_os16<10, 4><<<grid, 64, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
    else
      k_circ_os16<10, 6><<<grid, 64, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
    count_launch();
    return check_launch("k_circ_os16");
  }
  const char* eb = getenv("EDAK_CIRC_OS_MINB");
  const char* ep = getenv("EDAK_CIRC_OS_PREH");
  const bool preh = !(ep && atoi(ep) == 0) && logm == 10;
  const int mb = eb ? atoi(eb) : (preh ? 4 : 6);
  if (logm == 10 && preh && mb == 4)
    k_circ_os<10, 128, 4, true><<<grid, 128, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
  else if (logm == 10 && preh)
    k_circ_os<10, 128, 6, true><<<grid, 128, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
  else if (logm == 10 && mb == 8)
    k_circ_os<10, 128, 8><<<grid, 128, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
  else if (logm == 10 && mb == 6)
    k_circ_os<10, 128, 6><<<grid, 128, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
  else if (logm == 10)
    k_circ_os<10, 128><<<grid, 128, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
  else if (os16) {
    // M = 2048 (cfg5): register-pass variant (k_circ_os16), 128 threads
    const char* e2 = getenv("EDAK_CIRC_OS16_MINB");
    const int m2 = e2 ? atoi(e2) : 4;
    if (m2 == 3)
      k_circ_os16<11, 3><<<grid, 128, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
    else
      k_circ_os16<11, 4><<<grid, 128, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
  } else {
    // M = 2048 (cfg5): 166 registers at one CTA per SM left 8 warps per SM to
    // hide every load and barrier; 3 resident CTAs (80 registers): 435 ->
    // 321 us per 128 columns (A/B knob EDAK_CIRC_OS2_MINB)
    const char* e2 = getenv("EDAK_CIRC_OS2_MINB");
    const int m2 = e2 ? atoi(e2) : 3;
    if (m2 == 4)
      k_circ_os<11, 256, 4><<<grid, 256, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
    else if (m2 == 3)
      k_circ_os<11, 256, 3><<<grid, 256, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
    else if (m2 == 2)
      k_circ_os<11, 256, 2><<<grid, 256, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
    else
      k_circ_os<11, 256><<<grid, 256, 0, st>>>(n, L, V, ncols, T, H, in, out, ident, zadd, dotp, dtiles);
  }
  count_launch();
  return check_launch("k_circ_os");
}

}  // namespace edak
