// U_B v = irfft(symbol * rfft(v)) (covariance.py:41-45) as ONE kernel per
// column: the column's n reals are packed as N = n/2 complex values
// z_k = v_2k + i v_2k+1 in shared memory, transformed by a radix-8
// decimation-in-frequency FFT (natural -> bit-reversed order), the real-FFT
// split, the symbol and the inverse real-FFT merge are applied pairwise
// (k, N-k) in the bit-reversed domain, and a radix-8 decimation-in-time
// inverse FFT (bit-reversed -> natural) brings the product back; no
// bit-reversal permutation pass is ever needed.  ~5x fewer flops than the
// tap convolution at cfg4 (189 taps) and the same HBM traffic (one read,
// one write per element, plus zadd for I + A).
//
// Twiddles: one table T[k] = exp(-2 pi i k / n), k < n/2 (fp64, accurate
// host values).  A radix-8 group needs one lookup; its other twiddles are
// that value's square and fourth power times constant eighth roots of unity.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;
#include <cstdlib>

namespace edak {

constexpr int CF_NT = 512;

// one pad complex per 8: the stride-8 passes (the last DIF and first DIT
// radix-8 pass) become bank-conflict free for 16-byte accesses
__device__ __forceinline__ int pz(int j) { return j + (j >> 3); }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// a * (-i) and a * (+i)
__device__ __forceinline__ double2 cmul_mi(double2 a) { return make_double2(a.y, -a.x); }
__device__ __forceinline__ double2 cmul_pi(double2 a) { return make_double2(-a.y, a.x); }

// W_N^e = exp(-2 pi i e / N), N = n/2, from T[m] = exp(-2 pi i m / n)
__device__ __forceinline__ double2 tw_N(const double2* __restrict__ T, int e, int N) {
  const int m = 2 * e;
  if (m < N) return __ldg(T + m);
  const double2 v = __ldg(T + (m - N));
  return make_double2(-v.x, -v.y);
}

// multiply by the eighth roots exp(-+2 pi i m / 8), m = 1..3 (exact constants)
template <bool INV>
__device__ __forceinline__ double2 w8(double2 a, int m) {
  const double r = 0.70710678118654752440;
  if (m == 0) return a;
  if (m == 2) return INV ? cmul_pi(a) : cmul_mi(a);
  if (m == 1) {  // (1 -+ i) / sqrt2
    return INV ? make_double2(r * (a.x - a.y), r * (a.x + a.y)) : make_double2(r * (a.x + a.y), r * (a.y - a.x));
  }
  // m == 3: (-1 -+ i) / sqrt2
  return INV ? make_double2(-r * (a.x + a.y), r * (a.x - a.y)) : make_double2(r * (a.y - a.x), -r * (a.x + a.y));
}

__global__ void __launch_bounds__(CF_NT) k_circ_fft(int n, int logN, const double* __restrict__ sym,
                                                    const double2* __restrict__ T, const double* __restrict__ in,
                                                    double* __restrict__ out, double ident,
                                                    const double* __restrict__ zadd, double* __restrict__ dotp,
                                                    int dtiles) {
  extern __shared__ __align__(16) double2 Z[];
  __shared__ double red[CF_NT / 32];
  const int N = n >> 1, t = threadIdx.x, col = blockIdx.x;
  const double2* src = reinterpret_cast<const double2*>(in + (size_t)col * n);
  for (int k = t; k < N; k += CF_NT) Z[pz(k)] = src[k];
  __syncthreads();
  // ---- forward DIF: leading radix-2 stages, then radix-8 passes ----------
  int h = N >> 1;
  for (int r = 0; r < logN % 3; ++r, h >>= 1) {
    for (int p = t; p < N / 2; p += CF_NT) {
      const int j = (p / h) * 2 * h + p % h;
      const double2 x = Z[pz(j)], y = Z[pz(j + h)];
      Z[pz(j)] = cadd(x, y);
      Z[pz(j + h)] = cmul(csub(x, y), tw_N(T, (p % h) * (N / (2 * h)), N));
    }
    __syncthreads();
  }
  for (; h >= 4; h >>= 3) {
    const int q = h >> 2;
    for (int g = t; g < N / 8; g += CF_NT) {
      const int r0 = g % q, j0 = (g / q) * 2 * h + r0;
      double2 a[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) a[m] = Z[pz(j0 + m * q)];
      const double2 b1 = tw_N(T, r0 * (N / (2 * h)), N);
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
    }
    __syncthreads();
  }
  // ---- real split, symbol, inverse real merge (pairs k, N-k; bit-reversed)
  const int sh = 32 - logN;
  for (int k = t; k <= N / 2; k += CF_NT) {
    const int km = (N - k) & (N - 1);
    const int rk = __brev(k) >> sh, rm = __brev(km) >> sh;
    const double2 zk = Z[pz(rk)], zm = Z[pz(rm)];
    const double2 tk = __ldg(T + k);            // exp(-2 pi i k / n)
    const double2 tn = make_double2(-tk.x, tk.y);  // exp(-2 pi i (N-k) / n) = -conj(tk)
    // X_k = (zk + conj zm)/2 - i tk (zk - conj zm)/2, X_{N-k} likewise
    const double2 sk = cadd(zk, cconj(zm)), dk = csub(zk, cconj(zm));
    const double2 sm = cadd(zm, cconj(zk)), dm = csub(zm, cconj(zk));
    double2 Xk = cmul_mi(cmul(tk, dk));
    Xk = make_double2(0.5 * (sk.x + Xk.x), 0.5 * (sk.y + Xk.y));
    double2 Xm = cmul_mi(cmul(tn, dm));
    Xm = make_double2(0.5 * (sm.x + Xm.x), 0.5 * (sm.y + Xm.y));
    const double gk_s = __ldg(sym + k), gm_s = __ldg(sym + (N - k));
    const double2 Gk = make_double2(gk_s * Xk.x, gk_s * Xk.y);
    const double2 Gm = make_double2(gm_s * Xm.x, gm_s * Xm.y);
    // Y_k = (G_k + conj G_{N-k}) + i conj(tk) (G_k - conj G_{N-k})
    const double2 Yk = cadd(cadd(Gk, cconj(Gm)), cmul_pi(cmul(cconj(tk), csub(Gk, cconj(Gm)))));
    Z[pz(rk)] = Yk;
    if (km != k) {
      const double2 Ym = cadd(cadd(Gm, cconj(Gk)), cmul_pi(cmul(cconj(tn), csub(Gm, cconj(Gk)))));
      Z[pz(rm)] = Ym;
    }
  }
  __syncthreads();
  // ---- inverse DIT: radix-8 passes from span 1, then radix-2 stages --------
  const int full = logN - logN % 3;
  h = 1;
  for (; h < (1 << full); h <<= 3) {
    for (int g = t; g < N / 8; g += CF_NT) {
      const int r0 = g % h, j0 = (g / h) * 8 * h + r0;
      double2 a[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) a[m] = Z[pz(j0 + m * h)];
      const double2 c1 = cconj(tw_N(T, r0 * (N / (8 * h)), N));
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
    }
    __syncthreads();
  }
  for (; h < N; h <<= 1) {
    for (int p = t; p < N / 2; p += CF_NT) {
      const int j = (p / h) * 2 * h + p % h;
      const double2 x = Z[pz(j)], y = cmul(Z[pz(j + h)], cconj(tw_N(T, (p % h) * (N / (2 * h)), N)));
      Z[pz(j)] = cadd(x, y);
      Z[pz(j + h)] = csub(x, y);
    }
    __syncthreads();
  }
  // ---- unpack, scale 1/n, I + A epilogue, p.Hp partial ----------------------
  const double sc = 1.0 / (double)n;
  double2* dst = reinterpret_cast<double2*>(out + (size_t)col * n);
  const double2* za = zadd ? reinterpret_cast<const double2*>(zadd + (size_t)col * n) : nullptr;
  double dp = 0.0;
  for (int k = t; k < N; k += CF_NT) {
    double2 v = Z[pz(k)];
    v.x *= sc;
    v.y *= sc;
    if (za) {
      const double2 z = za[k];
      v.x = fma(ident, z.x, v.x);
      v.y = fma(ident, z.y, v.y);
      dp = fma(z.x, v.x, dp);
      dp = fma(z.y, v.y, dp);
    }
    dst[k] = v;
  }
  if (dotp) {  // fixed-order CTA reduction; the column's other tiles get 0
    dp = warp_sum(dp);
    if ((t & 31) == 0) red[t >> 5] = dp;
    __syncthreads();
    if (t == 0) {
      double s = 0.0;
      for (int w = 0; w < CF_NT / 32; ++w) s += red[w];
      dotp[(size_t)col * dtiles] = s;
    }
    for (int q = 1 + t; q < dtiles; q += CF_NT) dotp[(size_t)col * dtiles + q] = 0.0;
  }
}

// The same transform on a 2-CTA cluster: each CTA keeps one half of the N
// complex values (64 KB at n = 16384, so 3 CTAs fit an SM and a whole
// 200-column block runs in one wave instead of two).  Only the first DIF
// stage and the last DIT stage (span N/2) cross the halves -- through
// distributed shared memory; the radix-8 passes and the real split/merge
// (k and N-k have the same parity, so rev(k) and rev(N-k) share a half)
// stay local.  Needs logN = 1 (mod 3), e.g. n = 2048, 16384.
constexpr int CF2_MAXH = 4096;  // complex values per CTA (n <= 16384)
constexpr int CF2_NT = 256;     // 3 CTAs (74 KB smem each) per SM: 400 CTAs in one wave
constexpr int CF2_CH = 4;       // cross-stage values per thread and chunk (registers)

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(CF2_NT, 3)
    k_circ_fft2(int n, int logN, const double* __restrict__ sym, const double2* __restrict__ T,
                const double* __restrict__ in, double* __restrict__ out, double ident,
                const double* __restrict__ zadd, double* __restrict__ dotp, int dtiles) {
  extern __shared__ __align__(16) double2 Z[];
  __shared__ double red[CF2_NT / 32];
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank(), col = blockIdx.x >> 1, t = threadIdx.x;
  const int N = n >> 1, H = N >> 1, base = r * H;
  const int chunk = CF2_NT * CF2_CH;
  const double2* src = reinterpret_cast<const double2*>(in + (size_t)col * n) + base;
  for (int k = t; k < H; k += CF2_NT) Z[pz(k)] = src[k];
  cl.sync();
  const double2* Zo = cl.map_shared_rank(Z, r ^ 1);
  // DIF stage of span N/2 across the halves, chunk by chunk: every value of
  // a chunk is read from both halves (barrier) before either CTA rewrites it
  for (int c0 = 0; c0 < H; c0 += chunk) {
    double2 v[CF2_CH];
#pragma unroll
    for (int i = 0; i < CF2_CH; ++i) {
      const int k = c0 + t + i * CF2_NT;
      if (k < H) {
        const double2 mine = Z[pz(k)], other = Zo[pz(k)];
        v[i] = r == 0 ? cadd(mine, other) : cmul(csub(other, mine), tw_N(T, k, N));
      }
    }
    cl.sync();
#pragma unroll
    for (int i = 0; i < CF2_CH; ++i) {
      const int k = c0 + t + i * CF2_NT;
      if (k < H) Z[pz(k)] = v[i];
    }
  }
  __syncthreads();
  // local radix-8 DIF passes, spans N/4 .. 1
  for (int h = N >> 2; h >= 4; h >>= 3) {
    const int q = h >> 2;
    for (int gl = t; gl < N / 16; gl += CF2_NT) {
      const int g = r * (N / 16) + gl;
      const int r0 = g % q, j0 = (g / q) * 2 * h + r0 - base;
      double2 a[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) a[m] = Z[pz(j0 + m * q)];
      const double2 b1 = tw_N(T, r0 * (N / (2 * h)), N);
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const double2 x = a[m], y = a[m + 4];
        a[m] = cadd(x, y);
        a[m + 4] = cmul(w8<false>(csub(x, y), m), b1);
      }
      const double2 b2 = cmul(b1, b1);
#pragma unroll
      for (int mm = 0; mm < 4; ++mm) {
        const int m = (mm & 1) + 4 * (mm >> 1);
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
    }
    __syncthreads();
  }
  // real split / symbol / inverse merge: this CTA owns the k of parity r
  const int sh = 32 - logN;
  for (int k = r + 2 * t; k <= N / 2; k += 2 * CF2_NT) {
    const int km = (N - k) & (N - 1);
    const int rk = (__brev(k) >> sh) - base, rm = (__brev(km) >> sh) - base;
    const double2 zk = Z[pz(rk)], zm = Z[pz(rm)];
    const double2 tk = __ldg(T + k);
    const double2 tn = make_double2(-tk.x, tk.y);
    const double2 sk = cadd(zk, cconj(zm)), dk = csub(zk, cconj(zm));
    const double2 sm = cadd(zm, cconj(zk)), dm = csub(zm, cconj(zk));
    double2 Xk = cmul_mi(cmul(tk, dk));
    Xk = make_double2(0.5 * (sk.x + Xk.x), 0.5 * (sk.y + Xk.y));
    double2 Xm = cmul_mi(cmul(tn, dm));
    Xm = make_double2(0.5 * (sm.x + Xm.x), 0.5 * (sm.y + Xm.y));
    const double gk_s = __ldg(sym + k), gm_s = __ldg(sym + (N - k));
    const double2 Gk = make_double2(gk_s * Xk.x, gk_s * Xk.y);
    const double2 Gm = make_double2(gm_s * Xm.x, gm_s * Xm.y);
    Z[pz(rk)] = cadd(cadd(Gk, cconj(Gm)), cmul_pi(cmul(cconj(tk), csub(Gk, cconj(Gm)))));
    if (km != k) Z[pz(rm)] = cadd(cadd(Gm, cconj(Gk)), cmul_pi(cmul(cconj(tn), csub(Gm, cconj(Gk)))));
  }
  __syncthreads();
  // local radix-8 DIT passes, spans 1 .. N/4
  for (int h = 1; 8 * h <= H; h <<= 3) {
    for (int gl = t; gl < N / 16; gl += CF2_NT) {
      const int g = r * (N / 16) + gl;
      const int r0 = g % h, j0 = (g / h) * 8 * h + r0 - base;
      double2 a[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) a[m] = Z[pz(j0 + m * h)];
      const double2 c1 = cconj(tw_N(T, r0 * (N / (8 * h)), N));
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
    }
    __syncthreads();
  }
  // DIT stage of span N/2 across the halves (chunked as above), then unpack,
  // scale 1/n, I + A epilogue, p.Hp partial
  const double sc = 1.0 / (double)n;
  double2* dst = reinterpret_cast<double2*>(out + (size_t)col * n) + base;
  const double2* za = zadd ? reinterpret_cast<const double2*>(zadd + (size_t)col * n) + base : nullptr;
  double dp = 0.0;
  cl.sync();
  for (int c0 = 0; c0 < H; c0 += chunk) {
    double2 v[CF2_CH];
#pragma unroll
    for (int i = 0; i < CF2_CH; ++i) {
      const int k = c0 + t + i * CF2_NT;
      if (k < H) {
        const double2 x = r == 0 ? Z[pz(k)] : Zo[pz(k)];
        const double2 y = cmul(r == 0 ? Zo[pz(k)] : Z[pz(k)], cconj(tw_N(T, k, N)));
        v[i] = r == 0 ? cadd(x, y) : csub(x, y);
      }
    }
    cl.sync();  // the partner has read this chunk of both halves
#pragma unroll
    for (int i = 0; i < CF2_CH; ++i) {
      const int k = c0 + t + i * CF2_NT;
      if (k < H) {
        double2 w = make_double2(v[i].x * sc, v[i].y * sc);
        if (za) {
          const double2 z = za[k];
          w.x = fma(ident, z.x, w.x);
          w.y = fma(ident, z.y, w.y);
          dp = fma(z.x, w.x, dp);
          dp = fma(z.y, w.y, dp);
        }
        dst[k] = w;
      }
    }
  }
  if (dotp) {  // fixed-order CTA reduction -> tiles 0 / 1 of the column; the rest 0
    dp = warp_sum(dp);
    if ((t & 31) == 0) red[t >> 5] = dp;
    __syncthreads();
    if (t == 0) {
      double s2 = 0.0;
      for (int w = 0; w < CF2_NT / 32; ++w) s2 += red[w];
      dotp[(size_t)col * dtiles + r] = s2;
    }
    if (r == 0)
      for (int q = 2 + t; q < dtiles; q += CF2_NT) dotp[(size_t)col * dtiles + q] = 0.0;
  }
}

bool circ_fft_ok(const edak_problem* P) {
  const int n = P->n;
  return P->sym && P->fft_tw && n >= 1024 && n <= 16384 && (n & (n - 1)) == 0;
}

int launch_circ_fft(const edak_problem* P, const double* in, double* out, int ncols, double ident,
                    const double* zadd, cudaStream_t st, double* dotp, int dtiles) {
  const int n = P->n, N = n / 2;
  int logN = 0;
  while ((1 << logN) < N) ++logN;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_circ_fft, cudaFuncAttributeMaxDynamicSharedMemorySize, 9216 * (int)sizeof(double2));
    cudaFuncSetAttribute(k_circ_fft2, cudaFuncAttributeMaxDynamicSharedMemorySize, 4608 * (int)sizeof(double2));
    attr = true;
  }
  if (logN % 3 == 1 && dtiles >= 2 && !getenv("EDAK_CIRC_FFT1")) {
    const size_t smem2 = (size_t)(N / 2 + N / 16) * sizeof(double2);
    k_circ_fft2<<<2 * ncols, CF2_NT, smem2, st>>>(n, logN, P->sym, reinterpret_cast<const double2*>(P->fft_tw), in,
                                                 out, ident, zadd, dotp, dtiles);
    count_launch();
    return check_launch("k_circ_fft2");
  }
  const size_t smem = (size_t)(N + N / 8) * sizeof(double2);
  k_circ_fft<<<ncols, CF_NT, smem, st>>>(n, logN, P->sym, reinterpret_cast<const double2*>(P->fft_tw), in, out,
                                         ident, zadd, dotp, dtiles);
  count_launch();
  return check_launch("k_circ_fft");
}

}  // namespace edak
