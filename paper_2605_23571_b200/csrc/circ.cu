// Circulant background-covariance factor U_B applied column-wise
// (GridCovFactor.apply / apply_t, covariance.py:41-47).
//
// U_B is circulant with generator u = irfft(symbol); the host truncates u to
// the taps whose magnitude exceeds 2^-60 of the peak (the Gaussian factor
// decays like exp(-d^2/L^2), so 2w+1 ~ 12.5 L taps) or keeps all n taps.
//   out_i = sum_k taps[k] * in[(i + tap_w - k) mod n],  k < ntaps
// One CTA = one column x a tile of NT*R outputs.  The input segment (tile +
// halo) is staged in shared memory with one pad double per R (bank-conflict
// free strided reads); each thread keeps R consecutive outputs in registers
// and slides an R-wide window over the segment, so per tap it issues one
// shared load of the segment, one broadcast load of the tap and R DFMAs.
#include "common.cuh"
#include <cstdlib>

namespace edak {

constexpr int CIRC_R = 8;
constexpr int CIRC_NT = 128;
constexpr int CIRC_MAXTAPS = 4096;


template <int R, int NT>
__global__ void __launch_bounds__(NT) k_circ(int n, const double* __restrict__ taps, int K, int Kp, int w,
                                             const double* __restrict__ in, double* __restrict__ out,
                                             double ident, const double* __restrict__ zadd,
                                             double* __restrict__ dotp, int dtiles) {
  auto padi = [](int q) { return q + q / R; };
  extern __shared__ double sm[];
  double* st = sm;                      // reversed taps, Kp (zero padded)
  double* sg = sm + Kp;                 // segment, padded
  const int col = blockIdx.y;
  const int i0 = blockIdx.x * NT * R;
  const int t = threadIdx.x;
  const double* src = in + (size_t)col * n;
  // correlation form: out[i0+o] = sum_m T[m] * seg[o + m], T[m] = taps[K-1-m],
  // seg[q] = in[(i0 + w - K + 1 + q) mod n]
  for (int m = t; m < Kp; m += NT) st[m] = m < K ? taps[K - 1 - m] : 0.0;
  const int seglen = NT * R + Kp + R;
  int g0 = wrap(i0 + w - K + 1, n);
  if (seglen <= n) {  // the segment wraps the ring at most once: no modulo
    for (int q = t; q < seglen; q += NT) {
      int g = g0 + q;
      if (g >= n) g -= n;
      sg[padi(q)] = src[g];
    }
  } else {
    for (int q = t; q < seglen; q += NT) {
      int g = g0 + q % n;
      if (g >= n) g -= n;
      sg[padi(q)] = src[g];
    }
  }
  __syncthreads();

  double acc[R], cur[R], nxt[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    acc[r] = 0.0;
    cur[r] = sg[padi(t * R + r)];
  }
  for (int m0 = 0; m0 < Kp; m0 += R) {
#pragma unroll
    for (int r = 0; r < R; ++r) nxt[r] = sg[padi(t * R + m0 + R + r)];
#pragma unroll
    for (int mm = 0; mm < R; ++mm) {
      const double tm = st[m0 + mm];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = fma(tm, (r + mm < R) ? cur[r + mm] : nxt[r + mm - R], acc[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) cur[r] = nxt[r];
  }
  double* dst = out + (size_t)col * n;
  double dp = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = i0 + t * R + r;
    if (i < n) {
      double o = acc[r];
      if (zadd) {
        const double zi = zadd[(size_t)col * n + i];
        o += ident * zi;
        dp += zi * o;  // tile partial of zadd . out (PCG p . Hp, krylov.py:81)
      }
      dst[i] = o;
    }
  }
  if (dotp) {  // fixed-order CTA reduction -> dotp[col][tile]
    __syncthreads();
    dp = warp_sum(dp);
    if ((t & 31) == 0) sm[t >> 5] = dp;
    __syncthreads();
    if (t == 0) {
      double s = 0.0;
      for (int w = 0; w < NT / 32; ++w) s += sm[w];
      dotp[(size_t)col * dtiles + blockIdx.x] = s;
    }
    if (blockIdx.x == 0)  // slots past the last tile (circ_tiles counts 512-point tiles)
      for (int q = (int)gridDim.x + t; q < dtiles; q += NT) dotp[(size_t)col * dtiles + q] = 0.0;
  }
}

// out = U_B in (+ ident * zadd when zadd != NULL: the I + A of assim.py:70-72)
// dot-partial slots per column: one per 512 outputs, enough for the 1024-point
// tiles of the tap convolution and the >= 512-output blocks of circ_os.cu
int circ_tiles(int n) { return (n + 511) / 512; }

int launch_circ_os(const edak_problem* P, const double* in, double* out, int ncols, double ident,
                   const double* zadd, cudaStream_t st, double* dotp, int dtiles);

int launch_circ(const edak_problem* P, const double* in, double* out, int ncols, double ident,
                const double* zadd, cudaStream_t st, double* dotp) {
  // overlap-save block FFTs (circ_os.cu) when the factor carries their
  // tables; EDAK_CIRC_OS=0 forces the tap convolution
  const char* eo = getenv("EDAK_CIRC_OS");
  if (!(eo && atoi(eo) == 0) && P->os_spec) {
    const int rc = launch_circ_os(P, in, out, ncols, ident, zadd, st, dotp, circ_tiles(P->n));
    if (rc != EDAK_EUNSUPPORTED) return rc;
  }
  const int n = P->n, K = P->ntaps;
  if (K < 1 || K > CIRC_MAXTAPS) {
    set_error("circulant factor: tap count outside [1, 4096]");
    return EDAK_EUNSUPPORTED;
  }
  // register blocking: R outputs per thread, 8 or 16 (knob EDAK_CIRC_R); both
  // use 1024-output tiles, so the dot-partial layout is the same.  Measured
  // on B200 (tools/ab_knobs.py): R = 16 takes cfg5's 377-tap U_B pair from
  // ~2.2 to ~1.75 ms and cfg4's (189 taps) 3% faster, but is slower on
  // one-tile rings (cfg3, n = 1024), so it is the default for long tap lists
  // on long rings
  const char* er = getenv("EDAK_CIRC_R");
  const int R = er ? (atoi(er) == 16 ? 16 : CIRC_R) : (K >= 128 && n >= 8192 ? 16 : CIRC_R);
  const int NT = CIRC_NT * CIRC_R / R;
  const int Kp = (K + R - 1) / R * R;
  const int tile = NT * R;
  dim3 grid((n + tile - 1) / tile, ncols);
  const int seglen = tile + Kp + R;
  const size_t smem = (size_t)(Kp + seglen + seglen / R + 1) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_circ<CIRC_R, CIRC_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_circ<16, CIRC_NT / 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  if (R == 16)
    k_circ<16, CIRC_NT / 2><<<grid, NT, smem, st>>>(n, P->taps, K, Kp, P->tap_w, in, out, ident, zadd, dotp,
                                                   circ_tiles(n));
  else
    k_circ<CIRC_R, CIRC_NT><<<grid, NT, smem, st>>>(n, P->taps, K, Kp, P->tap_w, in, out, ident, zadd, dotp,
                                                   circ_tiles(n));
  count_launch();
  return check_launch("k_circ");
}

}  // namespace edak
