// Per-vector Lorenz-96 operators of model.py as device kernels -- the
// reference's building blocks below the fused sweeps, for callers that use
// them directly (the sweeps in l96.cu / sweep_tile.cu inline the same
// arithmetic):
//   tendency      f(x)       (model.py:20-22)
//   tendency_tlm  J(x) v     (model.py:25-28)
//   tendency_adj  J(x)^T w   (model.py:31-35)
// and the two vector combinations that step_tlm / step_adj / _rk4_stages
// (model.py:38-84) build from them.  Every operation is IEEE-rounded in the
// reference's numpy order (no FMA contraction), so the results are the
// reference's bit for bit.  Blocks of ncols vectors, column c at c * n;
// grid-stride over all elements.
#include "common.cuh"

namespace edak {

namespace l96op {
__device__ __forceinline__ int rot(int i, int k, int n) {  // index of np.roll(x, k)[i] = x[i - k]
  int j = i - k;
  j = j < 0 ? j + n : (j >= n ? j - n : j);
  return j;
}
}  // namespace l96op

// op 0: f(x); op 1: J(x) v; op 2: J(x)^T v
__global__ void __launch_bounds__(256) k_l96_tend(int op, int n, int64_t total, const double* __restrict__ x,
                                                  const double* __restrict__ v, double forcing,
                                                  double* __restrict__ out) {
  using namespace l96op;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / n;
    const int i = (int)(e - c * n);
    const double* X = x + c * n;
    const double* V = v ? v + c * n : nullptr;
    double r;
    if (op == 0) {  // (x[i+1] - x[i-2]) * x[i-1] - x + F
      r = __dadd_rn(__dsub_rn(__dmul_rn(__dsub_rn(X[rot(i, -1, n)], X[rot(i, 2, n)]), X[rot(i, 1, n)]), X[i]),
                    forcing);
    } else if (op == 1) {  // (v[i+1] - v[i-2]) x[i-1] + (x[i+1] - x[i-2]) v[i-1] - v
      const double a = __dmul_rn(__dsub_rn(V[rot(i, -1, n)], V[rot(i, 2, n)]), X[rot(i, 1, n)]);
      const double b = __dmul_rn(__dsub_rn(X[rot(i, -1, n)], X[rot(i, 2, n)]), V[rot(i, 1, n)]);
      r = __dsub_rn(__dadd_rn(a, b), V[i]);
    } else {  // x[i-2] w[i-1] + (x[i+2] - x[i-1]) w[i+1] - x[i+1] w[i+2] - w
      const double a = __dmul_rn(X[rot(i, 2, n)], V[rot(i, 1, n)]);
      const double b = __dmul_rn(__dsub_rn(X[rot(i, -2, n)], X[rot(i, 1, n)]), V[rot(i, -1, n)]);
      const double d = __dmul_rn(X[rot(i, -1, n)], V[rot(i, -2, n)]);
      r = __dsub_rn(__dsub_rn(__dadd_rn(a, b), d), V[i]);
    }
    out[e] = r;
  }
}

// op 0: out = y + c z; op 1: out = y + c (((a1 + 2 a2) + 2 a3) + a4); op 2: out = c z
// (model.py:41-47 and 58-63: the scalar c is formed on the host as numpy does)
__global__ void __launch_bounds__(256) k_l96_comb(int op, int64_t total, const double* __restrict__ y, double c,
                                                  const double* __restrict__ a1, const double* __restrict__ a2,
                                                  const double* __restrict__ a3, const double* __restrict__ a4,
                                                  double* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    if (op == 2) {
      out[e] = __dmul_rn(c, a1[e]);
      continue;
    }
    double s;
    if (op == 0) {
      s = a1[e];
    } else {
      s = __dadd_rn(__dadd_rn(__dadd_rn(a1[e], __dmul_rn(2.0, a2[e])), __dmul_rn(2.0, a3[e])), a4[e]);
    }
    out[e] = __dadd_rn(y[e], __dmul_rn(c, s));
  }
}

static unsigned grid_for(int64_t total) {
  const int64_t b = (total + 255) / 256;
  return (unsigned)(b < 148 * 8 ? (b > 0 ? b : 1) : 148 * 8);
}

int launch_l96_tend(int op, int n, int ncols, const double* x, const double* v, double forcing, double* out,
                    cudaStream_t st) {
  const int64_t total = (int64_t)n * ncols;
  k_l96_tend<<<grid_for(total), 256, 0, st>>>(op, n, total, x, v, forcing, out);
  count_launch();
  return check_launch("k_l96_tend");
}

int launch_l96_comb(int op, int64_t len, const double* y, double c, const double* a1, const double* a2,
                    const double* a3, const double* a4, double* out, cudaStream_t st) {
  k_l96_comb<<<grid_for(len), 256, 0, st>>>(op, len, y, c, a1, a2, a3, a4, out);
  count_launch();
  return check_launch("k_l96_comb");
}

}  // namespace edak
