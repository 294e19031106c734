// diag.cu — the pairwise-perturbation error monitor: column sums of squares of
// two K-column matrices and the per-column error ratios and bound certificate built from them.
//
// P:548 writes M^(n) as M_p^(n) + the first-order terms (what PP keeps) + every term that
// contracts X with two or more dA^(i) (what PP drops).  With p_i = ||a_p,k^(i)||, d_i =
// ||da_k^(i)|| and ||X ×_S v|| <= ||X||_F Π ||v|| (the tensor spectral norm is at most the
// Frobenius norm), the dropped part of column k is bounded by
//     ||m~_k − m_k|| <= ||X||_F Σ_{S ⊆ others, |S| >= 2} Π_{i∈S} d_i Π_{j∉S} p_j
// — the expansion in the proof of Thm 4.1 applied to M instead of H, with the
// matrix 2-norms replaced by ||X||_F.  Every quantity here is computed on the device.
#include <math_constants.h>

#include "internal.h"

namespace cppp {
namespace {

constexpr int CS_COLS = 32;   // columns per CTA (one per lane)
constexpr int CS_ROWS = 8;    // row groups per CTA

// sums[0][k] = Σ_y (a − b)², sums[1][k] = Σ_y b², sums[2][k] = Σ_y a²  (rows x K, row-major).
// Rows are visited in ascending order per row group and the 8 groups added in order: the
// result does not depend on the launch.
__global__ void colsq_kernel(const double* __restrict__ a, const double* __restrict__ b,
                             int64_t rows, int K, double* __restrict__ sums) {
  __shared__ double red[3][CS_ROWS][CS_COLS];
  const int kx = threadIdx.x, ry = threadIdx.y;
  const int k = blockIdx.x * CS_COLS + kx;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  if (k < K) {
    for (int64_t y = ry; y < rows; y += CS_ROWS) {
      const double av = a[y * K + k], bv = b[y * K + k], dv = av - bv;
      s0 = fma(dv, dv, s0);
      s1 = fma(bv, bv, s1);
      s2 = fma(av, av, s2);
    }
  }
  red[0][ry][kx] = s0;
  red[1][ry][kx] = s1;
  red[2][ry][kx] = s2;
  __syncthreads();
  if (ry < 3 && k < K) {
    double t = 0.0;
    for (int r = 0; r < CS_ROWS; ++r) t += red[ry][r][kx];
    sums[ry * K + k] = t;
  }
}

// One thread per (n, k).  msum[n] / asum[n]: the colsq sums of (M~^(n), M^(n)) and
// (A_p^(n), A^(n)).  Outputs [N][K]: err = ||m~ − m|| / ||m||, eps = ||da|| / ||a||,
// bound = the certificate above divided by ||m||.
__global__ void pp_error_final_kernel(const double* __restrict__ msum, const double* __restrict__ asum,
                                      int N, int K, double normX, double* __restrict__ err,
                                      double* __restrict__ eps, double* __restrict__ bound) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= N * K) return;
  const int n = idx / K, k = idx - n * K;
  auto ratio = [](double num, double den) {
    if (num == 0.0) return 0.0;
    return den > 0.0 ? sqrt(num / den) : CUDART_INF;
  };
  const double* ms = msum + static_cast<int64_t>(n) * 3 * K;
  const double* as = asum + static_cast<int64_t>(n) * 3 * K;
  err[idx] = ratio(ms[k], ms[K + k]);
  eps[idx] = ratio(as[k], as[K + k]);
  double p[CPPP_MAX_ORDER_], d[CPPP_MAX_ORDER_];
  int m = 0;
  for (int i = 0; i < N; ++i) {
    if (i == n) continue;
    const double* ai = asum + static_cast<int64_t>(i) * 3 * K;
    d[m] = sqrt(ai[k]);           // ||a_p − a|| = ||da||
    p[m] = sqrt(ai[2 * K + k]);   // ||a_p||
    ++m;
  }
  double tot = 0.0;
  for (unsigned S = 0; S < (1u << m); ++S) {   // subsets in ascending bit order
    if (__popc(S) < 2) continue;
    double t = 1.0;
    for (int i = 0; i < m; ++i) t *= (S >> i) & 1u ? d[i] : p[i];
    tot += t;
  }
  const double mn = sqrt(ms[K + k]);
  bound[idx] = tot == 0.0 ? 0.0 : (mn > 0.0 ? normX * tot / mn : CUDART_INF);
}

// The two data terms of the S:177 expansion for mode n (one CTA, fixed order):
//   fit[0] = Σ_y Σ_k M[y][k] A[y][k]                (rows in thread-strided order, k ascending)
//   fit[1] = Σ_{i,j} Γ^(n)[i][j] S^(n)[i][j],  Γ^(n) = Hadamard of S^(m), m != n ascending
// Per-thread partials are added by a fixed binary tree.
constexpr int FT_THREADS = 256;
__global__ void __launch_bounds__(FT_THREADS)
    fit_terms_kernel(const double* __restrict__ M, const double* __restrict__ A, int64_t rows, int K,
                     const double* __restrict__ S_all, int N, int n, double* __restrict__ fit) {
  __shared__ double red[2][FT_THREADS];
  double inner = 0.0, model = 0.0;
  for (int64_t y = threadIdx.x; y < rows; y += FT_THREADS) {
    double r = 0.0;
    for (int k = 0; k < K; ++k) r = fma(M[y * K + k], A[y * K + k], r);
    inner += r;
  }
  const int KK = K * K;
  for (int e = threadIdx.x; e < KK; e += FT_THREADS) {
    double g = 1.0;
    bool first = true;
    for (int m = 0; m < N; ++m) {
      if (m == n) continue;
      const double v = S_all[static_cast<int64_t>(m) * KK + e];
      g = first ? v : g * v;
      first = false;
    }
    model = fma(g, S_all[static_cast<int64_t>(n) * KK + e], model);
  }
  red[0][threadIdx.x] = inner;
  red[1][threadIdx.x] = model;
  __syncthreads();
  for (int w = FT_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      red[0][threadIdx.x] += red[0][threadIdx.x + w];
      red[1][threadIdx.x] += red[1][threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    fit[0] = red[0][0];
    fit[1] = red[1][0];
  }
}

// PP switching monitor (the "alternative schemes for switching" of P:1134): the
// largest certificate bound of pp_error_final_kernel over (n, k), with ||m_k|| taken from the
// sweep's M~ (msum[n][K..2K) = Σ m~²) instead of an exact MTTKRP -- O(N K 2^N) work, no tensor pass.
// One warp; out[0] = max bound (fixed-order shuffle max: exact).
__global__ void pp_bound_max_kernel(const double* __restrict__ msum, const double* __restrict__ asum,
                                    int N, int K, const double* __restrict__ normX_sq,
                                    double* __restrict__ out) {
  const double normX = sqrt(*normX_sq);
  double mx = 0.0;
  for (int idx = threadIdx.x; idx < N * K; idx += 32) {
    const int n = idx / K, k = idx - n * K;
    double p[CPPP_MAX_ORDER_], d[CPPP_MAX_ORDER_];
    int m = 0;
    for (int i = 0; i < N; ++i) {
      if (i == n) continue;
      const double* ai = asum + static_cast<int64_t>(i) * 3 * K;
      d[m] = sqrt(ai[k]);
      p[m] = sqrt(ai[2 * K + k]);
      ++m;
    }
    double tot = 0.0;
    for (unsigned S = 0; S < (1u << m); ++S) {
      if (__popc(S) < 2) continue;
      double t = 1.0;
      for (int i = 0; i < m; ++i) t *= (S >> i) & 1u ? d[i] : p[i];
      tot += t;
    }
    const double mn = sqrt(msum[static_cast<int64_t>(n) * 3 * K + K + k]);
    const double b = tot == 0.0 ? 0.0 : (mn > 0.0 ? normX * tot / mn : CUDART_INF);
    mx = fmax(mx, b);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (threadIdx.x == 0) out[0] = mx;
}

}  // namespace

cudaError_t launch_pp_bound_max(const double* msum, const double* asum, int N, int K,
                                const double* normX_sq, double* out, cudaStream_t st) {
  pp_bound_max_kernel<<<1, 32, 0, st>>>(msum, asum, N, K, normX_sq, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_fit_terms(const double* M, const double* A, int64_t rows, int K,
                             const double* S_all, int N, int n, double* fit, cudaStream_t st) {
  fit_terms_kernel<<<1, FT_THREADS, 0, st>>>(M, A, rows, K, S_all, N, n, fit);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_colsq(const double* a, const double* b, int64_t rows, int K, double* sums,
                         cudaStream_t st) {
  colsq_kernel<<<(K + CS_COLS - 1) / CS_COLS, dim3(CS_COLS, CS_ROWS), 0, st>>>(a, b, rows, K, sums);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pp_error_final(const double* msum, const double* asum, int N, int K,
                                  double normX, double* err, double* eps, double* bound,
                                  cudaStream_t st) {
  const int n = N * K;
  pp_error_final_kernel<<<(n + 127) / 128, 128, 0, st>>>(msum, asum, N, K, normX, err, eps, bound);
  note_launch();
  return cudaGetLastError();
}

}  // namespace cppp
