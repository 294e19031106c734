// solve.cu — the small dense part of every ALS step, on device (Alg. 1 P:393-399,
// Alg. 3, normal equations):
//   Γ^(n) = S^(1) ∗ … ∗ S^(n-1) ∗ S^(n+1) ∗ … ∗ S^(N)          (Hadamard, ascending m)
//   A_new = M Γ^†                                              (L13 pivot rule)
//   G^(n) = (A^(n) - A_new) Γ^(n)
//   S^(n) = A_newᵀ A_new
// plus ‖A‖², ‖dA‖², ‖G‖² per mode (the ε_pp test L7 and the stop metric) and the fitness
// expansion terms.  K <= 128.  Every reduction has a fixed order (deterministic).
#include "internal.h"

namespace cppp {
namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum, fixed order (warp tree, then warp 0 over warp partials).  All threads get it.
__device__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = lane < nw ? sh[lane] : 0.0;
    r = warp_sum(r);
    if (lane == 0) sh[0] = r;
  }
  __syncthreads();
  r = sh[0];
  __syncthreads();
  return r;
}

constexpr int GF_THREADS = 512;
constexpr double PIVOT_TAU = 1e-12;  // L13 / S:201
constexpr double PINV_TAU = 1e-12;

// Γ, Cholesky (right-looking, in shared memory) with the L13 pivot rule; on failure the
// cyclic-Jacobi eigen pseudo-inverse (Brent-Luk parallel ordering).  One CTA.
__global__ void __launch_bounds__(GF_THREADS)
    gamma_factor_kernel(const double* __restrict__ S_all, int N, int n, int K, double* Gamma,
                        double* Lout, int* mode, double* Vscratch) {
  extern __shared__ double W[];  // K x (K+1)
  __shared__ double sh[32];
  __shared__ int s_ok;
  const int P = K + 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  double dmax_local = 0.0;
  for (int e = tid; e < K * K; e += nt) {
    double v = 0.0;
    bool first = true;
    for (int m = 0; m < N; ++m) {
      if (m == n) continue;
      const double sv = S_all[(int64_t)m * K * K + e];
      v = first ? sv : v * sv;
      first = false;
    }
    Gamma[e] = v;
    const int i = e / K, j = e - i * K;
    W[i * P + j] = v;
    if (i == j) dmax_local = fmax(dmax_local, v);
  }
  // max diag (fixed order reduction via max is order independent)
  double dm = dmax_local;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
  if ((tid & 31) == 0) sh[tid >> 5] = dm;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int w = 0; w < (nt + 31) / 32; ++w) m = fmax(m, sh[w]);
    sh[0] = m;
    s_ok = 1;
  }
  __syncthreads();
  const double thresh = PIVOT_TAU * sh[0];
  // ---- Cholesky, right-looking
  for (int j = 0; j < K; ++j) {
    if (tid == 0) {
      const double d = W[j * P + j];
      if (!(d > thresh)) s_ok = 0;
      else W[j * P + j] = sqrt(d);
    }
    __syncthreads();
    if (!s_ok) break;
    const double ljj = W[j * P + j];
    for (int i = j + 1 + tid; i < K; i += nt) W[i * P + j] /= ljj;
    __syncthreads();
    const int m = K - j - 1;
    // trailing lower triangle (j < l <= i < K) as an m x m square, lower half only
    for (int e = tid; e < m * m; e += nt) {
      const int ii = e / m, ll = e - ii * m;
      if (ll <= ii) {
        const int i = j + 1 + ii, l = j + 1 + ll;
        W[i * P + l] -= W[i * P + j] * W[l * P + j];
      }
    }
    __syncthreads();
  }
  if (s_ok) {
    for (int e = tid; e < K * K; e += nt) {
      const int i = e / K, j = e - i * K;
      Lout[e] = (j <= i) ? W[i * P + j] : 0.0;
    }
    if (tid == 0) *mode = 0;
    return;
  }
  // ---- eigen pseudo-inverse: two-sided cyclic Jacobi on W (reloaded), V in global scratch
  for (int e = tid; e < K * K; e += nt) {
    const int i = e / K, j = e - i * K;
    W[i * P + j] = Gamma[e];
    Vscratch[e] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int Ke = (K + 1) & ~1;  // even number of players
  __shared__ double cs[64], sn[64];
  __shared__ int pp_[64], qq_[64];
  for (int sweep = 0; sweep < 40; ++sweep) {
    // convergence: off-diagonal mass relative to the diagonal
    double off = 0.0, dia = 0.0;
    for (int e = tid; e < K * K; e += nt) {
      const int i = e / K, j = e - i * K;
      const double v = W[i * P + j];
      if (i == j) dia += v * v; else off += v * v;
    }
    off = block_sum(off, sh);
    dia = block_sum(dia, sh);
    if (off <= 1e-30 * dia || dia == 0.0) break;
    for (int r = 0; r < Ke - 1; ++r) {
      if (tid < Ke / 2) {
        int p, q;
        if (tid == 0) { p = Ke - 1; q = r; }
        else { p = (r + tid) % (Ke - 1); q = (r - tid + Ke - 1) % (Ke - 1); }
        if (p > q) { int tmp = p; p = q; q = tmp; }
        double c = 1.0, s = 0.0;
        if (q < K) {
          const double apq = W[p * P + q];
          if (apq != 0.0) {
            const double tau = (W[q * P + q] - W[p * P + p]) / (2.0 * apq);
            const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        }
        cs[tid] = c; sn[tid] = s; pp_[tid] = p; qq_[tid] = q;
      }
      __syncthreads();
      // rows: W <- J^T W
      for (int e = tid; e < (Ke / 2) * K; e += nt) {
        const int pr = e / K, l = e - pr * K;
        const int p = pp_[pr], q = qq_[pr];
        if (q >= K) continue;
        const double c = cs[pr], s = sn[pr];
        const double wp = W[p * P + l], wq = W[q * P + l];
        W[p * P + l] = c * wp - s * wq;
        W[q * P + l] = s * wp + c * wq;
      }
      __syncthreads();
      // columns: W <- W J, V <- V J
      for (int e = tid; e < (Ke / 2) * K; e += nt) {
        const int pr = e / K, l = e - pr * K;
        const int p = pp_[pr], q = qq_[pr];
        if (q >= K) continue;
        const double c = cs[pr], s = sn[pr];
        const double wp = W[l * P + p], wq = W[l * P + q];
        W[l * P + p] = c * wp - s * wq;
        W[l * P + q] = s * wp + c * wq;
        const double vp = Vscratch[l * K + p], vq = Vscratch[l * K + q];
        Vscratch[l * K + p] = c * vp - s * vq;
        Vscratch[l * K + q] = s * vp + c * vq;
      }
      __syncthreads();
    }
  }
  // eigenvalues on the diagonal; λ⁺ with cutoff PINV_TAU * λmax
  __shared__ double lam[128];
  for (int i = tid; i < K; i += nt) lam[i] = W[i * P + i];
  __syncthreads();
  if (tid == 0) {
    double lmax = 0.0;
    for (int i = 0; i < K; ++i) lmax = fmax(lmax, lam[i]);
    sh[0] = lmax;
  }
  __syncthreads();
  const double lmax = sh[0];
  for (int i = tid; i < K; i += nt) {
    const double l = lam[i];
    lam[i] = (lmax > 0.0 && l > PINV_TAU * lmax) ? 1.0 / l : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < K * K; e += nt) {
    const int i = e / K, j = e - i * K;
    double v = 0.0;
    for (int l = 0; l < K; ++l) v += Vscratch[i * K + l] * lam[l] * Vscratch[j * K + l];
    Lout[e] = v;
  }
  if (tid == 0) *mode = 1;
}

// One warp per row y.  Lane c owns columns c, c+32, c+64, c+96.  Cholesky path: forward then
// back substitution with L staged in shared memory (pitch K+1, conflict-free columns);
// pinv path: a = m P.  Then g = (a_old - a_new) Γ, dA = a_new - ref, row norm partials.
constexpr int SR_WARPS = 16;

__global__ void __launch_bounds__(SR_WARPS * 32)
    solve_rows_kernel(const double* __restrict__ M, double* A, const double* ref, double* dA,
                      int64_t rows, int K, const double* __restrict__ Gamma,
                      const double* __restrict__ L, const int* __restrict__ mode_p,
                      double* __restrict__ rowstat) {
  extern __shared__ double Ls[];  // K x (K+1) when mode == 0
  const int P = K + 1;
  const int mode = *mode_p;
  if (mode == 0) {
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
      const int i = e / K, j = e - i * K;
      Ls[i * P + j] = L[e];
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t y = blockIdx.x * (int64_t)SR_WARPS + w; y < rows; y += (int64_t)gridDim.x * SR_WARPS) {
    double m[4], a[4], aold[4], rf[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int c = lane + 32 * s;
      m[s] = c < K ? M[y * K + c] : 0.0;
      aold[s] = c < K ? A[y * K + c] : 0.0;
      rf[s] = c < K ? ref[y * K + c] : 0.0;
    }
    if (mode == 0) {
      // forward: L z = m  (z overwrites m)
      for (int j = 0; j < K; ++j) {
        const int owner = j & 31, slot = j >> 5;
        double zj = 0.0;
        if (lane == owner) {
          double v = (slot == 0) ? m[0] : (slot == 1) ? m[1] : (slot == 2) ? m[2] : m[3];
          zj = v / Ls[j * P + j];
        }
        zj = __shfl_sync(0xffffffffu, zj, owner);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int c = lane + 32 * s;
          if (c == j) m[s] = zj;
          else if (c > j && c < K) m[s] -= Ls[c * P + j] * zj;
        }
      }
      // back: L^T a = z
      for (int j = K - 1; j >= 0; --j) {
        const int owner = j & 31, slot = j >> 5;
        double aj = 0.0;
        if (lane == owner) {
          double v = (slot == 0) ? m[0] : (slot == 1) ? m[1] : (slot == 2) ? m[2] : m[3];
          aj = v / Ls[j * P + j];
        }
        aj = __shfl_sync(0xffffffffu, aj, owner);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int c = lane + 32 * s;
          if (c == j) m[s] = aj;
          else if (c < j) m[s] -= Ls[j * P + c] * aj;
        }
      }
#pragma unroll
      for (int s = 0; s < 4; ++s) a[s] = (lane + 32 * s < K) ? m[s] : 0.0;
    } else {
#pragma unroll
      for (int s = 0; s < 4; ++s) a[s] = 0.0;
      for (int p = 0; p < K; ++p) {
        const int owner = p & 31, slot = p >> 5;
        double mp = (slot == 0) ? m[0] : (slot == 1) ? m[1] : (slot == 2) ? m[2] : m[3];
        mp = __shfl_sync(0xffffffffu, mp, owner);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int c = lane + 32 * s;
          if (c < K) a[s] = fma(mp, L[p * K + c], a[s]);
        }
      }
    }
    // gradient g = (a_old - a_new) Γ
    double g[4] = {0.0, 0.0, 0.0, 0.0};
    for (int p = 0; p < K; ++p) {
      const int owner = p & 31, slot = p >> 5;
      double dp = (slot == 0) ? aold[0] - a[0] : (slot == 1) ? aold[1] - a[1]
                : (slot == 2) ? aold[2] - a[2] : aold[3] - a[3];
      dp = __shfl_sync(0xffffffffu, dp, owner);
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int c = lane + 32 * s;
        if (c < K) g[s] = fma(dp, Gamma[p * K + c], g[s]);
      }
    }
    double na = 0.0, nd = 0.0, ng = 0.0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int c = lane + 32 * s;
      if (c < K) {
        const double d = a[s] - rf[s];
        A[y * K + c] = a[s];
        dA[y * K + c] = d;
        na += a[s] * a[s];
        nd += d * d;
        ng += g[s] * g[s];
      }
    }
    na = warp_sum(na);
    nd = warp_sum(nd);
    ng = warp_sum(ng);
    if (lane == 0) {
      rowstat[y * 3 + 0] = na;
      rowstat[y * 3 + 1] = nd;
      rowstat[y * 3 + 2] = ng;
    }
  }
}

// S = AᵀA: thread per (k1 <= k2), sum over rows ascending, mirrored (exactly symmetric).
// Block 0 also reduces the per-row norm partials in row order -> nrm[0..2].
__global__ void gram_norms_kernel(const double* __restrict__ A, int64_t rows, int K, double* S,
                                  const double* __restrict__ rowstat, double* nrm) {
  const int64_t pairs = (int64_t)K * K;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < pairs) {
    const int k1 = static_cast<int>(e / K), k2 = static_cast<int>(e % K);
    if (k1 <= k2) {
      double acc = 0.0;
      for (int64_t y = 0; y < rows; ++y) acc = fma(A[y * K + k1], A[y * K + k2], acc);
      S[k1 * K + k2] = acc;
      S[k2 * K + k1] = acc;
    }
  }
  if (rowstat != nullptr && blockIdx.x == 0) {
    __shared__ double sh[32];
    for (int c = 0; c < 3; ++c) {
      double v = 0.0;
      for (int64_t y = threadIdx.x; y < rows; y += blockDim.x) v += rowstat[y * 3 + c];
      v = block_sum(v, sh);
      if (threadIdx.x == 0) nrm[c] = v;
    }
  }
}

__global__ void fitness_terms_kernel(const double* __restrict__ M, const double* __restrict__ A,
                                     int64_t n, const double* __restrict__ Gm,
                                     const double* __restrict__ S, int64_t kk, double* out) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) v = fma(M[e], A[e], v);
  v = block_sum(v, sh);
  double w = 0.0;
  for (int64_t e = threadIdx.x; e < kk; e += blockDim.x) w = fma(Gm[e], S[e], w);
  w = block_sum(w, sh);
  if (threadIdx.x == 0) {
    out[0] = v;
    out[1] = w;
  }
}

__global__ void sqnorm_partial(const double* __restrict__ x, int64_t n, double* partial) {
  __shared__ double sh[32];
  double v = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const double a = __ldcs(x + i), b = __ldcs(x + i + stride);
    const double c = __ldcs(x + i + 2 * stride), d = __ldcs(x + i + 3 * stride);
    v = fma(a, a, v);
    v = fma(b, b, v);
    v = fma(c, c, v);
    v = fma(d, d, v);
  }
  for (; i < n; i += stride) {
    const double a = __ldcs(x + i);
    v = fma(a, a, v);
  }
  v = block_sum(v, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

__global__ void sum_final(const double* __restrict__ partial, int n, double* out) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += partial[i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) out[0] = v;
}

__global__ void sub_kernel(const double* a, const double* b, double* y, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    y[e] = a[e] - b[e];
}

__global__ void pad_rows_kernel(const double* F, int64_t S, int K, double* Fp, int ld) {
  const int64_t total = S * ld;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = e / ld;
    const int n = static_cast<int>(e - x * ld);
    Fp[e] = n < K ? F[x * K + n] : 0.0;
  }
}

int grid_for(int64_t n, int threads, int cap) {
  int64_t b = (n + threads - 1) / threads;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<int>(b);
}

}  // namespace

static unsigned long long g_launches = 0;
void note_launch() { __atomic_add_fetch(&g_launches, 1ull, __ATOMIC_RELAXED); }
uint64_t launch_count() { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

cudaError_t launch_gamma_factor(const double* S_all, int N, int n, int K, SolveWS ws,
                                cudaStream_t st) {
  const size_t smem = static_cast<size_t>(K) * (K + 1) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gamma_factor_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         128 * 129 * 8);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  // ws.L holds 2 K*K doubles: the factor / pseudo-inverse, then the Jacobi V scratch
  gamma_factor_kernel<<<1, GF_THREADS, smem, st>>>(S_all, N, n, K, ws.Gamma, ws.L, ws.mode,
                                                   ws.L + K * K);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_solve_rows(const double* M, double* A, const double* ref, double* dA,
                              int64_t rows, int K, SolveWS ws, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  const size_t smem = static_cast<size_t>(K) * (K + 1) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(solve_rows_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         128 * 129 * 8);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int blocks = grid_for(rows, SR_WARPS, 148);
  solve_rows_kernel<<<blocks, SR_WARPS * 32, smem, st>>>(M, A, ref, dA, rows, K, ws.Gamma, ws.L,
                                                         ws.mode, ws.rowstat);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gram_norms(const double* A, int64_t rows, int K, double* S,
                              const double* rowstat, double* nrm, cudaStream_t st) {
  const int blocks = grid_for((int64_t)K * K, 256, 1 << 20);
  gram_norms_kernel<<<blocks, 256, 0, st>>>(A, rows, K, S, rowstat, nrm);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gram(const double* A, int64_t rows, int K, double* S, cudaStream_t st) {
  return launch_gram_norms(A, rows, K, S, nullptr, nullptr, st);
}

cudaError_t launch_fitness_terms(const double* M, const double* A, int64_t rows, int K,
                                 const double* Gamma, const double* S, double* out,
                                 cudaStream_t st) {
  fitness_terms_kernel<<<1, 1024, 0, st>>>(M, A, rows * K, Gamma, S, (int64_t)K * K, out);
  note_launch();
  return cudaGetLastError();
}

int sqnorm_blocks(int64_t n) { return grid_for(n, 256, 1184); }

cudaError_t launch_sqnorm(const double* x, int64_t n, double* partial, int nblk, double* out,
                          cudaStream_t st) {
  sqnorm_partial<<<nblk, 256, 0, st>>>(x, n, partial);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  sum_final<<<1, 1024, 0, st>>>(partial, nblk, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_sub(const double* a, const double* b, double* y, int64_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  sub_kernel<<<grid_for(n, 256, 1184), 256, 0, st>>>(a, b, y, n);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pad_rows(const double* F, int64_t S, int K, double* Fp, int ld,
                            cudaStream_t st) {
  pad_rows_kernel<<<grid_for(S * ld, 256, 1184), 256, 0, st>>>(F, S, K, Fp, ld);
  note_launch();
  return cudaGetLastError();
}

}  // namespace cppp
