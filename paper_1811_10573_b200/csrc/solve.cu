// solve.cu — the small dense part of every ALS step, on device (Alg. 1 P:393-399,
// Alg. 3, normal equations):
//   Γ^(n) = S^(1) ∗ … ∗ S^(n-1) ∗ S^(n+1) ∗ … ∗ S^(N)          (Hadamard, ascending m)
//   A_new = M Γ^†                                              (L13 pivot rule)
//   G^(n) = (A^(n) - A_new) Γ^(n)
//   S^(n) = A_newᵀ A_new
// plus ‖A‖², ‖dA‖², ‖G‖² per mode (the ε_pp test L7 and the stop metric) and the fitness
// expansion terms.  K <= 128.  Every reduction has a fixed order (deterministic).
//
// Latency design: Γ^(n) only depends on the Grams, so its inverse is computed by
// ONE CTA (register-resident Gauss-Jordan, one barrier per pivot) on a side stream while the main
// stream computes M^(n); the main stream then runs one row kernel (A_new = M P, G, dA, norms and
// a per-block partial Gram, all from shared memory) and one tiny reduction.
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

constexpr double PIVOT_TAU = 1e-12;  // L13 / S:201
constexpr double PINV_TAU = 1e-12;
constexpr int GI_THREADS = 512;
constexpr int GI_MAXE = 32;          // K*K <= 16384 = 32 * 512 register-resident elements

// ---------------------------------------------------------------- Γ and its Cholesky factor
// Right-looking Cholesky Γ = L Lᵀ with the L13 pivot rule (accept iff every pivot d_j >
// τ·max diag Γ), the same factorization the oracle uses.  Thread (l = tid % 128, rg = tid / 128)
// keeps column l, rows 32 rg + v (v < 32) in registers.  Column j+1 is published (unscaled) at the
// end of step j, so step j+1 reads its pivot and scales on the fly: one barrier per pivot.
__global__ void __launch_bounds__(GI_THREADS, 1)
    gamma_chol_kernel(const double* __restrict__ S_all, int N, int n, int K, double* Gamma,
                      double* Lout, int* mode) {
  __shared__ __align__(16) double colb[2][128];
  __shared__ double piv_s[2][2];    // [buffer][-, 1/pivot]
  __shared__ int bad_s[2];
  __shared__ double sh[32];
  const int tid = threadIdx.x, KK = K * K;
  const int lane = tid & 31, wid = tid >> 5;
  // column l = 4 lane + (warp mod 4): every SM sub-partition owns every 4th column, so the
  // shrinking trailing matrix stays balanced; rg = warp / 4 selects rows 32 rg .. 32 rg + 31.
  const int l = 4 * lane + (wid & 3), rg = wid >> 2;
  const bool col_ok = l < K;
  double w[GI_MAXE];
#pragma unroll
  for (int v = 0; v < GI_MAXE; ++v) w[v] = 1.0;   // 1.0 * S^(first) is exactly S^(first)
  const int rows_here = min(GI_MAXE, max(0, K - 32 * rg));
  if (col_ok) {
    for (int m = 0; m < N; ++m) {
      if (m == n) continue;
      const double* Sm = S_all + (int64_t)m * KK + (32 * rg) * K + l;
#pragma unroll
      for (int v = 0; v < GI_MAXE; ++v)
        if (v < rows_here) w[v] *= __ldg(Sm + v * K);
    }
  }
  double dmax = 0.0;
#pragma unroll
  for (int v = 0; v < GI_MAXE; ++v) {
    const int i = 32 * rg + v;
    if (!(col_ok && v < rows_here)) w[v] = 0.0;
    else {
      Gamma[i * K + l] = w[v];
      if (i == l) dmax = fmax(dmax, w[v]);
    }
  }
  for (int i = tid; i < 2 * 128; i += GI_THREADS) (&colb[0][0])[i] = 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if (lane == 0) sh[wid] = dmax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < GI_THREADS / 32; ++i) m = fmax(m, sh[i]);
    sh[0] = m;
  }
  __syncthreads();
  const double thresh = PIVOT_TAU * sh[0];
  // Unscaled (LDLᵀ-form) elimination: column j keeps W[i][j] with d_j = W[j][j] the pivot, the
  // trailing update is W[i][l] -= W[i][j] W[l][j] / d_j, and L = W diag(d)^(-1/2) is applied at
  // the end, so only one reciprocal (no sqrt) sits on the per-pivot critical path.
  __shared__ double dpiv[128];
  if (l == 0) {
#pragma unroll
    for (int v = 0; v < GI_MAXE; ++v) colb[0][32 * rg + v] = w[v];
    if (rg == 0) {
      const double p = w[0];
      bad_s[0] = !(p > thresh);
      dpiv[0] = p;
      piv_s[0][1] = __drcp_rn(p);
    }
  }
  __syncthreads();
  bool ok = true;
  for (int j = 0; j < K; ++j) {
    const int b = j & 1;
    if (bad_s[b]) {
      ok = false;
      break;
    }
    if (col_ok && l > j && 32 * rg + 31 > j) {
      const double cl = colb[b][l] * piv_s[b][1];
#pragma unroll
      for (int v = 0; v < GI_MAXE; v += 2) {
        const double2 cc = *reinterpret_cast<const double2*>(&colb[b][32 * rg + v]);
        w[v] = fma(-cc.x, cl, w[v]);
        w[v + 1] = fma(-cc.y, cl, w[v + 1]);
      }
    }
    if (l == j + 1) {   // publish the next column (and, from its diagonal owner, the pivot)
#pragma unroll
      for (int v = 0; v < GI_MAXE; ++v) colb[b ^ 1][32 * rg + v] = w[v];
      if (rg == ((j + 1) >> 5)) {
        const double p = colb[b ^ 1][j + 1];   // this thread just wrote it
        bad_s[b ^ 1] = !(p > thresh);
        dpiv[j + 1] = p;
        piv_s[b ^ 1][1] = __drcp_rn(p);
      }
    }
    __syncthreads();
  }
  if (ok) {
    if (col_ok) {
      const double d = dpiv[l];
      const double r = sqrt(d);
      const double ri = 1.0 / r;
#pragma unroll
      for (int v = 0; v < GI_MAXE; ++v) {
        const int i = 32 * rg + v;
        if (i < K) Lout[i * K + l] = (i > l) ? w[v] * ri : (i == l ? r : 0.0);
      }
    }
    if (tid == 0) *mode = 0;
  } else if (tid == 0) {
    *mode = 1;   // gamma_pinv_kernel takes over
  }
}

// Eigen pseudo-inverse fallback (L13): runs after gamma_chol_kernel and exits at once unless
// the Gauss-Jordan pivot test failed.  Two-sided cyclic Jacobi, Brent-Luk parallel ordering.
__global__ void __launch_bounds__(GI_THREADS, 1)
    gamma_pinv_kernel(int K, const double* __restrict__ Gamma, double* Pout, const int* mode,
                      double* Vscratch) {
  if (*mode == 0) return;
  extern __shared__ double W[];  // K x (K+1)
  __shared__ double sh[32];
  const int tid = threadIdx.x, KK = K * K;
  // ---- eigen pseudo-inverse: two-sided cyclic Jacobi on W (from Γ), V in global scratch
  const int P = K + 1;
  const int nt = GI_THREADS;
  for (int e = tid; e < KK; e += nt) {
    const int i = e / K, j = e - i * K;
    W[i * P + j] = Gamma[e];
    Vscratch[e] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int Ke = (K + 1) & ~1;  // even number of players
  __shared__ double cs[64], sn[64];
  __shared__ int pp_[64], qq_[64];
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int e = tid; e < KK; e += nt) {
      const int i = e / K, j = e - i * K;
      const double v = W[i * P + j];
      if (i == j) dia += v * v;
      else off += v * v;
    }
    off = block_sum(off, sh);
    dia = block_sum(dia, sh);
    if (off <= 1e-30 * dia || dia == 0.0) break;
    for (int r = 0; r < Ke - 1; ++r) {
      if (tid < Ke / 2) {
        int p, q;
        if (tid == 0) {
          p = Ke - 1;
          q = r;
        } else {
          p = (r + tid) % (Ke - 1);
          q = (r - tid + Ke - 1) % (Ke - 1);
        }
        if (p > q) {
          const int tmp = p;
          p = q;
          q = tmp;
        }
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
        cs[tid] = c;
        sn[tid] = s;
        pp_[tid] = p;
        qq_[tid] = q;
      }
      __syncthreads();
      for (int e = tid; e < (Ke / 2) * K; e += nt) {  // rows: W <- Jᵀ W
        const int pr = e / K, l = e - pr * K;
        const int p = pp_[pr], q = qq_[pr];
        if (q >= K) continue;
        const double c = cs[pr], s = sn[pr];
        const double wp = W[p * P + l], wq = W[q * P + l];
        W[p * P + l] = c * wp - s * wq;
        W[q * P + l] = s * wp + c * wq;
      }
      __syncthreads();
      for (int e = tid; e < (Ke / 2) * K; e += nt) {  // columns: W <- W J, V <- V J
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
  for (int e = tid; e < KK; e += nt) {
    const int i = e / K, j = e - i * K;
    double v = 0.0;
    for (int l = 0; l < K; ++l) v += Vscratch[i * K + l] * lam[l] * Vscratch[j * K + l];
    Pout[e] = v;
  }
}

// ---------------------------------------------------------------- row solves + partial Gram
// One warp per row (16 rows per CTA).  Cholesky path (mode 0): forward then back substitution
// with L staged in shared memory (pitch K+1: column reads are conflict-free), as the oracle does;
// pinv path (mode 1): a = m P.  Then G = (a_old - a_new) Γ with Γ staged, dA, row norms and the
// CTA's partial Gram.  Lane c owns columns c + 32u.
constexpr int SR_WARPS = 8;

// stage a K x K row-major matrix into shared memory with row pitch `pitch`: 8-byte cp.async
// (LDGSTS) for every element, all in flight, no register round trip; the caller syncs.
__device__ __forceinline__ void stage_matrix(double* dst, int pitch, const double* __restrict__ src,
                                             int K) {
  const int KK = K * K;
  int i = threadIdx.x / K, j = threadIdx.x - (threadIdx.x / K) * K;
  const int di = blockDim.x / K, dj = blockDim.x - di * K;
  for (int e = threadIdx.x; e < KK; e += blockDim.x) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst + i * pitch + j));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src + e) : "memory");
    i += di;
    j += dj;
    if (j >= K) {
      j -= K;
      ++i;
    }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ double pick4(const double (&m)[4], int slot) {
  return slot == 0 ? m[0] : slot == 1 ? m[1] : slot == 2 ? m[2] : m[3];
}

__global__ void __launch_bounds__(SR_WARPS * 32)
    solve_rows_kernel(const double* __restrict__ M, double* A, const double* ref, double* dA,
                      int64_t rows, int K, const double* __restrict__ Gamma,
                      const double* __restrict__ Lm, const int* __restrict__ mode_p,
                      double* __restrict__ rowstat, double* __restrict__ gpart) {
  extern __shared__ double sm[];
  const int KK = K * K;
  const int P = K + 1;
  double* Ws = sm;                         // K*(K+1)
  double* dinv = Ws + K * P;               // K
  double* As = dinv + K;                   // SR_WARPS*K
  double* Ds = As + SR_WARPS * K;          // SR_WARPS*K
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t y = blockIdx.x * (int64_t)SR_WARPS + w;
  const bool valid = y < rows;
  const int mode = *mode_p;
  stage_matrix(Ws, mode == 0 ? P : K, Lm, K);
  double m[4], aold[4], rf[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = lane + 32 * u;
    const bool in = valid && c < K;
    aold[u] = in ? A[y * K + c] : 0.0;
    rf[u] = in ? ref[y * K + c] : 0.0;
    m[u] = in ? M[y * K + c] : 0.0;
  }
  __syncthreads();
  if (mode == 0) {
    for (int j = threadIdx.x; j < K; j += blockDim.x) dinv[j] = 1.0 / Ws[j * P + j];
    __syncthreads();
    // forward L z = m, blocked by 32 columns: in-block substitution (lane = column), then a
    // dependency-free update of the later column blocks
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (32 * b >= K) break;
      const int c = 32 * b + lane;
      for (int jj = 0; jj < 32; ++jj) {
        const int j = 32 * b + jj;
        if (j >= K) break;
        const double zj = __shfl_sync(0xffffffffu, m[b], jj) * dinv[j];
        if (lane == jj) m[b] = zj;
        else if (lane > jj && c < K) m[b] = fma(-Ws[c * P + j], zj, m[b]);
      }
#pragma unroll
      for (int u = b + 1; u < 4; ++u) {
        const int cu = lane + 32 * u;
        if (32 * u >= K) break;
        double acc = m[u];
        for (int jj = 0; jj < 32 && 32 * b + jj < K; ++jj) {
          const double zj = __shfl_sync(0xffffffffu, m[b], jj);
          if (cu < K) acc = fma(-Ws[cu * P + 32 * b + jj], zj, acc);
        }
        m[u] = acc;
      }
    }
    // back Lᵀ a = z, blocks in reverse
#pragma unroll
    for (int b = 3; b >= 0; --b) {
      if (32 * b >= K) continue;
      const int c = 32 * b + lane;
      const int jtop = min(31, K - 1 - 32 * b);
      for (int jj = jtop; jj >= 0; --jj) {
        const int j = 32 * b + jj;
        const double aj = __shfl_sync(0xffffffffu, m[b], jj) * dinv[j];
        if (lane == jj) m[b] = aj;
        else if (lane < jj) m[b] = fma(-Ws[j * P + c], aj, m[b]);
      }
#pragma unroll
      for (int u = 0; u < b; ++u) {
        const int cu = lane + 32 * u;
        double acc = m[u];
        for (int jj = 0; jj <= jtop; ++jj) {
          const double aj = __shfl_sync(0xffffffffu, m[b], jj);
          acc = fma(-Ws[(32 * b + jj) * P + cu], aj, acc);
        }
        m[u] = acc;
      }
    }
  } else {
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    for (int p = 0; p < K; ++p) {
      const double mp = __shfl_sync(0xffffffffu, pick4(m, p >> 5), p & 31);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = lane + 32 * u;
        if (c < K) a[u] = fma(mp, Ws[p * K + c], a[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) m[u] = a[u];
  }
  // m now holds a_new
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = lane + 32 * u;
    if (c < K) {
      As[w * K + c] = valid ? m[u] : 0.0;
      Ds[w * K + c] = valid ? aold[u] - m[u] : 0.0;
    }
  }
  __syncthreads();
  stage_matrix(Ws, K, Gamma, K);
  __syncthreads();
  double g[4] = {0.0, 0.0, 0.0, 0.0};
  for (int p = 0; p < K; ++p) {
    const double dp = Ds[w * K + p];
    const double* wr = Ws + p * K;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = lane + 32 * u;
      if (c < K) g[u] = fma(dp, wr[c], g[u]);
    }
  }
  double na = 0.0, nd = 0.0, ng = 0.0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = lane + 32 * u;
    if (valid && c < K) {
      const double d = m[u] - rf[u];
      A[y * K + c] = m[u];
      dA[y * K + c] = d;
      na = fma(m[u], m[u], na);
      nd = fma(d, d, nd);
      ng = fma(g[u], g[u], ng);
    }
  }
  na = warp_sum(na);
  nd = warp_sum(nd);
  ng = warp_sum(ng);
  if (valid && lane == 0) {
    rowstat[y * 3 + 0] = na;
    rowstat[y * 3 + 1] = nd;
    rowstat[y * 3 + 2] = ng;
  }
  // partial Gram of this CTA's rows (rows in ascending order), 2 outputs per thread per pass
  for (int e = threadIdx.x; e < KK; e += blockDim.x) {
    const int k1 = e / K, k2 = e - k1 * K;
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < SR_WARPS; ++r) s = fma(As[r * K + k1], As[r * K + k2], s);
    gpart[(int64_t)blockIdx.x * KK + e] = s;
  }
}

// partial Gram only (rows staged in shared memory), same partial layout as solve_rows
__global__ void __launch_bounds__(SR_WARPS * 32)
    gram_partial_kernel(const double* __restrict__ A, int64_t rows, int K,
                        double* __restrict__ gpart) {
  extern __shared__ double As[];  // SR_WARPS x K
  const int KK = K * K;
  const int64_t y0 = blockIdx.x * (int64_t)SR_WARPS;
  for (int e = threadIdx.x; e < SR_WARPS * K; e += blockDim.x) {
    const int64_t y = y0 + e / K;
    As[e] = y < rows ? A[y0 * K + e] : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < KK; e += blockDim.x) {
    const int k1 = e / K, k2 = e - k1 * K;
    double s = 0.0;
#pragma unroll 4
    for (int r = 0; r < SR_WARPS; ++r) s = fma(As[r * K + k1], As[r * K + k2], s);
    gpart[(int64_t)blockIdx.x * KK + e] = s;
  }
}

// S = Σ_b gpart[b] (ascending b); block 0 also reduces the row norms in row order.
__global__ void gram_reduce_kernel(const double* __restrict__ gpart, int nb, int K, double* S,
                                   const double* __restrict__ rowstat, int64_t rows, double* nrm) {
  const int KK = K * K;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < KK) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += gpart[(int64_t)b * KK + e];
    S[e] = s;
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
void note_launches(uint64_t n) { __atomic_add_fetch(&g_launches, n, __ATOMIC_RELAXED); }
uint64_t launch_count() { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int solve_row_blocks(int64_t rows) { return static_cast<int>((rows + SR_WARPS - 1) / SR_WARPS); }

cudaError_t launch_gamma_factor(const double* S_all, int N, int n, int K, double* Gamma, double* L,
                                int* mode, double* Vscratch, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(K) * (K + 1) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gamma_pinv_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 129 * 8);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  gamma_chol_kernel<<<1, GI_THREADS, 0, st>>>(S_all, N, n, K, Gamma, L, mode);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  gamma_pinv_kernel<<<1, GI_THREADS, smem, st>>>(K, Gamma, L, mode, Vscratch);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_solve_rows(const double* M, double* A, const double* ref, double* dA,
                              int64_t rows, int K, const double* Gamma, const double* L,
                              const int* mode, double* rowstat, double* gpart, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  const size_t smem = (static_cast<size_t>(K) * (K + 1) + K + 2 * SR_WARPS * K) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(solve_rows_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (128 * 129 + 128 + 2 * SR_WARPS * 128) * 8);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  solve_rows_kernel<<<solve_row_blocks(rows), SR_WARPS * 32, smem, st>>>(M, A, ref, dA, rows, K,
                                                                         Gamma, L, mode, rowstat,
                                                                         gpart);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gram_reduce(const double* gpart, int nb, int K, double* S,
                               const double* rowstat, int64_t rows, double* nrm, cudaStream_t st) {
  gram_reduce_kernel<<<grid_for((int64_t)K * K, 256, 1 << 20), 256, 0, st>>>(gpart, nb, K, S, rowstat,
                                                                            rows, nrm);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gram(const double* A, int64_t rows, int K, double* S, double* gpart,
                        cudaStream_t st) {
  const int nb = solve_row_blocks(rows);
  gram_partial_kernel<<<nb, SR_WARPS * 32, SR_WARPS * K * sizeof(double), st>>>(A, rows, K, gpart);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_gram_reduce(gpart, nb, K, S, nullptr, 0, nullptr, st);
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
