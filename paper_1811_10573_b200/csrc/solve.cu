// solve.cu — the small dense part of every ALS step, on device (Alg. 1 P:393-399,
// Alg. 3, normal equations):
//   Γ^(n) = S^(1) ∗ … ∗ S^(n-1) ∗ S^(n+1) ∗ … ∗ S^(N)          (Hadamard, ascending m)
//   A_new = M Γ^†                                              (L13 pivot rule)
//   G^(n) = (A^(n) - A_new) Γ^(n)
//   S^(n) = A_newᵀ A_new
// plus ‖A‖², ‖dA‖², ‖G‖² per mode (the ε_pp test L7 and the stop metric) and the fitness
// expansion terms.  K <= 128.  Every reduction has a fixed order (deterministic).
//
// Latency design: Γ^(n) only depends on the Grams, so its Cholesky factor is
// computed by ONE CTA (register-resident, one barrier per pivot) on a side stream while the main
// stream computes M^(n); the main stream then runs one row kernel (substitution solves, G, dA,
// per-row statistics; one warp per row) and one Gram kernel (S^(n), the fixed-order sums).
#include "internal.h"

#include <cstdlib>

namespace cppp {
#ifdef CPPP_PROBE_CYCLES   // tools/probe_solve only: per-phase clock64 deltas of CTA 0, thread 0
__device__ long long g_probe_cycles[16];
#define PROBE_T0() const long long probe_t0_ = clock64()
#define PROBE_T(slot) \
  if (threadIdx.x == 0 && blockIdx.x == 0) g_probe_cycles[slot] = clock64() - probe_t0_
#else
#define PROBE_T0() (void)0
#define PROBE_T(slot) (void)0
#endif
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

// NV block sums at once, each with block_sum's tree (same arithmetic, three barriers in all)
template <int NV>
__device__ void block_sum_n(double (&v)[NV], double* sh /* 32 NV */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int c = 0; c < NV; ++c) v[c] = warp_sum(v[c]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < NV; ++c) sh[32 * c + w] = v[c];
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int c = 0; c < NV; ++c) {
      double r = lane < nw ? sh[32 * c + lane] : 0.0;
      r = warp_sum(r);
      if (lane == 0) sh[32 * c] = r;
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NV; ++c) v[c] = sh[32 * c];
}

// L13 / S:201: the pivot rule and the pseudo-inverse cutoff take τ (cppp_opts.pinv_rel_tol,
// default 1e-12) as a kernel argument

// 1/d for the factorization's pivots: the hardware approximation (MUFU.RCP64H) refined by two
// Newton steps -- within an ulp of the correctly rounded value, and off the slow path that
// __drcp_rn takes on every call (the reciprocal sits on the per-pivot critical path)
__device__ __forceinline__ double pivot_rcp(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}
constexpr int GF_THREADS = 640;      // factorization: 20 warps = the lower-triangle 16x32 blocks
constexpr int GP_THREADS = 512;      // Jacobi fallback

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- Γ and its Cholesky factor
// Right-looking Cholesky Γ = L Lᵀ in unscaled (LDLᵀ) form with the L13 pivot rule (accept iff
// every pivot d_j > τ·max diag Γ), the factorization the oracle uses.  Step j updates
// W[i][l] -= W[i][j] · (W[l][j] / d_j) for i, l > j, then L = W diag(d)^(-1/2).
//
// Layout: a 128 x 128 Γ is cut into 16-row x 32-column blocks; the 20 blocks that touch the
// lower triangle get one warp each, and thread (block, lane) keeps W[16 rg + v][32 cg + lane],
// v < 16, in registers.  Blocks are dealt to warps in order of how long they stay active (a
// block retires once j passes its last row or column), so the four SM sub-partitions stay
// balanced while the trailing matrix shrinks; a retired warp skips the step.  Column j+1 and
// 1/d_(j+1) are published through a double-buffered shared column: one barrier per pivot.
//
// Γ is stored with row pitch ldt (K rounded up to 8; zero padding).  Output Tp (ldt x ldt, the
// row solves' packed factor; zero padding with a unit diagonal past K):
// Tp[j][j] = 1 / L[j][j];
// Tp[j][c] = L[c][j] for c > j (column j of L: the forward substitution reads row j);
// Tp[j][c] = L[j][c] for c < j (row j of L: the back substitution reads row j).
// warp -> lower block (rg | cg << 4), sorted by decreasing lifetime min(16 rg + 15, 32 cg + 31)
// (ties: ascending cg, then rg), dealt round-robin over the SM sub-partitions (wid % 4)
__constant__ unsigned char kCholBlock[20] = {
    7 | 3 << 4, 6 | 3 << 4, 5 | 2 << 4, 6 | 2 << 4, 7 | 2 << 4, 4 | 2 << 4, 3 | 1 << 4,
    4 | 1 << 4, 5 | 1 << 4, 6 | 1 << 4, 7 | 1 << 4, 2 | 1 << 4, 1,          2,
    3,          4,          5,          6,          7,          0};

template <bool transpose>
__global__ void __launch_bounds__(GF_THREADS, 1)
    gamma_chol_kernel(const double* __restrict__ S_all, int N, int n, int K, double* Gamma,
                      double* Tp, int ldt, int* mode, double tau) {
  PROBE_T0();
  pdl_wait();
  __shared__ __align__(16) double colb[2][128];
  __shared__ double rdv[2];
  __shared__ int bad_s;
  __shared__ double dpiv[128];
  __shared__ double sh[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int rg = kCholBlock[wid] & 15, cg = kCholBlock[wid] >> 4;
  const int r0 = 16 * rg, l = 32 * cg + lane;
  const bool col_ok = l < K;
  const bool lowerw = (r0 < K) && (32 * cg < K);   // every allocated block touches the lower part
  const bool has_diag = col_ok && l >= r0 && l < r0 + 16;   // this thread holds W[l][l]
  double w[16];
#pragma unroll
  for (int v = 0; v < 16; ++v) w[v] = 1.0;   // 1.0 * S^(first) is exactly S^(first)
  double diag = 1.0;                          // a second copy of W[l][l] (same operations)
  const int rows_here = min(16, max(0, K - r0));
  if (col_ok) {
    for (int m = 0; m < N; ++m) {
      if (m == n) continue;
      const double* Sm = S_all + (int64_t)m * K * K + r0 * K + l;
#pragma unroll
      for (int v = 0; v < 16; ++v)
        if (v < rows_here) w[v] *= __ldg(Sm + v * K);
      diag *= __ldg(S_all + (int64_t)m * K * K + l * K + l);
    }
  }
#pragma unroll
  for (int v = 0; v < 16; ++v) {
    const int i = r0 + v;
    if (!(col_ok && v < rows_here)) {
      w[v] = 0.0;
    } else {
      Gamma[i * ldt + l] = w[v];   // row i: 32 consecutive columns per store
      if constexpr (!transpose) Gamma[l * ldt + i] = w[v];   // small K: the mirror directly
    }
  }
  if constexpr (transpose) {
    // Γ is exactly symmetric (Grams are written mirrored): the lower blocks also fill the upper
    // triangle, transposed through shared memory so every store is a 128-byte row segment
    // (column-wise stores of the mirror cost ~10 k cycles of LSU issue at K = 100)
    extern __shared__ double gf_dyn[];   // [GF_THREADS / 32][16][33]
    double(*tb)[16][33] = reinterpret_cast<double(*)[16][33]>(gf_dyn);
#pragma unroll
    for (int v = 0; v < 16; ++v) tb[wid][v][lane] = w[v];
    __syncwarp();
    const int vi = lane & 15, half = lane >> 4;
    const int i = r0 + vi;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int lc = 2 * q + half;                 // column of the block = row of the mirror
      const int lm = 32 * cg + lc;
      if (lowerw && lm < K && vi < rows_here) Gamma[lm * ldt + i] = tb[wid][vi][lc];
    }
  }
  double dmax = has_diag ? diag : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if (lane == 0) sh[wid] = dmax;
  if (tid == 0) bad_s = 0;
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int i = 0; i < GF_THREADS / 32; ++i) mx = fmax(mx, sh[i]);
    sh[0] = mx;
  }
  __syncthreads();
  const double thresh = tau * sh[0];
  if (tid < ldt - K) Tp[(K + tid) * ldt + K + tid] = 1.0;   // unit diagonal of the padding
  if (l == 0) {   // publish column 0 and its pivot
#pragma unroll
    for (int v = 0; v < 16; ++v) colb[0][r0 + v] = w[v];
    if (rg == 0) {
      if (!(diag > thresh)) bad_s = 1;
      dpiv[0] = diag;
      rdv[0] = pivot_rcp(diag);
    }
  }
  __syncthreads();
  PROBE_T(0);
  // One pivot per step.  The diagonal owner of column j+1 updates its copy of W[j+1][j+1]
  // first, so the reciprocal overlaps the rest of the update.  A failed pivot test is recorded
  // (sticky) and acted on after the loop.
  // shared-window addresses computed once (the generic-pointer form re-derived the window base
  // with an S2R on every pivot, on the chain in front of the column load)
  uint32_t colb0 = smem_addr(&colb[0][0]), rdv0 = smem_addr(&rdv[0]);
  uint32_t my_l = colb0 + 8u * static_cast<uint32_t>(l), my_rows = colb0 + 8u * static_cast<uint32_t>(r0);
  // opaque to the compiler: otherwise it re-derives them from the shared window base (S2R
  // SR_CgaCtaId + LEA) inside the pivot loop, on the chain in front of every column load
  asm volatile("" : "+r"(rdv0), "+r"(my_l), "+r"(my_rows));
  for (int j = 0; j < K; ++j) {
    const uint32_t bo = (j & 1) ? 128u * 8u : 0u;   // colb[b] / colb[b ^ 1]
    if (lowerw && r0 + 15 > j && 32 * cg + 31 > j && l > j) {
      double cjl, rj;
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(cjl) : "r"(my_l + bo) : "memory");
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(rj) : "r"(rdv0 + ((j & 1) ? 8u : 0u)) : "memory");
      const double cl = cjl * rj;
      if (has_diag) {
        diag = fma(-cjl, cl, diag);
        if (l == j + 1) {
          if (!(diag > thresh)) bad_s = 1;
          dpiv[j + 1] = diag;
          const double rn = pivot_rcp(diag);
          asm volatile("st.shared.f64 [%0], %1;" ::"r"(rdv0 + ((j & 1) ? 0u : 8u)), "d"(rn) : "memory");
        }
      }
#pragma unroll
      for (int v = 0; v < 16; v += 2) {
        double cx, cy;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(cx), "=d"(cy) : "r"(my_rows + bo + 8u * v) : "memory");
        w[v] = fma(-cx, cl, w[v]);
        w[v + 1] = fma(-cy, cl, w[v + 1]);
      }
      if (l == j + 1) {   // publish column j+1
#pragma unroll
        for (int v = 0; v < 16; v += 2)
          asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(my_rows + (1024u - bo) + 8u * v), "d"(w[v]),
                       "d"(w[v + 1])
                       : "memory");
      }
    }
    __syncthreads();
  }
  if (!bad_s) {
    extern __shared__ double gf_dyn[];   // the mirror transposes again: column l of L as rows
    double(*tb)[16][33] = reinterpret_cast<double(*)[16][33]>(gf_dyn);
    if (col_ok) {
      const double d = dpiv[l];
      const double r = sqrt(d);
      const double ri = 1.0 / r;
#pragma unroll
      for (int v = 0; v < 16; ++v) {
        const int i = r0 + v;
        if (i < K && i > l) {
          const double x = w[v] * ri;
          Tp[i * ldt + l] = x;   // row i of L
          if constexpr (transpose) tb[wid][v][lane] = x;
          else Tp[l * ldt + i] = x;
        } else if (i == l) {
          Tp[l * ldt + l] = 1.0 / r;
        }
      }
    }
    __syncwarp();
    if constexpr (transpose) {   // column l of L below the diagonal into row l of Tp, 128-byte rows
      const int vi = lane & 15, half = lane >> 4;
      const int i = r0 + vi;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int lm = 32 * cg + 2 * q + half;
        if (lowerw && lm < K && i < K && i > lm) Tp[lm * ldt + i] = tb[wid][vi][2 * q + half];
      }
    }
    if (tid == 0) *mode = 0;
  } else if (tid == 0) {
    *mode = 1;   // gamma_post_kernel runs the pseudo-inverse fallback
  }
  PROBE_T(1);
}

// Inverses of the 32 x 32 diagonal blocks of L for the row solves (Q, right after Tp): warp b,
// lane c computes column c of inv(L_bb) right-looking with compile-time indices; Q[b][c][j] =
// inv(L_bb)[j][c] with row pitch 33.  Rows past ld are the identity.  Exits unless the Cholesky
// path was taken.
// Ls = the block (1 / L[i][i] on the diagonal, L below it; pitch 33), Q = its output rows.
// NB < 32: rows and columns >= NB of the block are the identity, so the substitution stops at
// NB and column c >= NB of the inverse is e_c.
template <int NB = 32>
__device__ __forceinline__ void block_inverse_smem(double (*Ls)[33], double* Q) {
  const int lane = threadIdx.x & 31, c = lane;
  double y[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) y[j] = (j >= NB && j == c) ? 1.0 : 0.0;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const double dinv = Ls[i][i];   // 1 / L[i][i]
    y[i] = i == c ? dinv : (i > c ? -y[i] * dinv : 0.0);
#pragma unroll
    for (int j = i + 1; j < NB; ++j) y[j] = fma(Ls[j][i], y[i], y[j]);   // L[j][i]
  }
  // Q[c][j] = y_c[j]: staged row-wise in shared memory (the block is no longer needed), then
  // written as 33-double rows by the whole warp (coalesced; lane-c row stores hit 32 sectors)
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 32; ++j) Ls[c][j] = y[j];
  __syncwarp();
#pragma unroll 4
  for (int r = 0; r < 32; ++r) Q[r * 33 + lane] = Ls[r][lane];
}

__device__ __forceinline__ void block_inverse_dev(double* Tp, int ldt) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nblk = (ldt + 31) >> 5;
  if (wid >= nblk) return;
  const int b0 = 32 * wid, c = lane;
  __shared__ double Ls[4][32][33];   // the diagonal block (coalesced rows), identity past ld
#pragma unroll 4
  for (int j = 0; j < 32; ++j) {
    const int gj = b0 + j, gc = b0 + c;
    Ls[wid][j][c] = (gj < ldt && gc < ldt) ? Tp[gj * ldt + gc] : (j == c ? 1.0 : 0.0);
  }
  __syncwarp();
  block_inverse_smem(Ls[wid], Tp + ldt * ldt + wid * 32 * 33);
}

// Eigen pseudo-inverse fallback (L13): runs after gamma_chol_kernel and exits at once unless
// the pivot test failed.  Two-sided cyclic Jacobi, Brent-Luk parallel ordering; the
// pseudo-inverse P goes to Tp (pitch ldt).
__device__ __forceinline__ void gamma_pinv_dev(int K, const double* __restrict__ Gamma,
                                               double* Pout, int ldt, double* Vscratch, double tau) {
  extern __shared__ double W[];  // K x (K+1)
  __shared__ double sh[32];
  const int tid = threadIdx.x, KK = K * K;
  const int P = K + 1;
  const int nt = blockDim.x;
  for (int e = tid; e < KK; e += nt) {
    const int i = e / K, j = e - i * K;
    W[i * P + j] = Gamma[i * ldt + j];
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
    lam[i] = (lmax > 0.0 && l > tau * lmax) ? 1.0 / l : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < KK; e += nt) {
    const int i = e / K, j = e - i * K;
    double v = 0.0;
    for (int l = 0; l < K; ++l) v += Vscratch[i * K + l] * lam[l] * Vscratch[j * K + l];
    Pout[i * ldt + j] = v;
  }
}

// After the factorization: the Cholesky path inverts the diagonal 32 x 32 blocks of L (warps
// 0-3), the pseudo-inverse path (failed pivot test) runs the Jacobi fallback — one launch
// either way (the two separate kernels cost a launch on the factorization chain per mode).
__global__ void __launch_bounds__(GP_THREADS, 1)
    gamma_post_kernel(int K, const double* __restrict__ Gamma, double* Tp, int ldt,
                      const int* mode, double* Vscratch, double tau) {
  pdl_wait();
  if (*mode == 0) {
    if (threadIdx.x < 128) block_inverse_dev(Tp, ldt);
  } else {
    gamma_pinv_dev(K, Gamma, Tp, ldt, Vscratch, tau);
  }
}

// K <= 32: the whole factorization in ONE warp, one launch (the chain above costs two launches
// and ~570 cycles of barrier + shared-memory round trip per pivot: C4's K = 30 took 21 us).
// Lane i keeps row i of W in registers; step j broadcasts row j by shuffles (W stays symmetric
// in exact arithmetic, so row j stands in for column j) and lane i > j updates
// W[i][k] -= (W[i][j] / d_j) W[j][k], k > j -- the same L13 pivot rule and output layout as
// gamma_chol_kernel, then the inverse of the single diagonal block (block_inverse_dev).  A
// failed pivot test runs the Jacobi pseudo-inverse, as gamma_post_kernel.
// one warp: a shuffle inside a warp-uniform branch of a larger CTA still compiles to the
// divergent-collective path (WARPSYNC/ENDCOLLECTIVE around every SHFL: 2x slower than the
// two-kernel chain); the rare pseudo-inverse fallback then runs on 32 threads
constexpr int GS_THREADS = 32;
template <int KP>   // K <= KP (8, 16 or 32): every loop is unrolled to KP
__global__ void __launch_bounds__(GS_THREADS, 1)
    gamma_small_kernel(const double* __restrict__ S_all, int N, int n, int K, double* Gamma,
                       double* Tp, int ldt, int* mode, double* Vscratch, double tau) {
  PROBE_T0();
  pdl_wait();
  __shared__ int bad_s;
  {
    const int i = threadIdx.x;
    const bool row_ok = i < K;
    double w[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) w[k] = 1.0;   // 1.0 * S^(first) is exactly S^(first)
    // two Grams per round, both rows loaded before either product (ascending m as before)
    for (int m = 0; m < N; ++m) {
      if (m == n) continue;
      int m2 = m + 1;
      if (m2 == n) ++m2;
      const double* Sa = S_all + (int64_t)m * K * K + (int64_t)(row_ok ? i : 0) * K;
      const double* Sb = S_all + (int64_t)(m2 < N ? m2 : m) * K * K + (int64_t)(row_ok ? i : 0) * K;
      double a[KP], b[KP];
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        a[k] = k < K ? __ldg(Sa + k) : 1.0;
        b[k] = k < K && m2 < N ? __ldg(Sb + k) : 1.0;
      }
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        w[k] *= a[k];
        if (m2 < N) w[k] *= b[k];
      }
      m = m2;
    }
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      if (!row_ok || k >= K) w[k] = 0.0;
      else Gamma[i * ldt + k] = w[k];
    }
    double dmax = 0.0;
#pragma unroll
    for (int k = 0; k < KP; ++k)
      if (k == i && row_ok) dmax = w[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    const double thresh = tau * dmax;
    PROBE_T(6);
    // every shuffle unconditional (a shuffle under a runtime condition compiles to the
    // divergent-collective path); steps j >= K only touch padding lanes and columns (their
    // zero pivots turn them into inf/NaN there), rows and columns < K are exact
    bool bad = false;
#pragma unroll
    for (int j = 0; j < KP; ++j) {
      const double d = __shfl_sync(0xffffffffu, w[j], j);
      if (j < K && !(d > thresh)) bad = true;
      const double cl = w[j] * pivot_rcp(d);
#pragma unroll
      for (int k = j + 1; k < KP; ++k) {
        const double rjk = __shfl_sync(0xffffffffu, w[k], j);
        if (i > j) w[k] = fma(-cl, rjk, w[k]);
      }
    }
    PROBE_T(7);
    if (!bad) {
      // L[i][j] = W[i][j] / sqrt(d_j): row i of L into row i of Tp and column i (the mirror);
      // d_j is lane j's W[j][j], untouched after step j: lane j forms 1 / sqrt(d_j) once
      __shared__ double Ls[32][33];   // the block for the inverse, straight from registers
      double own = 1.0;
#pragma unroll
      for (int k = 0; k < KP; ++k)
        if (k == i) own = w[k];
      const double rinv_own = row_ok ? 1.0 / sqrt(own) : 1.0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {   // Ls is the full 32 x 32 block (identity past KP)
        const double rinv = j < KP ? __shfl_sync(0xffffffffu, rinv_own, j) : 1.0;
        double x = 0.0;
        if (j < KP && j < K && row_ok && j < i) {
          x = w[j] * rinv;
          Tp[i * ldt + j] = x;
          Tp[j * ldt + i] = x;
        }
        Ls[i][j] = j == i ? rinv_own : x;
      }
      if (row_ok) Tp[i * ldt + i] = rinv_own;
      else if (i < ldt) Tp[i * ldt + i] = 1.0;   // unit diagonal of the padding
      PROBE_T(8);
      __syncwarp();
      block_inverse_smem<KP>(Ls, Tp + ldt * ldt);
      PROBE_T(9);
    }
    if (i == 0) {
      bad_s = bad ? 1 : 0;
      *mode = bad ? 1 : 0;
    }
  }
  __syncthreads();
  if (bad_s) gamma_pinv_dev(K, Gamma, Tp, ldt, Vscratch, tau);
}

// ---------------------------------------------------------------- row solves
// One warp per row, SR_WARPS rows per CTA (one CTA per SM: every row of a B200-sized mode runs
// at once).  The packed factor Tp (and Γ when it fits) arrive in shared memory by one bulk copy
// (cp.async.bulk + mbarrier) while the warps load their rows.  Lane c owns columns c + 32u.
//   Cholesky path (mode 0): forward L z = m, then back Lᵀ a = z, right-looking, one pivot per
//   step: z_j is broadcast by shuffle and every later column takes its fma (the oracle's
//   substitution, P:395 via L13).  pinv path (mode 1): a = m P.
//   Then G = (a_old - a_new) Γ, dA = a_new - ref, and the per-row statistics
//   rowstat[y] = (‖a_new‖², ‖dA‖², ‖g‖², Σ m∘a_new) for the norms and the fitness.
constexpr int SR_WARPS = 4;

__device__ __forceinline__ void bar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

// one bulk copy global -> shared, completing on `bar` (the caller arms it with bar_expect)
__device__ __forceinline__ void bulk_to_smem(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  }
}

__global__ void __launch_bounds__(SR_WARPS * 32, 1)
    solve_rows_kernel(const double* __restrict__ M, double* A, const double* ref, double* dA,
                      int64_t rows, int K, const double* __restrict__ Gamma,
                      const double* __restrict__ Tp, int ldt, int gamma_in_smem,
                      const int* __restrict__ mode_p, double* __restrict__ rowstat) {
  PROBE_T0();
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar;
  double* Ts = sm + 128;                                // ldt x ldt (+ 128 pad on each side)
  double* Qs = Ts + (int64_t)ldt * ldt + 256;           // 4 x 32 x 33 inverted diagonal blocks
  double* Gs = Qs + 4 * 32 * 33;                        // ldt x ldt (+ 128 pad), if staged
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t tbytes = static_cast<uint32_t>(ldt) * ldt * 8;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // Tp and Γ come from the factorization (a full, event dependency): stage them before the
    // programmatic wait on the kernel that produced M
    const uint32_t qbytes = static_cast<uint32_t>((ldt + 31) >> 5) * 32 * 33 * 8;
    bar_expect(&bar, (gamma_in_smem ? 2 * tbytes : tbytes) + qbytes);
    bulk_to_smem(Ts, Tp, tbytes, &bar);
    bulk_to_smem(Qs, Tp + (int64_t)ldt * ldt, qbytes, &bar);
    if (gamma_in_smem) bulk_to_smem(Gs, Gamma, tbytes, &bar);
  }
  __syncthreads();
  pdl_wait();
  const int64_t y = blockIdx.x * (int64_t)SR_WARPS + w;
  const bool valid = y < rows;
  double m[4], m0[4], aold[4], rf[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = lane + 32 * u;
    const bool in = valid && c < K;
    aold[u] = in ? A[y * K + c] : 0.0;
    rf[u] = in ? ref[y * K + c] : 0.0;
    m[u] = in ? M[y * K + c] : 0.0;
    m0[u] = m[u];
  }
  const int mode = *mode_p;
  bar_wait(&bar, 0);
  PROBE_T(2);
  // Tp / Γ are ldt x ldt (ldt = K rounded up to 8) with zero padding and a unit diagonal past K,
  // so every loop below runs ldt (a multiple of 8) steps: 8-step bodies with compile-time trip
  // counts; the padded steps change nothing (their m and factor entries are zero).
  const int kp = ldt;
  if (mode == 0) {
    // Blocked substitution with the inverted 32 x 32 diagonal blocks (Q, from the factorization):
    // forward L z = m block by block: z_u = inv(L_uu) m_u (32 independent shuffles and fmas,
    // two accumulators added in a fixed order), then the later blocks take -L[.][u] z_u
    // (rows of Tp's upper part, in ascending order).  Back Lᵀ a = z the same way, descending, with
    // inv(L_uu)ᵀ and the rows of Tp's lower part.  No per-pivot dependency chain.
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (32 * u >= kp) break;
      const double* Qu = Qs + u * 32 * 33;
      double z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int jj = 0; jj < 32; jj += 2) {
        z0 = fma(Qu[jj * 33 + lane], __shfl_sync(0xffffffffu, m[u], jj), z0);
        z1 = fma(Qu[(jj + 1) * 33 + lane], __shfl_sync(0xffffffffu, m[u], jj + 1), z1);
      }
      m[u] = z0 + z1;
      const int nb = min(32, kp - 32 * u);
      for (int j8 = 0; j8 < nb; j8 += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int jj = j8 + k;
          const double zj = __shfl_sync(0xffffffffu, m[u], jj);
          const double* tr = Ts + (32 * u + jj) * ldt + lane;
#pragma unroll
          for (int v = u + 1; v < 4; ++v) m[v] = fma(-tr[32 * v], zj, m[v]);
        }
      }
    }
#pragma unroll
    for (int u = 3; u >= 0; --u) {
      if (32 * u >= kp) continue;
      const double* Qu = Qs + u * 32 * 33 + lane * 33;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int jj = 0; jj < 32; jj += 2) {
        a0 = fma(Qu[jj], __shfl_sync(0xffffffffu, m[u], jj), a0);
        a1 = fma(Qu[jj + 1], __shfl_sync(0xffffffffu, m[u], jj + 1), a1);
      }
      m[u] = a0 + a1;
      const int nb = min(32, kp - 32 * u);
      for (int j8 = 0; j8 < nb; j8 += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int jj = j8 + k;
          const double aj = __shfl_sync(0xffffffffu, m[u], jj);
          const double* tr = Ts + (32 * u + jj) * ldt + lane;
#pragma unroll
          for (int v = 0; v < u; ++v) m[v] = fma(-tr[32 * v], aj, m[v]);
        }
      }
    }
  } else {
    double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (32 * u >= kp) break;
      const int nb = min(32, kp - 32 * u);
      for (int j8 = 0; j8 < nb; j8 += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int p = 32 * u + j8 + k;
          const double mp = __shfl_sync(0xffffffffu, m[u], j8 + k);
#pragma unroll
          for (int v = 0; v < 4; ++v) a[v] = fma(mp, Ts[p * ldt + 32 * v + lane], a[v]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) m[u] = a[u];
  }
  PROBE_T(3);
  // m now holds a_new (garbage in lanes c >= K)
  double d[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) d[u] = (lane + 32 * u < K) ? aold[u] - m[u] : 0.0;
  if (!gamma_in_smem) {   // K > 112: Γ replaces the factor in shared memory
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_expect(&bar, tbytes);
      bulk_to_smem(Ts, Gamma, tbytes, &bar);
    }
    bar_wait(&bar, 1);
  }
  const double* Gm = gamma_in_smem ? Gs : Ts;
  double g[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (32 * u >= kp) break;
    const int nb = min(32, kp - 32 * u);
    for (int j8 = 0; j8 < nb; j8 += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int p = 32 * u + j8 + k;
        const double dp = __shfl_sync(0xffffffffu, d[u], j8 + k);
#pragma unroll
        for (int v = 0; v < 4; ++v) g[v] = fma(dp, Gm[p * ldt + 32 * v + lane], g[v]);
      }
    }
  }
  double na = 0.0, nd = 0.0, ng = 0.0, in = 0.0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = lane + 32 * u;
    if (valid && c < K) {
      const double e = m[u] - rf[u];
      A[y * K + c] = m[u];
      dA[y * K + c] = e;
      na = fma(m[u], m[u], na);
      nd = fma(e, e, nd);
      ng = fma(g[u], g[u], ng);
      in = fma(m0[u], m[u], in);
    }
  }
  na = warp_sum(na);
  nd = warp_sum(nd);
  ng = warp_sum(ng);
  in = warp_sum(in);
  if (valid && lane == 0)
    *reinterpret_cast<double4*>(rowstat + y * 4) = make_double4(na, nd, ng, in);
  PROBE_T(4);
}

// ---------------------------------------------------------------- Gram S = AᵀA (+ statistics)
// CTA (tile pair t, split q): tile pair (ti <= tj) of S, rows [q R/ns, (q+1) R/ns) of A;
// thread (i, j) owns S[16ti+i][16tj+j] (and its mirror).  The two 16-column strips stream
// through shared memory GR_ROWS rows at a time: every thread issues its coalesced loads of the
// next chunk (all in flight) while the current chunk is consumed; rows are stored in pairs so
// one 16-byte load serves two rows; 4 accumulators (row mod 4) are combined in a fixed order.
// With ns > 1 the splits leave partial tiles and the last split to finish (per-tile ticket)
// sums them in split order.  With stats, the last tile to finish (global ticket) sums the
// per-row statistics in row order and the per-tile Σ Γ∘S partials in tile order
// (nrm[0..2] = Σ ‖a‖², ‖dA‖², ‖g‖²; fit[0] = Σ M∘A, fit[1] = 1ᵀ(Γ∗S)1).
// Every sum has a fixed order; the tickets only decide which CTA performs it.
constexpr int GR_ROWS = 128;
constexpr int GR_THREADS = 256;
constexpr int GR_LOADS = 2 * GR_ROWS * 16 / GR_THREADS;   // 16 per thread
constexpr size_t GR_SMEM = 2 * GR_ROWS * 16 * sizeof(double);   // 32 KiB
constexpr int GR_MAX_CTAS = 148;

__global__ void __launch_bounds__(GR_THREADS)
    gram_kernel(const double* __restrict__ A, int64_t rows, int K, int nsplit,
                double* __restrict__ S, const double* __restrict__ rowstat, double* nrm,
                const double* __restrict__ Gm, int ldt, double* fit, double* scratch,
                unsigned int* counters) {
  PROBE_T0();
  pdl_wait();
  extern __shared__ __align__(16) double gsm[];   // [2 strips][GR_ROWS / 2][16][2]
  __shared__ double sh[32];
  __shared__ int last_s;
  const int T = (K + 15) >> 4;
  const int ntiles = T * (T + 1) / 2;
  const int tile = blockIdx.x % ntiles, split = blockIdx.x / ntiles;
  int t = tile, ti = 0;   // tile pair -> (ti, tj), ti <= tj, row-major over the upper triangle
  while (t >= T - ti) {
    t -= T - ti;
    ++ti;
  }
  const int tj = ti + t;
  const int tid = threadIdx.x, i = tid >> 4, j = tid & 15;
  const int64_t rlo = rows * split / nsplit, rhi = rows * (split + 1) / nsplit;
  // loader: element e = tid + 256 q (q < GR_LOADS): strip = q >= GR_LOADS / 2,
  // row = (e >> 4) % GR_ROWS, column = e % 16  (a warp reads two 128-byte row segments)
  double pre[GR_LOADS];
  auto load = [&](int64_t r0) {
#pragma unroll
    for (int q = 0; q < GR_LOADS; ++q) {
      const int e = tid + GR_THREADS * q;
      const int strip = q >= GR_LOADS / 2;
      const int rr = (e >> 4) & (GR_ROWS - 1), cc = e & 15;
      const int col = 16 * (strip ? tj : ti) + cc;
      const int64_t r = r0 + rr;
      pre[q] = (r < rhi && col < K) ? __ldcg(A + r * K + col) : 0.0;
    }
  };
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (rlo < rhi) load(rlo);
  for (int64_t r0 = rlo; r0 < rhi; r0 += GR_ROWS) {
#pragma unroll
    for (int q = 0; q < GR_LOADS; ++q) {
      const int e = tid + GR_THREADS * q;
      const int strip = q >= GR_LOADS / 2;
      const int rr = (e >> 4) & (GR_ROWS - 1), cc = e & 15;
      gsm[strip * GR_ROWS * 16 + ((rr >> 1) * 16 + cc) * 2 + (rr & 1)] = pre[q];
    }
    __syncthreads();
    if (r0 + GR_ROWS < rhi) load(r0 + GR_ROWS);
    const int nr = static_cast<int>(rhi - r0 < GR_ROWS ? rhi - r0 : GR_ROWS);
    const double2* sa = reinterpret_cast<const double2*>(gsm);
    const double2* sb = reinterpret_cast<const double2*>(gsm + GR_ROWS * 16);
    for (int p = 0; p < (nr + 1) / 2; p += 2) {   // row pairs; rows past the end are zero
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double2 x = sa[(p + k) * 16 + i], y = sb[(p + k) * 16 + j];
        acc[2 * k] = fma(x.x, y.x, acc[2 * k]);
        acc[2 * k + 1] = fma(x.y, y.y, acc[2 * k + 1]);
      }
    }
    __syncthreads();
  }
  PROBE_T(5);
  double s = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  if (nsplit > 1) {   // partial tiles: the last split of this tile sums them in split order
    scratch[(int64_t)blockIdx.x * GR_THREADS + tid] = s;
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      last_s = atomicAdd(counters + tile, 1u) == static_cast<unsigned>(nsplit - 1);
    }
    __syncthreads();
    if (!last_s) return;
    __threadfence();
    s = 0.0;
    for (int q = 0; q < nsplit; ++q)
      s += __ldcg(scratch + (int64_t)(q * ntiles + tile) * GR_THREADS + tid);
    if (tid == 0) counters[tile] = 0u;
  }
  const int gi = 16 * ti + i, gj = 16 * tj + j;
  const bool ok = gi < K && gj < K;
  if (ok) {
    S[gi * K + gj] = s;
    S[gj * K + gi] = s;
  }
  if (nrm == nullptr) return;
  if (gridDim.x == 1) {
    // one CTA (K <= 16, rows <= GR_ROWS: C1): no tickets, and the row statistics and the Σ Γ∘S
    // term in one five-value block sum (the same per-value trees as below)
    __shared__ double sh5[5 * 32];
    double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t y = tid; y < rows; y += GR_THREADS) {
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] += __ldcg(rowstat + y * 4 + c);
    }
    if (Gm != nullptr && ok) v[4] = Gm[gi * ldt + gj] * s;
    block_sum_n<5>(v, sh5);
    if (tid == 0) {
      nrm[0] = v[0];
      nrm[1] = v[1];
      nrm[2] = v[2];
      if (Gm != nullptr) {
        fit[0] = v[3];
        fit[1] = 0.0 + v[4];   // the tile-order sum over one tile
      }
    }
    return;
  }
  double* tilepart = scratch + (int64_t)GR_MAX_CTAS * GR_THREADS;
  if (Gm != nullptr) {
    double v = ok ? Gm[gi * ldt + gj] * s : 0.0;
    if (ti != tj) v *= 2.0;   // the mirrored tile
    v = block_sum(v, sh);
    if (tid == 0) tilepart[tile] = v;
  }
  // last tile: fixed-order sums of the row statistics and of the tile partials
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    last_s = atomicAdd(counters + ntiles, 1u) == static_cast<unsigned>(ntiles - 1);
  }
  __syncthreads();
  if (!last_s) return;
  __threadfence();
  {   // the four row-statistic sums in one block reduction (block_sum's tree for each)
    __shared__ double sh4[4 * 32];
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t y = tid; y < rows; y += GR_THREADS) {
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] += __ldcg(rowstat + y * 4 + c);
    }
    block_sum_n<4>(v, sh4);
    if (tid == 0) {
      nrm[0] = v[0];
      nrm[1] = v[1];
      nrm[2] = v[2];
      if (Gm != nullptr) fit[0] = v[3];
    }
  }
  if (tid == 0) {
    if (Gm != nullptr) {
      double v = 0.0;
      for (int b = 0; b < ntiles; ++b) v += __ldcg(tilepart + b);
      fit[1] = v;
    }
    counters[ntiles] = 0u;
  }
}

// ---------------------------------------------------------------- one small mode, one launch
// K <= 32 and rows <= MS_MAX_ROWS (C1, C4, the paper's P6W / LAP shapes): the whole mode — Γ^(n)
// (P:364), its LDLᵀ factorization with the L13 pivot rule, the inverse of L, the row solves
// A_new = M Γ^†, G = (A_old − A_new) Γ, dA, S^(n) = A_newᵀ A_new, the
// norms and the S:177 fitness terms — in ONE CTA.  The three-kernel chain above spends most of a
// small mode's time in launch gaps and cross-stream hops (C4: a 30 µs factorization on the side
// stream, 2.6 µs event hops, 6 + 7 µs row / Gram kernels per mode).
//
// Every value is formed by the same IEEE operations in the same order as that chain
// (gamma_small_kernel -> solve_rows_kernel -> gram_kernel with one row split), so the two paths
// are bit-identical (tested); only the work is spread differently:
//   * factorization: warp i keeps row i of W, lane k column k (the one-warp kernel kept row i in
//     lane i).  Step j: row j (final after step j−1) is read from a double-buffered shared row,
//     W[i][j] by a shuffle inside warp i, and W[i][k] −= (W[i][j]·(1/d_j))·W[j][k] for i, k > j;
//     warp j+1 then publishes its row: one barrier per pivot, no per-pivot register sweep.
//   * inverse of L (block_inverse_smem's column recurrences): warp c runs column c, lane j keeps
//     y_j, so a step is one shuffle, one multiply and one fma instead of a 32-entry sweep.
//   * rows: warp w takes rows w, w + NW, …; the Gram and the statistics reductions replay
//     gram_kernel's 256-thread trees on warps 0-7.
// The pseudo-inverse fallback (failed pivot test) runs gamma_pinv_dev on the whole CTA; its
// Jacobi stopping test sums over the CTA's threads, so only that path may differ in rounding.
constexpr int MS_MAX_ROWS = 64;

template <int KP>
struct MsCfg {
  // warps: >= 8 (gram_kernel's 256-thread trees); K <= 32 keeps two rows of Γ per warp so the
  // CTA stays at 512 threads (128 registers a thread)
  static constexpr int NW = KP <= 8 ? 8 : 16;
  static constexpr int RW = KP / NW > 1 ? KP / NW : 1;       // rows of Γ per warp
};

// gram_kernel's block_sum over 256 threads (8 warps) replayed on warps 0-7 of a larger CTA;
// every thread must call it (barriers).  Result in all threads.
template <int NV>
__device__ __forceinline__ void sum256_n(double (&v)[NV], double* sh /* 32 NV */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < NV; ++c) v[c] = warp_sum(v[c]);
  __syncthreads();
  if (lane == 0 && w < 8) {
#pragma unroll
    for (int c = 0; c < NV; ++c) sh[32 * c + w] = v[c];
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int c = 0; c < NV; ++c) {
      double r = lane < 8 ? sh[32 * c + lane] : 0.0;
      r = warp_sum(r);
      if (lane == 0) sh[32 * c] = r;
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NV; ++c) v[c] = sh[32 * c];
  __syncthreads();
}

// warp_sum's xor butterfly for lane 0, replayed from the 32 lane values in shared memory:
// ((v_l + v_{l+16}) level by level down to one value (fadd commutes, so each level is exact)
__device__ __forceinline__ double butterfly32(const double* v) {
  double x[16];
#pragma unroll
  for (int l = 0; l < 16; ++l) x[l] = v[l] + v[l + 16];
#pragma unroll
  for (int o = 8; o > 0; o >>= 1)
#pragma unroll
    for (int l = 0; l < o; ++l) x[l] = x[l] + x[l + o];
  return x[0];
}

template <int KP>
__global__ void __launch_bounds__(MsCfg<KP>::NW * 32, 1)
    mode_small_kernel(const double* __restrict__ S_all, int N, int n, int K,
                      const double* __restrict__ M, double* A, const double* ref, double* dA,
                      int rows, double* Sn, double* nrm, double* fit, double* Gamma_g, double* P_g,
                      double* Vscratch, double tau) {
  constexpr int NW = MsCfg<KP>::NW, NT = NW * 32, RW = MsCfg<KP>::RW;
  PROBE_T0();
  // dynamic shared memory: [pinv overlay: K (K+1)] | M | A (old, then A_new in place) | ref
  // (unless ref == A) | z, then d | per-lane statistic terms [rows][4][32] | row statistics
  // [rows][4].  Row blocks are MS_MAX_ROWS x KP, zero past (rows, K): every loop below runs to
  // compile-time bounds without predicates (the zero terms are the ones solve_rows_kernel and
  // gram_kernel add too), and the rows are staged once (all loads in flight together).
  extern __shared__ __align__(16) double ms_dyn[];
  constexpr int RB = MS_MAX_ROWS * KP;
  double* Ms = ms_dyn + ((K * (K + 1) + 1) & ~1);
  double* Ao = Ms + RB;
  const bool ref_is_A = ref == A;
  double* Rf = ref_is_A ? Ao : Ao + RB;
  double* Zs = Ao + 2 * RB;
  double* Ps = Zs + RB;                     // [rows][4][32]
  double* rs = Ps + MS_MAX_ROWS * 128;      // [rows][4]
  __shared__ double Gs[32][33];   // Γ (zero past K)
  __shared__ double Ls[32][33];   // 1 / L[i][i] on the diagonal, L below it; identity past K
  __shared__ double Qs[32][33];   // Qs[c][j] = inv(L)[j][c] (pinv path: the pseudo-inverse)
  __shared__ double Ss[32][33];   // S^(n)
  __shared__ __align__(16) double Rb[2][32];
  __shared__ double rinv_s[32];
  __shared__ double red[7 * 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int ldt = (K + 7) & ~7;
  // Everything up to the factor's inverse reads only data of kernels two or more launches back
  // (the Grams, A^(n), the reference factor), so it runs BEFORE the programmatic wait: the
  // kernels that produce M^(n) trigger their dependents early (pdl_trigger) and this part
  // overlaps them.  Those reads go through L2 (ld.global.cg), M after the wait.

  // every load in flight at once: the N-1 Gram rows of Γ and the staged rows
  double sv[RW][CPPP_MAX_ORDER_ - 1];
#pragma unroll
  for (int t = 0; t < RW; ++t) {
    const int i = w * RW + t;
#pragma unroll
    for (int q = 0; q < CPPP_MAX_ORDER_ - 1; ++q) {
      const int m = q < n ? q : q + 1;   // ascending m != n
      sv[t][q] = (q < N - 1 && i < K && lane < K) ? __ldcg(S_all + (int64_t)m * K * K + i * K + lane) : 1.0;
    }
  }
  constexpr int LQ = RB / NT;
  double la[LQ], lr[LQ];
#pragma unroll
  for (int q = 0; q < LQ; ++q) {
    const int f = tid + q * NT, y = f / KP, c = f % KP;
    const bool in = y < rows && c < K;
    const int e = y * K + c;
    la[q] = in ? __ldcg(A + e) : 0.0;
    lr[q] = (in && !ref_is_A) ? __ldcg(ref + e) : 0.0;
  }
  // Γ^(n) = 1.0 · S^(m_0) · S^(m_1) · … (ascending m, as gamma_small_kernel); warp w keeps rows
  // w RW + t, lane k column k
  double g[RW];
  double dmax = 0.0;
#pragma unroll
  for (int t = 0; t < RW; ++t) {
    const int i = w * RW + t;
    g[t] = 0.0;
    if (i < K && lane < K) {
      double x = 1.0;
#pragma unroll
      for (int q = 0; q < CPPP_MAX_ORDER_ - 1; ++q)
        if (q < N - 1) x *= sv[t][q];
      g[t] = x;
    }
    Gs[i][lane] = g[t];
    if (i == lane && i < K) dmax = g[t];
  }
  for (int r = NW * RW + w; r < 32; r += NW) Gs[r][lane] = 0.0;
#pragma unroll
  for (int q = 0; q < LQ; ++q) {
    const int f = tid + q * NT;
    Ao[f] = la[q];
    if (!ref_is_A) Rf[f] = lr[q];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if (lane == 0) red[w] = dmax;
  if (w == 0) Rb[0][lane] = g[0];
  __syncthreads();
  double mx = 0.0;
  for (int q = 0; q < NW; ++q) mx = fmax(mx, red[q]);
  const double thresh = tau * mx;
  PROBE_T(10);

  // LDLᵀ, right-looking, one pivot per barrier (the one-warp kernel's operations element by
  // element: cl = W[i][j]·(1/d_j), W[i][k] = fma(−cl, W[j][k], W[i][k]) for i, k > j)
  bool bad = false;
  for (int j = 0; j < K; ++j) {
    const double d = Rb[j & 1][j];
    const double rjk = Rb[j & 1][lane];
    if (!(d > thresh)) bad = true;
    const double rd = pivot_rcp(d);
#pragma unroll
    for (int t = 0; t < RW; ++t) {
      const int i = w * RW + t;
      const double wij = __shfl_sync(0xffffffffu, g[t], j);
      const double cl = wij * rd;
      if (i < K && lane < K && i > j && lane > j) g[t] = fma(-cl, rjk, g[t]);
      if (i == j + 1) Rb[(j + 1) & 1][lane] = g[t];
    }
    __syncthreads();
  }
  PROBE_T(11);

  // L[i][j] = W[i][j] / sqrt(d_j) (d_j = W[j][j], untouched after step j); formed and inverted
  // whether or not the pivot test passed (a failed test replaces the result below)
#pragma unroll
  for (int t = 0; t < RW; ++t) {
    const int i = w * RW + t;
    if (i == lane && i < K) rinv_s[i] = 1.0 / sqrt(g[t]);
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < RW; ++t) {
    const int r = w * RW + t;
    double v;
    if (r == lane) v = r < K ? rinv_s[r] : 1.0;
    else v = (r < K && lane < K && lane < r) ? g[t] * rinv_s[lane] : 0.0;
    Ls[r][lane] = v;
  }
  for (int r = NW * RW + w; r < 32; r += NW) Ls[r][lane] = r == lane ? 1.0 : 0.0;
  __syncthreads();
  if (w == 0) {   // inv(L): block_inverse_smem<KP>'s recurrences, lane c = column c (no shuffles)
    const int c = lane;
    double y[KP];
#pragma unroll
    for (int j = 0; j < KP; ++j) y[j] = 0.0;
#pragma unroll
    for (int i = 0; i < KP; ++i) {
      const double dinv = Ls[i][i];
      y[i] = i == c ? dinv : (i > c ? -y[i] * dinv : 0.0);
#pragma unroll
      for (int j = i + 1; j < KP; ++j) y[j] = fma(Ls[j][i], y[i], y[j]);
    }
#pragma unroll
    for (int j = 0; j < KP; ++j) Qs[c][j] = y[j];
  }
  if (bad) {   // CTA-uniform (every thread tested the same pivots)
    // pseudo-inverse fallback (L13): Γ to global, gamma_pinv_dev on the whole CTA, P into Qs
    __syncthreads();
    for (int e = tid; e < K * ldt; e += NT) {
      const int i = e / ldt, j = e - i * ldt;
      Gamma_g[e] = j < K ? Gs[i][j] : 0.0;
    }
    __syncthreads();
    gamma_pinv_dev(K, Gamma_g, P_g, ldt, Vscratch, tau);
    __syncthreads();
    for (int r = w; r < 32; r += NW) Qs[r][lane] = (r < K && lane < K) ? P_g[r * ldt + lane] : 0.0;
  }
  pdl_wait();   // M^(n) comes from the kernel right before this one
#pragma unroll
  for (int q = 0; q < LQ; ++q) {
    const int f = tid + q * NT, y = f / KP, c = f % KP;
    Ms[f] = (y < rows && c < K) ? __ldcg(M + y * K + c) : 0.0;
  }
  __syncthreads();
  PROBE_T(12);

  // rows: warp w takes rows w, w + NW, …, lane c = column c (solve_rows_kernel's arithmetic).
  // The vector operand comes from shared memory (broadcast), the matrix operand from registers.
  // No shuffles (the sums are replayed below).
  //   pass 1: z = inv(L) m (even / odd accumulators)      [pinv: a = P m, one accumulator]
  //   pass 2: a = inv(L)ᵀ z; d = a_old − a, dA, A; the lane terms of ‖a‖², ‖dA‖², Σ m∘a
  //   pass 3: g = d Γ; the lane terms of ‖g‖²
  const int c = lane < KP ? lane : 0;
  {
    double qv[KP];
#pragma unroll
    for (int jj = 0; jj < KP; ++jj) qv[jj] = Qs[jj][lane];
    for (int y = w; y < MS_MAX_ROWS; y += NW) {
      const double* mrow = Ms + y * KP;
      double z;
      if (!bad) {
        double z0 = 0.0, z1 = 0.0;
#pragma unroll
        for (int jj = 0; jj < KP; jj += 2) {
          z0 = fma(qv[jj], mrow[jj], z0);
          z1 = fma(qv[jj + 1], mrow[jj + 1], z1);
        }
        z = z0 + z1;
      } else {
        double a = 0.0;
#pragma unroll
        for (int jj = 0; jj < KP; ++jj) a = fma(mrow[jj], qv[jj], a);
        z = a;
      }
      if (lane < KP) Zs[y * KP + lane] = lane < K ? z : 0.0;
      if (y + NW >= rows) break;
    }
  }
  __syncwarp();
  PROBE_T(1);
  {
    double qv[KP];
#pragma unroll
    for (int jj = 0; jj < KP; ++jj) qv[jj] = Qs[lane][jj];
    for (int y = w; y < MS_MAX_ROWS; y += NW) {
      const double* zrow = Zs + y * KP;
      double m;
      if (!bad) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int jj = 0; jj < KP; jj += 2) {
          a0 = fma(qv[jj], zrow[jj], a0);
          a1 = fma(qv[jj + 1], zrow[jj + 1], a1);
        }
        m = a0 + a1;
      } else {
        m = zrow[c];
      }
      const int f = y * KP + c;
      const bool in = y < rows && lane < K;
      const double aold = Ao[f], rf = Rf[f], m0 = Ms[f];
      __syncwarp();   // every lane has read row y of z before it is overwritten with d
      const double ev = m - rf;
      double na = 0.0, nd = 0.0, ip = 0.0;
      if (in) {
        const int e = y * K + lane;
        A[e] = m;
        dA[e] = ev;
        na = fma(m, m, na);
        nd = fma(ev, ev, nd);
        ip = fma(m0, m, ip);
      }
      if (lane < KP) {
        Ao[f] = in ? m : 0.0;            // A_new for the Gram (ref, when it aliases A, was read above)
        Zs[f] = in ? aold - m : 0.0;     // d for pass 3
      }
      Ps[y * 128 + 0 * 32 + lane] = na;
      Ps[y * 128 + 1 * 32 + lane] = nd;
      Ps[y * 128 + 3 * 32 + lane] = ip;
      if (y + NW >= rows) break;
    }
  }
  __syncwarp();
  PROBE_T(2);
  {
    double gv[KP];
#pragma unroll
    for (int p = 0; p < KP; ++p) gv[p] = Gs[p][lane];
    for (int y = w; y < MS_MAX_ROWS; y += NW) {
      const double* drow = Zs + y * KP;
      double gg = 0.0;
#pragma unroll
      for (int p = 0; p < KP; ++p) gg = fma(drow[p], gv[p], gg);
      Ps[y * 128 + 2 * 32 + lane] = lane < K ? fma(gg, gg, 0.0) : 0.0;
      if (y + NW >= rows) break;
    }
  }
  __syncthreads();
  // the per-row sums, warp_sum's tree (thread = (row, statistic))
  for (int e = tid; e < rows * 4; e += NT) rs[e] = butterfly32(Ps + e * 32);
  __syncthreads();
  PROBE_T(13);

  // S^(n) = A_newᵀ A_new (gram_kernel: 4 accumulators by row mod 4, rows in ascending order,
  // zero rows up to the row-pair loop's multiple of 4, (acc0 + acc1) + (acc2 + acc3))
  const int r4 = 4 * (((rows + 1) / 2 + 1) / 2);
  for (int e = tid; e < KP * KP; e += NT) {
    const int a = e / KP, b = e - a * KP;
    if (a > b || b >= K) continue;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r = 0; r < r4; r += 4) {   // rows past `rows` are zero in Ao
#pragma unroll
      for (int t = 0; t < 4; ++t) acc[t] = fma(Ao[(r + t) * KP + a], Ao[(r + t) * KP + b], acc[t]);
    }
    const double s = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    Ss[a][b] = s;
    Ss[b][a] = s;
    Sn[a * K + b] = s;
    Sn[b * K + a] = s;
  }
  if (nrm == nullptr) return;
  __syncthreads();
  PROBE_T(14);
  // gram_kernel's statistics, every sum with its 256-thread tree: the row sums (0.0 + one row per
  // virtual thread t < 256, rows <= 64) and, for the last mode, Σ Γ∘S by 16 x 16 tiles (thread
  // t = (i, j) = (t >> 4, t & 15); the mirrored tile counted twice), all in one reduction
  const int T = (K + 15) >> 4;
  double v[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (tid < 256) {
    if (tid < rows) {
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] += rs[4 * tid + c];
    }
    if (fit != nullptr) {
#pragma unroll
      for (int tile = 0; tile < 3; ++tile) {   // T <= 2: tile pairs (0,0), (0,1), (1,1)
        const int ti = tile == 2 ? 1 : 0, tj = tile == 0 ? 0 : 1;
        if (tj < T) {
          const int gi = 16 * ti + (tid >> 4), gj = 16 * tj + (tid & 15);
          double x = (gi < K && gj < K) ? Gs[gi][gj] * Ss[gi][gj] : 0.0;
          if (ti != tj) x *= 2.0;
          v[4 + tile] = x;
        }
      }
    }
  }
  sum256_n<7>(v, red);
  if (tid == 0) {
    nrm[0] = v[0];
    nrm[1] = v[1];
    nrm[2] = v[2];
    if (fit != nullptr) {
      fit[0] = v[3];
      double f = 0.0 + v[4];   // T == 1: 0.0 + the one tile, as gram_kernel's single-CTA path
      if (T == 2) f = (f + v[5]) + v[6];
      fit[1] = f;
    }
  }
  PROBE_T(15);
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

__global__ void add_kernel(const double* x, double* y, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    y[e] = y[e] + x[e];
}

__global__ void pad_rows_kernel(const double* F, int64_t S, int K, double* Fp, int ld) {
  pdl_wait();
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

static thread_local bool t_pdl_suppressed = false;
void pdl_suppress(bool on) { t_pdl_suppressed = on; }
bool pdl_enabled() {
  static const bool on = getenv("CPPP_NO_PDL") == nullptr;
  return on && !t_pdl_suppressed;
}

static unsigned long long g_launches = 0;
void note_launch() { __atomic_add_fetch(&g_launches, 1ull, __ATOMIC_RELAXED); }
void note_launches(uint64_t n) { __atomic_add_fetch(&g_launches, n, __ATOMIC_RELAXED); }
uint64_t launch_count() { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int solve_ld(int K) { return (K + 7) & ~7; }

cudaError_t launch_gamma_factor(const double* S_all, int N, int n, int K, double* Gamma, double* Tp,
                                int* mode, double* Vscratch, cudaStream_t st, double tau) {
  const int ldt = solve_ld(K);
  const size_t smem = static_cast<size_t>(K) * (K + 1) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gamma_post_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 129 * 8);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  static const bool no_small = getenv("CPPP_NO_SMALL_FACTOR") != nullptr;   // A/B
  if (K <= 32 && !no_small) {
    static bool small_attr = false;
    if (!small_attr) {
      for (auto f : {gamma_small_kernel<8>, gamma_small_kernel<16>, gamma_small_kernel<32>}) {
        cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 33 * 8);
        if (e != cudaSuccess) return e;
      }
      small_attr = true;
    }
    auto f = K <= 8 ? gamma_small_kernel<8> : K <= 16 ? gamma_small_kernel<16> : gamma_small_kernel<32>;
    cudaError_t e = launch_pdl(f, dim3(1), dim3(GS_THREADS), smem, st, S_all, N, n, K, Gamma, Tp, ldt,
                               mode, Vscratch, tau);
    note_launch();
    return e;
  }
  // K > 48: the mirrored halves of Γ and of the factor go out through shared-memory transposes
  // (coalesced rows); for small K the direct column stores are cheaper than the extra shared
  // memory (C1's K = 10 lost 3% to it; the opt-in attribute is only set once a large K needs it)
  constexpr size_t chol_smem = sizeof(double) * (GF_THREADS / 32) * 16 * 33;   // mirror transposes
  const bool transpose = K > 48;
  static bool chol_attr = false;
  if (transpose && !chol_attr) {
    cudaError_t e = cudaFuncSetAttribute(gamma_chol_kernel<true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chol_smem);
    if (e != cudaSuccess) return e;
    chol_attr = true;
  }
  cudaError_t e = transpose
                      ? launch_pdl(gamma_chol_kernel<true>, dim3(1), dim3(GF_THREADS), chol_smem, st,
                                   S_all, N, n, K, Gamma, Tp, ldt, mode, tau)
                      : launch_pdl(gamma_chol_kernel<false>, dim3(1), dim3(GF_THREADS), 0, st, S_all,
                                   N, n, K, Gamma, Tp, ldt, mode, tau);
  note_launch();
  if (e != cudaSuccess) return e;
  e = launch_pdl(gamma_post_kernel, dim3(1), dim3(GP_THREADS), smem, st, K,
                 static_cast<const double*>(Gamma), Tp, ldt, static_cast<const int*>(mode), Vscratch, tau);
  note_launch();
  return e;
}

cudaError_t launch_solve_rows(const double* M, double* A, const double* ref, double* dA,
                              int64_t rows, int K, const double* Gamma, const double* Tp,
                              const int* mode, double* rowstat, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  const int ldt = solve_ld(K);
  const size_t one = static_cast<size_t>(ldt) * ldt * sizeof(double);
  // layout: 128 pad | Tp | 256 pad | Q (4 x 32 x 33) | Γ | 128 pad
  const size_t qb = 4 * 32 * 33 * sizeof(double);
  const bool both = 2 * one + qb + 512 * sizeof(double) <= 220 * 1024;   // Γ staged too
  const size_t smem = (both ? 2 * one : one) + qb + 512 * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(solve_rows_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         220 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t blocks = (rows + SR_WARPS - 1) / SR_WARPS;
  cudaError_t e = launch_pdl(solve_rows_kernel, dim3((unsigned)blocks), dim3(SR_WARPS * 32), smem,
                             st, M, A, ref, dA, rows, K, Gamma, Tp, ldt, both ? 1 : 0, mode, rowstat);
  note_launch();
  return e;
}

bool mode_small_ok(int K, int64_t rows) { return K >= 1 && K <= 32 && rows >= 1 && rows <= MS_MAX_ROWS; }

cudaError_t launch_mode_small(const double* S_all, int N, int n, int K, const double* M, double* A,
                              const double* ref, double* dA, int64_t rows, double* Sn, double* nrm,
                              double* fit, double* Gamma, double* Tp, double* Vscratch,
                              cudaStream_t st, double tau) {
  if (!mode_small_ok(K, rows)) return cudaErrorInvalidValue;
  // [pinv overlay | M | A | ref | z/d | lane terms | row statistics] (mode_small_kernel)
  const int KP = K <= 8 ? 8 : K <= 16 ? 16 : 32;
  const size_t smem = sizeof(double) * ((((int64_t)K * (K + 1) + 1) & ~1) + 4 * MS_MAX_ROWS * KP + 132 * MS_MAX_ROWS);
  const size_t smem_max = sizeof(double) * (32 * 33 + 4 * MS_MAX_ROWS * 32 + 132 * MS_MAX_ROWS);
  static bool attr = false;
  if (!attr) {
    for (auto f : {mode_small_kernel<8>, mode_small_kernel<16>, mode_small_kernel<32>}) {
      cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
      if (e != cudaSuccess) return e;
    }
    attr = true;
  }
  cudaError_t e;
  if (K <= 8)
    e = launch_pdl(mode_small_kernel<8>, dim3(1), dim3(MsCfg<8>::NW * 32), smem, st, S_all, N, n, K, M, A,
                   ref, dA, (int)rows, Sn, nrm, fit, Gamma, Tp, Vscratch, tau);
  else if (K <= 16)
    e = launch_pdl(mode_small_kernel<16>, dim3(1), dim3(MsCfg<16>::NW * 32), smem, st, S_all, N, n, K, M,
                   A, ref, dA, (int)rows, Sn, nrm, fit, Gamma, Tp, Vscratch, tau);
  else
    e = launch_pdl(mode_small_kernel<32>, dim3(1), dim3(MsCfg<32>::NW * 32), smem, st, S_all, N, n, K, M,
                   A, ref, dA, (int)rows, Sn, nrm, fit, Gamma, Tp, Vscratch, tau);
  note_launch();
  return e;
}

int gram_tiles(int K) {
  const int T = (K + 15) / 16;
  return T * (T + 1) / 2;
}

size_t gram_scratch_doubles() { return (size_t)GR_MAX_CTAS * GR_THREADS + 64; }

cudaError_t launch_gram(const double* A, int64_t rows, int K, double* S, const double* rowstat,
                        double* nrm, const double* Gamma_model, double* fit, double* scratch,
                        unsigned int* counters, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(GR_SMEM));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int nt = gram_tiles(K);
  int64_t ns = (rows + GR_ROWS - 1) / GR_ROWS;
  const int64_t cap = GR_MAX_CTAS / nt;
  if (ns > cap) ns = cap;
  if (ns < 1) ns = 1;
  cudaError_t e = launch_pdl(gram_kernel, dim3((unsigned)(nt * ns)), dim3(GR_THREADS), GR_SMEM, st,
                             A, rows, K, (int)ns, S, rowstat, nrm, Gamma_model, solve_ld(K), fit,
                             scratch, counters);
  note_launch();
  return e;
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

__global__ void stagger_kernel(unsigned ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

cudaError_t launch_stagger(cudaStream_t st) {
  stagger_kernel<<<1, 32, 0, st>>>(3000u);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_sub(const double* a, const double* b, double* y, int64_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  sub_kernel<<<grid_for(n, 256, 1184), 256, 0, st>>>(a, b, y, n);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_add(const double* x, double* y, int64_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  add_kernel<<<grid_for(n, 256, 1184), 256, 0, st>>>(x, y, n);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pad_rows(const double* F, int64_t S, int K, double* Fp, int ld,
                            cudaStream_t st) {
  cudaError_t e = launch_pdl(pad_rows_kernel, dim3(grid_for(S * ld, 256, 1184)), dim3(256), 0, st,
                             F, S, K, Fp, ld);
  note_launch();
  return e;
}

}  // namespace cppp
