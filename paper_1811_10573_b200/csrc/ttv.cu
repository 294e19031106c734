// ttv.cu — multi-TTV: the rank-diagonal contraction of one mode of a partially contracted
// intermediate (PAPER.md Tree_Map_PP P:88-91: M(:,k) = M_parent(:,k) ×_i A^(i)(:,k)), used by the
// lower levels of the regular dimension tree and by the PP construction tree (Def. pptree).
//
//   out[b][r][k] = Σ_x P[b][x][r][k] · F[x][k]        parent viewed as [B][S][R][K], k last
//
// HBM-bound (2 flops per 8-byte parent element).  Each output element is owned by one thread,
// which walks x in ascending order (deterministic, no atomics); consecutive threads own
// consecutive (r, k) so every x step is a coalesced row read of the parent.
//
// The fused variant emits all children of one parent in ONE pass over the parent (the
// per-parent fan-out of Def. pptree is 3/2/1 at level 2): a CTA owns a [S0 x ... x S_{m-1}]
// block of one (b, tail, k) fibre set in shared memory and reduces it along each axis.
#include "internal.h"

namespace cppp {
namespace {

template <int U>
__global__ void ttv_kernel(const double* __restrict__ P, int64_t B, int64_t S, int64_t RK, int K,
                           const double* __restrict__ F, double* __restrict__ out) {
  const int64_t total = B * RK;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / RK;
    const int64_t rk = e - b * RK;
    const int k = static_cast<int>(rk % K);
    const double* p = P + b * S * RK + rk;
    const double* f = F + k;
    double acc = 0.0;
    int64_t x = 0;
    for (; x + U <= S; x += U) {
      double pv[U], fv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        pv[u] = __ldg(p + (x + u) * RK);
        fv[u] = __ldg(f + (x + u) * K);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc = fma(pv[u], fv[u], acc);
    }
    for (; x < S; ++x) acc = fma(__ldg(p + x * RK), __ldg(f + x * K), acc);
    out[e] = acc;
  }
}

// Small outputs (the lower tree levels of an order-3 tensor: s²K -> sK): split the x range
// over `xsplit` independent partial sums, then add them in a fixed order.
__global__ void ttv_split_kernel(const double* __restrict__ P, int64_t S, int64_t RK, int K,
                                 int64_t total, int xsplit, const double* __restrict__ F,
                                 double* __restrict__ part) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int p = blockIdx.y;
  if (e >= total) return;
  const int64_t b = e / RK;
  const int64_t rk = e - b * RK;
  const int k = static_cast<int>(rk % K);
  const int64_t x0 = S * p / xsplit, x1 = S * (p + 1) / xsplit;
  const double* pp = P + b * S * RK + rk;
  const double* f = F + k;
  double acc = 0.0;
  int64_t x = x0;
  for (; x + 4 <= x1; x += 4) {
    const double p0 = __ldcs(pp + x * RK), p1 = __ldcs(pp + (x + 1) * RK);
    const double p2 = __ldcs(pp + (x + 2) * RK), p3 = __ldcs(pp + (x + 3) * RK);
    acc = fma(p0, __ldg(f + x * K), acc);
    acc = fma(p1, __ldg(f + (x + 1) * K), acc);
    acc = fma(p2, __ldg(f + (x + 2) * K), acc);
    acc = fma(p3, __ldg(f + (x + 3) * K), acc);
  }
  for (; x < x1; ++x) acc = fma(__ldcs(pp + x * RK), __ldg(f + x * K), acc);
  part[p * total + e] = acc;
}

__global__ void ttv_combine_kernel(const double* __restrict__ part, int64_t total, int xsplit,
                                   double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < xsplit; ++p) s += part[p * total + e];
    out[e] = s;
  }
}

}  // namespace

size_t ttv_scratch_doubles() { return static_cast<size_t>(148) * 2048 * 16; }

cudaError_t launch_ttv(const double* P, int64_t B, int64_t S, int64_t R, int K, const double* F,
                       double* out, double* scratch, cudaStream_t st) {
  const int64_t RK = R * K;
  const int64_t total = B * RK;
  if (total == 0) return cudaSuccess;
  const int64_t target = 148LL * 2048;
  if (scratch != nullptr && total < target && S >= 32) {
    int64_t xs = (target + total - 1) / total;
    xs = xs > S / 8 ? S / 8 : xs;
    xs = xs > 64 ? 64 : xs;
    const int64_t cap = static_cast<int64_t>(ttv_scratch_doubles()) / total;
    xs = xs > cap ? cap : xs;
    if (xs >= 2) {
      dim3 grid((unsigned)((total + 255) / 256), (unsigned)xs);
      ttv_split_kernel<<<grid, 256, 0, st>>>(P, S, RK, K, total, (int)xs, F, scratch);
      note_launch();
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      int blocks = (int)((total + 255) / 256);
      ttv_combine_kernel<<<blocks, 256, 0, st>>>(scratch, total, (int)xs, out);
      note_launch();
      return cudaGetLastError();
    }
  }
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = 148LL * 16;
  if (blocks > cap) blocks = cap;
  ttv_kernel<8><<<(unsigned)blocks, 256, 0, st>>>(P, B, S, RK, K, F, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_ttv_multi(const TtvMulti& p, cudaStream_t st) {
  // Generic path: one pass per child.  Child c contracts middle axis c of
  // [B][S0]..[S_{m-1}][T][K]: view as [B*prod(S_<c)][S_c][prod(S_>c)*T][K].
  for (int c = 0; c < p.m; ++c) {
    int64_t Bc = p.B, Rc = p.T;
    for (int a = 0; a < c; ++a) Bc *= p.S[a];
    for (int a = c + 1; a < p.m; ++a) Rc *= p.S[a];
    cudaError_t e = launch_ttv(p.P, Bc, p.S[c], Rc, p.K, p.F[c], p.out[c], nullptr, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace cppp
