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

}  // namespace

cudaError_t launch_ttv(const double* P, int64_t B, int64_t S, int64_t R, int K, const double* F,
                       double* out, cudaStream_t st) {
  const int64_t RK = R * K;
  const int64_t total = B * RK;
  if (total == 0) return cudaSuccess;
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
    cudaError_t e = launch_ttv(p.P, Bc, p.S[c], Rc, p.K, p.F[c], p.out[c], st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace cppp
