// ttv.cu — multi-TTV: the rank-diagonal contraction of one mode of a partially contracted
// intermediate (PAPER.md Tree_Map_PP P:88-91: M(:,k) = M_parent(:,k) ×_i A^(i)(:,k)), used by the
// lower levels of the regular dimension tree and by the PP construction tree (Def. pptree).
//
//   out[b][r][k] = Σ_x P[b][x][r][k] · F[x][k]        parent viewed as [B][S][R][K], k last
//
// HBM-bound (2 flops per 8-byte parent element).  Each output element is owned by one thread,
// which walks its x range in ascending order (deterministic, no atomics); consecutive threads own
// consecutive (r, k) so every x step is a coalesced row read of the parent.
//
// Every child of a tree node is its own pass over the parent (a one-pass variant for all the
// children of a parent was analysed and not built: the children reduce along different axes, so
// a one-pass kernel needs partial outputs per block along each axis — DESIGN.md §11).
#include "internal.h"

#include <cstdio>
#include <cstdlib>

namespace cppp {
namespace {

// One kernel for every shape.  Thread = V consecutive outputs (V = 2: 16-byte loads of the
// parent and the factor when K is even); blockIdx.y = x-split index p of XS (gridDim.y) equal
// ranges.  XS > 1 launches (1, XS, 1) thread-block clusters: the XS partial sums of an output
// block meet in CTA rank 0's shared memory over DSMEM and are added in rank order
// (deterministic, no second kernel).  Loads are issued UNROLL x-steps ahead.
constexpr int TTV_THREADS = 256;

template <int V>
struct Vec;
template <>
struct Vec<1> {
  using T = double;
  static __device__ __forceinline__ T ld_stream(const double* p) { return __ldcs(p); }
  static __device__ __forceinline__ T ld(const double* p) { return __ldg(p); }
};
template <>
struct Vec<2> {
  using T = double2;
  static __device__ __forceinline__ T ld_stream(const double* p) {
    return __ldcs(reinterpret_cast<const double2*>(p));
  }
  static __device__ __forceinline__ T ld(const double* p) {
    return __ldg(reinterpret_cast<const double2*>(p));
  }
};
__device__ __forceinline__ void vfma(double& acc, double p, double f) { acc = fma(p, f, acc); }
__device__ __forceinline__ void vfma(double2& acc, double2 p, double2 f) {
  acc.x = fma(p.x, f.x, acc.x);
  acc.y = fma(p.y, f.y, acc.y);
}
__device__ __forceinline__ void vadd(double& a, double b) { a += b; }
__device__ __forceinline__ void vadd(double2& a, double2 b) {
  a.x += b.x;
  a.y += b.y;
}

template <int V, int TTV_UNROLL>
__global__ void __launch_bounds__(TTV_THREADS)
    ttv_kernel(const double* __restrict__ P, int64_t S, int64_t RK, int K, int64_t nvec,
               const double* __restrict__ F, double* __restrict__ out) {
  using T = typename Vec<V>::T;
  pdl_wait();
  __shared__ T red[TTV_THREADS];
  const int64_t e = blockIdx.x * (int64_t)TTV_THREADS + threadIdx.x;   // vector index
  const int p = blockIdx.y, xs = gridDim.y;
  T acc;
  if constexpr (V == 1) acc = 0.0;
  else acc = make_double2(0.0, 0.0);
  if (e < nvec) {
    const int64_t o = e * V;            // first output element
    const int64_t b = o / RK;
    const int64_t rk = o - b * RK;
    const int k = static_cast<int>(rk % K);
    const int64_t x0 = S * p / xs, x1 = S * (p + 1) / xs;
    const double* pp = P + b * S * RK + rk;
    const double* f = F + k;
    int64_t x = x0;
    for (; x + TTV_UNROLL <= x1; x += TTV_UNROLL) {
      T pv[TTV_UNROLL], fv[TTV_UNROLL];
#pragma unroll
      for (int u = 0; u < TTV_UNROLL; ++u) {
        pv[u] = Vec<V>::ld_stream(pp + (x + u) * RK);
        fv[u] = Vec<V>::ld(f + (x + u) * K);
      }
#pragma unroll
      for (int u = 0; u < TTV_UNROLL; ++u) vfma(acc, pv[u], fv[u]);
    }
    for (; x < x1; ++x) vfma(acc, Vec<V>::ld_stream(pp + x * RK), Vec<V>::ld(f + x * K));
  }
  if (xs == 1) {
    if (e < nvec) *reinterpret_cast<T*>(out + e * V) = acc;
    return;
  }
  // cluster reduction: rank r = p (cluster dims (1, xs, 1)); rank 0 adds ranks 0..xs-1 in order
  red[threadIdx.x] = acc;
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (p == 0 && e < nvec) {
    T s = acc;
    const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(&red[threadIdx.x]));
    for (int r = 1; r < xs; ++r) {
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(r));
      T v;
      if constexpr (V == 1) {
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote));
      } else {
        asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(remote));
      }
      vadd(s, v);
    }
    *reinterpret_cast<T*>(out + e * V) = s;
  }
  // keep every CTA's shared memory alive until rank 0 has read it
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int V, int U>
cudaError_t launch_v(const double* P, int64_t S, int64_t RK, int K, int64_t total, int xs,
                     const double* F, double* out, cudaStream_t st) {
  static bool attr_done = false;
  if (!attr_done) {   // clusters of up to 16 CTAs along the split axis
    cudaError_t e = cudaFuncSetAttribute(ttv_kernel<V, U>,
                                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const int64_t nvec = total / V;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((nvec + TTV_THREADS - 1) / TTV_THREADS), (unsigned)xs, 1);
  cfg.blockDim = dim3(TTV_THREADS, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = (unsigned)xs;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // see launch_pdl
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, ttv_kernel<V, U>, P, S, RK, K, nvec, F, out);
  note_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

size_t ttv_scratch_doubles() { return 0; }

// explicit configuration (tools/probe_ttv sweeps these): V outputs per thread (1, or 2 for even
// K), U x-steps in flight, xs x-splits (cluster size, <= 16)
cudaError_t launch_ttv_cfg(const double* P, int64_t B, int64_t S, int64_t R, int K,
                           const double* F, double* out, int V, int U, int xs, cudaStream_t st) {
  const int64_t RK = R * K, total = B * RK;
  if (total == 0) return cudaSuccess;
  if (V == 2 && U == 4) return launch_v<2, 4>(P, S, RK, K, total, xs, F, out, st);
  if (V == 2 && U == 8) return launch_v<2, 8>(P, S, RK, K, total, xs, F, out, st);
  if (V == 1 && U == 4) return launch_v<1, 4>(P, S, RK, K, total, xs, F, out, st);
  return launch_v<1, 8>(P, S, RK, K, total, xs, F, out, st);
}

cudaError_t launch_ttv(const double* P, int64_t B, int64_t S, int64_t R, int K, const double* F,
                       double* out, double* /*scratch*/, cudaStream_t st) {
  const int64_t RK = R * K;
  const int64_t total = B * RK;
  if (total == 0) return cudaSuccess;
  const bool v2 = (K % 2 == 0) && ((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(F) |
                                    reinterpret_cast<uintptr_t>(out)) % 16 == 0);
  const int V = v2 ? 2 : 1;
  // split x only when the outputs alone give fewer than ~2 CTAs per SM (tools/probe_ttv: larger
  // clusters and more splits lose to the cluster barriers; C2 level 2 -> xs = 4)
  const int64_t ctas = (total / V + TTV_THREADS - 1) / TTV_THREADS;
  int xs = 1;
  while (xs < 8 && ctas * xs < 148LL * 2 && S / (2 * xs) >= 16) xs *= 2;
  static const bool dbg = getenv("CPPP_DEBUG_TTM") != nullptr;
  if (dbg)
    fprintf(stderr, "ttv B %lld S %lld R %lld K %d: V %d xs %d\n", (long long)B, (long long)S,
            (long long)R, K, V, xs);
  return launch_ttv_cfg(P, B, S, R, K, F, out, V, 4, xs, st);
}

}  // namespace cppp
