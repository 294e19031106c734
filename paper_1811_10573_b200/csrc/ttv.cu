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
// Kernels: ttv_pipe_kernel (16-byte pairs, software-pipelined x loop) and ttv_kernel (odd K)
// for single contractions; ttv_batch_kernel (one launch per construction-tree level) and
// ttv_pair_kernel (two children of one parent that contract adjacent kept modes, one pass over
// the parent) for the batched jobs below.
#include "internal.h"

#include <cstdio>
#include <cstdlib>
#include <vector>

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
  pdl_trigger();
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

// The same contraction for 16-byte pairs, software-pipelined: the next U x-steps' loads are
// issued before the current ones are consumed, in 128-thread CTAs (so every CTA of an x split
// stays resident).  Each output is still ONE fma chain in ascending x (steps past the range load
// a valid row and multiply it by 0), the ranks' sums added in rank order: bit-identical to
// ttv_kernel<2, U> with the same split.  tools/probe_ttv2.cu, L2 flushed: C2's two level-2
// shapes (xs = 4) 35.1 / 32.9 -> 31.3 / 30.7 us; unsplit shapes: C3 73.9 / 75.9 / 71.9 ->
// 71.8 / 72.3 / 71.8 us, C5 2455 -> 2445 us, LAP's last-mode level 2 65.0 -> 49.1 us.
constexpr int TTVP_THREADS = 128;
template <int U>
__global__ void __launch_bounds__(TTVP_THREADS, 5)
    ttv_pipe_kernel(const double* __restrict__ P, int64_t S, int64_t RK, int K, int64_t nvec,
                    const double* __restrict__ F, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ double2 red[TTVP_THREADS];
  const int64_t e = blockIdx.x * (int64_t)TTVP_THREADS + threadIdx.x;
  const int p = blockIdx.y, xs = gridDim.y;
  double2 acc = make_double2(0.0, 0.0);
  if (e < nvec) {
    const int64_t o = e * 2;
    const int64_t b = o / RK;
    const int64_t rk = o - b * RK;
    const int k = static_cast<int>(rk % K);
    const int64_t x0 = S * p / xs, x1 = S * (p + 1) / xs;
    const double* pp = P + b * S * RK + rk;
    const double* f = F + k;
    double2 pa[U], fa[U], pb[U], fb[U];
    auto load = [&](double2 (&pv)[U], double2 (&fv)[U], int64_t x) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = x + u < x1;
        const int64_t xx = ok ? x + u : x0;
        pv[u] = __ldcs(reinterpret_cast<const double2*>(pp + xx * RK));
        fv[u] = ok ? __ldg(reinterpret_cast<const double2*>(f + xx * K)) : make_double2(0.0, 0.0);
      }
    };
    auto consume = [&](const double2 (&pv)[U], const double2 (&fv)[U]) {
#pragma unroll
      for (int u = 0; u < U; ++u) vfma(acc, pv[u], fv[u]);
    };
    if (x0 < x1) {
      load(pa, fa, x0);
      int64_t x = x0;
      while (true) {
        if (x + U < x1) load(pb, fb, x + U);
        consume(pa, fa);
        x += U;
        if (x >= x1) break;
        if (x + U < x1) load(pa, fa, x + U);
        consume(pb, fb);
        x += U;
        if (x >= x1) break;
      }
    }
  }
  if (xs == 1) {
    if (e < nvec) *reinterpret_cast<double2*>(out + e * 2) = acc;
    return;
  }
  // cluster reduction (rank order), as ttv_kernel
  red[threadIdx.x] = acc;
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (p == 0 && e < nvec) {
    double2 s = acc;
    const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(&red[threadIdx.x]));
    for (int r = 1; r < xs; ++r) {
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(r));
      double2 v;
      asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(remote));
      vadd(s, v);
    }
    *reinterpret_cast<double2*>(out + e * 2) = s;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

cudaError_t launch_pipe(const double* P, int64_t S, int64_t RK, int K, int64_t total, int xs,
                        const double* F, double* out, cudaStream_t st) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(ttv_pipe_kernel<4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const int64_t nvec = total / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((nvec + TTVP_THREADS - 1) / TTVP_THREADS), (unsigned)xs, 1);
  cfg.blockDim = dim3(TTVP_THREADS, 1, 1);
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, ttv_pipe_kernel<4>, P, S, RK, K, nvec, F, out);
  note_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
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

// ---------------------------------------------------------------- batched multi-TTV
// ONE launch for a list of jobs (all the contractions of one construction-tree level, or the N
// single-mode operators; SURVEY a2 "batched multi-TTV").  Job j views its parent as
// [Bo][Sa][Sb][IN] (IN = the kept extents after the contracted ones, times K) and computes
//   child b: outB[bo][xa][t] = Σ_xb P[bo][xa][xb][t] · Fb[xb][k]        (always)
//   child a: outA[bo][xb][t] = Σ_xa P[bo][xa][xb][t] · Fa[xa][k]        (pair jobs, Fa != null)
// A pair job reads its parent ONCE for two children contracting adjacent kept modes (Sb <= 32:
// child a's Sb partial sums stay in registers across the xa loop).  A single job has Sa = 1.
// Each output is owned by one thread and summed in ascending x (with the x split of
// launch_ttv: cluster partials added in rank order) -- the same fma chain as ttv_kernel.
// single jobs (Sa = 1): ttv_kernel's arithmetic per job, the x split over a (1, xs, 1) cluster
// (V = 2: 128-thread CTAs and ttv_pipe_kernel's software-pipelined x loop, the same fma chain)
template <int V, int THR = TTV_THREADS>
__global__ void __launch_bounds__(THR, THR == TTV_THREADS ? 1 : 5)
    ttv_batch_kernel(const __grid_constant__ TtvBatch bt) {
  using T = typename Vec<V>::T;
  pdl_wait();
  pdl_trigger();
  __shared__ T red[THR];
  int ji = 0;
  while (ji + 1 < bt.njobs && (int)blockIdx.x >= bt.j[ji + 1].cta0) ++ji;
  const double* __restrict__ P = bt.j[ji].P;
  const double* __restrict__ F = bt.j[ji].Fb;
  double* out = bt.j[ji].outB;
  const int64_t IN = bt.j[ji].IN, S = bt.j[ji].Sb, nvec = bt.j[ji].nvec;
  const bool stream = bt.j[ji].stream != 0;
  const int K = bt.K;
  const int64_t e = ((int64_t)blockIdx.x - bt.j[ji].cta0) * THR + threadIdx.x;
  const int p = blockIdx.y, xs = gridDim.y;
  T acc;
  if constexpr (V == 1) acc = 0.0;
  else acc = make_double2(0.0, 0.0);
  if (e < nvec) {
    const int64_t o = e * V;
    const int64_t b = o / IN;
    const int64_t t = o - b * IN;
    const int k = static_cast<int>(t % K);
    const int64_t x0 = S * p / xs, x1 = S * (p + 1) / xs;
    const double* pp = P + b * S * IN + t;
    const double* f = F + k;
    int64_t x = x0;
    if constexpr (THR != TTV_THREADS) {
      constexpr int U = 4;
      T pa[U], fa[U], pb[U], fb[U];
      auto load = [&](T (&pv)[U], T (&fv)[U], int64_t xb) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool ok = xb + u < x1;
          const int64_t xx = ok ? xb + u : x0;
          pv[u] = stream ? Vec<V>::ld_stream(pp + xx * IN) : Vec<V>::ld(pp + xx * IN);
          if (ok) fv[u] = Vec<V>::ld(f + xx * K);
          else if constexpr (V == 1) fv[u] = 0.0;
          else fv[u] = make_double2(0.0, 0.0);
        }
      };
      auto consume = [&](const T (&pv)[U], const T (&fv)[U]) {
#pragma unroll
        for (int u = 0; u < U; ++u) vfma(acc, pv[u], fv[u]);
      };
      if (x0 < x1) {
        load(pa, fa, x0);
        while (true) {
          if (x + U < x1) load(pb, fb, x + U);
          consume(pa, fa);
          x += U;
          if (x >= x1) break;
          if (x + U < x1) load(pa, fa, x + U);
          consume(pb, fb);
          x += U;
          if (x >= x1) break;
        }
      }
      x = x1;
    }
    for (; x + 4 <= x1; x += 4) {
      T pv[4], fv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        pv[u] = stream ? Vec<V>::ld_stream(pp + (x + u) * IN) : Vec<V>::ld(pp + (x + u) * IN);
        fv[u] = Vec<V>::ld(f + (x + u) * K);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) vfma(acc, pv[u], fv[u]);
    }
    for (; x < x1; ++x) vfma(acc, Vec<V>::ld(pp + x * IN), Vec<V>::ld(f + x * K));
  }
  if (xs == 1) {
    if (e < nvec) *reinterpret_cast<T*>(out + e * V) = acc;
    return;
  }
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
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// pair jobs: one pass over the parent for two children contracting adjacent kept modes
template <int MAXSB>
__global__ void __launch_bounds__(TTV_THREADS, 2)
    ttv_pair_kernel(const __grid_constant__ TtvBatch bt) {
  pdl_wait();
  pdl_trigger();
  int ji = 0;
  while (ji + 1 < bt.njobs && (int)blockIdx.x >= bt.j[ji + 1].cta0) ++ji;
  const double* __restrict__ P = bt.j[ji].P;
  const double* __restrict__ Fa = bt.j[ji].Fa;
  const double* __restrict__ Fb = bt.j[ji].Fb;
  double* outA = bt.j[ji].outA;
  double* outB = bt.j[ji].outB;
  const int64_t IN = bt.j[ji].IN, nvec = bt.j[ji].nvec;
  const int Sa = bt.j[ji].Sa, Sb = bt.j[ji].Sb;
  const bool stream = bt.j[ji].stream != 0;
  const int K = bt.K;
  const int64_t e = ((int64_t)blockIdx.x - bt.j[ji].cta0) * TTV_THREADS + threadIdx.x;
  if (e >= nvec) return;
  const int64_t bo = e / IN, t = e - bo * IN;
  const int k = static_cast<int>(t % K);
  double accA[MAXSB];
#pragma unroll
  for (int u = 0; u < MAXSB; ++u) accA[u] = 0.0;
  const double* pp = P + bo * (int64_t)Sa * Sb * IN + t;
  for (int xa = 0; xa < Sa; ++xa) {
    const double fa = __ldg(Fa + (int64_t)xa * K + k);
    const double* px = pp + (int64_t)xa * Sb * IN;
    const double* fb = Fb + k;
    double accB = 0.0;
    // every xb load of this xa in flight at once (registers: MAXSB accumulators + MAXSB loads);
    // running pointers (hoisted per-xb offsets would take 2 MAXSB more registers)
    double pv[MAXSB];
#pragma unroll
    for (int u = 0; u < MAXSB; ++u) {
      if (u < Sb) pv[u] = stream ? __ldcs(px) : __ldg(px);
      px += IN;
    }
#pragma unroll
    for (int u = 0; u < MAXSB; ++u) {
      if (u < Sb) {
        accB = fma(pv[u], __ldg(fb), accB);
        accA[u] = fma(pv[u], fa, accA[u]);
      }
      fb += K;
    }
    outB[(bo * Sa + xa) * IN + t] = accB;
  }
#pragma unroll
  for (int u = 0; u < MAXSB; ++u)
    if (u < Sb) outA[(bo * Sb + u) * IN + t] = accA[u];
}

template <typename Kern>
cudaError_t launch_batch_k(Kern kern, const TtvBatch& bt, int ctas, int xs, cudaStream_t st,
                           int threads = TTV_THREADS) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ctas, (unsigned)xs, 1);
  cfg.blockDim = dim3((unsigned)threads, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (xs > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 1;
    attr[na].val.clusterDim.y = (unsigned)xs;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, bt);
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
  static const bool no_pipe = getenv("CPPP_NO_TTV_PIPE") != nullptr;   // A/B: ttv_kernel
  if (V == 2 && !no_pipe) return launch_pipe(P, S, RK, K, total, xs, F, out, st);
  return launch_ttv_cfg(P, B, S, R, K, F, out, V, 4, xs, st);
}

}  // namespace cppp

namespace cppp {

// Batched multi-TTV: the pair jobs of jobs[0..n) in one launch and the single jobs in another
// (per TTV_MAX_JOBS).  Pair jobs need Sb <= 32 and use 8-byte loads; single jobs take 16-byte
// loads when K is even and every operand 16-byte aligned, and launch_ttv's x-split rule over
// the batch's total CTA count.
cudaError_t launch_ttv_batch(const TtvJob* jobs, int n, int K, cudaStream_t st) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(ttv_batch_kernel<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(ttv_batch_kernel<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(ttv_batch_kernel<2, TTVP_THREADS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  for (int pass = 0; pass < 2; ++pass) {   // 0: pairs, 1: singles
    std::vector<TtvJob> sel;
    for (int i = 0; i < n; ++i)
      if ((jobs[i].Fa != nullptr) == (pass == 0)) sel.push_back(jobs[i]);
    for (size_t b0 = 0; b0 < sel.size(); b0 += TTV_MAX_JOBS) {
      const int nb = (int)std::min(sel.size() - b0, (size_t)TTV_MAX_JOBS);
      bool v2 = pass == 1 && K % 2 == 0;
      int64_t minS = INT64_MAX;
      for (int i = 0; i < nb; ++i) {
        const TtvJob& J = sel[b0 + i];
        if (pass == 0 && (J.Sb > TTV_PAIR_MAXSB || J.Sb < 1)) return cudaErrorInvalidValue;
        if (pass == 1 && J.Sa != 1) return cudaErrorInvalidValue;
        const uintptr_t al = reinterpret_cast<uintptr_t>(J.P) | reinterpret_cast<uintptr_t>(J.Fb) |
                             reinterpret_cast<uintptr_t>(J.outB);
        if (al % 16) v2 = false;
        minS = std::min<int64_t>(minS, J.Sb);
      }
      const int V = v2 ? 2 : 1;
      TtvBatch bt;
      bt.njobs = nb;
      bt.K = K;
      int ctas = 0;
      for (int i = 0; i < nb; ++i) {
        bt.j[i] = sel[b0 + i];
        bt.j[i].nvec = bt.j[i].Bo * bt.j[i].IN / (pass == 0 ? 1 : V);
        bt.j[i].cta0 = ctas;
        ctas += (int)((bt.j[i].nvec + TTV_THREADS - 1) / TTV_THREADS);
      }
      if (ctas == 0) continue;
      cudaError_t e;
      if (pass == 0) {
        e = launch_batch_k(ttv_pair_kernel<TTV_PAIR_MAXSB>, bt, ctas, 1, st);
      } else {
        int xs = 1;
        while (xs < 8 && (int64_t)ctas * xs < 148LL * 2 && minS / (2 * xs) >= 16) xs *= 2;
        static const bool no_pipe = getenv("CPPP_NO_TTV_PIPE") != nullptr;   // A/B
        if (V == 2 && !no_pipe) {   // the same split, 128-thread CTAs
          int c128 = 0;
          for (int i = 0; i < nb; ++i) {
            bt.j[i].cta0 = c128;
            c128 += (int)((bt.j[i].nvec + TTVP_THREADS - 1) / TTVP_THREADS);
          }
          e = launch_batch_k(ttv_batch_kernel<2, TTVP_THREADS>, bt, c128, xs, st, TTVP_THREADS);
        } else {
          e = V == 2 ? launch_batch_k(ttv_batch_kernel<2>, bt, ctas, xs, st)
                     : launch_batch_k(ttv_batch_kernel<1>, bt, ctas, xs, st);
        }
      }
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace cppp
