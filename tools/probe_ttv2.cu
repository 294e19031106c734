// probe_ttv2.cu — multi-TTV with several output rows per thread (the factor row F[x][k] loaded
// once for NR parent rows) against the library's ttv_kernel, on the workload shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe_ttv2 \
//        tools/probe_ttv2.cu paper_1811_10573_b200/csrc/ttv.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <string>
#include <cuda_runtime.h>
#include "../paper_1811_10573_b200/csrc/internal.h"

namespace cppp {
bool pdl_enabled() { return false; }
void note_launch() {}
cudaError_t launch_ttv_cfg(const double* P, int64_t B, int64_t S, int64_t R, int K,
                           const double* F, double* out, int V, int U, int xs, cudaStream_t st);
}  // namespace cppp

constexpr int TH = 256;

// out[rho][k] = sum_x P[b][x][r][k] F[x][k], rho = b R + r; thread = NR rows x 2 columns
template <int NR, int U>
__global__ void __launch_bounds__(TH) ttv_rows(const double* __restrict__ P, int64_t S, int64_t R,
                                              int K, int64_t rows, const double* __restrict__ F,
                                              double* __restrict__ out) {
  __shared__ double2 red[NR][TH];
  const int KH = K / 2;
  const int64_t e = blockIdx.x * (int64_t)TH + threadIdx.x;
  const int64_t ngrp = (rows + NR - 1) / NR;
  const int p = blockIdx.y, xs = gridDim.y;
  const int64_t RK = R * K;
  double2 acc[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j] = make_double2(0.0, 0.0);
  const bool live = e < ngrp * KH;
  if (live) {
    const int64_t g = e / KH;
    const int c = static_cast<int>(e - g * KH);
    const double* base[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      int64_t rho = g * NR + j;
      if (rho >= rows) rho = rows - 1;
      const int64_t b = rho / R, r = rho - b * R;
      base[j] = P + b * S * RK + r * K + 2 * c;
    }
    const double* f = F + 2 * c;
    const int64_t x0 = S * p / xs, x1 = S * (p + 1) / xs;
    int64_t x = x0;
    for (; x + U <= x1; x += U) {
      double2 pv[U][NR], fv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int j = 0; j < NR; ++j)
          pv[u][j] = __ldcs(reinterpret_cast<const double2*>(base[j] + (x + u) * RK));
        fv[u] = __ldg(reinterpret_cast<const double2*>(f + (x + u) * K));
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          acc[j].x = fma(pv[u][j].x, fv[u].x, acc[j].x);
          acc[j].y = fma(pv[u][j].y, fv[u].y, acc[j].y);
        }
    }
    for (; x < x1; ++x) {
      const double2 fv = __ldg(reinterpret_cast<const double2*>(f + x * K));
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const double2 pv = __ldcs(reinterpret_cast<const double2*>(base[j] + x * RK));
        acc[j].x = fma(pv.x, fv.x, acc[j].x);
        acc[j].y = fma(pv.y, fv.y, acc[j].y);
      }
    }
  }
  if (xs == 1) {
    if (live) {
      const int64_t g = e / KH;
      const int c = static_cast<int>(e - g * KH);
#pragma unroll
      for (int j = 0; j < NR; ++j)
        if (g * NR + j < rows)
          *reinterpret_cast<double2*>(out + (g * NR + j) * K + 2 * c) = acc[j];
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < NR; ++j) red[j][threadIdx.x] = acc[j];
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  // rank p adds entries [p E / xs, (p+1) E / xs) of all ranks in rank order
  constexpr int E = NR * TH;
  const int i0 = p * E / xs, i1 = (p + 1) * E / xs;
  for (int i = i0 + threadIdx.x; i < i1; i += TH) {
    const int j = i / TH, t = i - j * TH;
    const int64_t et = blockIdx.x * (int64_t)TH + t;
    if (et >= ngrp * KH) continue;
    const int64_t g = et / KH;
    const int c = static_cast<int>(et - g * KH);
    if (g * NR + j >= rows) continue;
    const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(&red[j][t]));
    double2 s = make_double2(0.0, 0.0);
    for (int r = 0; r < xs; ++r) {
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(r));
      double2 v;
      asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(remote));
      if (r == 0) s = v;
      else { s.x += v.x; s.y += v.y; }
    }
    *reinterpret_cast<double2*>(out + (g * NR + j) * K + 2 * c) = s;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int NR, int U>
cudaError_t launch_rows(const double* P, int64_t B, int64_t S, int64_t R, int K, const double* F,
                        double* out, int xs) {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(ttv_rows<NR, U>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    done = true;
  }
  const int64_t rows = B * R, ngrp = (rows + NR - 1) / NR;
  const int64_t th = ngrp * (K / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((th + TH - 1) / TH), (unsigned)xs, 1);
  cfg.blockDim = dim3(TH, 1, 1);
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = 1;
  a[0].val.clusterDim.y = (unsigned)xs;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ttv_rows<NR, U>, P, S, R, K, rows, F, out);
}

// software-pipelined: round i+1's loads are issued before round i is consumed; predicated tail
template <int U, int THR, int MINB>
__global__ void __launch_bounds__(THR, MINB) ttv_pipe(const double* __restrict__ P, int64_t S, int64_t RK,
                                               int K, int64_t nvec, const double* __restrict__ F,
                                               double* __restrict__ out) {
  __shared__ double2 red[THR];
  const int64_t e = blockIdx.x * (int64_t)THR + threadIdx.x;
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
#define LOADB(PV, FV, X)                                                                     \
  _Pragma("unroll") for (int u = 0; u < U; ++u) {                                             \
    const bool ok = (X) + u < x1;                                                             \
    const int64_t xx = ok ? (X) + u : x0;                                                     \
    PV[u] = __ldcs(reinterpret_cast<const double2*>(pp + xx * RK));                           \
    FV[u] = ok ? __ldg(reinterpret_cast<const double2*>(f + xx * K)) : make_double2(0.0, 0.0); \
  }
#define CONS(PV, FV)                                   \
  _Pragma("unroll") for (int u = 0; u < U; ++u) {      \
    acc.x = fma(PV[u].x, FV[u].x, acc.x);              \
    acc.y = fma(PV[u].y, FV[u].y, acc.y);              \
  }
    LOADB(pa, fa, x0);
    int64_t x = x0;
    while (true) {
      if (x + U < x1) { LOADB(pb, fb, x + U); }
      CONS(pa, fa);
      x += U;
      if (x >= x1) break;
      if (x + U < x1) { LOADB(pa, fa, x + U); }
      CONS(pb, fb);
      x += U;
      if (x >= x1) break;
    }
  }
  if (xs == 1) {
    if (e < nvec) *reinterpret_cast<double2*>(out + e * 2) = acc;
    return;
  }
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
      s.x += v.x; s.y += v.y;
    }
    *reinterpret_cast<double2*>(out + e * 2) = s;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <int U, int THR, int MINB>
cudaError_t launch_pipe(const double* P, int64_t B, int64_t S, int64_t R, int K, const double* F,
                        double* out, int xs) {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(ttv_pipe<U, THR, MINB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    done = true;
  }
  const int64_t nvec = B * R * K / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((nvec + THR - 1) / THR), (unsigned)xs, 1);
  cfg.blockDim = dim3(THR, 1, 1);
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = 1;
  a[0].val.clusterDim.y = (unsigned)xs;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ttv_pipe<U, THR, MINB>, P, S, R * K, K, nvec, F, out);
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint32_t b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_expect(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint32_t b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(b), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// bulk-staged multi-TTV: CTA = (item = (b, column block cb of W), x part p of a (1, xs, 1) cluster);
// units of XG x rows: W == RK -> one contiguous bulk copy per unit; else per-x segments from
// the 16-byte boundary (pitch W + 2).  Thread = (column pair c, x phase j of TPC).
struct TB { const double* P; const double* F; double* out; int64_t B, S, RK; int K, W, XG, ncb, NS; };
__global__ void __launch_bounds__(256) ttv_bulk(const TB a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(16) double2 red[256];
  __shared__ uint64_t full[4];
  const int tid = threadIdx.x;
  const int P2 = a.W == a.RK ? a.W : a.W + 2;   // stage pitch
  const int64_t item = blockIdx.x;
  const int64_t b = item / a.ncb;
  const int64_t c0 = (item - b * a.ncb) * a.W;
  const int wv = (int)(a.RK - c0 < a.W ? a.RK - c0 : a.W);
  const int np = a.W / 2, tpc = 256 / np;
  const int cp = tid % np, j = tid / np;
  const bool act = j < tpc && 2 * cp < wv;
  const int p = blockIdx.y, xs = gridDim.y;
  const int64_t x0 = a.S * p / xs, x1 = a.S * (p + 1) / xs;
  const int nu = (int)((x1 - x0 + a.XG - 1) / a.XG);
  const double* base = a.P + b * a.S * a.RK + c0;
  const bool whole = a.W == a.RK;
  const int k = (int)((c0 + 2 * cp) % a.K);
  double* fsm = sm + (int64_t)a.NS * a.XG * P2;   // [NS][XG][K] factor rows
  auto issue = [&](int u, int st, uint64_t pol) {
    const int64_t xa = x0 + (int64_t)u * a.XG, xb = xa + a.XG < x1 ? xa + a.XG : x1;
    double* dst = sm + (int64_t)st * a.XG * P2;
    const uint32_t fbytes = (uint32_t)((xb - xa) * a.K * 8);
    if (whole) {
      const uint32_t bytes = (uint32_t)((xb - xa) * a.RK * 8);
      mb_expect(su32(&full[st]), bytes + fbytes);
      bulk(su32(fsm + (int64_t)st * a.XG * a.K), a.F + xa * a.K, fbytes, su32(&full[st]), pol);
      bulk(su32(dst), base + xa * a.RK, bytes, su32(&full[st]), pol);
    } else {
      uint32_t tot = fbytes;
      for (int64_t x = xa; x < xb; ++x) {
        const double* src = base + x * a.RK;
        const int off = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
        tot += (uint32_t)(((wv + off) * 8 + 15) & ~15);
      }
      mb_expect(su32(&full[st]), tot);
      bulk(su32(fsm + (int64_t)st * a.XG * a.K), a.F + xa * a.K, fbytes, su32(&full[st]), pol);
      for (int64_t x = xa; x < xb; ++x) {
        const double* src = base + x * a.RK;
        const int off = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
        bulk(su32(dst + (x - xa) * P2), src - off, (uint32_t)(((wv + off) * 8 + 15) & ~15), su32(&full[st]), pol);
      }
    }
  };
  uint64_t pol = 0;
  if (tid == 0) {
    pol = pol_first();
    for (int s = 0; s < a.NS; ++s) mb_init(su32(&full[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < a.NS && s < nu; ++s) issue(s, s, pol);
  }
  __syncthreads();
  double2 acc = make_double2(0.0, 0.0);
  uint32_t phase = 0;
  for (int u = 0; u < nu; ++u) {
    const int st = u % a.NS;
    const int64_t xa = x0 + (int64_t)u * a.XG, xb = xa + a.XG < x1 ? xa + a.XG : x1;
    mb_wait(su32(&full[st]), (phase >> st) & 1);
    phase ^= 1u << st;
    if (act) {
      const double* stg = sm + (int64_t)st * a.XG * P2;
      const double* fst = fsm + (int64_t)st * a.XG * a.K;
      int64_t x = xa + j;
      double2 acc2 = make_double2(0.0, 0.0);
      for (; x + tpc < xb; x += 2 * tpc) {
        const double* r0 = stg + (x - xa) * P2;
        const double* r1 = r0 + tpc * P2;
        const int o0 = whole ? 0 : (int)((reinterpret_cast<uintptr_t>(base + x * a.RK) >> 3) & 1);
        const int o1 = whole ? 0 : (int)((reinterpret_cast<uintptr_t>(base + (x + tpc) * a.RK) >> 3) & 1);
        const double v0 = r0[o0 + 2 * cp], v1 = r0[o0 + 2 * cp + 1];
        const double w0 = r1[o1 + 2 * cp], w1 = r1[o1 + 2 * cp + 1];
        const double2 f = *reinterpret_cast<const double2*>(fst + (x - xa) * a.K + k);
        const double2 g = *reinterpret_cast<const double2*>(fst + (x + tpc - xa) * a.K + k);
        acc.x = fma(v0, f.x, acc.x);
        acc.y = fma(v1, f.y, acc.y);
        acc2.x = fma(w0, g.x, acc2.x);
        acc2.y = fma(w1, g.y, acc2.y);
      }
      for (; x < xb; x += tpc) {
        const double* row = stg + (x - xa) * P2;
        const int off = whole ? 0 : (int)((reinterpret_cast<uintptr_t>(base + x * a.RK) >> 3) & 1);
        const double2 f = *reinterpret_cast<const double2*>(fst + (x - xa) * a.K + k);
        acc.x = fma(row[off + 2 * cp], f.x, acc.x);
        acc.y = fma(row[off + 2 * cp + 1], f.y, acc.y);
      }
      acc.x += acc2.x;
      acc.y += acc2.y;
    }
    __syncthreads();
    if (tid == 0 && u + a.NS < nu) issue(u + a.NS, st, pol);
  }
  red[tid] = acc;
  __syncthreads();
  double2 s = make_double2(0.0, 0.0);
  if (j == 0 && act) {
    s = red[cp];
    for (int jj = 1; jj < tpc; ++jj) { s.x += red[jj * np + cp].x; s.y += red[jj * np + cp].y; }
  }
  if (xs == 1) {
    if (j == 0 && act) *reinterpret_cast<double2*>(a.out + b * a.RK + c0 + 2 * cp) = s;
    return;
  }
  __syncthreads();
  if (j == 0) red[cp] = s;
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (p == 0 && j == 0 && act) {
    const uint32_t local = su32(&red[cp]);
    for (int r = 1; r < xs; ++r) {
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(r));
      double2 v;
      asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(remote));
      s.x += v.x; s.y += v.y;
    }
    *reinterpret_cast<double2*>(a.out + b * a.RK + c0 + 2 * cp) = s;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
void run_bulk(const double* P, int64_t B, int64_t S, int64_t R, int K, const double* F, double* out,
              int W, int XG, int NS, int xs) {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(ttv_bulk, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(ttv_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    done = true;
  }
  TB a;
  a.P = P; a.F = F; a.out = out; a.B = B; a.S = S; a.RK = R * K; a.K = K;
  a.W = W > a.RK ? (int)a.RK : W;
  a.XG = XG; a.NS = NS;
  a.ncb = (int)((a.RK + a.W - 1) / a.W);
  const int P2 = a.W == a.RK ? a.W : a.W + 2;
  const size_t smem = 8ull * NS * XG * P2 + 8ull * NS * XG * K;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(B * a.ncb), (unsigned)xs, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = (unsigned)xs;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, ttv_bulk, a);
}

__global__ void fill(double* p, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z = (z ^ (z >> 31)) * 0xBF58476D1CE4E5B9ull;
    z ^= z >> 29;
    p[i] = (double)(z >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  struct Shape { const char* name; int64_t B, S, R; int K; };
  Shape shapes[] = {{"C3 lvl2 (100^3 x50 mid)", 100, 100, 100, 50},
                    {"C3 lvl2 last", 10000, 100, 1, 50},
                    {"C3 lvl2 first", 1, 100, 10000, 50},
                    {"C5 lvl2 (256^3 x128 mid)", 256, 256, 256, 128},
                    {"LAP lvl2 last (25^4 x 25 x 2)", 390625, 25, 1, 2},
                    {"LAP lvl2 first (25 x 25^4 x 2)", 1, 25, 390625, 2}};
  const int64_t PN = 256ll * 256 * 256 * 128;
  double *P, *F, *out, *ref, *flush;
  cudaMalloc(&P, 8 * PN);
  cudaMalloc(&F, 8 * 400 * 128);
  cudaMalloc(&out, 8ll * 256 * 256 * 128);
  cudaMalloc(&ref, 8ll * 256 * 256 * 128);
  const int64_t FL = 300ll << 20;
  cudaMalloc(&flush, FL);
  fill<<<4096, 256>>>(P, PN, 1);
  fill<<<64, 256>>>(F, 400 * 128, 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (const Shape& s : shapes) {
    const double bytes = 8.0 * (s.B * s.S * s.R * s.K + s.B * s.R * s.K);
    if (s.B * s.S * s.R * s.K > PN) continue;
    printf("%s  (%.1f MB)\n", s.name, bytes / 1e6);
    cppp::launch_ttv_cfg(P, s.B, s.S, s.R, s.K, F, ref, 2, 4, 1, 0);   // unsplit reference
    cudaDeviceSynchronize();
    std::vector<double> hr(s.B * s.R * s.K), ho(hr.size());
    cudaMemcpy(hr.data(), ref, 8 * hr.size(), cudaMemcpyDeviceToHost);
    auto run = [&](const char* nm, auto&& f) {
      for (int cold = 1; cold < 2; ++cold) {
        float tot = 0;
        const int reps = 10;
        for (int i = 0; i < reps + 2; ++i) {
          if (cold) cudaMemsetAsync(flush, i & 0xff, FL);
          cudaEventRecord(a);
          f();
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (i >= 2) tot += ms;
        }
        cudaError_t e = cudaGetLastError();
        cudaMemcpy(ho.data(), out, 8 * ho.size(), cudaMemcpyDeviceToHost);
        double md = 0, mr = 0;
        for (size_t i = 0; i < ho.size(); ++i) {
          md = fmax(md, fabs(ho[i] - hr[i]));
          mr = fmax(mr, fabs(hr[i]));
        }
        const double us = 1e3 * tot / reps;
        printf("  %-22s %s %7.1f us %6.2f TB/s  err %.1e %s\n", nm, cold ? "cold" : "warm", us,
               bytes / us / 1e6, md / mr, e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    };
    run("lib xs1", [&] { cppp::launch_ttv_cfg(P, s.B, s.S, s.R, s.K, F, out, 2, 4, 1, 0); });
    run("pipe U4 T128 m5 xs1", [&] { launch_pipe<4, 128, 5>(P, s.B, s.S, s.R, s.K, F, out, 1); });
    run("pipe U4 T256 m2 xs1", [&] { launch_pipe<4, 256, 2>(P, s.B, s.S, s.R, s.K, F, out, 1); });
    run("pipe U2 T128 m8 xs1", [&] { launch_pipe<2, 128, 8>(P, s.B, s.S, s.R, s.K, F, out, 1); });
    run("pipe U8 T128 m2 xs1", [&] { launch_pipe<8, 128, 2>(P, s.B, s.S, s.R, s.K, F, out, 1); });
  }
  return 0;
}
