// probe_skinny.cu — the skinny (K <= 16, odd-stride) TTMs of the compact Laplacian (s = 25, K = 2)
// fed by 1-D bulk async copies (cp.async.bulk + mbarrier ring) against the library's
// register-load kernels (launch_ttm_simt -> ttm_skinny_{kc,mc}_kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe_skinny \
//        tools/probe_skinny.cu paper_1811_10573_b200/csrc/ttm.cu paper_1811_10573_b200/csrc/solve.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1811_10573_b200/csrc/internal.h"

namespace cppp {
cudaError_t launch_ttm_simt(const double* X, int64_t B, int64_t S, int64_t R, const double* F,
                            int K, double* out, cudaStream_t st);
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

// R == 1: chunk = CH consecutive rows of S doubles (one contiguous run, CH even so every full
// chunk starts 16-byte aligned); thread = row; the factor in shared memory.
template <int KB, int CH, int NS>
__global__ void __launch_bounds__(CH) kc_bulk(const double* __restrict__ X, int64_t B, int S,
                                             const double* __restrict__ F, int K, double* __restrict__ out) {
  extern __shared__ __align__(16) double sm[];
  double* fs = sm + (int64_t)NS * CH * S;
  uint64_t* full = reinterpret_cast<uint64_t*>(fs + ((S * K + 1) & ~1));
  const int tid = threadIdx.x;
  const int64_t nch = (B + CH - 1) / CH, nfull = B / CH;
  const uint32_t bytes = (uint32_t)CH * S * 8;
  uint64_t pol = 0;
  if (tid == 0) {
    pol = pol_first();
    for (int s = 0; s < NS; ++s) mb_init(su32(&full[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NS; ++s) {
      const int64_t c = blockIdx.x + (int64_t)s * gridDim.x;
      if (c < nfull) {
        mb_expect(su32(&full[s]), bytes);
        bulk(su32(sm + (int64_t)s * CH * S), X + c * CH * S, bytes, su32(&full[s]), pol);
      }
    }
  }
  for (int e = tid; e < S * K; e += CH) fs[e] = F[e];
  __syncthreads();
  int it = 0;
  uint32_t phase = 0;   // per-stage parity bits (a plain-load chunk leaves its stage's barrier as is)
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
    const int st = it % NS;
    double* stage = sm + (int64_t)st * CH * S;
    const int nr = (int)(B - c * CH < CH ? B - c * CH : CH);
    if (c < nfull) {
      mb_wait(su32(&full[st]), (phase >> st) & 1);
      phase ^= 1u << st;
    } else {
      for (int e = tid; e < nr * S; e += CH) stage[e] = __ldcs(X + c * CH * S + e);
      __syncthreads();
    }
    if (tid < nr) {
      const double* row = stage + tid * S;
      double acc[KB];
#pragma unroll
      for (int n = 0; n < KB; ++n) acc[n] = 0.0;
      for (int x = 0; x < S; ++x) {
        const double v = row[x];
#pragma unroll
        for (int n = 0; n < KB; ++n)
          if (n < K) acc[n] = fma(v, fs[x * K + n], acc[n]);
      }
      double* o = out + (c * CH + tid) * K;
#pragma unroll
      for (int n = 0; n < KB; ++n)
        if (n < K) o[n] = acc[n];
    }
    __syncthreads();
    if (tid == 0) {
      const int64_t cn = c + (int64_t)NS * gridDim.x;
      if (cn < nfull) {
        mb_expect(su32(&full[st]), bytes);
        bulk(su32(stage), X + cn * CH * S, bytes, su32(&full[st]), pol);
      }
    }
  }
}

// R > 1: chunk = (b, CR consecutive r): S row segments X[b][x][r0 .. r0+CR), each copied from
// the 16-byte boundary at or below its start (odd R: every other x is 8 bytes off), pitch CR + 2.
template <int KB, int CR, int NS>
__global__ void __launch_bounds__(CR) mc_bulk(const double* __restrict__ X, int64_t B, int S, int64_t R,
                                             const double* __restrict__ F, int K, double* __restrict__ out) {
  extern __shared__ __align__(16) double sm[];
  constexpr int P = CR + 2;
  double* fs = sm + (int64_t)NS * S * P;
  uint64_t* full = reinterpret_cast<uint64_t*>(fs + ((S * K + 1) & ~1));
  const int tid = threadIdx.x;
  const int64_t nrb = (R + CR - 1) / CR, nch = B * nrb;
  const double* Xend = X + B * S * R;
  auto safe = [&](int64_t c) {   // a full r block whose rounded-up copies stay inside X
    const int64_t b = c / nrb, r0 = (c - b * nrb) * CR;
    return r0 + CR <= R && X + ((b * S + S - 1) * R + r0 + CR + 2) <= Xend;
  };
  auto issue = [&](int64_t c, int s, uint64_t pol) {
    const int64_t b = c / nrb, r0 = (c - b * nrb) * CR;
    uint32_t tot = 0;
    for (int x = 0; x < S; ++x) {
      const double* src = X + (b * S + x) * R + r0;
      const int off = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
      tot += (uint32_t)(((CR + off) * 8 + 15) & ~15);
    }
    mb_expect(su32(&full[s]), tot);
    for (int x = 0; x < S; ++x) {
      const double* src = X + (b * S + x) * R + r0;
      const int off = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
      bulk(su32(sm + ((int64_t)s * S + x) * P), src - off, (uint32_t)(((CR + off) * 8 + 15) & ~15),
           su32(&full[s]), pol);
    }
  };
  uint64_t pol = 0;
  if (tid == 0) {
    pol = pol_first();
    for (int s = 0; s < NS; ++s) mb_init(su32(&full[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NS; ++s) {
      const int64_t c = blockIdx.x + (int64_t)s * gridDim.x;
      if (c < nch && safe(c)) issue(c, s, pol);
    }
  }
  for (int e = tid; e < S * K; e += CR) fs[e] = F[e];
  __syncthreads();
  int it = 0;
  uint32_t phase = 0;   // per-stage parity bits (a plain-load chunk leaves its stage's barrier as is)
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
    const int st = it % NS;
    const int64_t b = c / nrb, r0 = (c - b * nrb) * CR;
    const int nr = (int)(R - r0 < CR ? R - r0 : CR);
    double* stage = sm + (int64_t)st * S * P;
    const bool bulk_c = safe(c);
    if (bulk_c) {
      mb_wait(su32(&full[st]), (phase >> st) & 1);
      phase ^= 1u << st;
    } else {
      for (int x = 0; x < S; ++x) {
        const double* src = X + (b * S + x) * R + r0;
        const int off = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
        if (tid < nr) stage[x * P + off + tid] = __ldcs(src + tid);
      }
      __syncthreads();
    }
    if (tid < nr) {
      double acc[KB];
#pragma unroll
      for (int n = 0; n < KB; ++n) acc[n] = 0.0;
      for (int x = 0; x < S; ++x) {
        const double* src = X + (b * S + x) * R + r0;
        const int off = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
        const double v = stage[x * P + off + tid];
#pragma unroll
        for (int n = 0; n < KB; ++n)
          if (n < K) acc[n] = fma(v, fs[x * K + n], acc[n]);
      }
      double* o = out + (b * R + r0 + tid) * K;
#pragma unroll
      for (int n = 0; n < KB; ++n)
        if (n < K) o[n] = acc[n];
    }
    __syncthreads();
    if (tid == 0) {
      const int64_t cn = c + (int64_t)NS * gridDim.x;
      if (cn < nch && safe(cn)) issue(cn, st, pol);
    }
  }
}

template <int CH, int NS>
void run_kc(const double* X, int64_t B, int S, const double* F, int K, double* out, int per_sm) {
  const size_t smem = 8 * ((size_t)NS * CH * S + ((S * K + 1) & ~1)) + 8 * NS;
  cudaFuncSetAttribute(kc_bulk<2, CH, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t nch = (B + CH - 1) / CH;
  int64_t g = 148 * per_sm;
  if (g > nch) g = nch;
  kc_bulk<2, CH, NS><<<(unsigned)g, CH, smem>>>(X, B, S, F, K, out);
}
template <int CR, int NS>
void run_mc(const double* X, int64_t B, int S, int64_t R, const double* F, int K, double* out, int per_sm) {
  const size_t smem = 8 * ((size_t)NS * S * (CR + 2) + ((S * K + 1) & ~1)) + 8 * NS;
  cudaFuncSetAttribute(mc_bulk<2, CR, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t nch = B * ((R + CR - 1) / CR);
  int64_t g = 148 * per_sm;
  if (g > nch) g = nch;
  mc_bulk<2, CR, NS><<<(unsigned)g, CR, smem>>>(X, B, S, R, F, K, out);
}

// R > 1, long segments: a unit = (b, CR consecutive r, XG consecutive x): XG row segments of CR
// doubles (copied from the 16-byte boundary at or below their start, pitch CR + 2); a CTA runs
// the x groups of one r block in order, so each thread's RT accumulators persist across units.
template <int KB, int CR, int XG, int NS>
__global__ void __launch_bounds__(256) mc2_bulk(const double* __restrict__ X, int64_t B, int S, int64_t R,
                                               const double* __restrict__ F, int K, double* __restrict__ out) {
  extern __shared__ __align__(16) double sm[];
  constexpr int P = CR + 2, RT = CR / 256;
  double* fs = sm + (int64_t)NS * XG * P;
  uint64_t* full = reinterpret_cast<uint64_t*>(fs + ((S * K + 1) & ~1));
  const int tid = threadIdx.x;
  const int ng = (S + XG - 1) / XG;
  const int64_t nrb = (R + CR - 1) / CR, nch = B * nrb;
  const double* Xend = X + B * S * R;
  auto safe = [&](int64_t c) {
    const int64_t b = c / nrb, r0 = (c - b * nrb) * CR;
    return r0 + CR <= R && X + ((b * S + S - 1) * R + r0 + CR + 2) <= Xend;
  };
  // unit u of this CTA: chunk blockIdx.x + (u / ng) gridDim.x, x group u % ng
  const int64_t my = nch > blockIdx.x ? (nch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nunits = my * ng;
  auto issue = [&](int64_t u, int s, uint64_t pol) {
    const int64_t c = blockIdx.x + (u / ng) * gridDim.x;
    if (!safe(c)) return;
    const int g = (int)(u % ng);
    const int64_t b = c / nrb, r0 = (c - b * nrb) * CR;
    const int xa = g * XG, xb = xa + XG < S ? xa + XG : S;
    uint32_t tot = 0;
    for (int x = xa; x < xb; ++x) {
      const double* src = X + (b * S + x) * R + r0;
      const int off = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
      tot += (uint32_t)(((CR + off) * 8 + 15) & ~15);
    }
    mb_expect(su32(&full[s]), tot);
    for (int x = xa; x < xb; ++x) {
      const double* src = X + (b * S + x) * R + r0;
      const int off = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
      bulk(su32(sm + ((int64_t)s * XG + (x - xa)) * P), src - off, (uint32_t)(((CR + off) * 8 + 15) & ~15),
           su32(&full[s]), pol);
    }
  };
  uint64_t pol = 0;
  if (tid == 0) {
    pol = pol_first();
    for (int s = 0; s < NS; ++s) mb_init(su32(&full[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NS && s < nunits; ++s) issue(s, s, pol);
  }
  for (int e = tid; e < S * K; e += 256) fs[e] = F[e];
  __syncthreads();
  uint32_t phase = 0;
  double acc[RT][KB];
  for (int64_t u = 0; u < nunits; ++u) {
    const int st = (int)(u % NS);
    const int64_t c = blockIdx.x + (u / ng) * gridDim.x;
    const int g = (int)(u % ng);
    const int64_t b = c / nrb, r0 = (c - b * nrb) * CR;
    const int nr = (int)(R - r0 < CR ? R - r0 : CR);
    const int xa = g * XG, xb = xa + XG < S ? xa + XG : S;
    double* stage = sm + (int64_t)st * XG * P;
    if (safe(c)) {
      mb_wait(su32(&full[st]), (phase >> st) & 1);
      phase ^= 1u << st;
    } else {
      for (int x = xa; x < xb; ++x) {
        const double* src = X + (b * S + x) * R + r0;
        const int off = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
        for (int t = tid; t < nr; t += 256) stage[(x - xa) * P + off + t] = __ldcs(src + t);
      }
      __syncthreads();
    }
    if (g == 0) {
#pragma unroll
      for (int j = 0; j < RT; ++j)
#pragma unroll
        for (int n = 0; n < KB; ++n) acc[j][n] = 0.0;
    }
    const double* row0 = X + (b * S + xa) * R + r0;
    for (int x = xa; x < xb; ++x) {
      const int off = (int)((reinterpret_cast<uintptr_t>(row0 + (int64_t)(x - xa) * R) >> 3) & 1);
      const double* srow = stage + (x - xa) * P + off;
      double f[KB];
#pragma unroll
      for (int n = 0; n < KB; ++n) f[n] = n < K ? fs[x * K + n] : 0.0;
#pragma unroll
      for (int j = 0; j < RT; ++j) {
        const double v = srow[tid + 256 * j];
#pragma unroll
        for (int n = 0; n < KB; ++n)
          if (n < K) acc[j][n] = fma(v, f[n], acc[j][n]);
      }
    }
    if (g == ng - 1) {
#pragma unroll
      for (int j = 0; j < RT; ++j) {
        const int r = tid + 256 * j;
        if (r < nr) {
          double* o = out + (b * R + r0 + r) * K;
#pragma unroll
          for (int n = 0; n < KB; ++n)
            if (n < K) o[n] = acc[j][n];
        }
      }
    }
    __syncthreads();
    if (tid == 0 && u + NS < nunits) issue(u + NS, st, pol);
  }
}
template <int CR, int XG, int NS>
void run_mc2(const double* X, int64_t B, int S, int64_t R, const double* F, int K, double* out, int per_sm) {
  const size_t smem = 8 * ((size_t)NS * XG * (CR + 2) + ((S * K + 1) & ~1)) + 8 * NS;
  cudaFuncSetAttribute(mc2_bulk<2, CR, XG, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t nch = B * ((R + CR - 1) / CR);
  int64_t g = 148 * per_sm;
  if (g > nch) g = nch;
  mc2_bulk<2, CR, XG, NS><<<(unsigned)g, 256, smem>>>(X, B, S, R, F, K, out);
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
  const int64_t s = 25, N6 = s * s * s * s * s * s;
  double *X, *F, *out, *ref, *flush;
  cudaMalloc(&X, 8 * N6);
  cudaMalloc(&F, 8 * 64 * 16);
  cudaMalloc(&out, 8 * N6 / s * 2 + 64);
  cudaMalloc(&ref, 8 * N6 / s * 2 + 64);
  const int64_t FL = 300ll << 20;
  cudaMalloc(&flush, FL);
  fill<<<4096, 256>>>(X, N6, 1);
  fill<<<4, 256>>>(F, 64 * 16, 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Shape { const char* name; int64_t B, S, R; };
  Shape shapes[] = {{"kc 25^5 x 25", s * s * s * s * s, s, 1},
                    {"mc 25 x 25^5", 1, s, s * s * s * s * s},
                    {"mc 25 x 25 x 25^4", s, s, s * s * s * s},
                    {"kc odd B (25^5 - 7)", s * s * s * s * s - 7, s, 1},
                    {"mc odd (1 x 25 x 25^5-3)", 1, s, s * s * s * s * s - 3}};
  const int K = 2;
  for (const Shape& sh : shapes) {
    const double bytes = 8.0 * (sh.B * sh.S * sh.R + sh.B * sh.R * K);
    printf("%s  (%.1f MB)\n", sh.name, bytes / 1e6);
    cppp::launch_ttm_simt(X, sh.B, sh.S, sh.R, F, K, ref, 0);
    cudaDeviceSynchronize();
    std::vector<double> hr(sh.B * sh.R * K), ho(hr.size());
    cudaMemcpy(hr.data(), ref, 8 * hr.size(), cudaMemcpyDeviceToHost);
    auto run = [&](const char* nm, auto&& f) {
      float tot = 0;
      const int reps = 6;
      cudaMemset(out, 0, 8 * hr.size());
      for (int i = 0; i < reps + 1; ++i) {
        cudaMemsetAsync(flush, i & 0xff, FL);
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (i >= 1) tot += ms;
      }
      cudaError_t e = cudaGetLastError();
      cudaMemcpy(ho.data(), out, 8 * ho.size(), cudaMemcpyDeviceToHost);
      double md = 0, mr = 0;
      for (size_t i = 0; i < ho.size(); ++i) {
        md = fmax(md, fabs(ho[i] - hr[i]));
        mr = fmax(mr, fabs(hr[i]));
      }
      const double us = 1e3 * tot / reps;
      printf("  %-26s %8.1f us %6.2f TB/s  maxdiff %.1e %s\n", nm, us, bytes / us / 1e6, md / mr,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    run("lib", [&] { cppp::launch_ttm_simt(X, sh.B, sh.S, sh.R, F, K, out, 0); });
    if (sh.R == 1) {
      run("kc_bulk CH256 NS2 x2", [&] { run_kc<256, 2>(X, sh.B, (int)sh.S, F, K, out, 2); });
      run("kc_bulk CH128 NS2 x4", [&] { run_kc<128, 2>(X, sh.B, (int)sh.S, F, K, out, 4); });
      run("kc_bulk CH256 NS1 x4", [&] { run_kc<256, 1>(X, sh.B, (int)sh.S, F, K, out, 4); });
      run("kc_bulk CH128 NS2 x3", [&] { run_kc<128, 2>(X, sh.B, (int)sh.S, F, K, out, 3); });
      run("kc_bulk CH256 NS2 x2 (again)", [&] { run_kc<256, 2>(X, sh.B, (int)sh.S, F, K, out, 2); });
    } else {
      run("mc2 CR1024 XG5 NS2 x2", [&] { run_mc2<1024, 5, 2>(X, sh.B, (int)sh.S, sh.R, F, K, out, 2); });
      run("mc2 CR512 XG5 NS2 x3", [&] { run_mc2<512, 5, 2>(X, sh.B, (int)sh.S, sh.R, F, K, out, 3); });
      run("mc2 CR1024 XG3 NS2 x3", [&] { run_mc2<1024, 3, 2>(X, sh.B, (int)sh.S, sh.R, F, K, out, 3); });
      run("mc2 CR2048 XG2 NS2 x2", [&] { run_mc2<2048, 2, 2>(X, sh.B, (int)sh.S, sh.R, F, K, out, 2); });
      run("mc2 CR1024 XG3 NS3 x2", [&] { run_mc2<1024, 3, 3>(X, sh.B, (int)sh.S, sh.R, F, K, out, 2); });
      run("mc2 CR512 XG5 NS2 x4", [&] { run_mc2<512, 5, 2>(X, sh.B, (int)sh.S, sh.R, F, K, out, 4); });
      run("mc2 CR1024 XG5 NS1 x4", [&] { run_mc2<1024, 5, 1>(X, sh.B, (int)sh.S, sh.R, F, K, out, 4); });
      run("mc2 CR2048 XG5 NS1 x2", [&] { run_mc2<2048, 5, 1>(X, sh.B, (int)sh.S, sh.R, F, K, out, 2); });
    }
  }
  return 0;
}
