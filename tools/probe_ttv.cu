// probe_ttv.cu — TTV configurations on the workload shapes (GB/s of algorithmic traffic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o tools/probe_ttv \
//        tools/probe_ttv.cu paper_1811_10573_b200/csrc/ttv.cu paper_1811_10573_b200/csrc/solve.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1811_10573_b200/csrc/internal.h"

// round-1 baseline: split-x partial sums + a combine kernel
__global__ void old_split(const double* __restrict__ P, int64_t S, int64_t RK, int K, int64_t total,
                          int xsplit, const double* __restrict__ F, double* __restrict__ part) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int p = blockIdx.y;
  if (e >= total) return;
  const int64_t b = e / RK, rk = e - b * RK;
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
__global__ void old_combine(const double* __restrict__ part, int64_t total, int xsplit,
                            double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < xsplit; ++p) s += part[p * total + e];
    out[e] = s;
  }
}

int main() {
  using namespace cppp;
  struct Shape { const char* name; int64_t B, S, R; int K; };
  Shape shapes[] = {{"C2 M0 (contract middle)", 400, 400, 1, 100},
                    {"C2 M1 (contract first)", 1, 400, 400, 100},
                    {"C4 level-2 (20^4 x 20 x 30)", 160000, 20, 1, 30},
                    {"C4 first-mode (20 x 20^4)", 1, 20, 160000, 30},
                    {"C3 lvl2 (100x100x100x50 mid)", 100, 100, 100, 50},
                    {"C5 lvl2 (256^3 x128 mid)", 256, 256, 256, 128}};
  double *P, *F, *out, *part;
  cudaMalloc(&P, 8ll * 256 * 256 * 256 * 128);
  cudaMalloc(&F, 8 * 256 * 128);
  cudaMalloc(&out, 8ll * 256 * 256 * 128);
  cudaMalloc(&part, 8ll * 16 * 400 * 400 * 100);
  cudaMemset(P, 0, 8ll * 256 * 256 * 256 * 128);
  cudaMemset(F, 0, 8 * 256 * 128);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (auto& sh : shapes) {
    const int64_t total = sh.B * sh.R * sh.K;
    const double bytes = 8.0 * (sh.B * sh.S * sh.R * sh.K + total);
    auto time = [&](auto fn) {
      for (int r = 0; r < 3; ++r) fn();
      cudaEventRecord(a);
      for (int r = 0; r < 10; ++r) fn();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      return ms * 1e3 / 10;
    };
    printf("%s: %.0f MB\n", sh.name, bytes / 1e6);
    if (total < 148ll * 2048) {
      for (int xs : {4, 8, 16}) {
        const double us = time([&] {
          dim3 g((unsigned)((total + 255) / 256), xs);
          old_split<<<g, 256>>>(P, sh.S, sh.R * sh.K, sh.K, total, xs, F, part);
          old_combine<<<(unsigned)((total + 255) / 256), 256>>>(part, total, xs, out);
        });
        printf("   old split+combine xs %2d: %7.1f us %6.0f GB/s\n", xs, us, bytes / us / 1e3);
      }
    }
    for (int V : {1, 2}) {
      if (V == 2 && sh.K % 2) continue;
      for (int U : {4, 8})
        for (int xs : {1, 2, 4, 8, 16}) {
          if (sh.S / xs < 4) continue;
          const double us = time([&] { launch_ttv_cfg(P, sh.B, sh.S, sh.R, sh.K, F, out, V, U, xs, 0); });
          printf("   V %d U %d xs %2d: %7.1f us %6.0f GB/s\n", V, U, xs, us, bytes / us / 1e3);
        }
    }
    const double us = time([&] { launch_ttv(P, sh.B, sh.S, sh.R, sh.K, F, out, nullptr, 0); });
    printf("   default: %7.1f us %6.0f GB/s   [%s]\n", us, bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
