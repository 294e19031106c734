// probe_bar.cu — what does one pivot step of a 512-thread single-CTA kernel cost on B200?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(double* o, int n) { double a = threadIdx.x; for (int i = 0; i < n; ++i) a = fma(a, 1.0000001, 1e-9); if (a == 0.5) o[0] = a; }

template <int MODE>
__global__ void __launch_bounds__(512, 1) steps(double* out, int K) {
  __shared__ __align__(16) double rowb[2][128], colb[2][128];
  const int tid = threadIdx.x, l = tid & 127, rg = tid >> 7;
  double w[32];
#pragma unroll
  for (int v = 0; v < 32; ++v) w[v] = 1.0 + 1e-3 * (v + l);
  for (int j = 0; j < K; ++j) {
    const int b = j & 1;
    if (MODE >= 1 && l == j) {
#pragma unroll
      for (int v = 0; v < 32; ++v) colb[b][32 * rg + v] = w[v];
    }
    if (MODE >= 1 && rg == (j >> 5)) rowb[b][l] = w[0];
    __syncthreads();
    if (MODE >= 2) {
      const double p = rowb[b][j] + 2.0;
      const double inv = MODE >= 3 ? __drcp_rn(p) : 0.5;
      const double rl = rowb[b][l] * inv;
#pragma unroll
      for (int v = 0; v < 32; v += 2) {
        const double2 cc = *reinterpret_cast<const double2*>(&colb[b][32 * rg + v]);
        w[v] = fma(-cc.x, rl, w[v]);
        w[v + 1] = fma(-cc.y, rl, w[v + 1]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int v = 0; v < 32; ++v) s += w[v];
  out[tid] = s;
}

template <int MODE>
void run(double* o, int K) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  steps<MODE><<<1, 512>>>(o, K);
  cudaEventRecord(a);
  for (int r = 0; r < 20; ++r) steps<MODE><<<1, 512>>>(o, K);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("{\"mode\": %d, \"K\": %d, \"us\": %.2f, \"us_per_step\": %.4f}\n", MODE, K, ms * 1e3 / 20, ms * 1e3 / 20 / K);
}

int main() {
  double* o; cudaMalloc(&o, 8 * 1024);
  for (int r = 0; r < 40; ++r) spin<<<148 * 8, 256>>>(o, 1 << 16);
  cudaDeviceSynchronize();
  for (int K : {32, 128}) { run<0>(o, K); run<1>(o, K); run<2>(o, K); run<3>(o, K); }
  return 0;
}
