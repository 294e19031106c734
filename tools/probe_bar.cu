// probe_bar.cu — cost of one pivot step (publish, barrier, broadcast loads, rank-1 FMA update) of a
// single-CTA register-resident factorization on B200, for several thread/row layouts.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(double* o, int n) { double a = threadIdx.x; for (int i = 0; i < n; ++i) a = fma(a, 1.0000001, 1e-9); if (a == 0.5) o[0] = a; }

// T threads, R rows per thread (T*R/128 >= K), LDSV: 0 = no smem loads, 1 = LDS.128 pairs
template <int T, int R, int LDSV>
__global__ void __launch_bounds__(T, 1) steps(double* out, int K) {
  __shared__ __align__(16) double colb[2][128];
  const int tid = threadIdx.x, l = tid & 127, rg = tid / 128;
  double w[R];
#pragma unroll
  for (int v = 0; v < R; ++v) w[v] = 1.0 + 1e-3 * (v + l);
  if (tid < 256) (&colb[0][0])[tid] = 1e-3 * tid;
  __syncthreads();
  for (int j = 0; j < K; ++j) {
    const int b = j & 1;
    const double cl = colb[b][l] * 1e-3;
    if (LDSV) {
#pragma unroll
      for (int v = 0; v < R; v += 2) {
        const double2 cc = *reinterpret_cast<const double2*>(&colb[b][(R * rg + v) & 127]);
        w[v] = fma(-cc.x, cl, w[v]);
        w[v + 1] = fma(-cc.y, cl, w[v + 1]);
      }
    } else {
#pragma unroll
      for (int v = 0; v < R; ++v) w[v] = fma(-w[(v + 1) % R], cl, w[v]);
    }
    if (l == (j & 127)) colb[b ^ 1][rg] = w[0];
    __syncthreads();
  }
  double s = 0;
#pragma unroll
  for (int v = 0; v < R; ++v) s += w[v];
  out[tid] = s;
}

template <int T, int R, int LDSV>
void run(double* o, int K) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  steps<T, R, LDSV><<<1, T>>>(o, K);
  cudaEventRecord(a);
  for (int r = 0; r < 20; ++r) steps<T, R, LDSV><<<1, T>>>(o, K);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("{\"T\": %d, \"R\": %d, \"lds\": %d, \"K\": %d, \"us_per_step\": %.4f, \"cycles_per_step\": %.0f}\n", T, R, LDSV, K,
         ms * 1e3 / 20 / K, ms * 1e3 / 20 / K * 1965);
}

int main() {
  double* o; cudaMalloc(&o, 8 * 1024);
  for (int r = 0; r < 40; ++r) spin<<<148 * 8, 256>>>(o, 1 << 16);
  cudaDeviceSynchronize();
  const int K = 128;
  run<512, 32, 1>(o, K); run<512, 32, 0>(o, K);
  run<1024, 16, 1>(o, K); run<1024, 16, 0>(o, K);
  run<256, 64, 1>(o, K); run<256, 64, 0>(o, K);
  run<512, 8, 1>(o, K); run<512, 2, 1>(o, K);
  return 0;
}
