// fp64_peak.cu — measures the FP64 roofline denominators on this B200 (not in
// MEASURED_PEAKS.json, which only has bf16 and HBM): register-resident DMMA.8x8x4
// (mma.sync m8n8k4 f64) and DFMA throughput, burst (best of 10) and sustained (~3 s loop).
// Prints one JSON line.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;

__global__ void dmma_loop(double* out, int iters) {
  double acc[CHAINS][2];
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  for (int c = 0; c < CHAINS; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double acc[CHAINS];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  for (int c = 0; c < CHAINS; ++c) acc[c] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.0) out[0] = s;
}

template <typename F>
double run(F launch, double flops_per_launch, double seconds_target, double* best_out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  double best = 0;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double tf = flops_per_launch / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  *best_out = best;
  // sustained: back-to-back for ~seconds_target
  int n = 0;
  cudaEventRecord(a);
  float ms = 0;
  while (true) {
    launch();
    ++n;
    if (n % 20 == 0) {
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (ms > seconds_target * 1e3) break;
    }
  }
  return flops_per_launch * n / (ms * 1e-3) / 1e12;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 256, iters = 4096;
  const double dmma_flops = 2.0 * 256 * CHAINS * (double)iters * (threads / 32) * blocks;  // 8x8x4 MACs per warp-op
  const double dfma_flops = 2.0 * CHAINS * (double)iters * threads * blocks;
  double dmma_burst, dfma_burst;
  double dmma_sus = run([&] { dmma_loop<<<blocks, threads>>>(out, iters); }, dmma_flops, 3.0, &dmma_burst);
  double dfma_sus = run([&] { dfma_loop<<<blocks, threads>>>(out, iters); }, dfma_flops, 3.0, &dfma_burst);
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"sms\": %d, \"dmma_tflops_burst\": %.3f, \"dmma_tflops_sustained\": %.3f, "
         "\"dfma_tflops_burst\": %.3f, \"dfma_tflops_sustained\": %.3f, \"cuda\": \"%s\"}\n",
         sms, dmma_burst, dmma_sus, dfma_burst, dfma_sus, cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
