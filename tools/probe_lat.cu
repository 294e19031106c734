// probe_lat.cu — FP64 / shuffle / shared / barrier latencies on this GPU (cycles), to size the
// latency-bound small-solve kernels.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_lat tools/probe_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 1024;

__global__ void lat_kernel(double* out, long long* cyc, double seed) {
  __shared__ double sm[1024];
  __shared__ int chase[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) {
    sm[i] = 1.0 + i * 1e-9;
    chase[i] = (i + 33) & 1023;
  }
  __syncthreads();
  double a = seed + tid, b = 1.0000001, c = 1e-9;
  long long t0, t1;
  // 0: DFMA chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) a = fma(a, b, c);
  t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
  // 1: DMUL chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) a = a * b;
  t1 = clock64();
  if (tid == 0) cyc[1] = t1 - t0;
  // 2: DADD chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) a = a + c;
  t1 = clock64();
  if (tid == 0) cyc[2] = t1 - t0;
  // 3: shfl of a double (2 SHFL) chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) a = __shfl_sync(0xffffffffu, a, (tid + 1) & 31);
  t1 = clock64();
  if (tid == 0) cyc[3] = t1 - t0;
  // 4: LDS (int pointer chase)
  int p = tid & 1023;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) p = chase[p];
  t1 = clock64();
  if (tid == 0) cyc[4] = t1 - t0;
  // 5: LDS double dependent (address from value)
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) a = sm[(__double2int_rz(a) + i) & 1023];
  t1 = clock64();
  if (tid == 0) cyc[5] = t1 - t0;
  // 6: __drcp_rn chain
  double r = a + 2.0;
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) r = __drcp_rn(r) + 1.5;
  t1 = clock64();
  if (tid == 0) cyc[6] = t1 - t0;
  // 7: 1.0 / x chain (IEEE division)
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) r = 1.0 / r + 1.5;
  t1 = clock64();
  if (tid == 0) cyc[7] = t1 - t0;
  // 8: sqrt chain
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) r = sqrt(r) + 1.5;
  t1 = clock64();
  if (tid == 0) cyc[8] = t1 - t0;
  // 9: __syncthreads loop (blockDim threads)
  t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    __syncthreads();
  }
  t1 = clock64();
  if (tid == 0) cyc[9] = t1 - t0;
  // 10: STS then barrier then LDS of another warp's value (publish round trip)
  t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    if (tid == (i & 31)) sm[i & 1023] = a;
    __syncthreads();
    a = sm[i & 1023] * b;
  }
  t1 = clock64();
  if (tid == 0) cyc[10] = t1 - t0;
  // 11: 32 independent DFMA per thread, all warps (throughput)
  double v[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = a + k;
  t0 = clock64();
  for (int i = 0; i < 64; ++i) {
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = fma(v[k], b, c);
  }
  t1 = clock64();
  if (tid == 0) cyc[11] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int k = 0; k < 32; ++k) s += v[k];
  out[blockIdx.x * blockDim.x + tid] = a + r + p + s;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 64 * sizeof(long long));
  const char* names[] = {"dfma", "dmul", "dadd", "shfl64", "lds32 chase", "lds64 dep", "drcp_rn+add",
                         "div+add", "sqrt+add", "bar.sync", "sts-bar-lds", "32 dfma x64 (per iter)"};
  for (int threads : {32, 128, 512, 1024}) {
    for (int rep = 0; rep < 3; ++rep) lat_kernel<<<1, threads>>>(out, cyc, 0.5);
    cudaDeviceSynchronize();
    printf("threads %d:", threads);
    for (int k = 0; k < 12; ++k)
      printf("  %s %.1f", names[k], (double)cyc[k] / (k == 11 ? 64 : ITERS));
    printf("\n");
  }
  return 0;
}
