// probe_chain.cu — cycles per step of the substitution dependency chain (one warp), variants.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_chain tools/probe_chain.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int STEPS = 1024;
__global__ void chain(double* out, long long* cyc, const double* tab) {
  __shared__ double ts[STEPS + 64];
  for (int i = threadIdx.x; i < STEPS + 64; i += blockDim.x) ts[i] = tab[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double m = 1.0 + lane, src = m, acc = 0;
  long long t0, t1;
  // A: shfl -> mul -> fma -> select (the rows kernel)
  t0 = clock64();
  for (int j = 0; j < STEPS; ++j) {
    const int jj = j & 31;
    const double zj = __shfl_sync(0xffffffffu, src, jj) * ts[j];
    const double t = fma(-ts[j + 1], zj, m);
    src = t;
    m = lane == jj ? zj : (lane > jj ? t : m);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  acc += m;
  // B: shfl -> fma only
  t0 = clock64();
  for (int j = 0; j < STEPS; ++j) {
    const int jj = j & 31;
    src = fma(-ts[j + 1], __shfl_sync(0xffffffffu, src, jj), src);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  acc += src;
  // C: shfl only (double)
  t0 = clock64();
  for (int j = 0; j < STEPS; ++j) src = __shfl_sync(0xffffffffu, src, j & 31);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
  acc += src;
  // D: smem broadcast instead of shfl: lane jj writes, syncwarp, all read
  __shared__ double bc[32];
  t0 = clock64();
  for (int j = 0; j < STEPS; ++j) {
    const int jj = j & 31;
    if (lane == jj) bc[jj] = src;
    __syncwarp();
    src = fma(-ts[j + 1], bc[jj], src);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
  acc += src;
  // E: float shfl chain (1 SHFL)
  float f = lane;
  t0 = clock64();
  for (int j = 0; j < STEPS; ++j) f = __shfl_sync(0xffffffffu, f, j & 31) * 1.0001f + 0.5f;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
  // F: A plus the three later-block updates per step (the rows kernel's full step)
  double m1 = 2.0 + lane, m2 = 3.0 + lane, m3 = 4.0 + lane;
  src = m;
  t0 = clock64();
  for (int j = 0; j < STEPS; ++j) {
    const int jj = j & 31;
    const double* tr = ts + j + lane;
    const double zj = __shfl_sync(0xffffffffu, src, jj) * ts[j];
    const double t = fma(-tr[0], zj, m);
    src = t;
    m = lane == jj ? zj : (lane > jj ? t : m);
    m1 = fma(-tr[1], zj, m1);
    m2 = fma(-tr[2], zj, m2);
    m3 = fma(-tr[3], zj, m3);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
  acc += m + m1 + m2 + m3;
  // G: F with a runtime trip count and unroll 2 (as compiled in the kernel)
  const int nsteps = (int)tab[STEPS + 63] + STEPS;   // runtime (tab is zero)
  t0 = clock64();
#pragma unroll 2
  for (int j = 0; j < nsteps; ++j) {
    const int jj = j & 31;
    const double* tr = ts + j + lane;
    const double zj = __shfl_sync(0xffffffffu, src, jj) * ts[j];
    const double t = fma(-tr[0], zj, m);
    src = t;
    m = lane == jj ? zj : (lane > jj ? t : m);
    m1 = fma(-tr[1], zj, m1);
    m2 = fma(-tr[2], zj, m2);
    m3 = fma(-tr[3], zj, m3);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = t1 - t0;
  acc += m + m1 + m2 + m3;
  out[threadIdx.x] = acc + f;
}
int main() {
  double *out, *tab;
  long long* cyc;
  cudaMalloc(&out, 4096);
  cudaMalloc(&tab, 8 * (STEPS + 64));
  cudaMemset(tab, 0, 8 * (STEPS + 64));
  cudaMallocManaged(&cyc, 64);
  for (int w : {32, 128}) {
    for (int r = 0; r < 3; ++r) chain<<<1, w>>>(out, cyc, tab);
    cudaDeviceSynchronize();
    printf("threads %d: A shfl-mul-fma-sel %.1f  B shfl-fma %.1f  D smem-bcast-fma %.1f  F full step %.1f  G runtime-trip %.1f\n",
           w, cyc[0] / (double)STEPS, cyc[1] / (double)STEPS, cyc[3] / (double)STEPS, cyc[5] / (double)STEPS, cyc[6] / (double)STEPS);
  }
  return 0;
}
