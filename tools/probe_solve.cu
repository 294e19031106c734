// probe_solve.cu — standalone timing/correctness probe of the small-solve kernels (solve.cu):
// Γ inverse (Gauss-Jordan / Jacobi), row solves, Gram reduce.  Prints one JSON line per K.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe_solve tools/probe_solve.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_1811_10573_b200/csrc/solve.cu"

__global__ void spin(double* o, int n) {
  double a = threadIdx.x;
  for (int i = 0; i < n; ++i) a = fma(a, 1.0000001, 1e-9);
  if (a == 0.5) o[0] = a;
}

int main() {
  using namespace cppp;
  {
    double* o;
    cudaMalloc(&o, 8);
    for (int r = 0; r < 40; ++r) spin<<<148 * 8, 256>>>(o, 1 << 16);   // ramp the SM clock
    cudaDeviceSynchronize();
  }
  for (int K : {10, 30, 50, 100, 128}) {
    const int N = 3, s = 400;
    std::vector<double> A(s * K), S(N * K * K);
    srand(1);
    for (auto& v : A) v = rand() / (double)RAND_MAX - 0.5;
    for (int m = 0; m < N; ++m)
      for (int i = 0; i < K; ++i)
        for (int j = 0; j < K; ++j) {
          double acc = 0;
          for (int y = 0; y < s; ++y) acc += A[y * K + i] * A[y * K + j] * (1.0 + 0.1 * m);
          S[m * K * K + i * K + j] = acc;
        }
    double *dS, *dG, *dP, *dV, *dM, *dA, *dD, *drs, *dgp, *dSn, *dn;
    int* dmode;
    cudaMalloc(&dS, 8 * N * K * K); cudaMalloc(&dG, 8 * K * K); cudaMalloc(&dP, 8 * K * K);
    cudaMalloc(&dV, 8 * K * K); cudaMalloc(&dmode, 4); cudaMalloc(&dM, 8 * s * K);
    cudaMalloc(&dA, 8 * s * K); cudaMalloc(&dD, 8 * s * K); cudaMalloc(&drs, 8 * s * 3);
    cudaMalloc(&dgp, 8 * 64 * K * K); cudaMalloc(&dSn, 8 * K * K); cudaMalloc(&dn, 8 * 3);
    cudaMemcpy(dS, S.data(), 8 * N * K * K, cudaMemcpyHostToDevice);
    cudaMemcpy(dM, A.data(), 8 * s * K, cudaMemcpyHostToDevice);
    cudaMemcpy(dA, A.data(), 8 * s * K, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    launch_gamma_factor(dS, N, 0, K, dG, dP, dmode, dV, 0);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) launch_gamma_factor(dS, N, 0, K, dG, dP, dmode, dV, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms_inv; cudaEventElapsedTime(&ms_inv, a, b);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) {
      launch_solve_rows(dM, dA, dA, dD, s, K, dG, dP, dmode, drs, dgp, 0);
      launch_gram_reduce(dgp, solve_row_blocks(s), K, dSn, drs, s, dn, 0);
    }
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms_rows; cudaEventElapsedTime(&ms_rows, a, b);
    std::vector<double> G(K * K), P(K * K);
    int mode = -1;
    cudaMemcpy(G.data(), dG, 8 * K * K, cudaMemcpyDeviceToHost);
    cudaMemcpy(P.data(), dP, 8 * K * K, cudaMemcpyDeviceToHost);
    cudaMemcpy(&mode, dmode, 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < K; ++i)
      for (int j = 0; j < K; ++j) {
        double acc = 0;
        for (int l = 0; l < K; ++l) acc += P[i * K + l] * P[j * K + l];
        err = fmax(err, fabs(acc - G[i * K + j]) / fabs(G[i * K + i]));
      }
    printf("{\"K\": %d, \"mode\": %d, \"inv_err\": %.3e, \"gamma_factor_us\": %.2f, \"rows_plus_reduce_us\": %.2f, \"cuda\": \"%s\"}\n",
           K, mode, err, ms_inv * 1e3 / 20, ms_rows * 1e3 / 20, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
