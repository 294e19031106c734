// probe_solve.cu — standalone timing/correctness probe of the small-solve kernels (solve.cu):
// Γ inverse (Gauss-Jordan / Jacobi), row solves, Gram reduce.  Prints one JSON line per K.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe_solve tools/probe_solve.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#define CPPP_PROBE_CYCLES 1
#include "../paper_1811_10573_b200/csrc/solve.cu"

__global__ void spin(double* o, int n) {
  double a = threadIdx.x;
  for (int i = 0; i < n; ++i) a = fma(a, 1.0000001, 1e-9);
  if (a == 0.5) o[0] = a;
}

int main(int argc, char** argv) {
  const int only_k = argc > 1 ? atoi(argv[1]) : 0;
  using namespace cppp;
  {
    double* o;
    cudaMalloc(&o, 8);
    for (int r = 0; r < 40; ++r) spin<<<148 * 8, 256>>>(o, 1 << 16);   // ramp the SM clock
    cudaDeviceSynchronize();
  }
  for (int K : {10, 30, 50, 100, 128}) {
    if (only_k && K != only_k) continue;
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
    const int ldt = solve_ld(K);
    double *dS, *dG, *dP, *dV, *dM, *dA, *dD, *drs, *dtp, *dSn, *dn, *dfit;
    unsigned* dcnt;
    int* dmode;
    cudaMalloc(&dS, 8 * N * K * K); cudaMalloc(&dG, 8 * ldt * ldt); cudaMalloc(&dP, 8 * (ldt * ldt + 4 * 32 * 33));
    cudaMemset(dG, 0, 8 * ldt * ldt); cudaMemset(dP, 0, 8 * (ldt * ldt + 4 * 32 * 33));
    cudaMalloc(&dV, 8 * K * K); cudaMalloc(&dmode, 4); cudaMalloc(&dM, 8 * s * K);
    cudaMalloc(&dA, 8 * s * K); cudaMalloc(&dD, 8 * s * K); cudaMalloc(&drs, 8 * s * 4);
    cudaMalloc(&dtp, 8 * gram_scratch_doubles()); cudaMalloc(&dSn, 8 * K * K); cudaMalloc(&dn, 8 * 3);
    cudaMalloc(&dfit, 8 * 2); cudaMalloc(&dcnt, 256); cudaMemset(dcnt, 0, 256);
    cudaMemcpy(dS, S.data(), 8 * N * K * K, cudaMemcpyHostToDevice);
    cudaMemcpy(dM, A.data(), 8 * s * K, cudaMemcpyHostToDevice);
    cudaMemcpy(dA, A.data(), 8 * s * K, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    launch_gamma_factor(dS, N, 0, K, dG, dP, dmode, dV, 0, 1e-12);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) launch_gamma_factor(dS, N, 0, K, dG, dP, dmode, dV, 0, 1e-12);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms_inv; cudaEventElapsedTime(&ms_inv, a, b);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) launch_solve_rows(dM, dA, dA, dD, s, K, dG, dP, dmode, drs, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms_rows; cudaEventElapsedTime(&ms_rows, a, b);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) launch_gram(dA, s, K, dSn, drs, dn, dG, dfit, dtp, dcnt, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms_gram; cudaEventElapsedTime(&ms_gram, a, b);
    // one solve from the original M to check A_new Γ = M
    cudaMemcpy(dA, A.data(), 8 * s * K, cudaMemcpyHostToDevice);
    launch_solve_rows(dM, dA, dA, dD, s, K, dG, dP, dmode, drs, 0);
    std::vector<double> An(s * K);
    cudaMemcpy(An.data(), dA, 8 * s * K, cudaMemcpyDeviceToHost);
    launch_gamma_factor(dS, N, 0, K, dG, dP, dmode, dV, 0, 1e-12);
    cudaDeviceSynchronize();
    long long cyc[16];
    cudaMemcpyFromSymbol(cyc, g_probe_cycles, sizeof(cyc));
    std::vector<double> Tp(K * ldt), Gh(K * ldt);
    cudaMemcpy(Tp.data(), dP, 8 * K * ldt, cudaMemcpyDeviceToHost);
    cudaMemcpy(Gh.data(), dG, 8 * K * ldt, cudaMemcpyDeviceToHost);
    // L from the packed factor: lower part = L, diag = 1/Tp[j][j]; check L Lᵀ = Γ and Tp upper = Lᵀ
    double lerr = 0, terr = 0;
    for (int i = 0; i < K; ++i)
      for (int j = 0; j <= i; ++j) {
        double acc = 0;
        for (int p = 0; p <= j; ++p) {
          const double li = p == i ? 1.0 / Tp[i * ldt + i] : Tp[i * ldt + p];
          const double lj = p == j ? 1.0 / Tp[j * ldt + j] : Tp[j * ldt + p];
          acc += li * lj;
        }
        lerr = fmax(lerr, fabs(acc - Gh[i * ldt + j]) / Gh[i * ldt + i]);
        if (j < i) terr = fmax(terr, fabs(Tp[j * ldt + i] - Tp[i * ldt + j]));
      }
    printf("small-factor cycles: hadamard %lld loop %lld tp %lld inverse %lld\n", cyc[6], cyc[7], cyc[8], cyc[9]);
    printf("K %d: LLt err %.3e, upper-vs-lower %.3e; cycles chol setup %lld total %lld; rows staged %lld subst %lld total %lld; gram loop %lld\n",
           K, lerr, terr, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5]);
    std::vector<double> G(K * ldt);
    int mode = -1;
    cudaMemcpy(G.data(), dG, 8 * K * ldt, cudaMemcpyDeviceToHost);
    cudaMemcpy(&mode, dmode, 4, cudaMemcpyDeviceToHost);
    double err = 0, nrm = 0;
    for (int y = 0; y < s; ++y)
      for (int c = 0; c < K; ++c) {
        double acc = 0;
        for (int l = 0; l < K; ++l) acc += An[y * K + l] * G[l * ldt + c];
        err = fmax(err, fabs(acc - A[y * K + c]));
        nrm = fmax(nrm, fabs(A[y * K + c]));
      }
    printf("{\"K\": %d, \"mode\": %d, \"resid\": %.3e, \"gamma_factor_us\": %.2f, \"rows_us\": %.2f, \"gram_us\": %.2f, \"cuda\": \"%s\"}\n",
           K, mode, err / nrm, ms_inv * 1e3 / 20, ms_rows * 1e3 / 20, ms_gram * 1e3 / 20, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
