// probe_small.cu — standalone timing of the fused small-mode kernel (launch_mode_small) against
// the factorization + row-solve + Gram chain it replaces, with per-phase clock64 deltas of CTA 0.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe_small tools/probe_small.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#define CPPP_PROBE_CYCLES 1
#include "../paper_1811_10573_b200/csrc/solve.cu"

int main() {
  using namespace cppp;
  struct Case { int K, N, rows; };
  for (Case cs : {Case{10, 3, 40}, Case{30, 6, 20}, Case{4, 6, 32}, Case{32, 4, 64}, Case{16, 3, 64}}) {
    const int K = cs.K, N = cs.N, s = cs.rows;
    std::vector<double> A(s * K), S(N * K * K);
    srand(1);
    for (auto& v : A) v = rand() / (double)RAND_MAX - 0.5;
    for (int m = 0; m < N; ++m)
      for (int i = 0; i < K; ++i)
        for (int j = 0; j < K; ++j) {
          double acc = 0;
          for (int y = 0; y < s; ++y) acc += A[y * K + i] * A[y * K + j] * (1.0 + 0.1 * m);
          S[m * K * K + i * K + j] = acc + (i == j ? 1.0 : 0.0);
        }
    const int ldt = solve_ld(K);
    double *dS, *dG, *dP, *dM, *dA, *dD, *drs, *dtp, *dSn, *dn, *dfit;
    unsigned* dcnt;
    int* dmode;
    cudaMalloc(&dS, 8 * N * K * K); cudaMalloc(&dG, 8 * ldt * ldt);
    cudaMalloc(&dP, 8 * (ldt * ldt + 4 * 32 * 33 + 128 * 128));
    cudaMemset(dG, 0, 8 * ldt * ldt); cudaMemset(dP, 0, 8 * (ldt * ldt + 4 * 32 * 33));
    cudaMalloc(&dmode, 4); cudaMalloc(&dM, 8 * s * K);
    cudaMalloc(&dA, 8 * s * K); cudaMalloc(&dD, 8 * s * K); cudaMalloc(&drs, 8 * s * 4);
    cudaMalloc(&dtp, 8 * gram_scratch_doubles()); cudaMalloc(&dSn, 8 * K * K); cudaMalloc(&dn, 8 * 3);
    cudaMalloc(&dfit, 8 * 2); cudaMalloc(&dcnt, 256); cudaMemset(dcnt, 0, 256);
    cudaMemcpy(dS, S.data(), 8 * N * K * K, cudaMemcpyHostToDevice);
    cudaMemcpy(dM, A.data(), 8 * s * K, cudaMemcpyHostToDevice);
    cudaMemcpy(dA, A.data(), 8 * s * K, cudaMemcpyHostToDevice);
    double* dV = dP + ldt * ldt + 4 * 32 * 33;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    auto chain = [&]() {
      launch_gamma_factor(dS, N, 0, K, dG, dP, dmode, dV, 0, 1e-12);
      launch_solve_rows(dM, dA, dA, dD, s, K, dG, dP, dmode, drs, 0);
      launch_gram(dA, s, K, dSn, drs, dn, dG, dfit, dtp, dcnt, 0);
    };
    auto fused = [&]() {
      launch_mode_small(dS, N, 0, K, dM, dA, dA, dD, s, dSn, dn, dfit, dG, dP, dV, 0, 1e-12);
    };
    for (int r = 0; r < 5; ++r) { chain(); fused(); }
    cudaDeviceSynchronize();
    float t[2];
    for (int v = 0; v < 2; ++v) {
      cudaEventRecord(a);
      for (int r = 0; r < 50; ++r) { if (v) fused(); else chain(); }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&t[v], a, b);
    }
    fused();
    cudaDeviceSynchronize();
    long long cyc[16];
    cudaMemcpyFromSymbol(cyc, g_probe_cycles, sizeof(cyc));
    printf("{\"K\": %d, \"N\": %d, \"rows\": %d, \"chain_us\": %.2f, \"fused_us\": %.2f, \"cycles\": "
           "[%lld, %lld, %lld, %lld, %lld, %lld, %lld, %lld], \"err\": \"%s\"}\n",
           K, N, s, t[0] * 1000 / 50, t[1] * 1000 / 50, cyc[10], cyc[11], cyc[12], cyc[1], cyc[2], cyc[13], cyc[14], cyc[15],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
