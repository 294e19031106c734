// probe_ttm.cu — per-unit timeline of one DMMA TTM launch (C2 shape by default): which SM ran
// which unit when, tile durations, the tail.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o tools/probe_ttm \
//        tools/probe_ttm.cu paper_1811_10573_b200/csrc/solve.cu -lcuda
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#define CPPP_PROBE_TTM 1
#include "../paper_1811_10573_b200/csrc/ttm.cu"

__global__ void spin(double* o, int n) {
  double a = threadIdx.x;
  for (int i = 0; i < n; ++i) a = fma(a, 1.0000001, 1e-9);
  if (a == 0.5) o[0] = a;
}

int main(int argc, char** argv) {
  using namespace cppp;
  // probe_ttm B S R K   (X viewed as [B][S][R]; R == 1 contracts the last mode)
  const int64_t B = argc > 1 ? atoll(argv[1]) : 160000;
  const int64_t S = argc > 2 ? atoll(argv[2]) : 400;
  const int64_t R = argc > 3 ? atoll(argv[3]) : 1;
  const int K = argc > 4 ? atoi(argv[4]) : 100;
  const int mc = R > 1;
  double *X, *F, *out, *scr, *o;
  cudaMalloc(&X, 8 * B * S * R);
  cudaMalloc(&F, 8 * S * K);
  cudaMalloc(&out, 8 * B * R * K);
  const size_t nscr = ttm_scratch_doubles(S);
  cudaMalloc(&scr, 8 * nscr);
  cudaMemset(scr, 0, 8 * nscr);
  cudaMemset(X, 0, 8 * B * S * R);
  cudaMemset(F, 0, 8 * S * K);
  cudaMalloc(&o, 8);
  for (int r = 0; r < 20; ++r) spin<<<148 * 8, 256>>>(o, 1 << 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int r = 0; r < 3; ++r) launch_ttm(X, B, S, R, F, K, out, scr, false, 0);
  cudaEventRecord(a);
  launch_ttm(X, B, S, R, F, K, out, scr, false, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  static unsigned long long tr[1 << 16][3];
  cudaMemcpyFromSymbol(tr, g_ttm_trace, sizeof(tr));
  const int64_t ntiles = ((mc ? R : B) + 127) / 128;
  unsigned long long t0 = ~0ull, t1 = 0;
  int nunits = 0;
  for (int u = 0; u < (1 << 16); ++u) {
    if (tr[u][1] == 0) continue;   // stream-K unit ids are sparse
    t0 = std::min(t0, tr[u][1]);
    t1 = std::max(t1, tr[u][2]);
    ++nunits;
  }
  std::vector<double> per_sm_end(160, 0), per_sm_busy(160, 0), dur;
  for (int u = 0; u < (1 << 16); ++u) {
    if (tr[u][1] == 0) continue;
    const int sm = (int)tr[u][0];
    per_sm_end[sm] = std::max(per_sm_end[sm], (tr[u][2] - t0) * 1e-3);
    per_sm_busy[sm] += (tr[u][2] - tr[u][1]) * 1e-3;
    dur.push_back((tr[u][2] - tr[u][1]) * 1e-3);
  }
  std::vector<double> ends;
  for (int i = 0; i < 160; ++i)
    if (per_sm_end[i] > 0) ends.push_back(per_sm_end[i]);
  std::sort(ends.begin(), ends.end());
  std::vector<double> d2 = dur;
  std::sort(d2.begin(), d2.end());
  const double flops = 2.0 * B * R * S * K;
  const double bytes = 8.0 * (B * S * R + B * R * K);
  printf("B %lld S %lld R %lld K %d: %.1f us (event), span %.1f us, %.2f TF/s, %.0f GB/s; tiles %lld units %d SMs %zu\n",
         (long long)B, (long long)S, (long long)R, K, ms * 1e3, (t1 - t0) * 1e-3,
         flops / (ms * 1e-3) / 1e12, bytes / (ms * 1e-3) / 1e9, (long long)ntiles, nunits, ends.size());
  printf("  SM end times: min %.1f p10 %.1f median %.1f p90 %.1f max %.1f us\n", ends.front(),
         ends[ends.size() / 10], ends[ends.size() / 2], ends[ends.size() * 9 / 10], ends.back());
  printf("  unit durations: min %.2f median %.2f p90 %.2f max %.2f us; first unit %.2f us\n", d2.front(),
         d2[d2.size() / 2], d2[d2.size() * 9 / 10], d2.back(), dur[0]);
  double first_start = 1e9, last_first_start = 0;
  for (int u = 0; u < std::min(nunits, 148); ++u) {
    first_start = std::min(first_start, (tr[u][1] - t0) * 1e-3);
    last_first_start = std::max(last_first_start, (tr[u][1] - t0) * 1e-3);
  }
  printf("  first-wave starts: %.2f .. %.2f us\n", first_start, last_first_start);
  printf("  %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
