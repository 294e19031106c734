// probe_pp.cu — PP-update kernels on the C2 shape (2 terms, s = 400, K = 100, 256 MB of operators)
// against a plain streaming-read reduction over the same bytes (the achievable read ceiling).
#include <cstdio>
#include <vector>
#include "../paper_1811_10573_b200/csrc/ppupdate.cu"
namespace cppp { void note_launch() {} bool pdl_enabled() { return false; } }
__global__ void spin(double* o, int n) { double a = threadIdx.x; for (int i = 0; i < n; ++i) a = fma(a, 1.0000001, 1e-9); if (a == 0.5) o[0] = a; }
template <int U>
__global__ void stream_read(const double* __restrict__ x, int64_t n, double* out) {
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(x + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 1.2345) out[0] = acc;
}
__global__ void stream_read2(const double2* __restrict__ x, int64_t n2, double* out) {
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 v0 = __ldcs(x + i), v1 = __ldcs(x + i + stride), v2 = __ldcs(x + i + 2 * stride), v3 = __ldcs(x + i + 3 * stride);
    acc += v0.x + v0.y + v1.x + v1.y + v2.x + v2.y + v3.x + v3.y;
  }
  if (acc == 1.2345) out[0] = acc;
}
template <typename F> float timeit(F f, int reps = 10) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / reps;
}
int main() {
  using namespace cppp;
  double* o; cudaMalloc(&o, 8 * 1024);
  for (int r = 0; r < 40; ++r) spin<<<148 * 8, 256>>>(o, 1 << 16);
  const int64_t s = 400, K = 100;
  const int64_t opn = s * s * K;
  double *op1, *op2, *dA, *Mp, *out, *part;
  cudaMalloc(&op1, 8 * opn); cudaMalloc(&op2, 8 * opn); cudaMalloc(&dA, 8 * s * K);
  cudaMalloc(&Mp, 8 * s * K); cudaMalloc(&out, 8 * s * K); cudaMalloc(&part, 8 * 16 * s * K);
  cudaMemset(op1, 0, 8 * opn); cudaMemset(op2, 0, 8 * opn); cudaMemset(dA, 0, 8 * s * K); cudaMemset(Mp, 0, 8 * s * K);
  const double bytes = 2.0 * opn * 8;
  for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
    float ms = timeit([&] { stream_read<8><<<blocks, 256>>>(op1, 2 * opn > opn ? opn : opn, o); stream_read<8><<<blocks, 256>>>(op2, opn, o); });
    printf("{\"kernel\": \"stream_read U8\", \"blocks\": %d, \"GBps\": %.0f}\n", blocks, bytes / (ms * 1e-3) / 1e9);
    ms = timeit([&] { stream_read2<<<blocks, 256>>>((const double2*)op1, opn / 2, o); stream_read2<<<blocks, 256>>>((const double2*)op2, opn / 2, o); });
    printf("{\"kernel\": \"stream_read double2 U4\", \"blocks\": %d, \"GBps\": %.0f}\n", blocks, bytes / (ms * 1e-3) / 1e9);
  }
  PPUpdateArgs a;
  a.Mp = Mp; a.extra = nullptr; a.ny = s; a.K = K; a.out = out; a.partial = part; a.nterms = 2;
  for (int t = 0; t < 2; ++t) { a.t[t].op = t ? op2 : op1; a.t[t].dA = dA; a.t[t].sx = K; a.t[t].sy = s * K; a.t[t].nx = s; }
  float ms = timeit([&] { launch_pp_update(a, 0); });
  printf("{\"kernel\": \"launch_pp_update (partial+combine)\", \"GBps\": %.0f, \"us\": %.1f}\n", bytes / (ms * 1e-3) / 1e9, ms * 1e3);
  auto v4 = [&](auto kern, const char* name, int yg) {
    for (int xs : {2, 4, 6, 8}) {
      const int64_t items = ((s + yg - 1) / yg) * xs;
      for (int g : {148 * 2, 148 * 3, 148 * 4}) {
        int gg = items < g ? (int)items : g;
        float m = timeit([&] { kern<<<gg, 256>>>(a, xs); });
        printf("{\"kernel\": \"%s\", \"xsplit\": %d, \"grid\": %d, \"GBps\": %.0f, \"us\": %.1f}\n", name, xs, gg, bytes / (m * 1e-3) / 1e9, m * 1e3);
      }
    }
  };
  v4(pp_update_partial_v4<2, 2>, "v4 YG2 U2", 2);
  for (int t = 0; t < 2; ++t) { a.t[t].sx = s * K; a.t[t].sy = K; }   // native [x][y][k] orientation
  v4(pp_update_partial_v4<2, 2>, "v4 YG2 U2 strided", 2);
  v4(pp_update_partial_v4<4, 1>, "v4 YG4 U1 strided", 4);
  for (int t = 0; t < 2; ++t) { a.t[t].sx = K; a.t[t].sy = s * K; }
  v4(pp_update_partial_v4<4, 2>, "v4 YG4 U2", 4);
  v4(pp_update_partial_v4<2, 4>, "v4 YG2 U4", 2);
  v4(pp_update_partial_v4<4, 1>, "v4 YG4 U1", 4);
  ms = timeit([&] { pp_update_combine<<<(s * K + 255) / 256, 256>>>(a, 6); });
  printf("{\"kernel\": \"combine xsplit 6\", \"us\": %.1f}\n", ms * 1e3);
  printf("{\"cuda\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
