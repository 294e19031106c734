// gen.cu — device twin of synthgen (the seeded input generator).
// Same counter-based Philox4x32-10 stream and the same per-element formulas:
//   X_true(i) = Σ_r ((A0(i0,r)·A1(i1,r))·A2(i2,r))·…   summed r = 0..K-1 from 0.0, no FMA
//   Z(e)      = sqrt(-2 log(1 - res53(x0,x1))) · cos(2π res53(x2,x3)),  Philox(e, stream=N, seed)
//   X         = X_true + scale · Z,   scale = noise (absolute) or η‖X_true‖/‖Z‖ (relative, L19)
// Models P:343-344 (CP model) and P:1040-1063 (the paper's synthetic families).
#include "internal.h"

namespace cppp {
namespace {

struct Fac {
  const double* A[8];
};

__device__ __forceinline__ void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
    const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

__device__ __forceinline__ double res53(uint32_t a, uint32_t b) {
  const double hi = static_cast<double>(a >> 5), lo = static_cast<double>(b >> 6);
  return __dmul_rn(__dadd_rn(__dmul_rn(hi, 67108864.0), lo), 1.0 / 9007199254740992.0);
}

__device__ __forceinline__ double normal_at(uint64_t e, uint32_t stream, uint64_t seed) {
  uint32_t c[4] = {static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32), stream, 0u};
  philox(c, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  const double u1 = res53(c[0], c[1]), u2 = res53(c[2], c[3]);
  return __dmul_rn(sqrt(__dmul_rn(-2.0, log(__dadd_rn(1.0, -u1)))),
                   cos(__dmul_rn(6.283185307179586, u2)));
}

// One CTA per fibre (i0..i_{N-2}) of the slab; q_r = Π_{n<N-1} A_n(i_n, r) staged in smem.
__global__ void gen_kruskal_kernel(double* __restrict__ X, int N, Dims d, int K, Fac f,
                                   int64_t row_lo, int64_t nfib) {
  __shared__ double q[128];
  const int64_t sl = d.s[N - 1];
  for (int64_t fib = blockIdx.x; fib < nfib; fib += gridDim.x) {
    // decompose the local fibre index into (i0 - row_lo, i1, ..., i_{N-2})
    int64_t rem = fib;
    int64_t idx[8];
    for (int n = N - 2; n >= 1; --n) {
      idx[n] = rem % d.s[n];
      rem /= d.s[n];
    }
    idx[0] = rem + row_lo;
    __syncthreads();
    for (int r = threadIdx.x; r < K; r += blockDim.x) {
      double p = f.A[0][idx[0] * K + r];
      for (int n = 1; n < N - 1; ++n) p = __dmul_rn(p, f.A[n][idx[n] * K + r]);
      q[r] = p;
    }
    __syncthreads();
    const double* Al = f.A[N - 1];
    for (int64_t i = threadIdx.x; i < sl; i += blockDim.x) {
      double acc = 0.0;
      for (int r = 0; r < K; ++r) acc = __dadd_rn(acc, __dmul_rn(q[r], Al[i * K + r]));
      X[fib * sl + i] = acc;
    }
  }
}

constexpr int CHUNKS = 64;

// per (row, chunk): Σ X_true², Σ Z² ; partials[row][chunk][2]
__global__ void gen_rowsq_kernel(const double* __restrict__ X, int64_t rowlen, uint32_t stream,
                                 uint64_t seed, int64_t row_lo, double* partials) {
  __shared__ double shx[32], shz[32];
  const int64_t row = blockIdx.x / CHUNKS;
  const int ch = blockIdx.x % CHUNKS;
  const int64_t c0 = rowlen * ch / CHUNKS, c1 = rowlen * (ch + 1) / CHUNKS;
  double vx = 0.0, vz = 0.0;
  const uint64_t ebase = static_cast<uint64_t>(row_lo + row) * rowlen;
  for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
    const double x = X[row * rowlen + i];
    const double z = normal_at(ebase + i, stream, seed);
    vx = fma(x, x, vx);
    vz = fma(z, z, vz);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    vx += __shfl_xor_sync(0xffffffffu, vx, o);
    vz += __shfl_xor_sync(0xffffffffu, vz, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    shx[w] = vx;
    shz[w] = vz;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      a += shx[i];
      b += shz[i];
    }
    partials[(row * CHUNKS + ch) * 2 + 0] = a;
    partials[(row * CHUNKS + ch) * 2 + 1] = b;
  }
}

__global__ void gen_rowsq_final(const double* partials, int64_t nrows, int64_t row_lo,
                                double* rowsq_x, double* rowsq_z) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0, b = 0.0;
    for (int c = 0; c < CHUNKS; ++c) {
      a += partials[(r * CHUNKS + c) * 2 + 0];
      b += partials[(r * CHUNKS + c) * 2 + 1];
    }
    rowsq_x[row_lo + r] = a;
    rowsq_z[row_lo + r] = b;
  }
}

__global__ void gen_scale_kernel(const double* rowsq_x, const double* rowsq_z, int64_t s0,
                                 double eta, double* scale) {
  double a = 0.0, b = 0.0;
  for (int64_t r = 0; r < s0; ++r) {
    a += rowsq_x[r];
    b += rowsq_z[r];
  }
  scale[0] = eta * sqrt(a) / sqrt(b);
}

__global__ void gen_noise_add_kernel(double* __restrict__ X, int64_t n, uint64_t ebase,
                                     uint32_t stream, uint64_t seed, const double* scale_dev,
                                     double abs_scale) {
  const double sc = scale_dev ? scale_dev[0] : abs_scale;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n;
       l += (int64_t)gridDim.x * blockDim.x) {
    const double z = normal_at(ebase + l, stream, seed);
    X[l] = __dadd_rn(X[l], __dmul_rn(sc, z));
  }
}

}  // namespace

cudaError_t launch_gen_kruskal(double* X, int N, const int64_t* s, int K, const double* const* A_dev,
                               int64_t row_lo, int64_t row_hi, cudaStream_t st) {
  Dims d;
  Fac f;
  for (int n = 0; n < N; ++n) {
    d.s[n] = s[n];
    f.A[n] = A_dev[n];
  }
  int64_t nfib = row_hi - row_lo;
  for (int n = 1; n < N - 1; ++n) nfib *= s[n];
  if (nfib == 0) return cudaSuccess;
  int64_t blocks = nfib < 148 * 32 ? nfib : 148 * 32;
  gen_kruskal_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, N, d, K, f, row_lo, nfib);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_noise_rowsq(double* X, const int64_t* s, int N, uint64_t seed, int64_t row_lo,
                                   int64_t row_hi, double* rowsq_x, double* rowsq_z,
                                   double* partials, cudaStream_t st) {
  int64_t rowlen = 1;
  for (int n = 1; n < N; ++n) rowlen *= s[n];
  const int64_t nrows = row_hi - row_lo;
  if (nrows == 0) return cudaSuccess;
  gen_rowsq_kernel<<<(unsigned)(nrows * CHUNKS), 256, 0, st>>>(X, rowlen, (uint32_t)N, seed, row_lo,
                                                                partials);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  gen_rowsq_final<<<(unsigned)((nrows + 127) / 128), 128, 0, st>>>(partials, nrows, row_lo,
                                                                     rowsq_x, rowsq_z);
  note_launch();
  return cudaGetLastError();
}

size_t gen_partials_doubles(int64_t nrows) { return static_cast<size_t>(nrows) * CHUNKS * 2; }

cudaError_t launch_gen_scale(const double* rowsq_x, const double* rowsq_z, int64_t s0, double eta,
                             double* scale_dev, cudaStream_t st) {
  gen_scale_kernel<<<1, 1, 0, st>>>(rowsq_x, rowsq_z, s0, eta, scale_dev);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gen_noise_add(double* X, const int64_t* s, int N, uint64_t seed, int64_t row_lo,
                                 int64_t row_hi, const double* scale_dev, double abs_scale,
                                 cudaStream_t st) {
  int64_t rowlen = 1;
  for (int n = 1; n < N; ++n) rowlen *= s[n];
  const int64_t n = (row_hi - row_lo) * rowlen;
  if (n == 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  gen_noise_add_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, n, static_cast<uint64_t>(row_lo) * rowlen,
                                                          (uint32_t)N, seed, scale_dev, abs_scale);
  note_launch();
  return cudaGetLastError();
}

}  // namespace cppp
