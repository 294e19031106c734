// ppupdate.cu — the pairwise-perturbation update (Alg. 3):
//
//   M~^(n)(y,k) = M_p^(n)(y,k) + Σ_{i≠n} Σ_x M_p^(i,n)(x,y,k) · dA^(i)(x,k)
//
// All N-1 operator terms of one mode in ONE launch (plus a tiny deterministic combine).  The
// operators are stored once per unordered pair as [x_min][x_max][k] (L5), so a term reads its
// operator either as [x][y][k] (i < n: stride of x = s_n K) or [y][x][k] (i > n: stride K).
// HBM-bound: 8 bytes read per 2 flops; the operator bytes dominate (N(N-1) s² K per sweep).
//
// Work split: CTA (y, part) reduces a contiguous x-range of every term for one output row y.
// Threads are laid out as [G][K] (G = 256 / K x-groups), so each thread keeps one k and walks
// x with stride G: every load instruction of the CTA touches G contiguous K-runs.  The G
// partial sums of each k are reduced in shared memory in a fixed order, the `part` partials in
// the combine kernel in a fixed order: bit-reproducible run to run.
#include "internal.h"

namespace cppp {
namespace {

constexpr int NT = 256;

__global__ void __launch_bounds__(NT)
    pp_update_partial(PPUpdateArgs a, int xsplit) {
  pdl_wait();
  const int64_t y = blockIdx.x;
  const int part = blockIdx.y;
  const int K = a.K;
  const int G = NT / K;
  const int tid = threadIdx.x;
  const int k = tid % K;
  const int xg = tid / K;
  double acc = 0.0;
  if (xg < G) {
    for (int ti = 0; ti < a.nterms; ++ti) {
      const PPTerm t = a.t[ti];
      const int64_t x0 = (t.nx * part) / xsplit;
      const int64_t x1 = (t.nx * (part + 1)) / xsplit;
      const double* op = t.op + y * t.sy + k;
      const double* d = t.dA + k;
      int64_t x = x0 + xg;
      for (; x + 7 * G < x1; x += 8 * G) {
        double o[8], dd[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          o[u] = __ldcs(op + (x + u * G) * t.sx);
          dd[u] = __ldg(d + (x + u * G) * K);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = fma(o[u], dd[u], acc);
      }
      for (; x < x1; x += G) acc = fma(__ldcs(op + x * t.sx), __ldg(d + x * K), acc);
    }
  }
  __shared__ double red[NT];
  red[tid] = acc;
  __syncthreads();
  if (tid < K) {
    double s = 0.0;
    for (int j = 0; j < G; ++j) s += red[j * K + tid];
    a.partial[(static_cast<int64_t>(part) * a.ny + y) * K + tid] = s;
  }
}

// v4 (even K, 16-byte aligned K-runs; both operator orientations): an item is (group of YG output rows, x-part).  For
// each x the warp loads the dA row pair once and the YG operator runs op(y, x, :) of its rows,
// U x-steps at a time, so YG*U 16-byte loads of operator data are in flight per lane.
template <int YG, int U>
__global__ void __launch_bounds__(256, (YG * U > 8) ? 2 : 3)
    pp_update_partial_v4(PPUpdateArgs a, int xsplit) {
  pdl_wait();
  __shared__ double red[8][YG][128];
  const int64_t ngroups = (a.ny + YG - 1) / YG;
  const int64_t items = ngroups * xsplit;
  const int K = a.K;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k0 = 2 * lane, k1 = 64 + 2 * lane;
  const bool h0 = k0 < K, h1 = k1 < K;
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int part = static_cast<int>(item / ngroups);
    const int64_t y0 = (item - static_cast<int64_t>(part) * ngroups) * YG;
    double acc[YG][4];
#pragma unroll
    for (int g = 0; g < YG; ++g) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.0;
    for (int ti = 0; ti < a.nterms; ++ti) {
      const PPTerm t = a.t[ti];
      const int64_t x0 = (t.nx * part) / xsplit, x1 = (t.nx * (part + 1)) / xsplit;
      const double* opb[YG];
#pragma unroll
      for (int g = 0; g < YG; ++g) opb[g] = t.op + min(y0 + g, a.ny - 1) * t.sy;
      int64_t x = x0 + w;
      for (; x + (U - 1) * 8 < x1; x += U * 8) {
        double2 o[U][YG][2], d[U][2];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t xx = x + u * 8;
          const double* dr = t.dA + xx * K;
          d[u][0] = h0 ? __ldg(reinterpret_cast<const double2*>(dr + k0)) : make_double2(0.0, 0.0);
          d[u][1] = h1 ? __ldg(reinterpret_cast<const double2*>(dr + k1)) : make_double2(0.0, 0.0);
#pragma unroll
          for (int g = 0; g < YG; ++g) {
            const double* run = opb[g] + xx * t.sx;
            o[u][g][0] = h0 ? __ldcs(reinterpret_cast<const double2*>(run + k0)) : make_double2(0.0, 0.0);
            o[u][g][1] = h1 ? __ldcs(reinterpret_cast<const double2*>(run + k1)) : make_double2(0.0, 0.0);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int g = 0; g < YG; ++g) {
            acc[g][0] = fma(o[u][g][0].x, d[u][0].x, acc[g][0]);
            acc[g][1] = fma(o[u][g][0].y, d[u][0].y, acc[g][1]);
            acc[g][2] = fma(o[u][g][1].x, d[u][1].x, acc[g][2]);
            acc[g][3] = fma(o[u][g][1].y, d[u][1].y, acc[g][3]);
          }
      }
      for (; x < x1; x += 8) {
        const double* dr = t.dA + x * K;
        const double2 d0 = h0 ? __ldg(reinterpret_cast<const double2*>(dr + k0)) : make_double2(0.0, 0.0);
        const double2 d1 = h1 ? __ldg(reinterpret_cast<const double2*>(dr + k1)) : make_double2(0.0, 0.0);
#pragma unroll
        for (int g = 0; g < YG; ++g) {
          const double* run = opb[g] + x * t.sx;
          const double2 o0 = h0 ? __ldcs(reinterpret_cast<const double2*>(run + k0)) : make_double2(0.0, 0.0);
          const double2 o1 = h1 ? __ldcs(reinterpret_cast<const double2*>(run + k1)) : make_double2(0.0, 0.0);
          acc[g][0] = fma(o0.x, d0.x, acc[g][0]);
          acc[g][1] = fma(o0.y, d0.y, acc[g][1]);
          acc[g][2] = fma(o1.x, d1.x, acc[g][2]);
          acc[g][3] = fma(o1.y, d1.y, acc[g][3]);
        }
      }
    }
#pragma unroll
    for (int g = 0; g < YG; ++g) {
      if (h0) {
        red[w][g][k0] = acc[g][0];
        red[w][g][k0 + 1] = acc[g][1];
      }
      if (h1) {
        red[w][g][k1] = acc[g][2];
        red[w][g][k1 + 1] = acc[g][3];
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < YG * K; e += blockDim.x) {
      const int g = e / K, k = e - g * K;
      if (y0 + g < a.ny) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) s += red[j][g][k];
        a.partial[(static_cast<int64_t>(part) * a.ny + y0 + g) * K + k] = s;
      }
    }
    __syncthreads();
  }
}

__global__ void pp_update_combine(PPUpdateArgs a, int xsplit) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = a.ny * a.K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int p = 0; p < xsplit; ++p) v += a.partial[p * total + e];
    double m = a.Mp ? a.Mp[e] : 0.0;   // Mp may be null (sharded exchange terms)
    if (a.extra) m += a.extra[e];
    a.out[e] = m + v;
  }
}

// The combine of a PP update split in two partial launches (the early terms computed during the
// previous mode's window, the late term after it): out = (M_p [+ extra]) + (Σ early parts + Σ late
// parts), every sum in a fixed order.
__global__ void pp_update_combine2(PPUpdateArgs a, const double* __restrict__ pE, int xsE,
                                   const double* __restrict__ pL, int xsL) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = a.ny * a.K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int p = 0; p < xsE; ++p) v += pE[p * total + e];
    for (int p = 0; p < xsL; ++p) v += pL[p * total + e];
    double m = a.Mp ? a.Mp[e] : 0.0;
    if (a.extra) m += a.extra[e];
    a.out[e] = m + v;
  }
}

int choose_xsplit(int64_t ny, int64_t max_nx) {
  // the aligned kernel walks (y, part) items grid-stride with 4 CTAs/SM: make ~4 items per CTA
  // slot; keep >= 8 x per part
  const int64_t cap = 148 * 4 * 4;
  int64_t want = (cap + ny - 1) / ny;
  const int64_t lim = max_nx / 8;
  if (want > lim) want = lim;
  if (want > 16) want = 16;
  if (want < 1) want = 1;
  return static_cast<int>(want);
}

}  // namespace

size_t pp_update_scratch_doubles(int64_t ny, int K, int64_t max_nx) {
  (void)max_nx;
  return static_cast<size_t>(16) * ny * K;
}

cudaError_t launch_pp_partial(const PPUpdateArgs& a, double* partial, int grid_cap, int* xs_used,
                              cudaStream_t st);

cudaError_t launch_pp_update(const PPUpdateArgs& a, cudaStream_t st) {
  if (a.ny == 0) return cudaSuccess;
  if (a.K > NT) return cudaErrorInvalidValue;
  int64_t max_nx = 1;
  for (int i = 0; i < a.nterms; ++i) max_nx = a.t[i].nx > max_nx ? a.t[i].nx : max_nx;
  const int xsplit = choose_xsplit(a.ny, max_nx);
  bool aligned = (a.K % 2) == 0;
  for (int i = 0; i < a.nterms; ++i)
    aligned = aligned && (a.t[i].sx % 2 == 0) && (a.t[i].sy % 2 == 0) &&
              (reinterpret_cast<uintptr_t>(a.t[i].op) % 16 == 0) &&
              (reinterpret_cast<uintptr_t>(a.t[i].dA) % 16 == 0);
  int xs_used = xsplit;
  if (aligned) {
    // v4 sizing (tools/probe_pp, C2 shape): ~3 items of (2 rows, x-part) per SM, one per CTA
    const int64_t ngroups = (a.ny + 1) / 2;
    int64_t xs = (148 * 3 + ngroups / 2) / ngroups;
    const int64_t lim = max_nx / 16;
    if (xs > lim) xs = lim;
    if (xs > 16) xs = 16;
    if (xs < 1) xs = 1;
    xs_used = static_cast<int>(xs);
    const int64_t items = ngroups * xs;
    const int64_t grid = items < 148 * 3 ? items : 148 * 3;
    // launched without a programmatic edge: a PP sweep's side-stream factorization must be able
    // to take an SM before these CTAs occupy every SM (measured: +23 µs per mode on C2 otherwise)
    pp_update_partial_v4<2, 2><<<(unsigned)grid, 256, 0, st>>>(a, xs_used);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  } else {
    dim3 grid((unsigned)a.ny, (unsigned)xsplit);
    pp_update_partial<<<grid, NT, 0, st>>>(a, xsplit);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  note_launch();
  int64_t total = a.ny * a.K;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  cudaError_t e = launch_pdl(pp_update_combine, dim3(blocks), dim3(256), 0, st, a, xs_used);
  note_launch();
  return e;
}

// The partial kernel alone, into `partial` (>= 16 ny K doubles); *xs_used = its x parts (0 when
// there are no terms: nothing launched).  grid_cap > 0 caps the CTAs (a side-stream launch that
// must leave room on every SM).
cudaError_t launch_pp_partial(const PPUpdateArgs& a, double* partial, int grid_cap, int* xs_used,
                              cudaStream_t st) {
  *xs_used = 0;
  if (a.ny == 0 || a.nterms == 0) return cudaSuccess;
  if (a.K > NT) return cudaErrorInvalidValue;
  PPUpdateArgs b = a;
  b.partial = partial;
  int64_t max_nx = 1;
  for (int i = 0; i < b.nterms; ++i) max_nx = b.t[i].nx > max_nx ? b.t[i].nx : max_nx;
  bool aligned = (b.K % 2) == 0;
  for (int i = 0; i < b.nterms; ++i)
    aligned = aligned && (b.t[i].sx % 2 == 0) && (b.t[i].sy % 2 == 0) &&
              (reinterpret_cast<uintptr_t>(b.t[i].op) % 16 == 0) &&
              (reinterpret_cast<uintptr_t>(b.t[i].dA) % 16 == 0);
  if (aligned) {
    const int64_t ngroups = (b.ny + 1) / 2;
    int64_t xs = (148 * 3 + ngroups / 2) / ngroups;
    const int64_t lim = max_nx / 16;
    if (xs > lim) xs = lim;
    if (xs > 16) xs = 16;
    if (xs < 1) xs = 1;
    const int64_t items = ngroups * xs;
    int64_t grid = items < 148 * 3 ? items : 148 * 3;
    if (grid_cap > 0 && grid > grid_cap) grid = grid_cap;
    pp_update_partial_v4<2, 2><<<(unsigned)grid, 256, 0, st>>>(b, static_cast<int>(xs));
    *xs_used = static_cast<int>(xs);
  } else {
    const int xsplit = choose_xsplit(b.ny, max_nx);
    dim3 grid((unsigned)b.ny, (unsigned)xsplit);
    pp_update_partial<<<grid, NT, 0, st>>>(b, xsplit);
    *xs_used = xsplit;
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pp_combine2(const PPUpdateArgs& a, const double* pE, int xsE, const double* pL,
                               int xsL, cudaStream_t st) {
  if (a.ny == 0) return cudaSuccess;
  const int64_t total = a.ny * a.K;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  cudaError_t e = launch_pdl(pp_update_combine2, dim3(blocks), dim3(256), 0, st, a, pE, xsE, pL, xsL);
  note_launch();
  return e;
}

}  // namespace cppp
