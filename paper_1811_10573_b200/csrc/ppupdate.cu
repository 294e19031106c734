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

// Even K: every (x, y) pair of a term is a contiguous K-run op(x, y, 0..K).  A warp streams whole
// runs with 16-byte loads (lane owns k-pairs 2l and 64 + 2l) for x = x0 + warp, x0 + warp + 8, ...,
// four runs in flight per lane; the 8 warps' partial sums are reduced in shared memory in a fixed
// order.  Works for both operator orientations (only the run's base address differs).
constexpr int V2_WARPS = 8;

__global__ void __launch_bounds__(V2_WARPS * 32, 6)
    pp_update_partial_v2(PPUpdateArgs a, int xsplit) {
  const int64_t y = blockIdx.x;
  const int part = blockIdx.y;
  const int K = a.K;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k0 = 2 * lane, k1 = 64 + 2 * lane;
  const bool h0 = k0 < K, h1 = k1 < K;
  double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
  for (int ti = 0; ti < a.nterms; ++ti) {
    const PPTerm t = a.t[ti];
    const int64_t x0 = (t.nx * part) / xsplit;
    const int64_t x1 = (t.nx * (part + 1)) / xsplit;
    const double* opy = t.op + y * t.sy;
    int64_t x = x0 + w;
    for (; x + 3 * V2_WARPS < x1; x += 4 * V2_WARPS) {
      double2 o0[4], o1[4], d0[4], d1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t xx = x + u * V2_WARPS;
        const double* run = opy + xx * t.sx;
        const double* dr = t.dA + xx * K;
        o0[u] = h0 ? __ldcs(reinterpret_cast<const double2*>(run + k0)) : make_double2(0.0, 0.0);
        o1[u] = h1 ? __ldcs(reinterpret_cast<const double2*>(run + k1)) : make_double2(0.0, 0.0);
        d0[u] = h0 ? __ldg(reinterpret_cast<const double2*>(dr + k0)) : make_double2(0.0, 0.0);
        d1[u] = h1 ? __ldg(reinterpret_cast<const double2*>(dr + k1)) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc0.x = fma(o0[u].x, d0[u].x, acc0.x);
        acc0.y = fma(o0[u].y, d0[u].y, acc0.y);
        acc1.x = fma(o1[u].x, d1[u].x, acc1.x);
        acc1.y = fma(o1[u].y, d1[u].y, acc1.y);
      }
    }
    for (; x < x1; x += V2_WARPS) {
      const double* run = opy + x * t.sx;
      const double* dr = t.dA + x * K;
      if (h0) {
        const double2 o = __ldcs(reinterpret_cast<const double2*>(run + k0));
        const double2 d = __ldg(reinterpret_cast<const double2*>(dr + k0));
        acc0.x = fma(o.x, d.x, acc0.x);
        acc0.y = fma(o.y, d.y, acc0.y);
      }
      if (h1) {
        const double2 o = __ldcs(reinterpret_cast<const double2*>(run + k1));
        const double2 d = __ldg(reinterpret_cast<const double2*>(dr + k1));
        acc1.x = fma(o.x, d.x, acc1.x);
        acc1.y = fma(o.y, d.y, acc1.y);
      }
    }
  }
  __shared__ double red[V2_WARPS][128];
  if (h0) {
    red[w][k0] = acc0.x;
    red[w][k0 + 1] = acc0.y;
  }
  if (h1) {
    red[w][k1] = acc1.x;
    red[w][k1 + 1] = acc1.y;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < V2_WARPS; ++j) s += red[j][k];
    a.partial[(static_cast<int64_t>(part) * a.ny + y) * K + k] = s;
  }
}

// v3 (even K, 16-byte aligned runs): the same warp-per-run walk as v2, but every lane streams its
// own 16-byte chunks (k-pairs 2l and 64 + 2l) of op and dA through a private 6-stage cp.async
// ring in shared memory, so the bytes in flight live in smem instead of registers.
constexpr int V3_WARPS = 8;
constexpr int V3_STAGES = 6;

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool pred) {
  const int n = pred ? 16 : 0;   // src-size 0 fills zeros
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}

__global__ void __launch_bounds__(V3_WARPS * 32)
    pp_update_partial_v3(PPUpdateArgs a, int xsplit) {
  // per lane and stage: op pair 0, op pair 1, dA pair 0, dA pair 1 (4 x 16 B) — dynamic smem
  extern __shared__ __align__(16) double v3_smem[];
  double (*ring)[V3_WARPS * 32][8] = reinterpret_cast<double (*)[V3_WARPS * 32][8]>(v3_smem);
  __shared__ double red[V3_WARPS][128];
  const int64_t y = blockIdx.x;
  const int part = blockIdx.y;
  const int K = a.K;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k0 = 2 * lane, k1 = 64 + 2 * lane;
  const bool h0 = k0 < K, h1 = k1 < K;
  double acc0x = 0.0, acc0y = 0.0, acc1x = 0.0, acc1y = 0.0;
  for (int ti = 0; ti < a.nterms; ++ti) {
    const double* op = a.t[ti].op;
    const double* dA = a.t[ti].dA;
    const int64_t sx = a.t[ti].sx, nx = a.t[ti].nx;
    const int64_t x0 = (nx * part) / xsplit, x1 = (nx * (part + 1)) / xsplit;
    const double* opy = op + y * a.t[ti].sy;
    // runs of this warp: x = x0 + w + V3_WARPS * r, r = 0 .. nr-1
    const int64_t nr = (x1 - x0 - w + V3_WARPS - 1) / V3_WARPS;
    auto issue = [&](int64_t r) {
      const int s = static_cast<int>(r % V3_STAGES);
      const int64_t x = x0 + w + V3_WARPS * r;
      const double* run = opy + x * sx;
      const double* dr = dA + x * K;
      const uint32_t base =
          static_cast<uint32_t>(__cvta_generic_to_shared(&ring[s][threadIdx.x][0]));
      cp16(base, run + (h0 ? k0 : 0), h0);
      cp16(base + 16, run + (h1 ? k1 : 0), h1);
      cp16(base + 32, dr + (h0 ? k0 : 0), h0);
      cp16(base + 48, dr + (h1 ? k1 : 0), h1);
    };
    for (int64_t r = 0; r < V3_STAGES - 1; ++r) {
      if (r < nr) issue(r);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int64_t r = 0; r < nr; ++r) {
      if (r + V3_STAGES - 1 < nr) issue(r + V3_STAGES - 1);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(V3_STAGES - 1) : "memory");
      const double* sl = &ring[r % V3_STAGES][threadIdx.x][0];
      const double2 o0 = *reinterpret_cast<const double2*>(sl);
      const double2 o1 = *reinterpret_cast<const double2*>(sl + 2);
      const double2 d0 = *reinterpret_cast<const double2*>(sl + 4);
      const double2 d1 = *reinterpret_cast<const double2*>(sl + 6);
      acc0x = fma(o0.x, d0.x, acc0x);
      acc0y = fma(o0.y, d0.y, acc0y);
      acc1x = fma(o1.x, d1.x, acc1x);
      acc1y = fma(o1.y, d1.y, acc1y);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  if (h0) {
    red[w][k0] = acc0x;
    red[w][k0 + 1] = acc0y;
  }
  if (h1) {
    red[w][k1] = acc1x;
    red[w][k1 + 1] = acc1y;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < V3_WARPS; ++j) s += red[j][k];
    a.partial[(static_cast<int64_t>(part) * a.ny + y) * K + k] = s;
  }
}

__global__ void pp_update_combine(PPUpdateArgs a, int xsplit) {
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

int choose_xsplit(int64_t ny, int64_t max_nx) {
  // one full wave of resident CTAs (148 SMs x 2 CTAs of the 96 KB cp.async ring) when ny
  // allows it (no tail wave); keep >= 8 x per part
  const int64_t cap = 148 * 2;
  int64_t want = ny >= cap ? 1 : cap / ny;
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

cudaError_t launch_pp_update(const PPUpdateArgs& a, cudaStream_t st) {
  if (a.ny == 0) return cudaSuccess;
  if (a.K > NT) return cudaErrorInvalidValue;
  int64_t max_nx = 1;
  for (int i = 0; i < a.nterms; ++i) max_nx = a.t[i].nx > max_nx ? a.t[i].nx : max_nx;
  const int xsplit = choose_xsplit(a.ny, max_nx);
  dim3 grid((unsigned)a.ny, (unsigned)xsplit);
  bool aligned = (a.K % 2) == 0;
  for (int i = 0; i < a.nterms; ++i)
    aligned = aligned && (a.t[i].sx % 2 == 0) && (a.t[i].sy % 2 == 0) &&
              (reinterpret_cast<uintptr_t>(a.t[i].op) % 16 == 0) &&
              (reinterpret_cast<uintptr_t>(a.t[i].dA) % 16 == 0);
  constexpr int v3_smem = V3_STAGES * V3_WARPS * 32 * 8 * sizeof(double);
  static bool v3_attr = false;
  if (aligned && !v3_attr) {
    cudaError_t e = cudaFuncSetAttribute(pp_update_partial_v3,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, v3_smem);
    if (e != cudaSuccess) return e;
    v3_attr = true;
  }
  if (aligned) pp_update_partial_v3<<<grid, V3_WARPS * 32, v3_smem, st>>>(a, xsplit);
  else pp_update_partial<<<grid, NT, 0, st>>>(a, xsplit);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int64_t total = a.ny * a.K;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  pp_update_combine<<<blocks, 256, 0, st>>>(a, xsplit);
  note_launch();
  return cudaGetLastError();
}

}  // namespace cppp
