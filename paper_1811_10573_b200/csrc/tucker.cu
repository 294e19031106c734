// tucker.cu — the PP-Tucker contraction path (include/cppp_tucker.h).
//
// Tucker-ALS needs, per mode n, the TTMc Y^(n) = X ×_{m≠n} A^(m)T; pairwise
// perturbation replaces it by Y~^(n) = Y_p^(n) + Σ_i Y_p^(i,n) ×_i dA^(i)T with the
// operators Y_p^(i,j) of Def. 3.2.  Every edge of both trees is one mode product
// X ×_u A^(u)T, i.e. the same GEMM as the CP path's first level — out[b][r][z] = Σ_x P[b][x][r]
// A[x][z] with the parent viewed as [B][S][R] — so every contraction here runs on the DMMA
// kernel of ttm.cu (SIMT kernel for odd shapes).
//
// Layouts.  The GEMM appends z last, so an intermediate keeps its uncontracted x axes in mode
// order followed by its z axes in contraction order (a Lay records the memory order).  Results
// handed out (Y^(n), operators, Y_p^(n), Y~^(n)) are permuted into the canonical layout (every
// mode in place) by one gather kernel; those tensors are the small ones (s² R^(N-2) at
// most), so the permutation costs one pass over them.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "cppp_tucker.h"
#include "internal.h"

namespace cppp {
namespace {

struct Lay {
  int n = 0;
  int mode[CPPP_MAX_ORDER_];
  bool z[CPPP_MAX_ORDER_];
};

struct PermArgs {
  int nd;
  int64_t odim[CPPP_MAX_ORDER_];
  int64_t istride[CPPP_MAX_ORDER_];
};

// out (canonical, row-major over odim) [+]= in gathered through istride
__global__ void permute_kernel(const double* __restrict__ in, double* __restrict__ out, PermArgs p,
                               int64_t total, int accumulate) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e, off = 0;
    for (int a = p.nd - 1; a >= 0; --a) {
      const int64_t i = r % p.odim[a];
      r /= p.odim[a];
      off += i * p.istride[a];
    }
    const double v = in[off];
    out[e] = accumulate ? out[e] + v : v;
  }
}

bool dev_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace
}  // namespace cppp

using cppp::Lay;

struct tk_ctx {
  int N = 0;
  int64_t s[CPPP_MAX_ORDER] = {};
  int R[CPPP_MAX_ORDER] = {};
  unsigned flags = 0;
  cudaStream_t st = nullptr;
  const double* X = nullptr;
  double* Xown = nullptr;
  double* A[CPPP_MAX_ORDER] = {};
  double* Ap[CPPP_MAX_ORDER] = {};
  double* dA[CPPP_MAX_ORDER] = {};
  double* ops[CPPP_MAX_ORDER][CPPP_MAX_ORDER] = {};   // canonical Y_p^(i,j), i < j
  double* Yp[CPPP_MAX_ORDER] = {};                    // canonical Y_p^(n)
  double* Fpad = nullptr;                              // TTM scratch (padded factor, scheduler)
  double* out = nullptr;                               // canonical result scratch (max Y^(n))
  bool factors_set = false, ops_valid = false;
  std::string err;
  std::vector<void*> owned;
};

namespace {

cppp_status tfail(tk_ctx* c, cppp_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return s;
}

#define TKCU(c, expr)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess) return tfail(c, CPPP_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)
#define TKST(expr)                     \
  do {                                 \
    cppp_status s_ = (expr);           \
    if (s_ != CPPP_OK) return s_;      \
  } while (0)

int64_t axis_dim(const tk_ctx* c, const Lay& l, int a) {
  return l.z[a] ? c->R[l.mode[a]] : c->s[l.mode[a]];
}
int64_t lay_elems(const tk_ctx* c, const Lay& l) {
  int64_t e = 1;
  for (int a = 0; a < l.n; ++a) e *= axis_dim(c, l, a);
  return e;
}
Lay root_lay(const tk_ctx* c) {
  Lay l;
  l.n = c->N;
  for (int m = 0; m < c->N; ++m) {
    l.mode[m] = m;
    l.z[m] = false;
  }
  return l;
}
// canonical element count with the modes in `kept` as x, the rest as z
int64_t canon_elems(const tk_ctx* c, uint32_t kept) {
  int64_t e = 1;
  for (int m = 0; m < c->N; ++m) e *= (kept >> m) & 1u ? c->s[m] : c->R[m];
  return e;
}

cppp_status dalloc(tk_ctx* c, double** p, int64_t doubles) {
  void* q = nullptr;
  TKCU(c, cudaMalloc(&q, sizeof(double) * std::max<int64_t>(doubles, 1)));
  c->owned.push_back(q);
  *p = static_cast<double*>(q);
  return CPPP_OK;
}
cppp_status talloc(tk_ctx* c, double** p, int64_t doubles) {
  void* q = nullptr;
  TKCU(c, cudaMallocAsync(&q, sizeof(double) * std::max<int64_t>(doubles, 1), c->st));
  *p = static_cast<double*>(q);
  return CPPP_OK;
}
cppp_status tfree(tk_ctx* c, double* p) {
  if (p) TKCU(c, cudaFreeAsync(p, c->st));
  return CPPP_OK;
}

// out = in ×_u F^T: contract axis x_u of `in` (layout l) with F (s_u x R_u); z_u appended last
cppp_status contract(tk_ctx* c, const double* in, const Lay& l, int u, const double* F, double* out,
                     Lay* lo) {
  int p = -1;
  for (int a = 0; a < l.n; ++a)
    if (l.mode[a] == u && !l.z[a]) p = a;
  if (p < 0) return tfail(c, CPPP_EINVAL, "internal: mode %d not kept", u);
  int64_t B = 1, R = 1;
  for (int a = 0; a < p; ++a) B *= axis_dim(c, l, a);
  for (int a = p + 1; a < l.n; ++a) R *= axis_dim(c, l, a);
  TKCU(c, cppp::launch_ttm(in, B, c->s[u], R, F, c->R[u], out, c->Fpad,
                           (c->flags & CPPP_FLAG_SIMT_TTM) != 0, c->st));
  Lay o;
  for (int a = 0; a < l.n; ++a) {
    if (a == p) continue;
    o.mode[o.n] = l.mode[a];
    o.z[o.n] = l.z[a];
    ++o.n;
  }
  o.mode[o.n] = u;
  o.z[o.n] = true;
  ++o.n;
  *lo = o;
  return CPPP_OK;
}

// canonical out [+]= in (layout l, one axis per mode)
cppp_status to_canonical(tk_ctx* c, const double* in, const Lay& l, double* out, bool accumulate) {
  cppp::PermArgs p{};
  p.nd = c->N;
  int64_t stride[CPPP_MAX_ORDER];
  int64_t st = 1;
  for (int a = l.n - 1; a >= 0; --a) {
    stride[a] = st;
    st *= axis_dim(c, l, a);
  }
  for (int m = 0; m < c->N; ++m) {
    int a = -1;
    for (int b = 0; b < l.n; ++b)
      if (l.mode[b] == m) a = b;
    if (a < 0) return tfail(c, CPPP_EINVAL, "internal: mode %d missing", m);
    p.odim[m] = axis_dim(c, l, a);
    p.istride[m] = stride[a];
  }
  const int64_t total = st;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  cppp::permute_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, c->st>>>(
      in, out, p, total, accumulate ? 1 : 0);
  cppp::note_launch();
  TKCU(c, cudaGetLastError());
  return CPPP_OK;
}

cppp_status copy_out(tk_ctx* c, double* dst, const double* src, int64_t n) {
  TKCU(c, cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDefault, c->st));
  if (!cppp::dev_ptr(dst)) TKCU(c, cudaStreamSynchronize(c->st));
  return CPPP_OK;
}

// Binary dimension tree: node keeps modes [lo, hi]; the left half is reached by
// contracting the right half's modes and vice versa; a leaf is Y^(lo).
struct TDT {
  tk_ctx* c;
  double* const* Y;

  cppp_status leaf(const double* d, const Lay& l, int n) {
    TKST(to_canonical(c, d, l, c->out, false));
    if (Y && Y[n]) TKST(copy_out(c, Y[n], c->out, canon_elems(c, 1u << n)));
    return CPPP_OK;
  }

  // contract modes [a, b] of (d, l) one by one (ascending), then recurse on [lo, hi]
  cppp_status half(const double* d, const Lay& l, int a, int b, int lo, int hi) {
    const double* cur = d;
    Lay cl = l;
    std::vector<double*> tmp;
    for (int u = a; u <= b; ++u) {
      Lay nl;
      Lay probe = cl;
      // output size: the contracted x_u becomes z_u
      int64_t e = lay_elems(c, probe) / c->s[u] * c->R[u];
      double* o = nullptr;
      TKST(talloc(c, &o, e));
      TKST(contract(c, cur, cl, u, c->A[u], o, &nl));
      if (cur != d) TKST(tfree(c, const_cast<double*>(cur)));
      cur = o;
      cl = nl;
    }
    cppp_status s = range(cur, cl, lo, hi);
    TKST(tfree(c, const_cast<double*>(cur)));
    return s;
  }

  cppp_status range(const double* d, const Lay& l, int lo, int hi) {
    if (lo == hi) return leaf(d, l, lo);
    const int mid = lo + (hi - lo + 1 + 1) / 2 - 1;
    TKST(half(d, l, mid + 1, hi, lo, mid));
    TKST(half(d, l, lo, mid, mid + 1, hi));
    return CPPP_OK;
  }
};

// Def. pptree over tree modes 0..N-1 mapped to modes by tau (largest dimension first):
// a node at level l with contracted tree set mu has children mu ∪ {w}, w ∈ (max mu, l+2], each
// one mode product of the parent (Ttmc_Map_PP P:170-192); the leaves (level N-2) are the
// operators.
struct TTree {
  tk_ctx* c;
  int tau[CPPP_MAX_ORDER];

  cppp_status visit(const double* d, const Lay& l, uint32_t mu, int level) {
    const int N = c->N;
    if (level == N - 2) {
      int i = -1, j = -1;
      for (int a = 0; a < l.n; ++a)
        if (!l.z[a]) (i < 0 ? i : j) = l.mode[a];
      if (i > j) std::swap(i, j);
      return to_canonical(c, d, l, c->ops[i][j], false);
    }
    int maxmu = -1;
    for (int t = 0; t < N; ++t)
      if (mu & (1u << t)) maxmu = t;
    for (int w = maxmu + 1; w <= level + 2; ++w) {
      const int u = tau[w];
      double* o = nullptr;
      TKST(talloc(c, &o, lay_elems(c, l) / c->s[u] * c->R[u]));
      Lay nl;
      TKST(contract(c, d, l, u, c->Ap[u], o, &nl));
      cppp_status s = visit(o, nl, mu | (1u << w), level + 1);
      TKST(tfree(c, o));
      TKST(s);
    }
    return CPPP_OK;
  }
};

Lay canon_lay(const tk_ctx* c, uint32_t kept) {
  Lay l;
  l.n = c->N;
  for (int m = 0; m < c->N; ++m) {
    l.mode[m] = m;
    l.z[m] = !((kept >> m) & 1u);
  }
  return l;
}

cppp_status load_factors(tk_ctx* c, const double* const* A) {
  if (!A) return tfail(c, CPPP_EINVAL, "null factor list");
  for (int n = 0; n < c->N; ++n) {
    if (!A[n]) return tfail(c, CPPP_EINVAL, "null factor %d", n);
    TKCU(c, cudaMemcpyAsync(c->A[n], A[n], sizeof(double) * c->s[n] * c->R[n], cudaMemcpyDefault,
                            c->st));
  }
  TKCU(c, cudaStreamSynchronize(c->st));
  return CPPP_OK;
}

}  // namespace

extern "C" {

cppp_status tk_init(tk_ctx** out, const double* X, int N, const int64_t* s, const int* R,
                    void* stream, unsigned flags) {
  if (!out) return CPPP_EINVAL;
  *out = nullptr;
  if (!X || !s || !R || N < 3 || N > CPPP_MAX_ORDER) return CPPP_EINVAL;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return CPPP_ENODEV;
  }
  tk_ctx* c = new tk_ctx;
  c->N = N;
  c->flags = flags;
  c->st = static_cast<cudaStream_t>(stream);
  int64_t numel = 1, smax = 1;
  for (int n = 0; n < N; ++n) {
    if (s[n] < 1 || R[n] < 1 || R[n] > s[n]) {
      delete c;
      return CPPP_EINVAL;
    }
    c->s[n] = s[n];
    c->R[n] = R[n];
    numel *= s[n];
    smax = std::max(smax, s[n]);
  }
  auto bail = [&](cppp_status st) {
    tk_destroy(c);
    return st;
  };
  if (flags & CPPP_FLAG_BORROW_TENSOR) {
    if (!cppp::dev_ptr(X)) return bail(CPPP_EINVAL);
    c->X = X;
  } else {
    if (dalloc(c, &c->Xown, numel) != CPPP_OK) return bail(CPPP_ENOMEM);
    if (cudaMemcpyAsync(c->Xown, X, sizeof(double) * numel, cudaMemcpyDefault, c->st) != cudaSuccess)
      return bail(CPPP_ECUDA);
    c->X = c->Xown;
  }
  int64_t ymax = 1;
  for (int n = 0; n < N; ++n) {
    if (dalloc(c, &c->A[n], s[n] * R[n]) != CPPP_OK || dalloc(c, &c->Ap[n], s[n] * R[n]) != CPPP_OK ||
        dalloc(c, &c->dA[n], s[n] * R[n]) != CPPP_OK || dalloc(c, &c->Yp[n], canon_elems(c, 1u << n)) != CPPP_OK)
      return bail(CPPP_ENOMEM);
    ymax = std::max(ymax, canon_elems(c, 1u << n));
    for (int j = n + 1; j < N; ++j)
      if (dalloc(c, &c->ops[n][j], canon_elems(c, (1u << n) | (1u << j))) != CPPP_OK)
        return bail(CPPP_ENOMEM);
  }
  if (dalloc(c, &c->out, ymax) != CPPP_OK) return bail(CPPP_ENOMEM);
  const size_t nscr = cppp::ttm_scratch_doubles(smax);
  if (dalloc(c, &c->Fpad, (int64_t)nscr) != CPPP_OK) return bail(CPPP_ENOMEM);
  if (cudaMemsetAsync(c->Fpad, 0, sizeof(double) * nscr, c->st) != cudaSuccess ||
      cudaStreamSynchronize(c->st) != cudaSuccess)
    return bail(CPPP_ECUDA);
  *out = c;
  return CPPP_OK;
}

cppp_status tk_set_factors(tk_ctx* c, const double* const* A) {
  if (!c) return CPPP_EINVAL;
  TKST(load_factors(c, A));
  c->factors_set = true;
  c->ops_valid = false;
  return CPPP_OK;
}

cppp_status tk_update_factors(tk_ctx* c, const double* const* A) {
  if (!c) return CPPP_EINVAL;
  if (!c->factors_set) return tfail(c, CPPP_ESTATE, "tk_update_factors before tk_set_factors");
  return load_factors(c, A);
}

cppp_status tk_ttmc(tk_ctx* c, double* const* Y) {
  if (!c) return CPPP_EINVAL;
  if (!c->factors_set) return tfail(c, CPPP_ESTATE, "tk_ttmc before tk_set_factors");
  TDT t{c, Y};
  TKST(t.range(c->X, root_lay(c), 0, c->N - 1));
  TKCU(c, cudaStreamSynchronize(c->st));
  return CPPP_OK;
}

cppp_status tk_pp_build(tk_ctx* c) {
  if (!c) return CPPP_EINVAL;
  if (!c->factors_set) return tfail(c, CPPP_ESTATE, "tk_pp_build before tk_set_factors");
  const int N = c->N;
  for (int n = 0; n < N; ++n) {
    TKCU(c, cudaMemcpyAsync(c->Ap[n], c->A[n], sizeof(double) * c->s[n] * c->R[n],
                            cudaMemcpyDeviceToDevice, c->st));
    TKCU(c, cudaMemsetAsync(c->dA[n], 0, sizeof(double) * c->s[n] * c->R[n], c->st));
  }
  TTree t{c, {}};
  for (int n = 0; n < N; ++n) t.tau[n] = n;
  std::stable_sort(t.tau, t.tau + N, [&](int a, int b) { return c->s[a] > c->s[b]; });
  TKST(t.visit(c->X, root_lay(c), 0u, 0));
  // Y_p^(n) = Y_p^(j,n) ×_j A_p^(j)T, j = min{j != n}
  for (int n = 0; n < N; ++n) {
    const int j = n == 0 ? 1 : 0;
    const int a = std::min(j, n), b = std::max(j, n);
    const Lay l = canon_lay(c, (1u << a) | (1u << b));
    double* o = nullptr;
    TKST(talloc(c, &o, canon_elems(c, 1u << n)));
    Lay nl;
    TKST(contract(c, c->ops[a][b], l, j, c->Ap[j], o, &nl));
    TKST(to_canonical(c, o, nl, c->Yp[n], false));
    TKST(tfree(c, o));
  }
  TKCU(c, cudaStreamSynchronize(c->st));
  c->ops_valid = true;
  return CPPP_OK;
}

cppp_status tk_pp_get_operator(tk_ctx* c, int i, int j, double* out) {
  if (!c) return CPPP_EINVAL;
  if (i < 0 || j >= c->N || i >= j) return tfail(c, CPPP_EINVAL, "operator (%d,%d): need 0<=i<j<N", i, j);
  if (!c->ops_valid) return tfail(c, CPPP_ESTATE, "no PP operators (call tk_pp_build)");
  if (!out) return tfail(c, CPPP_EINVAL, "null output");
  return copy_out(c, out, c->ops[i][j], canon_elems(c, (1u << i) | (1u << j)));
}

cppp_status tk_pp_get_single(tk_ctx* c, int n, double* out) {
  if (!c) return CPPP_EINVAL;
  if (n < 0 || n >= c->N) return tfail(c, CPPP_EINVAL, "mode %d out of range", n);
  if (!c->ops_valid) return tfail(c, CPPP_ESTATE, "no PP operators (call tk_pp_build)");
  if (!out) return tfail(c, CPPP_EINVAL, "null output");
  return copy_out(c, out, c->Yp[n], canon_elems(c, 1u << n));
}

cppp_status tk_pp_update(tk_ctx* c, int n, double* Y_tilde) {
  if (!c) return CPPP_EINVAL;
  if (n < 0 || n >= c->N) return tfail(c, CPPP_EINVAL, "mode %d out of range", n);
  if (!c->ops_valid) return tfail(c, CPPP_ESTATE, "tk_pp_update before tk_pp_build");
  const int N = c->N;
  for (int i = 0; i < N; ++i)
    TKCU(c, cppp::launch_sub(c->A[i], c->Ap[i], c->dA[i], c->s[i] * c->R[i], c->st));
  const int64_t ne = canon_elems(c, 1u << n);
  TKCU(c, cudaMemcpyAsync(c->out, c->Yp[n], sizeof(double) * ne, cudaMemcpyDeviceToDevice, c->st));
  double* o = nullptr;
  TKST(talloc(c, &o, ne));
  for (int i = 0; i < N; ++i) {
    if (i == n) continue;
    const int a = std::min(i, n), b = std::max(i, n);
    Lay nl;
    TKST(contract(c, c->ops[a][b], canon_lay(c, (1u << a) | (1u << b)), i, c->dA[i], o, &nl));
    TKST(to_canonical(c, o, nl, c->out, true));
  }
  TKST(tfree(c, o));
  if (Y_tilde) TKST(copy_out(c, Y_tilde, c->out, ne));
  TKCU(c, cudaStreamSynchronize(c->st));
  return CPPP_OK;
}

const char* tk_last_error(const tk_ctx* c) { return c ? c->err.c_str() : "null context"; }

void tk_destroy(tk_ctx* c) {
  if (!c) return;
  cudaStreamSynchronize(c->st);
  for (void* p : c->owned) cudaFree(p);
  delete c;
}

}  // extern "C"
