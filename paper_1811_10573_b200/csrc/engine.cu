// engine.cu — the host-side engine behind the C ABI (include/cppp.h): workspace planning, the
// regular dimension tree, the PP construction tree (Def. pptree), the Alg. 3 phase machine,
// slab sharding with NCCL all-reduce, kernel-class profiling.
//
// Citations: P:n = PAPER.md line n; Lnn = SURVEY.md §8(c) / DESIGN.md reading nn.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cppp.h"
#include "internal.h"

using namespace cppp;

namespace {

constexpr size_t ALIGN = 256;
inline size_t align_up(size_t x) { return (x + ALIGN - 1) & ~(ALIGN - 1); }

// ---------------------------------------------------------------- NCCL (dlopen'ed on demand)
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool load() {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    getErrorString = (decltype(getErrorString))dlsym(h, "ncclGetErrorString");
    return getUniqueId && commInitRank && allReduce && commDestroy && getErrorString;
  }
};
Nccl g_nccl;

// ---------------------------------------------------------------- bump/stack allocator
struct Stack {
  char* base = nullptr;
  size_t top = 0, peak = 0, cap = 0;
  bool dry = true;
  double* push(size_t doubles) {
    size_t off = top;
    top = align_up(top + doubles * sizeof(double));
    peak = std::max(peak, top);
    return dry ? reinterpret_cast<double*>(ALIGN) : reinterpret_cast<double*>(base + off);
  }
  size_t mark() const { return top; }
  void release(size_t m) { top = m; }
};

struct Node {
  uint32_t mask;   // kept modes
  double* data;    // kept modes ascending, then K; root: X (no K)
  bool root;
};

struct ProfPending {
  int cls;
  cudaEvent_t a, b;
  double flops, bytes;
};

}  // namespace

struct cppp_ctx {
  // problem
  int N = 0, K = 0;
  int64_t s[CPPP_MAX_ORDER] = {};    // global sizes
  int64_t dl[CPPP_MAX_ORDER] = {};   // local sizes
  int q = -1;                        // sharded mode (-1 none)
  int64_t qoff = 0, qext = 0;
  unsigned flags = 0;
  int device = 0;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  // memory
  char* ws = nullptr;
  char* ws_alloc = nullptr;
  size_t ws_bytes = 0;
  bool own_ws = false;
  double* X = nullptr;
  int64_t numel_local = 0;
  double *A[CPPP_MAX_ORDER] = {}, *Ap[CPPP_MAX_ORDER] = {}, *dA[CPPP_MAX_ORDER] = {};
  double *M[CPPP_MAX_ORDER] = {}, *Mp[CPPP_MAX_ORDER] = {}, *T[CPPP_MAX_ORDER] = {};
  double* S_all = nullptr;   // N x K x K
  double* Gamma = nullptr;   // K x K (of the mode being solved)
  double* L = nullptr;       // 2 K x K: Γ^(-1) or Γ^†, then Jacobi scratch
  int* lmode = nullptr;
  double* gram_scratch = nullptr;   // Gram split partials + per-tile Σ Γ∘S partials
  unsigned int* gram_counters = nullptr;
  cudaStream_t st2 = nullptr;           // side stream: Γ^(n) inverse overlapped with M^(n)
  cudaStream_t st3 = nullptr;           // order-3 DT: the second first-level TTM, overlapped
  cudaEvent_t ev_F = nullptr, ev_T = nullptr;   // st3 fork / join
  cudaStream_t st4 = nullptr;           // PP sweep: the next mode's early update terms
  cudaEvent_t ev_pf = nullptr, ev_pe[2] = {nullptr, nullptr};   // st4 fork / joins
  cudaEvent_t ev_S = nullptr, ev_P = nullptr;
  int prefetched = -1;                  // mode whose Γ inverse is issued on st2
  double* rowstat = nullptr; // max local rows x 4
  double* stats = nullptr;   // N x 3 norms, then fitness terms [2], then ||X||² [1]
  double* Fpad = nullptr;    // max s x 128
  double* ops[CPPP_MAX_ORDER][CPPP_MAX_ORDER] = {};   // i<j: [x_i][x_j][k]
  // sharded runs: the operators that contract the slab mode (i, j != q) are laid out back to back
  // (padding between them is zero), so the build all-reduces them in ONE call (SURVEY C-b)
  double* ops_red = nullptr;
  size_t ops_red_count = 0;
  // the PP sweep's exchange terms T_m, m != q, likewise in one call (C-c)
  // the slab mode's staging block [8 norms | K x K Gram]: its Gram kernel writes both here so
  // that they are all-reduced in one call (C-d), then they are copied to S_all[q] / stats
  double* qhdr = nullptr;
  double* pp_partial = nullptr;
  double* pp_part_early[2] = {nullptr, nullptr};   // split PP update: early-term partials
  double* sq_partial = nullptr;
  double* gath = nullptr;    // gather scratch (max s x K)
  double* chk = nullptr;     // pp_error: M~ scratch (max s x K), [N][3][K] sums x 2, [3][N][K] out
  double* ttv_scratch = nullptr;
  double* gen_scratch = nullptr;
  Stack stack;
  // state
  double normX_sq = 0.0;
  bool ops_valid = false;
  // order 3: ops[1][2] holds X ×_0 A^(0) for the CURRENT factors (the last sweep was a regular
  // one, which wrote it), so a PP build can take it instead of recomputing M_p^(1,2)
  bool op12_fresh = false;
  bool factors_set = false;
  bool borrowed = false;        // X is the caller's device buffer (CPPP_FLAG_BORROW_TENSOR)
  int next_phase = CPPP_PHASE_DT;
  int override_phase = CPPP_PHASE_AUTO;
  int policy = CPPP_POLICY_EPS_PP;   // PP switching policy (cp_set_pp_policy)
  double pinv_tol = 1e-12;           // τ of L13 (cppp_opts.pinv_rel_tol)
  double policy_tol = 0.0;
  int sweep = 0, restarts = 0;
  double last_fitness = NAN;
  double* host_stats = nullptr;  // pinned
  // comm
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  int (*host_ar)(double*, size_t, void*) = nullptr;
  void* host_ar_user = nullptr;
  double* host_ar_buf = nullptr;   // pinned staging
  size_t host_ar_cap = 0;
  // profiling
  std::vector<ProfPending> pending;
  std::vector<ProfPending> pending_graph;     // graph-owned events to read after a replay
  std::vector<cudaEvent_t> evpool;
  cppp_kernel_stat kstat[CPPP_K_COUNT] = {};
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  std::string err;
  bool dry = false;   // planning pass: no launches
  // CUDA graphs of whole sweeps, one per phase (captured on the phase's second use)
  bool capturing = false;
  std::vector<ProfPending> capture_prof;       // external event-record nodes of the capture
  struct SweepGraph {
    cudaGraphExec_t exec = nullptr;
    std::vector<ProfPending> prof;
    int uses = 0;
    uint64_t launches = 0;   // kernel nodes captured (credited to cppp_launch_count per replay)
  } graphs[3];
  // als_run: one graph for a whole run (a device-side WHILE over sweeps, a SWITCH over phases)
  struct RunGraph {
    cudaGraphExec_t exec = nullptr;
    cudaGraphConditionalHandle hw = 0, hs = 0;
    uint64_t launches_per_sweep[3] = {0, 0, 0};
    bool failed = false;   // capture not possible here: als_run falls back to als_sweep calls
  } run;
  struct RunState* run_dev = nullptr;   // device (workspace)
  struct RunState* run_host = nullptr;  // pinned
};

// Device-side Alg. 3 phase machine state for als_run (the same decisions als_sweep takes on the
// host, L7-L11, same IEEE operations in the same order).
struct RunInfo {
  double fitness, residual_sq, gsum, maxrel, bound;
  int phase, next_phase, restarts, converged;
};
// the communicating (sharded) code paths run with several ranks, or with one rank under
// CPPP_FLAG_FORCE_COMM (a one-rank NCCL communicator: the transport exercised on one GPU)
inline bool comm_on(const cppp_ctx* c) {
  return c->world > 1 || (c->flags & CPPP_FLAG_FORCE_COMM);
}

constexpr int RUN_MAX = 1024;   // sweeps per als_run call
struct RunState {
  double eps, eps_pp, normX_sq, policy_tol;
  int max_sweeps, done, phase, restarts, N, policy;
  RunInfo info[RUN_MAX];
};

namespace {

// ---------------------------------------------------------------- error plumbing
cppp_status fail(cppp_ctx* c, cppp_status s, const char* fmt, ...) {
  if (c) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    c->err = buf;
  }
  return s;
}

#define CUCHK(c, expr)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail((c), CPPP_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                    \
  } while (0)
#define STCHK(expr)                    \
  do {                                 \
    cppp_status s_ = (expr);           \
    if (s_ != CPPP_OK) return s_;      \
  } while (0)

// ---------------------------------------------------------------- profiling
cudaEvent_t get_event(cppp_ctx* c) {
  if (!c->evpool.empty()) {
    cudaEvent_t e = c->evpool.back();
    c->evpool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
struct Prof {
  cppp_ctx* c;
  int cls;
  double flops, bytes;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  Prof(cppp_ctx* c_, int cls_, double f, double b, cudaStream_t s = nullptr)
      : c(c_), cls(cls_), flops(f), bytes(b), st(s ? s : c_->st) {
    if (!c->dry && (c->flags & CPPP_FLAG_PROFILE)) {
      if (c->capturing) {   // graph-owned event, recorded by an event-record node on every replay
        cudaEventCreate(&a);
        cudaEventRecordWithFlags(a, st, cudaEventRecordExternal);
      } else {
        a = get_event(c);
        cudaEventRecord(a, st);
      }
    }
  }
  ~Prof() {
    if (!a) return;
    if (c->capturing) {
      cudaEvent_t b;
      cudaEventCreate(&b);
      cudaEventRecordWithFlags(b, st, cudaEventRecordExternal);
      c->capture_prof.push_back({cls, a, b, flops, bytes});
    } else {
      cudaEvent_t b = get_event(c);
      cudaEventRecord(b, st);
      c->pending.push_back({cls, a, b, flops, bytes});
    }
  }
};
// CPPP_TRACE=1 (debugging aid): every profiled scope of a sweep is printed to stderr as
// "trace <class> <start us> <end us>" relative to the sweep's first event.
void prof_trace(cppp_ctx* c, const char* tag, cudaEvent_t a, cudaEvent_t b, int cls) {
  static const bool on = getenv("CPPP_TRACE") != nullptr;
  if (!on) return;
  float t0 = 0.f, t1 = 0.f;
  cudaEventElapsedTime(&t0, c->ev_a, a);
  cudaEventElapsedTime(&t1, c->ev_a, b);
  fprintf(stderr, "trace %s %d %.1f %.1f\n", tag, cls, t0 * 1e3f, t1 * 1e3f);
}

void prof_collect(cppp_ctx* c) {
  for (auto& p : c->pending_graph) {
    float ms = 0.f;
    cudaEventSynchronize(p.b);
    cudaEventElapsedTime(&ms, p.a, p.b);
    prof_trace(c, "g", p.a, p.b, p.cls);
    auto& k = c->kstat[p.cls];
    k.launches += 1;
    k.total_ms += ms;
    k.flops += p.flops;
    k.bytes += p.bytes;
  }
  c->pending_graph.clear();
  if (c->pending.empty()) return;
  for (auto& p : c->pending) {
    float ms = 0.f;
    cudaEventSynchronize(p.b);
    cudaEventElapsedTime(&ms, p.a, p.b);
    prof_trace(c, "e", p.a, p.b, p.cls);
    auto& k = c->kstat[p.cls];
    k.launches += 1;
    k.total_ms += ms;
    k.flops += p.flops;
    k.bytes += p.bytes;
    c->evpool.push_back(p.a);
    c->evpool.push_back(p.b);
  }
  c->pending.clear();
}

// ---------------------------------------------------------------- comm
cppp_status allreduce(cppp_ctx* c, double* buf, size_t count) {
  if (!comm_on(c) || c->dry || count == 0) return CPPP_OK;
  if (c->host_ar) {
    if (count > c->host_ar_cap) {
      if (c->host_ar_buf) cudaFreeHost(c->host_ar_buf);
      c->host_ar_buf = nullptr;
      if (cudaMallocHost(&c->host_ar_buf, count * sizeof(double)) != cudaSuccess)
        return fail(c, CPPP_ENOMEM, "host all-reduce staging of %zu doubles", count);
      c->host_ar_cap = count;
    }
    CUCHK(c, cudaMemcpyAsync(c->host_ar_buf, buf, count * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CUCHK(c, cudaStreamSynchronize(c->st));
    if (c->host_ar(c->host_ar_buf, count, c->host_ar_user) != 0)
      return fail(c, CPPP_ENCCL, "host all-reduce callback failed");
    CUCHK(c, cudaMemcpyAsync(buf, c->host_ar_buf, count * sizeof(double), cudaMemcpyHostToDevice, c->st));
    CUCHK(c, cudaStreamSynchronize(c->st));
    return CPPP_OK;
  }
  ncclResult_t r = g_nccl.allReduce(buf, buf, count, ncclDouble, ncclSum, c->comm, c->st);
  if (r != ncclSuccess) return fail(c, CPPP_ENCCL, "ncclAllReduce: %s", g_nccl.getErrorString(r));
  return CPPP_OK;
}

// ---------------------------------------------------------------- geometry helpers
const double* fac_local(cppp_ctx* c, double* const* F, int u) {
  return F[u] + (u == c->q ? c->qoff * c->K : 0);
}
// Order 3, unsharded: a regular sweep's right-half TTM X ×_0 A^(0) (A^(0) already final for the
// sweep) is written straight into the operator slot M_p^(1,2); the PP build that follows a
// regular sweep (Alg. 3: always, unless a phase is forced) has A_p = A, so that TTM IS its
// M_p^(1,2) = X ×_0 A_p^(0) — one of the build's three full-tensor TTMs is skipped.  Same kernel,
// same shape: the operator is bit-identical to a recomputed one (tested).
// The order-3 GEMM that runs beside latency-bound work: two SMs without a persistent CTA (the
// factorization's 640-thread CTA cannot share an SM with a GEMM CTA).  A shallower ring (so a
// row-solve CTA could share an SM with a GEMM CTA) costs the GEMM < 1% (CPPP_TTM_STAGES in
// tools/probe_ttm) but buys nothing: the row solve stages Γ and its factor in ~207 KB of shared
// memory, and the Gram kernel's registers do not fit beside a GEMM CTA either.
// CPPP_TTM_RESERVE / CPPP_SIDE_STAGES: A/B.
TtmOpts side_gemm_opts() {
  static const TtmOpts o = [] {
    TtmOpts t;
    const char* r = getenv("CPPP_TTM_RESERVE");
    const char* st = getenv("CPPP_SIDE_STAGES");
    t.reserve_sms = r ? atoi(r) : 2;
    t.max_stages = st ? atoi(st) : 0;
    return t;
  }();
  return o;
}

bool reuse12(const cppp_ctx* c) {
  return c->N == 3 && c->q < 0 && !(c->flags & CPPP_FLAG_NO_OP_REUSE);
}
int64_t node_elems(cppp_ctx* c, uint32_t mask) {
  int64_t e = c->K;
  for (int v = 0; v < c->N; ++v)
    if (mask & (1u << v)) e *= c->dl[v];
  return e;
}

// out = contraction of `src` along mode u with factor F (local rows)
cppp_status contract(cppp_ctx* c, const Node& src, int u, const double* F, double* out,
                     cudaStream_t st = nullptr, TtmOpts topt = TtmOpts{}) {
  if (!st) st = c->st;
  int64_t B = 1, R = 1;
  for (int v = 0; v < c->N; ++v) {
    if (!(src.mask & (1u << v)) || v == u) continue;
    if (v < u) B *= c->dl[v];
    else R *= c->dl[v];
  }
  const int64_t S = c->dl[u];
  if (c->dry) return CPPP_OK;
  const int K = c->K;
  if (src.root) {
    const double flops = 2.0 * B * S * R * K;
    const double bytes = 8.0 * (B * S * R + B * R * K);
    const bool simt = (c->flags & CPPP_FLAG_SIMT_TTM) != 0;
    // factors live in the workspace (more buffers follow each), so the GEMM can read them in
    // place; CPPP_PAD_FACTOR keeps the padded copy (A/B)
    static const bool pad_env = getenv("CPPP_PAD_FACTOR") != nullptr;
    if (ttm_uses_dmma(B, S, R, K, simt)) {
      // (the side-stream GEMM keeps its pad kernel: it delays the GEMM's CTAs by a launch, and
      // without it C2 ran 2% slower -- mode 1's factorization chain then dispatches later; a
      // 3 us spacer kernel in its place measured the same as the pad)
      if (!pad_env && topt.reserve_sms == 0 && ttm_direct_ok(F, K)) topt.direct_factor = true;
      else CUCHK(c, ttm_prepare(S, F, K, c->Fpad, st));
    }
    Prof p(c, CPPP_K_TTM, flops, bytes, st);
    CUCHK(c, launch_ttm_core(src.data, B, S, R, F, K, out, c->Fpad, simt, st, topt));
  } else {
    const double flops = 2.0 * B * S * R * K;
    const double bytes = 8.0 * (B * S * R * K + B * R * K);
    Prof p(c, CPPP_K_TTV, flops, bytes, st);
    CUCHK(c, launch_ttv(src.data, B, S, R, K, F, out, c->ttv_scratch, st));
  }
  return CPPP_OK;
}

// Batched multi-TTV jobs (ttv.cu launch_ttv_batch): the contraction of a non-root node `src`
// along mode u into `out` (same geometry as contract()), and the one-pass pair of two children
// contracting modes u1 < u2 that are adjacent among src's kept modes.
TtvJob single_job(cppp_ctx* c, const Node& src, int u, const double* F, double* out) {
  TtvJob j;
  int64_t B = 1, R = 1;
  for (int v = 0; v < c->N; ++v) {
    if (!(src.mask & (1u << v)) || v == u) continue;
    if (v < u) B *= c->dl[v];
    else R *= c->dl[v];
  }
  j.P = src.data;
  j.Fb = F;
  j.outB = out;
  j.Bo = B;
  j.Sa = 1;
  j.Sb = (int)c->dl[u];
  j.IN = R * c->K;
  return j;
}
TtvJob pair_job(cppp_ctx* c, const Node& src, int u1, const double* F1, double* out1, int u2,
                const double* F2, double* out2) {
  TtvJob j;
  int64_t B = 1, R = 1;
  for (int v = 0; v < c->N; ++v) {
    if (!(src.mask & (1u << v)) || v == u1 || v == u2) continue;
    if (v < u1) B *= c->dl[v];
    else R *= c->dl[v];
  }
  j.P = src.data;
  j.Fa = F1;     // child a contracts u1 (the outer of the two)
  j.outA = out1;
  j.Fb = F2;     // child b contracts u2
  j.outB = out2;
  j.Bo = B;
  j.Sa = (int)c->dl[u1];
  j.Sb = (int)c->dl[u2];
  j.IN = R * c->K;
  return j;
}
bool ttv_batch_on(const cppp_ctx* c) {
  static const bool off = getenv("CPPP_NO_TTV_BATCH") != nullptr;   // A/B: one launch per child
  return !off && !(c->flags & CPPP_FLAG_NO_FUSED_TTV);
}
cppp_status run_ttv_jobs(cppp_ctx* c, const std::vector<TtvJob>& jobs) {
  if (c->dry || jobs.empty()) return CPPP_OK;
  double flops = 0.0, bytes = 0.0;
  for (const TtvJob& j : jobs) {
    const double pe = (double)j.Bo * j.Sa * j.Sb * j.IN;
    const int nch = j.Fa ? 2 : 1;
    flops += 2.0 * pe * nch;
    bytes += 8.0 * (pe + (double)j.Bo * j.Sa * j.IN + (j.Fa ? (double)j.Bo * j.Sb * j.IN : 0.0));
  }
  Prof p(c, CPPP_K_TTV, flops, bytes, c->st);
  CUCHK(c, launch_ttv_batch(jobs.data(), (int)jobs.size(), c->K, c->st));
  return CPPP_OK;
}

// Multi-mode first level: contract the consecutive modes `modes` (ascending) of X in ONE GEMM
// with their Khatri-Rao product (P:78-80 applied to a whole half of the tree at once; same
// 2 s^N R flops as a single-mode TTM, but no s^(N-1) R intermediate and no multi-TTV pass over
// it).  Returns false (nothing done) when the DMMA GEMM cannot take the shape.
bool contract_multi(cppp_ctx* c, const Node& src, const std::vector<int>& modes, double* out,
                    cppp_status* st, double* const* F = nullptr) {
  *st = CPPP_OK;
  int64_t B = 1, S = 1, R = 1;
  for (int v = 0; v < c->N; ++v) {
    if (v < modes.front()) B *= c->dl[v];
    else if (v > modes.back()) R *= c->dl[v];
    else S *= c->dl[v];
  }
  const int K = c->K;
  if (!ttm_uses_dmma(B, S, R, K, (c->flags & CPPP_FLAG_SIMT_TTM) != 0)) return false;
  if (c->dry) return true;
  KrpArgs a{};
  a.nm = static_cast<int>(modes.size());
  a.K = K;
  for (int j = 0; j < a.nm; ++j) {
    a.F[j] = fac_local(c, F ? F : c->A, modes[j]);
    a.dims[j] = c->dl[modes[j]];
  }
  cudaError_t e = ttm_prepare_krp(a, c->Fpad, c->st);
  if (e != cudaSuccess) {
    *st = fail(c, CPPP_ECUDA, "khatri-rao: %s", cudaGetErrorString(e));
    return true;
  }
  Prof p(c, CPPP_K_TTM, 2.0 * B * S * R * K, 8.0 * (B * S * R + B * R * K));
  e = launch_ttm_padded(src.data, B, S, R, K, out, c->Fpad, c->st);
  if (e != cudaSuccess) *st = fail(c, CPPP_ECUDA, "multi-mode TTM: %s", cudaGetErrorString(e));
  return true;
}

// ---------------------------------------------------------------- small solve of one mode
// A_new = M Γ^†, G, dA = A_new - ref, S^(n), norms (Alg. 1 P:393-399 / Alg. 3).
// Issue Γ^(n) and its inverse on the side stream once every S^(m), m != n, is final (ev_S).
// K <= 32 with every (local) mode <= 64 rows: each mode's solve is ONE launch on the main stream
// (launch_mode_small: Γ, factorization, rows, Gram, statistics; bit-identical to the chain of
// gamma factorization on the side stream + row solves + Gram), so nothing is prefetched.  The
// kernels that produce M^(n) trigger it early (pdl_trigger), so its Γ / factorization part runs
// beside them, as the side-stream factorization did.  Measured (20-sweep runs, A/B with
// CPPP_NO_FUSED_SOLVE and a build without the early trigger): C4 1784 -> 1848 sweeps/s fused,
// 2107 -> 2189 with the trigger (after the pair tree); C1 14.9 k (chain) -> 13.7 k fused without
// the trigger, 15.4 k with it; the LAP / P6W PP-approximated sweeps 208 -> 182 us.
bool small_modes(const cppp_ctx* c) {
  static const bool off = getenv("CPPP_NO_FUSED_SOLVE") != nullptr;   // A/B
  if (off || (c->flags & CPPP_FLAG_NO_FUSED_SOLVE)) return false;
  for (int n = 0; n < c->N; ++n)
    if (!mode_small_ok(c->K, c->dl[n])) return false;
  return true;
}

cppp_status prefetch_inverse(cppp_ctx* c, int n) {
  if (c->dry || c->prefetched == n || small_modes(c)) return CPPP_OK;
  CUCHK(c, cudaStreamWaitEvent(c->st2, c->ev_S, 0));
  {   // (the scope closes before ev_P: every side-stream node must be joined)
    Prof p(c, CPPP_K_FACTOR, (double)c->K * c->K * c->K / 3.0, 8.0 * c->K * c->K * c->N, c->st2);
    CUCHK(c, launch_gamma_factor(c->S_all, c->N, n, c->K, c->Gamma, c->L, c->lmode,
                                 c->L + (int64_t)solve_ld(c->K) * solve_ld(c->K) + 4 * 32 * 33,
                                 c->st2, c->pinv_tol));
  }
  CUCHK(c, cudaEventRecord(c->ev_P, c->st2));
  c->prefetched = n;
  return CPPP_OK;
}

// Drop a pending prefetch before the Grams are rewritten outside a sweep.
cppp_status drain_prefetch(cppp_ctx* c) {
  if (c->prefetched >= 0) CUCHK(c, cudaStreamWaitEvent(c->st, c->ev_P, 0));
  c->prefetched = -1;
  return CPPP_OK;
}

// A_new = M Γ^†, G, dA = A_new - ref, S^(n), norms (Alg. 1 P:393-399 / Alg. 3).
cppp_status finish_mode(cppp_ctx* c, int n, const double* Mn, bool pp_phase) {
  if (c->dry) return CPPP_OK;
  const int K = c->K;
  const int64_t rows = c->dl[n];
  const int64_t off = (n == c->q) ? c->qoff : 0;
  const bool fused = small_modes(c);
  if (!fused) {
    STCHK(prefetch_inverse(c, n));
    CUCHK(c, cudaStreamWaitEvent(c->st, c->ev_P, 0));
  }
  c->prefetched = -1;
  {
    Prof p(c, CPPP_K_SOLVE, 4.0 * rows * K * K, 8.0 * rows * K * 5);
    double* An = c->A[n] + off * K;
    const double* ref = pp_phase ? (c->Ap[n] + off * K) : An;
    const bool last = (n == c->N - 1);
    // the slab mode (q = 0) writes its norms into qhdr, right before S^(q) = S_all's first block
    const bool packq = (n == c->q) && comm_on(c) && !c->dry;
    double* nrm = packq ? c->qhdr : c->stats + 3 * n;
    double* Sn = packq ? c->qhdr + 8 : c->S_all + (int64_t)n * K * K;
    if (fused) {
      const int ld = solve_ld(K);
      CUCHK(c, launch_mode_small(c->S_all, c->N, n, K, Mn, An, ref, c->dA[n] + off * K, rows, Sn, nrm,
                                 last ? (packq ? c->qhdr + 3 : c->stats + 3 * c->N) : nullptr, c->Gamma,
                                 c->L, c->L + (int64_t)ld * ld + 4 * 32 * 33, c->st, c->pinv_tol));
    } else {
      CUCHK(c, launch_solve_rows(Mn, An, ref, c->dA[n] + off * K, rows, K, c->Gamma, c->L, c->lmode,
                                 c->rowstat, c->st));
      // S^(n), the norms and (last mode) the fitness terms in one kernel; Γ^(n) is still in place
      // (the next factorization starts after ev_S below)
      // (the slab mode's fitness terms, when it is the last mode, are partial sums too: qhdr[3..4])
      CUCHK(c, launch_gram(An, rows, K, Sn, c->rowstat, nrm, last ? c->Gamma : nullptr,
                           last ? (packq ? c->qhdr + 3 : c->stats + 3 * c->N) : nullptr, c->gram_scratch,
                           c->gram_counters, c->st));
    }
  }
  if (n == c->q && comm_on(c) && !c->dry) {
    // S^(q), its norms (and fitness terms) in ONE all-reduce (SURVEY C-d), then into their slots
    STCHK(allreduce(c, c->qhdr, (size_t)K * K + 8));
    CUCHK(c, cudaMemcpyAsync(c->S_all + (int64_t)n * K * K, c->qhdr + 8, sizeof(double) * K * K,
                             cudaMemcpyDeviceToDevice, c->st));
    CUCHK(c, cudaMemcpyAsync(c->stats + 3 * n, c->qhdr, 3 * sizeof(double), cudaMemcpyDeviceToDevice,
                             c->st));
    if (n == c->N - 1)
      CUCHK(c, cudaMemcpyAsync(c->stats + 3 * c->N, c->qhdr + 3, 2 * sizeof(double), cudaMemcpyDeviceToDevice,
                               c->st));
  }
  CUCHK(c, cudaEventRecord(c->ev_S, c->st));
  // the next mode's factorization starts right away on the side stream; inside a captured sweep
  // the wrap-around to mode 0 of the next sweep is left out (every fork must join in the graph)
  if (c->capturing && n == c->N - 1) return CPPP_OK;
  return prefetch_inverse(c, (n + 1) % c->N);
}

// ---------------------------------------------------------------- regular dimension tree
// DT sweep (Alg. 1 with a binary dimension tree; leading cost 4 s^N R).  Node `nd`
// keeps exactly modes [lo, hi].  Left half first (Gauss-Seidel order n = 0..N-1): its modes
// are reached by contracting the right half with the not-yet-updated factors; the right half
// is then reached by contracting the (now updated) left half.
struct DT {
  cppp_ctx* c;
  bool update;
  double* const* Mout;   // where M^(n) goes (c->M or caller buffers)

  std::vector<int> chain_order(const Node& nd, int lo, int hi) {
    std::vector<int> m;
    for (int v = lo; v <= hi; ++v) m.push_back(v);
    // keep the natural GEMM orientation for the first-level TTM: contract the last mode first
    // when it is in the chain, else the first; never contract the sharded mode first (SURVEY
    // §8(e)): it goes last so every big intermediate stays exact for the local rows.
    bool has_last = false;
    int last_kept = -1;
    for (int v = 0; v < c->N; ++v)
      if (nd.mask & (1u << v)) last_kept = v;
    for (int v : m) has_last |= (v == last_kept);
    if (has_last) std::reverse(m.begin(), m.end());
    auto it = std::find(m.begin(), m.end(), c->q);
    if (it != m.end()) {
      m.erase(it);
      m.push_back(c->q);
    }
    return m;
  }

  // contract `modes` (in order) out of nd; the final node goes to `final_dst` if given.  From
  // the root of an order >= 4 tensor, a half of two or more modes (none of them sharded) is
  // contracted in one multi-mode GEMM (contract_multi) unless CPPP_FLAG_NO_KRP.  (Order 3
  // keeps the single-mode TTM: its level-1 node feeds two leaves, and the multi-mode GEMM
  // would have only s/128 output tiles.)
  cppp_status chain(const Node& nd, const std::vector<int>& modes, double* final_dst, Node* out) {
    // (a half that contains the slab mode q is contracted the same way: with A^(q) restricted to
    // the local rows the GEMM's output is this rank's partial sum, every later contraction is
    // linear, and every leaf n != q is all-reduced anyway -- SURVEY §8(e))
    if (nd.root && modes.size() >= 2 && c->N >= 4 && !(c->flags & CPPP_FLAG_NO_KRP)) {
      std::vector<int> asc = modes;
      std::sort(asc.begin(), asc.end());
      uint32_t nm = nd.mask;
      for (int v : asc) nm &= ~(1u << v);
      const size_t mk = c->stack.mark();
      double* dst = final_dst ? final_dst : c->stack.push(node_elems(c, nm));
      cppp_status st;
      if (contract_multi(c, nd, asc, dst, &st)) {
        STCHK(st);
        *out = Node{nm, dst, false};
        return CPPP_OK;
      }
      c->stack.release(mk);
    }
    Node cur = nd;
    for (size_t i = 0; i < modes.size(); ++i) {
      const int u = modes[i];
      const uint32_t nm = cur.mask & ~(1u << u);
      double* dst = (i + 1 == modes.size() && final_dst) ? final_dst
                                                         : c->stack.push(node_elems(c, nm));
      if (update && reuse12(c) && nd.root && i == 0 && u == 0 && modes.size() == 2)
        dst = c->ops[1][2];   // (the stack slot stays pushed: sizing is the same either way)
      STCHK(contract(c, cur, u, fac_local(c, c->A, u), dst));
      cur = Node{nm, dst, false};
    }
    *out = cur;
    return CPPP_OK;
  }

  cppp_status leaf(int n, const double* Mn) {
    if (Mout != c->M && !c->dry) {
      CUCHK(c, cudaMemcpyAsync(Mout[n], Mn, sizeof(double) * c->dl[n] * c->K,
                               cudaMemcpyDeviceToDevice, c->st));
    }
    if (n != c->q) STCHK(allreduce(c, Mout[n], (size_t)c->dl[n] * c->K));
    if (update) STCHK(finish_mode(c, n, Mout[n], false));
    return CPPP_OK;
  }

  // Order 3, unsharded: the right half's first-level TTM (X ×_0 A^(0)) needs only A^(0), so it
  // runs on st3 beside mode 1's work (its multi-TTV, the Γ factorization and the row solves),
  // which are latency-bound and leave the tensor cores idle.  Same contractions, same order of
  // factor updates as range(); T01 and T12 are both live.
  cppp_status range3_overlap(const Node& nd) {
    const size_t mk = c->stack.mark();
    double* T01 = c->stack.push(node_elems(c, 0x3u));
    STCHK(contract(c, nd, 2, fac_local(c, c->A, 2), T01));
    const Node L{0x3u, T01, false};
    STCHK(contract(c, L, 1, fac_local(c, c->A, 1), c->M[0]));
    STCHK(leaf(0, c->M[0]));
    double* T12 = c->stack.push(node_elems(c, 0x6u));
    if (update && reuse12(c)) T12 = c->ops[1][2];
    if (!c->dry) {
      CUCHK(c, cudaEventRecord(c->ev_F, c->st));
      CUCHK(c, cudaStreamWaitEvent(c->st3, c->ev_F, 0));
    }
    // two SMs stay free of the GEMM's persistent CTAs: mode 1's factorization, row solves and
    // Gram and mode 2's factorization (latency-bound, one CTA or a few rows at a time) run there
    // meanwhile instead of waiting for the GEMM to end
    STCHK(contract(c, nd, 0, fac_local(c, c->A, 0), T12, c->st3, side_gemm_opts()));
    if (!c->dry) CUCHK(c, cudaEventRecord(c->ev_T, c->st3));
    STCHK(contract(c, L, 0, fac_local(c, c->A, 0), c->M[1]));
    STCHK(leaf(1, c->M[1]));
    if (!c->dry) CUCHK(c, cudaStreamWaitEvent(c->st, c->ev_T, 0));
    const Node Rn{0x6u, T12, false};
    STCHK(contract(c, Rn, 1, fac_local(c, c->A, 1), c->M[2]));
    STCHK(leaf(2, c->M[2]));
    c->stack.release(mk);
    return CPPP_OK;
  }

  cppp_status range(const Node& nd, int lo, int hi) {
    if (nd.root && c->N == 3 && lo == 0 && hi == 2 && c->q < 0 &&
        !(c->flags & CPPP_FLAG_NO_OVERLAP))
      return range3_overlap(nd);
    const int mid = lo + (hi - lo + 1 + 1) / 2 - 1;  // left half has ceil(len/2) modes
    // ---- left: modes [lo, mid]
    {
      const size_t mk = c->stack.mark();
      std::vector<int> ord = chain_order(nd, mid + 1, hi);
      Node L;
      if (lo == mid) {
        STCHK(chain(nd, ord, c->M[lo], &L));
        STCHK(leaf(lo, c->M[lo]));
      } else {
        STCHK(chain(nd, ord, nullptr, &L));
        STCHK(range(L, lo, mid));
      }
      c->stack.release(mk);
    }
    // ---- right: modes [mid+1, hi]
    {
      const size_t mk = c->stack.mark();
      std::vector<int> ord = chain_order(nd, lo, mid);
      Node R;
      if (mid + 1 == hi) {
        STCHK(chain(nd, ord, c->M[hi], &R));
        STCHK(leaf(hi, c->M[hi]));
      } else {
        STCHK(chain(nd, ord, nullptr, &R));
        STCHK(range(R, mid + 1, hi));
      }
      c->stack.release(mk);
    }
    return CPPP_OK;
  }
};

cppp_status run_dt(cppp_ctx* c, bool update, double* const* Mout) {
  DT dt{c, update, Mout};
  Node root{(1u << c->N) - 1, c->X, true};
  return dt.range(root, 0, c->N - 1);
}

// ---------------------------------------------------------------- PP construction tree
// Def. pptree over tree modes 0..N-1 mapped to physical modes by tau (tree mode N-1
// is the sharded mode when sharded, so it is contracted only at the leaves).  A node at level
// l has contracted set mu ⊂ {0..l+1}, |mu| = l; its children are mu ∪ {w}, w ∈ (max mu, l+2],
// each computed from it by contracting tau[w] (Tree_Map_PP P:77-91: i = max mu(t)).
struct PPTree {
  cppp_ctx* c;
  bool have12 = false;   // ops[1][2] already holds X ×_0 A_p^(0) (reuse12)
  int tau[CPPP_MAX_ORDER];

  void init() {
    const int N = c->N;
    int k = 0;
    for (int v = 0; v < N; ++v)
      if (v != c->q) tau[k++] = v;
    // largest dimensions contracted first: stable sort by decreasing global size; among
    // equal sizes, modes whose level-1 TTM tiles cleanly come first (the first and last modes,
    // and middle modes whose trailing extent R is a multiple of 16, which the GEMM tiles over
    // the flattened (b, r) rows) — only tau[0..2] are contracted from X, so a middle mode with a
    // ragged R (C3's mode 2: R = 100, 28 of every 128 tile rows idle) moves out of level 1
    auto ragged = [&](int m) {
      if (m == 0 || m == c->N - 1) return 0;
      int64_t R = 1;
      for (int v = m + 1; v < c->N; ++v) R *= c->dl[v];
      return R % 16 != 0 ? 1 : 0;
    };
    std::stable_sort(tau, tau + k, [&](int a, int b) {
      if (c->s[a] != c->s[b]) return c->s[a] > c->s[b];
      return ragged(a) < ragged(b);
    });
    if (c->q >= 0) tau[k++] = c->q;
  }

  uint32_t kept_of(uint32_t mu_tree) {
    uint32_t kept = (1u << c->N) - 1;
    for (int t = 0; t < c->N; ++t)
      if (mu_tree & (1u << t)) kept &= ~(1u << tau[t]);
    return kept;
  }

  double* op_ptr(uint32_t kept) {
    int i = -1, j = -1;
    for (int v = 0; v < c->N; ++v)
      if (kept & (1u << v)) {
        if (i < 0) i = v;
        else j = v;
      }
    return c->ops[i][j];
  }

  cppp_status visit(const Node& nd, uint32_t mu, int level) {
    const int N = c->N;
    if (level == N - 2) return CPPP_OK;  // leaf
    int maxmu = -1;
    for (int t = 0; t < N; ++t)
      if (mu & (1u << t)) maxmu = t;
    const bool child_leaf = (level + 1 == N - 2);
    if (nd.root) {
      // level-1 nodes are full-size TTMs: one at a time, depth first
      for (int w = maxmu + 1; w <= level + 2; ++w) {
        const uint32_t cmu = mu | (1u << w);
        const uint32_t kept = kept_of(cmu);
        if (w == 2 && !child_leaf && ttv_batch_on(c)) {
          cppp_status st = CPPP_OK;
          if (level2_from_x(nd, cmu | (1u << 3), &st)) {
            STCHK(st);
            continue;
          }
        }
        const size_t mk = c->stack.mark();
        double* dst = child_leaf ? op_ptr(kept) : c->stack.push(node_elems(c, kept));
        if (!(have12 && child_leaf && kept == 0x6u))
          STCHK(contract(c, nd, tau[w], fac_local(c, c->Ap, tau[w]), dst));
        if (!child_leaf && ttv_batch_on(c)) STCHK(subtree_batched(Node{kept, dst, false}, cmu));
        else STCHK(visit(Node{kept, dst, false}, cmu, level + 1));
        c->stack.release(mk);
      }
      return CPPP_OK;
    }
    // deeper: all children of this parent together (one pass over the parent when fused)
    const size_t mk = c->stack.mark();
    std::vector<Node> kids;
    std::vector<uint32_t> kmu;
    for (int w = maxmu + 1; w <= level + 2; ++w) {
      const uint32_t cmu = mu | (1u << w);
      const uint32_t kept = kept_of(cmu);
      double* dst = child_leaf ? op_ptr(kept) : c->stack.push(node_elems(c, kept));
      kids.push_back(Node{kept, dst, false});
      kmu.push_back(cmu);
    }
    STCHK(emit_children(nd, mu, maxmu, level, kids));
    for (size_t i = 0; i < kids.size(); ++i) STCHK(visit(kids[i], kmu[i], level + 1));
    c->stack.release(mk);
    return CPPP_OK;
  }

  // The last level-1 node of Def. pptree, {2}, has ONE child, {2, 3}.  When the two modes it
  // contracts are neighbours in X's layout, that level-2 node comes straight from X in one
  // multi-mode (Khatri-Rao) GEMM -- the same contraction of X with A_p^(tau 2) and A_p^(tau 3)
  // (L24: any tree gives the same values) -- and the s^(N-1) K level-1 node is
  // neither written nor read back (C4: a 768 MB node, its 307 us TTM and a 130 us multi-TTV pass,
  // against one GEMM whose output is 38 MB).  Unsharded, order >= 4, not with CPPP_FLAG_NO_KRP.
  bool level2_from_x(const Node& root, uint32_t mu2, cppp_status* st) {
    const int N = c->N;
    if (N < 4 || c->q >= 0 || (c->flags & CPPP_FLAG_NO_KRP)) return false;
    static const bool off = getenv("CPPP_NO_L2_FROM_X") != nullptr;   // A/B
    if (off) return false;
    const int u = std::min(tau[2], tau[3]), v = std::max(tau[2], tau[3]);
    if (v != u + 1) return false;
    const uint32_t kept = kept_of(mu2);
    const bool leaf = (N == 4);
    const size_t mk = c->stack.mark();
    double* dst = leaf ? op_ptr(kept) : c->stack.push(node_elems(c, kept));
    if (!contract_multi(c, root, std::vector<int>{u, v}, dst, st, c->Ap)) {
      c->stack.release(mk);
      return false;
    }
    if (*st == CPPP_OK && !leaf) *st = subtree_batched(Node{kept, dst, false}, mu2, 2);
    c->stack.release(mk);
    return true;
  }

  // Below a level-1 node, level by level (SURVEY a2 "batched multi-TTV"): every contraction of a
  // level in one batched launch (two when a parent feeds a one-pass pair), instead of one launch
  // per child depth first.  Same nodes and values as Def. pptree's traversal (L24); the nodes of
  // the subtree stay on the stack until its leaves are written.  (level0: the level of the node
  // the subtree hangs from -- 1, or 2 for a level-2 node contracted straight from X.)
  cppp_status subtree_batched(const Node& l1, uint32_t mu1, int level0 = 1) {
    const int N = c->N;
    struct Item {
      Node nd;
      uint32_t mu;
    };
    std::vector<Item> cur{{l1, mu1}};
    for (int level = level0; level < N - 2; ++level) {
      const bool child_leaf = (level + 1 == N - 2);
      std::vector<Item> next;
      std::vector<TtvJob> jobs;
      for (const Item& it : cur) {
        int maxmu = -1;
        for (int t = 0; t < N; ++t)
          if (it.mu & (1u << t)) maxmu = t;
        struct Kid {
          int u;
          double* dst;
        };
        std::vector<Kid> kid;
        for (int w = maxmu + 1; w <= level + 2; ++w) {
          const uint32_t cmu = it.mu | (1u << w);
          const uint32_t kept = kept_of(cmu);
          double* dst = child_leaf ? op_ptr(kept) : c->stack.push(node_elems(c, kept));
          next.push_back(Item{Node{kept, dst, false}, cmu});
          kid.push_back(Kid{tau[w], dst});
        }
        // one pair per parent: two children contracting kept modes adjacent in the parent (no
        // kept mode between them), the inner one with extent <= TTV_PAIR_MAXSB; the innermost such pair
        std::vector<bool> used(kid.size(), false);
        int best_a = -1, best_b = -1;
        for (size_t x = 0; x < kid.size(); ++x)
          for (size_t y = 0; y < kid.size(); ++y) {
            const int u1 = kid[x].u, u2 = kid[y].u;
            if (u1 >= u2 || c->dl[u2] > TTV_PAIR_MAXSB) continue;
            bool adjacent = true;
            for (int v = u1 + 1; v < u2; ++v)
              if (it.nd.mask & (1u << v)) adjacent = false;
            if (!adjacent) continue;
            if (best_a < 0 || u2 > kid[best_b].u) {
              best_a = (int)x;
              best_b = (int)y;
            }
          }
        const bool big = (double)node_elems(c, it.nd.mask) * 8.0 > 64.0 * (1 << 20);
        // pairs only for parents beyond L2 with enough columns to fill the GPU: on L2-resident
        // parents the batched singles share the parent through L2 anyway, and a pair job's few
        // long threads lost there (C4 level 4: 49 vs 12 us); C4 level 2 (768 MB parents):
        // node {1} 243 -> 186 us, node {0} 356 -> 317 us
        const bool pair_ok = big && best_a >= 0 &&
                             node_elems(c, it.nd.mask) / (c->dl[kid[best_a].u] * c->dl[kid[best_b].u]) >= 65536;
        if (pair_ok && !pair_off()) {
          const int u1 = kid[best_a].u, u2 = kid[best_b].u;
          TtvJob j = pair_job(c, it.nd, u1, fac_local(c, c->Ap, u1), kid[best_a].dst, u2,
                              fac_local(c, c->Ap, u2), kid[best_b].dst);
          j.stream = big;
          jobs.push_back(j);
          used[best_a] = used[best_b] = true;
        }
        for (size_t x = 0; x < kid.size(); ++x) {
          if (used[x]) continue;
          TtvJob j = single_job(c, it.nd, kid[x].u, fac_local(c, c->Ap, kid[x].u), kid[x].dst);
          j.stream = big;
          jobs.push_back(j);
        }
      }
      STCHK(run_ttv_jobs(c, jobs));
      cur.swap(next);
    }
    return CPPP_OK;
  }

  static bool pair_off() {
    static const bool off = getenv("CPPP_NO_TTV_PAIR") != nullptr;   // A/B
    return off;
  }

  cppp_status emit_children(const Node& nd, uint32_t mu, int maxmu, int level,
                            const std::vector<Node>& kids) {
    size_t i = 0;
    for (int w = maxmu + 1; w <= level + 2; ++w, ++i)
      STCHK(contract(c, nd, tau[w], fac_local(c, c->Ap, tau[w]), kids[i].data));
    (void)mu;
    return CPPP_OK;
  }

  cppp_status run() {
    init();
    Node root{(1u << c->N) - 1, c->X, true};
    return visit(root, 0u, 0);
  }
};

// M_p^(n) = M_p^(j,n) ×_j A_p^(j), j = min{j ∉ {n, q}}
cppp_status build_singles(cppp_ctx* c) {
  const int N = c->N, K = c->K;
  std::vector<TtvJob> jobs;
  for (int n = 0; n < N; ++n) {
    int j = -1;
    for (int v = 0; v < N; ++v)
      if (v != n && v != c->q) {
        j = v;
        break;
      }
    const int a = std::min(j, n), b = std::max(j, n);
    Node op{(1u << a) | (1u << b), c->ops[a][b], false};
    if (ttv_batch_on(c)) {
      TtvJob jb = single_job(c, op, j, fac_local(c, c->Ap, j), c->Mp[n]);
      jb.stream = (double)node_elems(c, op.mask) * 8.0 > 64.0 * (1 << 20);
      jobs.push_back(jb);
    } else {
      STCHK(contract(c, op, j, fac_local(c, c->Ap, j), c->Mp[n]));
    }
  }
  STCHK(run_ttv_jobs(c, jobs));   // the N single-mode operators in one batched launch
  (void)K;
  return CPPP_OK;
}

// Order 4, unsharded, s_3 % 128 == 0 (C5): the construction tree's level 1 -> level 2 fused into
// three GEMMs.  Level-1 node "contract a" (a = 0, 1, 2; kept modes in physical
// order, the last one f = 3) feeds two of its leaves from the GEMM epilogue: the FAST leaf
// (contract f) and the LOOP leaf (contract l); the third kept mode is o.  The choice (a, l, o) =
// (0, 1, 2), (1, 2, 0), (2, 0, 1) covers the six leaves exactly once:
//   a=0: (1,2) fast, (2,3) loop;  a=1: (0,2) fast, (0,3) loop;  a=2: (0,1) fast, (1,3) loop.
// Def. pptree's leaves are the same operators (L24: any tree gives the same values);
// no s^3 K level-1 node is ever written (C5: 16 GiB).  CPPP_FLAG_NO_FUSED_TTV: the plain tree.
bool fused_build_ok(const cppp_ctx* c) {
  if (c->N != 4 || c->q >= 0 || (c->flags & (CPPP_FLAG_NO_FUSED_TTV | CPPP_FLAG_SIMT_TTM))) return false;
  for (int a = 0; a < 3; ++a) {
    int64_t B = 1, R = 1;
    for (int v = 0; v < 4; ++v) {
      if (v < a) B *= c->dl[v];
      if (v > a) R *= c->dl[v];
    }
    if (!ttm_fused_ok(B, c->dl[a], R, c->K, c->dl[3])) return false;
  }
  return true;
}

cppp_status run_fused_build(cppp_ctx* c) {
  const int K = c->K;
  const int64_t* d = c->dl;
  static const int cover[3][2] = {{1, 2}, {2, 0}, {0, 1}};   // (l, o) per contracted mode a
  for (int a = 0; a < 3; ++a) {
    const int l = cover[a][0], o = cover[a][1], f = 3;
    int64_t B = 1, R = 1;
    for (int v = 0; v < 4; ++v) {
      if (v < a) B *= d[v];
      if (v > a) R *= d[v];
    }
    const int64_t S = d[a];
    auto tile_stride = [&](int v) {   // flattened kept index stride of mode v, in 128-row tiles
      int64_t st = 1;
      for (int u = v + 1; u < 4; ++u)
        if (u != a) st *= d[u];
      return st / 128;
    };
    TtmFused fz;
    fz.o_str = tile_stride(o);
    fz.l_str = tile_stride(l);
    fz.n_o = d[o];
    fz.n_l = d[l];
    fz.sf = d[f];
    const int64_t units0 = d[o] * (d[f] / 128);
    fz.nP = std::max<int64_t>(1, std::min<int64_t>(d[l], (148 * 7 + units0 - 1) / units0));
    {   // equal chunks of the x_l range, none empty (an empty chunk would leave its partial unwritten)
      const int64_t run = (d[l] + fz.nP - 1) / fz.nP;
      fz.nP = (d[l] + run - 1) / run;
    }
    fz.Af = c->Ap[f];
    fz.Al = c->Ap[l];
    fz.fl_o = o < l ? d[l] : 1;
    fz.fl_l = l < o ? d[o] : 1;
    const int64_t fast_rows = d[o] * d[l], loop_rows = d[o] * d[f];
    const size_t mk = c->stack.mark();
    fz.fast = c->stack.push((size_t)(d[f] / 128) * fast_rows * K);
    fz.loop = c->stack.push((size_t)fz.nP * loop_rows * K);
    if (!c->dry) {
      CUCHK(c, ttm_prepare(S, c->Ap[a], K, c->Fpad, c->st));
      {
        Prof p(c, CPPP_K_TTM, 2.0 * B * S * R * K + 4.0 * B * R * K,
               8.0 * (B * S * R + ((d[f] / 128) * fast_rows + fz.nP * loop_rows) * K));
        CUCHK(c, launch_ttm_fused(c->X, B, S, R, K, c->Fpad, fz, c->st));
      }
      const int lo = std::min(o, l), hi = std::max(o, l);
      {
        const double n1 = (double)fast_rows * K, n2 = (double)loop_rows * K;
        Prof p(c, CPPP_K_TTV, n1 * (d[f] / 128 - 1) + n2 * (fz.nP - 1),
               8.0 * (n1 * (d[f] / 128 + 1) + n2 * (fz.nP + 1)));
        CUCHK(c, launch_sum_parts(fz.fast, (int)(d[f] / 128), fast_rows * K, c->ops[lo][hi], c->st));
        CUCHK(c, launch_sum_parts(fz.loop, (int)fz.nP, loop_rows * K, c->ops[o][f], c->st));
      }
    }
    c->stack.release(mk);
  }
  return CPPP_OK;
}

// Order >= 6, unsharded: a construction tree whose level-2 nodes are the neighbour pairs of modes
// (0,1), (2,3), (4,5), ... each contracted straight from X in ONE Khatri-Rao GEMM (P:78-80 over two
// modes at once), with no s^(N-1) K level-1 node.  Every leaf M_p^(a,b) keeps two modes, so it
// contracts N-2 >= 4 of them, and those always include one whole pair of the matching ({a, b}
// meets at most two of the >= 3 pairs): the leaf hangs below the first pair disjoint from {a, b},
// from which its remaining N-4 modes are contracted in ascending order by batched multi-TTVs
// over the s^(N-2) K pair node (intermediate nodes shared between leaves, one launch per level).
// Def. pptree and this tree compute the same operators (L24: any tree gives the same values).
// C4: three GEMMs with 38 MB outputs instead of Def. pptree's three 768 MB level-1 nodes and
// their level-2 passes.  CPPP_NO_PAIR_BUILD (A/B) and the flags below select Def. pptree.
bool pair_build_ok(const cppp_ctx* c) {
  static const bool off = getenv("CPPP_NO_PAIR_BUILD") != nullptr;
  if (off || c->N < 6 || c->q >= 0 ||
      (c->flags & (CPPP_FLAG_NO_KRP | CPPP_FLAG_NO_FUSED_TTV | CPPP_FLAG_SIMT_TTM)))
    return false;
  for (int u = 0; u + 1 < c->N; u += 2) {
    int64_t B = 1, R = 1;
    for (int v = 0; v < c->N; ++v) {
      if (v < u) B *= c->dl[v];
      if (v > u + 1) R *= c->dl[v];
    }
    if (!ttm_uses_dmma(B, c->dl[u] * c->dl[u + 1], R, c->K, false)) return false;
  }
  return true;
}

cppp_status run_pair_build(cppp_ctx* c) {
  const int N = c->N;
  const uint32_t full = (1u << N) - 1;
  auto owner = [&](int a, int b) {   // the first pair (2p, 2p+1) disjoint from {a, b}
    for (int u = 0; u + 1 < N; u += 2)
      if (a != u && a != u + 1 && b != u && b != u + 1) return u;
    return -1;
  };
  for (int u = 0; u + 1 < N; u += 2) {
    std::vector<std::pair<int, int>> leaves;
    for (int a = 0; a < N; ++a)
      for (int b = a + 1; b < N; ++b)
        if (owner(a, b) == u) leaves.emplace_back(a, b);
    if (leaves.empty()) continue;
    const uint32_t kept2 = full & ~(3u << u);
    const size_t mk = c->stack.mark();
    double* P2 = c->stack.push(node_elems(c, kept2));
    cppp_status st = CPPP_OK;
    if (!contract_multi(c, Node{full, c->X, true}, std::vector<int>{u, u + 1}, P2, &st, c->Ap))
      return fail(c, CPPP_EINVAL, "pair build: GEMM shape");   // pair_build_ok checked the shapes
    STCHK(st);
    std::vector<std::pair<uint32_t, double*>> nodes{{kept2, P2}};
    auto find = [&](uint32_t m) -> double* {
      for (auto& x : nodes)
        if (x.first == m) return x.second;
      return nullptr;
    };
    for (int step = 0; step < N - 4; ++step) {
      std::vector<TtvJob> jobs;
      std::vector<std::pair<uint32_t, double*>> made;
      for (const auto& lf : leaves) {
        std::vector<int> seq;   // the modes this leaf contracts below the pair node, ascending
        for (int v = 0; v < N; ++v)
          if ((kept2 & (1u << v)) && v != lf.first && v != lf.second) seq.push_back(v);
        uint32_t parent = kept2;
        for (int t = 0; t < step; ++t) parent &= ~(1u << seq[t]);
        const uint32_t child = parent & ~(1u << seq[step]);
        bool dup = false;
        for (auto& x : made) dup |= (x.first == child);
        if (dup) continue;
        double* dst = (step == N - 5) ? c->ops[lf.first][lf.second] : c->stack.push(node_elems(c, child));
        TtvJob j = single_job(c, Node{parent, find(parent), false}, seq[step], fac_local(c, c->Ap, seq[step]), dst);
        j.stream = (double)node_elems(c, parent) * 8.0 > 64.0 * (1 << 20);
        jobs.push_back(j);
        made.emplace_back(child, dst);
      }
      STCHK(run_ttv_jobs(c, jobs));
      for (auto& x : made) nodes.push_back(x);
    }
    c->stack.release(mk);
  }
  return CPPP_OK;
}

cppp_status run_pp_build(cppp_ctx* c, bool have12 = false) {
  const int N = c->N, K = c->K;
  if (!c->dry) {
    for (int n = 0; n < N; ++n) {
      CUCHK(c, cudaMemcpyAsync(c->Ap[n], c->A[n], sizeof(double) * c->s[n] * K,
                               cudaMemcpyDeviceToDevice, c->st));
      CUCHK(c, cudaMemsetAsync(c->dA[n], 0, sizeof(double) * c->s[n] * K, c->st));
    }
  }
  if (fused_build_ok(c)) {
    STCHK(run_fused_build(c));
  } else if (pair_build_ok(c)) {
    STCHK(run_pair_build(c));
  } else {
    PPTree t{c};
    t.have12 = have12 && reuse12(c);
    STCHK(t.run());
  }
  // leaves that contracted the sharded mode hold partial sums: all-reduce them, one call over
  // their contiguous span (SURVEY C-b)
  if (c->q >= 0) STCHK(allreduce(c, c->ops_red, c->ops_red_count));
  STCHK(build_singles(c));
  if (!c->dry) c->ops_valid = true;
  return CPPP_OK;
}

// One PP term list for mode n (operator reads per L5: (i,n) is the transpose of (n,i)).
// terms i with dA^(i) known to be exactly zero (zero_mask bit i) are left out: they add +0.0
void pp_terms(cppp_ctx* c, int n, bool skip_q, PPUpdateArgs* a, uint32_t zero_mask = 0u) {
  const int K = c->K;
  a->nterms = 0;
  for (int i = 0; i < c->N; ++i) {
    if (i == n || (skip_q && i == c->q) || (zero_mask & (1u << i))) continue;
    PPTerm t;
    const int lo = std::min(i, n), hi = std::max(i, n);
    t.op = c->ops[lo][hi];
    t.dA = fac_local(c, c->dA, i);
    t.nx = c->dl[i];
    if (i < n) {  // stored [x_i][y][k]
      t.sx = c->dl[n] * K;
      t.sy = K;
    } else {      // stored [y][x_i][k]
      t.sx = K;
      t.sy = c->dl[i] * K;
    }
    a->t[a->nterms++] = t;
  }
}

cppp_status pp_update_mode(cppp_ctx* c, int n, double* out, const double* extra, bool skip_q,
                           const double* Mp, uint32_t zero_mask = 0u) {
  if (c->dry) return CPPP_OK;
  PPUpdateArgs a;
  a.Mp = Mp;
  a.extra = extra;
  a.ny = c->dl[n];
  a.K = c->K;
  a.out = out;
  a.partial = c->pp_partial;
  pp_terms(c, n, skip_q, &a, zero_mask);
  double bytes = 8.0 * (2.0 * a.ny * a.K);
  double flops = 0.0;
  for (int i = 0; i < a.nterms; ++i) {
    bytes += 8.0 * (a.t[i].nx * a.ny * a.K + a.t[i].nx * a.K);
    flops += 2.0 * a.t[i].nx * a.ny * a.K;
  }
  Prof p(c, CPPP_K_PPUPDATE, flops, bytes);
  CUCHK(c, launch_pp_update(a, c->st));
  return CPPP_OK;
}

// PP sweep (Alg. 3).  Sharded: the mode-q terms of the other modes depend only on
// dA^(q) (mode q is updated first), so they are formed once and all-reduced once (SURVEY C-c).
// after_build: the sweep that follows a PP build starts from A = A_p, so dA^(i) = 0 for every
// mode not yet updated in this sweep (i > n); those terms are left out, and the first mode's
// M~ is M_p itself (no launch).
// A PP sweep starts with mode 0's factorization (side stream) and its PP update (main stream)
// at the same instant; when the update's CTAs reach the SMs first, the factorization's one CTA
// finds no room until they drain.  A ~3 µs one-thread kernel ahead of the update lets the
// factorization land first (CPPP_NO_STAGGER: off, for A/B).
// (only when the operators are large enough for the PP update to fill the GPU: on C1's 384 KB
// of operators the spacer only added its own latency, C1 -2.2%; C2 +0.6%, C3 +0.2%, C4 even)
bool pp_stagger(const cppp_ctx* c) {
  static const bool off = getenv("CPPP_NO_STAGGER") != nullptr;
  if (off) return false;
  double bytes = 0.0;
  for (int i = 0; i < c->N; ++i)
    for (int j = i + 1; j < c->N; ++j) bytes += 8.0 * c->dl[i] * c->dl[j] * c->K;
  return bytes >= (1 << 20);
}

cppp_status pp_monitor(cppp_ctx* c);

// The slab mode's exchange terms T_m = M_p^(q,m) ×_q dA^(q) (partial over the local rows of mode q)
// for m0 <= m < m1, m != q, then ONE all-reduce over their contiguous buffers (SURVEY C-c).
cppp_status pp_exchange_terms(cppp_ctx* c, int m0, int m1) {
  const int q = c->q;
  int f = -1, l = -1;
  for (int m = m0; m < m1; ++m) {
    if (m == q) continue;
    if (f < 0) f = m;
    l = m;
    if (c->dry) continue;
    PPUpdateArgs a;
    a.Mp = nullptr;
    a.extra = nullptr;
    a.ny = c->dl[m];
    a.K = c->K;
    a.out = c->T[m];
    a.partial = c->pp_partial;
    a.nterms = 1;
    const int lo = std::min(q, m), hi = std::max(q, m);
    PPTerm t;
    t.op = c->ops[lo][hi];
    t.dA = fac_local(c, c->dA, q);
    t.nx = c->dl[q];
    if (q < m) { t.sx = c->dl[m] * c->K; t.sy = c->K; }
    else { t.sx = c->K; t.sy = c->dl[q] * c->K; }
    a.t[0] = t;
    CUCHK(c, launch_pp_update(a, c->st));
  }
  if (f < 0) return CPPP_OK;
  return allreduce(c, c->T[f], (size_t)(c->T[l] - c->T[f]) + (size_t)c->dl[l] * c->K);
}

// Split PP update (unsharded, small operators): mode n's terms other than i = n-1 need only
// factors final before mode n-1's solve, so they are issued on st4 right after mode n-1's own
// update (capped to one CTA per SM, so that mode n-1's solves still find room); at mode n only
// the i = n-1 term is on the chain, then a combine of both partial sets.  Measured (A/B with
// CPPP_NO_PP_SPLIT): PP sweeps LAP 96 -> 78 us, P6W 97 -> 79 us; with large operators the
// capped early launch is too slow for its window (C2's 128 MB operators: 207 -> 279 us, C3's
// 4 MB: 164 -> 170 us), so only operators of at most 1 MiB take it.
bool pp_split_on(const cppp_ctx* c) {
  static const bool off = getenv("CPPP_NO_PP_SPLIT") != nullptr;
  if (off || c->q >= 0 || c->N < 3) return false;
  for (int i = 0; i < c->N; ++i)
    for (int j = i + 1; j < c->N; ++j)
      if (8.0 * c->dl[i] * c->dl[j] * c->K > (1 << 20)) return false;
  return true;
}

// the terms of mode n in `sel` (bit i: term i) into a
void pp_terms_sel(cppp_ctx* c, int n, uint32_t sel, PPUpdateArgs* a) {
  pp_terms(c, n, false, a, ~sel);
}

cppp_status pp_sweep_split(cppp_ctx* c, bool after_build) {
  const int N = c->N;
  const uint32_t all = (1u << N) - 1;
  int xsE[2] = {0, 0};
  auto zero_of = [&](int n) {
    uint32_t z = 0u;
    if (after_build)
      for (int i = n + 1; i < N; ++i) z |= 1u << i;
    return z;
  };
  auto early_mask = [&](int n) {   // mode n's terms except i = n-1 (all of them for n = 0)
    uint32_t m = all & ~(1u << n) & ~zero_of(n);
    if (n > 0) m &= ~(1u << (n - 1));
    return m;
  };
  auto base_args = [&](int n, PPUpdateArgs* a) {
    a->Mp = c->Mp[n];
    a->extra = nullptr;
    a->ny = c->dl[n];
    a->K = c->K;
    a->out = c->M[n];
    a->partial = c->pp_partial;
  };
    // the early terms of mode m, on st4 after everything issued so far on the main stream
  auto issue_early = [&](int m) -> cppp_status {
    xsE[m & 1] = 0;
    if (m >= N) return CPPP_OK;
    PPUpdateArgs a;
    base_args(m, &a);
    pp_terms_sel(c, m, early_mask(m), &a);
    if (a.nterms == 0 || c->dry) return CPPP_OK;
    CUCHK(c, cudaEventRecord(c->ev_pf, c->st));
    CUCHK(c, cudaStreamWaitEvent(c->st4, c->ev_pf, 0));
    {
      double bytes = 0.0, flops = 0.0;
      for (int i = 0; i < a.nterms; ++i) {
        bytes += 8.0 * (a.t[i].nx * a.ny * a.K + a.t[i].nx * a.K);
        flops += 2.0 * a.t[i].nx * a.ny * a.K;
      }
      Prof p(c, CPPP_K_PPUPDATE, flops, bytes, c->st4);
      CUCHK(c, launch_pp_partial(a, c->pp_part_early[m & 1], 148, &xsE[m & 1], c->st4));
    }
    CUCHK(c, cudaEventRecord(c->ev_pe[m & 1], c->st4));
    return CPPP_OK;
  };
  for (int n = 0; n < N; ++n) {
    PPUpdateArgs a;
    base_args(n, &a);
    if (n == 0) {
      pp_terms(c, 0, false, &a, zero_of(0));
      if (a.nterms == 0) {   // after a build: M~^(0) = M_p^(0)
        STCHK(issue_early(1));
        STCHK(finish_mode(c, 0, c->Mp[0], true));
        continue;
      }
      if (!c->dry && pp_stagger(c)) CUCHK(c, launch_stagger(c->st));
      STCHK(pp_update_mode(c, 0, c->M[0], nullptr, false, c->Mp[0], zero_of(0)));
      STCHK(issue_early(1));
      STCHK(finish_mode(c, 0, c->M[0], true));
      continue;
    }
    // the late term (i = n-1) on the main stream, then the early ones of mode n+1 beside it
    uint32_t late = (1u << (n - 1)) & ~zero_of(n);
    PPUpdateArgs al;
    base_args(n, &al);
    pp_terms_sel(c, n, late, &al);
    int xsL = 0;
    if (!c->dry) {
      double bytes = 8.0 * 2.0 * al.ny * al.K, flops = 0.0;
      for (int i = 0; i < al.nterms; ++i) {
        bytes += 8.0 * (al.t[i].nx * al.ny * al.K + al.t[i].nx * al.K);
        flops += 2.0 * al.t[i].nx * al.ny * al.K;
      }
      Prof p(c, CPPP_K_PPUPDATE, flops, bytes);
      CUCHK(c, launch_pp_partial(al, c->pp_partial, 0, &xsL, c->st));
      if (xsE[n & 1] > 0) CUCHK(c, cudaStreamWaitEvent(c->st, c->ev_pe[n & 1], 0));
      CUCHK(c, launch_pp_combine2(al, c->pp_part_early[n & 1], xsE[n & 1], c->pp_partial, xsL, c->st));
    }
    STCHK(issue_early(n + 1));
    STCHK(finish_mode(c, n, c->M[n], true));
  }
  if (c->policy == CPPP_POLICY_BOUND) STCHK(pp_monitor(c));
  return CPPP_OK;
}

cppp_status run_pp_sweep(cppp_ctx* c, bool after_build) {
  const int N = c->N, q = c->q;
  const bool sh = q >= 0 && comm_on(c);
  if (!sh && pp_split_on(c)) return pp_sweep_split(c, after_build);
  // Modes n < q see the current dA^(q) (the previous PP sweep's): form their exchange terms here,
  // from the live dA^(q), so nothing written to T between sweeps (pp_update, pp_second_order) can
  // leak in.  After a build dA^(q) = 0 and those terms vanish.
  if (sh && q > 0 && !after_build) STCHK(pp_exchange_terms(c, 0, q));
  for (int n = 0; n < N; ++n) {
    const double* extra = nullptr;
    if (sh && n != q && !(after_build && n < q)) extra = c->T[n];
    uint32_t zero = 0u;
    if (after_build)
      for (int i = n + 1; i < N; ++i) zero |= 1u << i;
    if (after_build && n == 0 && extra == nullptr) {
      // every term is zero (dA^(i) = 0 for i > 0): M~^(0) = M_p^(0)
      STCHK(finish_mode(c, n, c->Mp[n], true));
    } else {
      if (n == 0 && !c->dry && pp_stagger(c)) CUCHK(c, launch_stagger(c->st));
      STCHK(pp_update_mode(c, n, c->M[n], extra, sh && n != q, c->Mp[n], zero));
      STCHK(finish_mode(c, n, c->M[n], true));
    }
    // modes n > q see the dA^(q) just formed
    if (sh && n == q) STCHK(pp_exchange_terms(c, q + 1, N));
  }
  if (c->policy == CPPP_POLICY_BOUND) STCHK(pp_monitor(c));
  return CPPP_OK;
}

// The switching monitor of CPPP_POLICY_BOUND (after every PP sweep): column sums of squares of the
// sweep's M~^(n) and of (A_p, A) per mode, then the largest certificate bound into stats[3N+6].
// The slab mode's rows are local: its sums are all-reduced.
cppp_status pp_monitor(cppp_ctx* c) {
  if (c->dry) return CPPP_OK;
  const int N = c->N, K = c->K;
  int64_t smax = 0;
  for (int n = 0; n < N; ++n) smax = std::max(smax, c->s[n]);
  double* msum = c->chk + smax * K;
  double* asum = msum + 3 * N * K;
  for (int n = 0; n < N; ++n) {
    const int64_t off = (n == c->q) ? c->qoff * K : 0;
    CUCHK(c, launch_colsq(c->M[n], c->M[n], c->dl[n], K, msum + (int64_t)n * 3 * K, c->st));
    CUCHK(c, launch_colsq(c->Ap[n] + off, c->A[n] + off, c->dl[n], K, asum + (int64_t)n * 3 * K, c->st));
  }
  if (c->q >= 0 && comm_on(c)) {
    STCHK(allreduce(c, msum + (int64_t)c->q * 3 * K, (size_t)3 * K));
    STCHK(allreduce(c, asum + (int64_t)c->q * 3 * K, (size_t)3 * K));
  }
  CUCHK(c, launch_pp_bound_max(msum, asum, N, K, c->stats + 3 * N + 2, c->stats + 3 * N + 6, c->st));
  return CPPP_OK;
}

// ---------------------------------------------------------------- one sweep of a phase
cppp_status run_phase_eager(cppp_ctx* c, int phase, bool have12 = true) {
  // inside a capture the side stream must fork from an event recorded in the capture
  if (c->capturing) CUCHK(c, cudaEventRecord(c->ev_S, c->st));
  STCHK(prefetch_inverse(c, 0));
  if (phase == CPPP_PHASE_DT) {
    STCHK(run_dt(c, true, c->M));
  } else {
    if (phase == CPPP_PHASE_PP_BUILD) STCHK(run_pp_build(c, have12));
    STCHK(run_pp_sweep(c, phase == CPPP_PHASE_PP_BUILD));
  }
  return CPPP_OK;
}

// Whole sweeps replay as CUDA graphs (captured on a phase's second use, so the first use sets
// every kernel attribute eagerly).  Not used with several ranks (collectives stay eager).
cppp_status run_phase(cppp_ctx* c, int phase) {
  // NCCL collectives are captured with the sweep (a host all-reduce hook is not capturable)
  const bool graphs = !(c->flags & CPPP_FLAG_NO_GRAPH) && !(comm_on(c) && c->host_ar);
  auto& g = c->graphs[phase];
  // the captured PP-build sweep takes M_p^(1,2) from the preceding regular sweep; a build
  // forced anywhere else recomputes it, eagerly
  const bool full_build = phase == CPPP_PHASE_PP_BUILD && reuse12(c) && !c->op12_fresh;
  if (!full_build) g.uses++;
  if (full_build) {
    STCHK(run_phase_eager(c, phase, false));
  } else if (!graphs || g.uses < 2) {
    STCHK(run_phase_eager(c, phase));
  } else {
    if (!g.exec) {
      // a pending prefetch on the side stream belongs to the previous sweep: join it first
      STCHK(drain_prefetch(c));
      cudaGraph_t graph = nullptr;
      CUCHK(c, cudaStreamBeginCapture(c->st, cudaStreamCaptureModeRelaxed));
      c->capturing = true;
      c->capture_prof.clear();
      const uint64_t l0 = launch_count();
      cppp_status s = run_phase_eager(c, phase);
      g.launches = launch_count() - l0;
      note_launches(0ull - g.launches);   // captured, not executed
      c->capturing = false;
      cudaError_t e = cudaStreamEndCapture(c->st, &graph);
      if (s != CPPP_OK) {
        if (graph) cudaGraphDestroy(graph);
        return s;
      }
      if (e != cudaSuccess) return fail(c, CPPP_ECUDA, "graph capture: %s", cudaGetErrorString(e));
      e = cudaGraphInstantiate(&g.exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return fail(c, CPPP_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
      g.prof = c->capture_prof;
      c->capture_prof.clear();
      c->prefetched = -1;   // the graph starts with its own mode-0 factorization
    } else {
      STCHK(drain_prefetch(c));
    }
    CUCHK(c, cudaGraphLaunch(g.exec, c->st));
    note_launches(g.launches);
    // events recorded inside a capture cannot be waited on outside it: re-arm them eagerly
    // (after the replay the Grams are final and no factorization is pending)
    CUCHK(c, cudaEventRecord(c->ev_S, c->st));
    CUCHK(c, cudaEventRecord(c->ev_P, c->st));
    c->prefetched = -1;
    for (auto& p : g.prof) c->pending_graph.push_back(p);
  }
  if (phase == CPPP_PHASE_PP_BUILD) c->ops_valid = true;
  if (reuse12(c)) {
    c->op12_fresh = phase == CPPP_PHASE_DT;
    if (phase == CPPP_PHASE_DT) c->ops_valid = false;   // M_p^(1,2) was overwritten
  }
  return CPPP_OK;
}

// ||X||² (all-reduced), kept on the host for the fitness (L17)
cppp_status tensor_norm(cppp_ctx* c) {
  const int N = c->N;
  {
    Prof pr(c, CPPP_K_OTHER, 2.0 * c->numel_local, 8.0 * c->numel_local);
    const int nb = sqnorm_blocks(c->numel_local);
    CUCHK(c, launch_sqnorm(c->X, c->numel_local, c->sq_partial, nb, c->stats + 3 * N + 2, c->st));
  }
  STCHK(allreduce(c, c->stats + 3 * N + 2, 1));
  CUCHK(c, cudaMemcpyAsync(c->host_stats, c->stats + 3 * N + 2, sizeof(double),
                           cudaMemcpyDeviceToHost, c->st));
  CUCHK(c, cudaStreamSynchronize(c->st));
  prof_collect(c);
  c->normX_sq = c->host_stats[0];
  return CPPP_OK;
}


// ---------------------------------------------------------------- als_run: the device loop
// A run of sweeps as ONE graph launch: run_prologue_kernel arms a WHILE node; its body is a
// SWITCH over the three phase graphs (the same captured sweeps als_sweep replays) followed by
// run_decide_kernel, which takes Alg. 3's decision on the device (the statistics als_sweep
// reads back to the host) and sets both conditions.  No host round trip per sweep.
__global__ void run_prologue_kernel(RunState* rs, cudaGraphConditionalHandle hw,
                                    cudaGraphConditionalHandle hs) {
  cudaGraphSetConditional(hs, static_cast<unsigned>(rs->phase));
  cudaGraphSetConditional(hw, rs->max_sweeps > 0 ? 1u : 0u);
}

__global__ void run_decide_kernel(RunState* rs, const double* __restrict__ stats,
                                  cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hs) {
  // the operations and their order are those of als_sweep (host), no contraction
  const int N = rs->N;
  double maxrel = 0.0, gsum = 0.0;
  for (int n = 0; n < N; ++n) {
    const double na = stats[3 * n], nd = stats[3 * n + 1], ng = stats[3 * n + 2];
    const double rel = na > 0.0 ? __ddiv_rn(sqrt(nd), sqrt(na)) : (nd > 0.0 ? INFINITY : 0.0);
    maxrel = fmax(maxrel, rel);
    gsum = __dadd_rn(gsum, sqrt(ng));
  }
  const double inner = stats[3 * N], model = stats[3 * N + 1];
  const double r2 = __dadd_rn(__dsub_rn(rs->normX_sq, __dmul_rn(2.0, inner)), model);
  const double fit = __dsub_rn(1.0, __ddiv_rn(sqrt(fmax(0.0, r2)), sqrt(rs->normX_sq)));
  const bool small = maxrel < rs->eps_pp;
  const int phase = rs->phase;
  int next = phase == CPPP_PHASE_DT ? (small ? CPPP_PHASE_PP_BUILD : CPPP_PHASE_DT)
                                    : (small ? CPPP_PHASE_PP : CPPP_PHASE_DT);
  const double bound = (rs->policy == CPPP_POLICY_BOUND && phase != CPPP_PHASE_DT) ? stats[3 * N + 6] : NAN;
  if (next == CPPP_PHASE_PP && bound >= rs->policy_tol) next = CPPP_PHASE_DT;
  if (phase == CPPP_PHASE_PP_BUILD) rs->restarts++;
  const int d = rs->done;
  RunInfo& in = rs->info[d];
  in.fitness = fit;
  in.residual_sq = r2;
  in.gsum = gsum;
  in.maxrel = maxrel;
  in.bound = bound;
  in.phase = phase;
  in.next_phase = next;
  in.restarts = rs->restarts;
  in.converged = gsum <= rs->eps;
  rs->done = d + 1;
  rs->phase = next;
  cudaGraphSetConditional(hs, static_cast<unsigned>(next));
  cudaGraphSetConditional(hw, (d + 1 < rs->max_sweeps && !in.converged) ? 1u : 0u);
}

cppp_status build_run_graph(cppp_ctx* c) {
  auto& R = c->run;
  cudaGraph_t G = nullptr;
  cudaGraphNode_t pro = nullptr, wn = nullptr, sn = nullptr, dn = nullptr;
  auto bail = [&](const char* what, cudaError_t e) {
    if (G) cudaGraphDestroy(G);
    cudaGetLastError();
    c->capturing = false;
    R.failed = true;
    return fail(c, CPPP_ECUDA, "als_run graph (%s): %s", what, cudaGetErrorString(e));
  };
  cudaError_t e = cudaGraphCreate(&G, 0);
  if (e != cudaSuccess) return bail("create", e);
  if ((e = cudaGraphConditionalHandleCreate(&R.hw, G, 0, 0)) != cudaSuccess) return bail("handle", e);
  {
    cudaKernelNodeParams kp = {};
    void* args[3] = {&c->run_dev, &R.hw, &R.hs};
    kp.func = reinterpret_cast<void*>(run_prologue_kernel);
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.kernelParams = args;
    // R.hs is created below, inside the WHILE body; the prologue's copy of it is patched after
    if ((e = cudaGraphAddKernelNode(&pro, G, nullptr, 0, &kp)) != cudaSuccess)
      return bail("prologue", e);
  }
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = R.hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  if ((e = cudaGraphAddNode(&wn, G, &pro, 1, &wp)) != cudaSuccess) return bail("while", e);
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  if ((e = cudaGraphConditionalHandleCreate(&R.hs, body, 0, 0)) != cudaSuccess)
    return bail("switch handle", e);
  cudaGraphNodeParams sp = {};
  sp.type = cudaGraphNodeTypeConditional;
  sp.conditional.handle = R.hs;
  sp.conditional.type = cudaGraphCondTypeSwitch;
  sp.conditional.size = 3;
  if ((e = cudaGraphAddNode(&sn, body, nullptr, 0, &sp)) != cudaSuccess) return bail("switch", e);
  // the three phase bodies, captured from the eager sweep code (no profiling, no PDL edges)
  for (int ph = 0; ph < 3; ++ph) {
    STCHK(drain_prefetch(c));
    e = cudaStreamBeginCaptureToGraph(c->st, sp.conditional.phGraph_out[ph], nullptr, nullptr, 0,
                                      cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) return bail("capture", e);
    c->capturing = true;
    c->capture_prof.clear();
    const uint64_t l0 = launch_count();
    pdl_suppress(getenv("CPPP_RUN_NO_PDL") != nullptr);
    cppp_status s = run_phase_eager(c, ph);
    pdl_suppress(false);
    R.launches_per_sweep[ph] = launch_count() - l0;
    note_launches(0ull - R.launches_per_sweep[ph]);
    c->capturing = false;
    cudaGraph_t out = nullptr;
    e = cudaStreamEndCapture(c->st, &out);
    c->prefetched = -1;
    if (s != CPPP_OK) {
      if (G) cudaGraphDestroy(G);
      R.failed = true;
      return s;
    }
    if (e != cudaSuccess) return bail("end capture", e);
  }
  {
    cudaKernelNodeParams kp = {};
    void* args[4] = {&c->run_dev, &c->stats, &R.hw, &R.hs};
    kp.func = reinterpret_cast<void*>(run_decide_kernel);
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.kernelParams = args;
    if ((e = cudaGraphAddKernelNode(&dn, body, &sn, 1, &kp)) != cudaSuccess)
      return bail("decide", e);
  }
  {  // the prologue node was added before hs existed: set its final arguments
    cudaKernelNodeParams kp = {};
    void* args[3] = {&c->run_dev, &R.hw, &R.hs};
    kp.func = reinterpret_cast<void*>(run_prologue_kernel);
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.kernelParams = args;
    if ((e = cudaGraphKernelNodeSetParams(pro, &kp)) != cudaSuccess) return bail("prologue args", e);
  }
  e = cudaGraphInstantiate(&R.exec, G, 0);
  cudaGraphDestroy(G);
  G = nullptr;
  if (e != cudaSuccess) return bail("instantiate", e);
  return CPPP_OK;
}

// ---------------------------------------------------------------- workspace plan
struct Plan {
  size_t total = 0;
  size_t off_X = 0, off_fac = 0, off_small = 0, off_ops = 0, off_stack = 0;
  size_t stack_bytes = 0;
};

cppp_status assign_buffers(cppp_ctx* c, bool borrow, Plan* plan) {
  // sizes (bytes)
  const int N = c->N, K = c->K;
  int64_t smax = 0;
  for (int n = 0; n < N; ++n) smax = std::max(smax, c->s[n]);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  size_t oX = borrow ? 0 : take(sizeof(double) * c->numel_local);
  size_t oA[CPPP_MAX_ORDER], oAp[CPPP_MAX_ORDER], odA[CPPP_MAX_ORDER], oM[CPPP_MAX_ORDER],
      oMp[CPPP_MAX_ORDER], oT[CPPP_MAX_ORDER];
  // A and A_p feed the first-level GEMM in place (TtmOpts::direct_factor): its TMA view of the
  // last row reads up to ttm_ld(K) - K doubles past the factor (into columns the epilogue drops),
  // so each of them owns that much slack
  const size_t fac_slack = sizeof(double) * (size_t)ttm_ld(K);
  for (int n = 0; n < N; ++n) {
    oA[n] = take(sizeof(double) * c->s[n] * K + fac_slack);
    oAp[n] = take(sizeof(double) * c->s[n] * K + fac_slack);
    odA[n] = take(sizeof(double) * c->s[n] * K + fac_slack);   // (pp_second_order's GEMMs read dA)
    oM[n] = take(sizeof(double) * c->dl[n] * K);
    oMp[n] = take(sizeof(double) * c->dl[n] * K);
  }
  for (int n = 0; n < N; ++n) oT[n] = take(sizeof(double) * c->dl[n] * K);   // back to back (C-c)
  const size_t oQh = take(sizeof(double) * (8 + (size_t)K * K));   // qhdr staging
  size_t oS = take(sizeof(double) * N * K * K);
  size_t oG = take(sizeof(double) * solve_ld(K) * solve_ld(K));
  // packed factor, inverted 32 x 32 diagonal blocks, Jacobi V
  size_t oL = take(sizeof(double) * (solve_ld(K) * solve_ld(K) + 4 * 32 * 33 + K * K));
  size_t oGp = take(sizeof(double) * gram_scratch_doubles() + 64 * sizeof(unsigned int));
  size_t oLm = take(sizeof(int) * 4);
  size_t oRow = take(sizeof(double) * smax * 4);
  size_t oStats = take(sizeof(double) * (3 * N + 8));
  size_t oRun = take(sizeof(RunState));
  // TTM scratch: the padded factor of the widest first-level GEMM (a single mode, or the
  // Khatri-Rao product of a whole half: S = Π of its extents) + scheduler + split partials
  int64_t maxS = smax;
  {
    const int mid = (c->N + 1) / 2 - 1;   // DT::range's split of [0, N-1]
    int64_t sl = 1, sr = 1;
    for (int v = 0; v <= mid; ++v) sl *= c->dl[v];
    for (int v = mid + 1; v < c->N; ++v) sr *= c->dl[v];
    maxS = std::max(maxS, std::max(sl, sr));
    // the PP build's level-2 node straight from X (PPTree::level2_from_x): two neighbour modes
    if (c->N >= 4)
      for (int v = 0; v + 1 < c->N; ++v) maxS = std::max(maxS, c->dl[v] * c->dl[v + 1]);
  }
  size_t oFpad = take(sizeof(double) * ttm_scratch_doubles(maxS));   // TTM factor + scheduler
  size_t oOps[CPPP_MAX_ORDER][CPPP_MAX_ORDER];
  size_t red_lo = 0, red_hi = 0;
  for (int pass = 0; pass < 2; ++pass)   // the operators not involving q first, back to back (C-b)
    for (int i = 0; i < N; ++i)
      for (int j = i + 1; j < N; ++j) {
        const bool withq = (i == c->q || j == c->q);
        if (withq != (pass == 1)) continue;
        oOps[i][j] = take(sizeof(double) * c->dl[i] * c->dl[j] * K);
        if (pass == 0) {
          if (red_hi == 0) red_lo = oOps[i][j];
          red_hi = oOps[i][j] + sizeof(double) * c->dl[i] * c->dl[j] * K;
        }
      }
  size_t oPP = take(sizeof(double) * pp_update_scratch_doubles(smax, K, smax));
  size_t oPE0 = take(sizeof(double) * pp_update_scratch_doubles(smax, K, smax));
  size_t oPE1 = take(sizeof(double) * pp_update_scratch_doubles(smax, K, smax));
  size_t oSq = take(sizeof(double) * 2048);
  size_t oGath = take(sizeof(double) * smax * K);
  size_t oChk = take(sizeof(double) * (smax * K + 9 * N * K));
  size_t oTtv = take(sizeof(double) * ttv_scratch_doubles());
  size_t oStack = off;
  plan->off_stack = oStack;
  // dry-run the DT sweep and the PP build to size the stack
  c->dry = true;
  c->stack = Stack{};
  c->stack.dry = true;
  cppp_status s1 = run_dt(c, true, c->M);
  cppp_status s2 = run_pp_build(c);
  c->dry = false;
  if (s1 != CPPP_OK) return s1;
  if (s2 != CPPP_OK) return s2;
  plan->stack_bytes = c->stack.peak;
  plan->total = oStack + align_up(c->stack.peak) + ALIGN;
  if (!c->ws) return CPPP_OK;  // sizing only
  char* b = c->ws;
  c->X = borrow ? c->X : reinterpret_cast<double*>(b + oX);
  for (int n = 0; n < N; ++n) {
    c->A[n] = reinterpret_cast<double*>(b + oA[n]);
    c->Ap[n] = reinterpret_cast<double*>(b + oAp[n]);
    c->dA[n] = reinterpret_cast<double*>(b + odA[n]);
    c->M[n] = reinterpret_cast<double*>(b + oM[n]);
    c->Mp[n] = reinterpret_cast<double*>(b + oMp[n]);
    c->T[n] = reinterpret_cast<double*>(b + oT[n]);
  }
  c->S_all = reinterpret_cast<double*>(b + oS);
  c->Gamma = reinterpret_cast<double*>(b + oG);
  c->L = reinterpret_cast<double*>(b + oL);
  c->gram_scratch = reinterpret_cast<double*>(b + oGp);
  c->gram_counters = reinterpret_cast<unsigned int*>(b + oGp + sizeof(double) * gram_scratch_doubles());
  c->lmode = reinterpret_cast<int*>(b + oLm);
  c->rowstat = reinterpret_cast<double*>(b + oRow);
  c->stats = reinterpret_cast<double*>(b + oStats);
  c->run_dev = reinterpret_cast<RunState*>(b + oRun);
  c->Fpad = reinterpret_cast<double*>(b + oFpad);
  for (int i = 0; i < N; ++i)
    for (int j = i + 1; j < N; ++j) c->ops[i][j] = reinterpret_cast<double*>(b + oOps[i][j]);
  c->ops_red = reinterpret_cast<double*>(b + red_lo);
  c->ops_red_count = (red_hi - red_lo) / sizeof(double);
  c->qhdr = reinterpret_cast<double*>(b + oQh);
  c->pp_partial = reinterpret_cast<double*>(b + oPP);
  c->pp_part_early[0] = reinterpret_cast<double*>(b + oPE0);
  c->pp_part_early[1] = reinterpret_cast<double*>(b + oPE1);
  c->sq_partial = reinterpret_cast<double*>(b + oSq);
  c->gath = reinterpret_cast<double*>(b + oGath);
  c->chk = reinterpret_cast<double*>(b + oChk);
  c->ttv_scratch = reinterpret_cast<double*>(b + oTtv);
  c->stack = Stack{};
  c->stack.base = b + oStack;
  c->stack.cap = c->ws_bytes - oStack;
  c->stack.dry = false;
  return CPPP_OK;
}

cppp_status validate(cppp_ctx* c, int N, const int64_t* s, int K, const cppp_opts* o) {
  if (N < 3 || N > CPPP_MAX_ORDER)
    return fail(c, CPPP_EINVAL, "order N=%d out of range [3, %d]", N, CPPP_MAX_ORDER);
  if (K < 1 || K > CPPP_MAX_RANK)
    return fail(c, CPPP_EINVAL, "rank K=%d out of range [1, %d]", K, CPPP_MAX_RANK);
  if (!s) return fail(c, CPPP_EINVAL, "null sizes");
  for (int n = 0; n < N; ++n)
    if (s[n] < 1) return fail(c, CPPP_EINVAL, "dimension mismatch: s[%d]=%lld < 1", n, (long long)s[n]);
  if (o && o->shard_mode != -1) {
    const int q = o->shard_mode;
    if (q < 0 || q >= N) return fail(c, CPPP_EINVAL, "shard mode %d outside [0, %d)", q, N);
    if (o->shard_offset < 0 || o->shard_extent < 1 || o->shard_offset + o->shard_extent > s[q])
      return fail(c, CPPP_EINVAL, "shard [%lld, +%lld) outside mode %d of size %lld",
                  (long long)o->shard_offset, (long long)o->shard_extent, q, (long long)s[q]);
  }
  return CPPP_OK;
}

void setup_dims(cppp_ctx* c, int N, const int64_t* s, int K, const cppp_opts* o) {
  c->N = N;
  c->K = K;
  c->flags = o ? o->flags : 0u;   // the plan (tree shapes) depends on the flags
  for (int n = 0; n < N; ++n) c->s[n] = c->dl[n] = s[n];
  c->q = -1;
  if (o && o->shard_mode >= 0 && o->shard_mode < N) {
    c->q = o->shard_mode;
    c->qoff = o->shard_offset;
    c->qext = o->shard_extent;
    c->dl[c->q] = o->shard_extent;
  }
  c->numel_local = 1;
  for (int n = 0; n < N; ++n) c->numel_local *= c->dl[n];
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Host sources go up in 16 MiB pieces: the copy engine serves its queue in order, so a large
// upload for one context (the next tensor of a serving loop) must not hold a small transfer of
// another context (its factors) for the whole 0.5-32 GB copy.
cppp_status copy_in(cppp_ctx* c, double* dst, const double* src, size_t n) {
  const size_t chunk = is_device_ptr(src) ? n : (size_t(16) << 20) / sizeof(double);
  for (size_t o = 0; o < n; o += chunk) {
    const size_t m = std::min(chunk, n - o);
    CUCHK(c, cudaMemcpyAsync(dst + o, src + o, m * sizeof(double), cudaMemcpyDefault, c->st));
  }
  return CPPP_OK;
}
cppp_status copy_out(cppp_ctx* c, double* dst, const double* src, size_t n) {
  CUCHK(c, cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDefault, c->st));
  if (!is_device_ptr(dst)) CUCHK(c, cudaStreamSynchronize(c->st));
  return CPPP_OK;
}

// gather the sharded factor's rows: zero everything but the local rows, all-reduce
cppp_status gather_rows(cppp_ctx* c, double* buf) {
  if (c->q < 0 || !comm_on(c)) return CPPP_OK;
  const int K = c->K;
  CUCHK(c, cudaMemsetAsync(c->gath, 0, sizeof(double) * c->s[c->q] * K, c->st));
  CUCHK(c, cudaMemcpyAsync(c->gath + c->qoff * K, buf + c->qoff * K, sizeof(double) * c->qext * K,
                           cudaMemcpyDeviceToDevice, c->st));
  STCHK(allreduce(c, c->gath, (size_t)c->s[c->q] * K));
  CUCHK(c, cudaMemcpyAsync(buf, c->gath, sizeof(double) * c->s[c->q] * K, cudaMemcpyDeviceToDevice,
                           c->st));
  return CPPP_OK;
}

}  // namespace

// =====================================================================================
// C ABI
// =====================================================================================
extern "C" {

void cppp_default_opts(cppp_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->device = 0;
  o->shard_mode = -1;
  o->rank = 0;
  o->world = 1;
}

const char* cppp_status_string(int s) {
  switch (s) {
    case CPPP_OK: return "ok";
    case CPPP_EINVAL: return "invalid argument";
    case CPPP_ENOMEM: return "out of memory / workspace too small";
    case CPPP_ECUDA: return "CUDA error";
    case CPPP_ENCCL: return "NCCL error";
    case CPPP_ESTATE: return "call out of order";
    case CPPP_ENODEV: return "no CUDA device";
  }
  return "unknown status";
}

const char* cppp_version(void) { return "cppp 0.1 sm_100a"; }

uint64_t cppp_launch_count(void) { return launch_count(); }

const char* cp_last_error(const cppp_ctx* c) { return c ? c->err.c_str() : "null context"; }

size_t cppp_workspace_bytes(int N, const int64_t* s, int K, const cppp_opts* o) {
  cppp_ctx tmp;
  if (validate(&tmp, N, s, K, o) != CPPP_OK) return 0;
  setup_dims(&tmp, N, s, K, o);
  Plan p;
  const bool borrow = o && (o->flags & CPPP_FLAG_BORROW_TENSOR);
  if (assign_buffers(&tmp, borrow, &p) != CPPP_OK) return 0;
  return p.total;
}

cppp_status cppp_nccl_unique_id(void* out128) {
  if (!out128) return CPPP_EINVAL;
  if (!g_nccl.load()) return CPPP_ENCCL;
  ncclUniqueId id;
  if (g_nccl.getUniqueId(&id) != ncclSuccess) return CPPP_ENCCL;
  std::memcpy(out128, &id, sizeof(id));
  return CPPP_OK;
}

cppp_status cp_init(cppp_ctx** out, const double* X, int N, const int64_t* s, int K,
                    const cppp_opts* o_in) {
  if (!out) return CPPP_EINVAL;
  *out = nullptr;
  cppp_opts o;
  if (o_in) o = *o_in;
  else cppp_default_opts(&o);
  cppp_ctx* c = new cppp_ctx();
  *out = c;
  STCHK(validate(c, N, s, K, &o));
  if (!X) return fail(c, CPPP_EINVAL, "null tensor");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(c, CPPP_ENODEV, "no CUDA device visible");
  }
  if (o.device < 0 || o.device >= ndev) return fail(c, CPPP_EINVAL, "device %d of %d", o.device, ndev);
  c->device = o.device;
  CUCHK(c, cudaSetDevice(c->device));
  c->flags = o.flags;
  if (o.pinv_rel_tol < 0.0 || !(o.pinv_rel_tol < 1.0))
    return fail(c, CPPP_EINVAL, "pinv_rel_tol %g outside [0, 1)", o.pinv_rel_tol);
  c->pinv_tol = o.pinv_rel_tol > 0.0 ? o.pinv_rel_tol : 1e-12;
  setup_dims(c, N, s, K, &o);
  if (o.stream) c->st = static_cast<cudaStream_t>(o.stream);
  else {
    CUCHK(c, cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  // comm
  c->rank = o.rank;
  c->world = o.world < 1 ? 1 : o.world;
  c->host_ar = o.host_allreduce;
  c->host_ar_user = o.host_allreduce_user;
  if (comm_on(c) && !c->host_ar) {
    if (!o.nccl_unique_id)
      return fail(c, CPPP_EINVAL, "a communicating context needs nccl_unique_id or host_allreduce");
    // the sweeps' collectives are captured into CUDA graphs: every connection is set up when the
    // communicator is created, not lazily inside a capture (a caller's setting wins)
    setenv("NCCL_RUNTIME_CONNECT", "0", 0);
    if (!g_nccl.load()) return fail(c, CPPP_ENCCL, "cannot dlopen libnccl.so.2");
    ncclUniqueId id;
    std::memcpy(&id, o.nccl_unique_id, sizeof(id));
    ncclResult_t r = g_nccl.commInitRank(&c->comm, c->world, id, c->rank);
    if (r != ncclSuccess) return fail(c, CPPP_ENCCL, "ncclCommInitRank: %s", g_nccl.getErrorString(r));
  }
  const bool x_dev = is_device_ptr(X);
  const bool borrow = (o.flags & CPPP_FLAG_BORROW_TENSOR) && x_dev;
  if ((o.flags & CPPP_FLAG_BORROW_TENSOR) && !x_dev)
    return fail(c, CPPP_EINVAL, "CPPP_FLAG_BORROW_TENSOR needs a device pointer");
  if (borrow) c->X = const_cast<double*>(X);
  Plan p;
  STCHK(assign_buffers(c, borrow, &p));
  if (o.workspace) {
    if (o.workspace_bytes < p.total)
      return fail(c, CPPP_ENOMEM, "workspace of %zu bytes < required %zu bytes", o.workspace_bytes,
                  p.total);
    c->ws = static_cast<char*>(o.workspace);
    c->ws_bytes = o.workspace_bytes;
  } else {
    void* m = nullptr;
    if (cudaMalloc(&m, p.total) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, CPPP_ENOMEM, "cudaMalloc(%zu) failed", p.total);
    }
    c->ws = static_cast<char*>(m);
    c->ws_alloc = c->ws;
    c->ws_bytes = p.total;
    c->own_ws = true;
  }
  c->ws = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(c->ws)));
  c->ws_bytes -= ALIGN;
  if (borrow) c->X = const_cast<double*>(X);
  STCHK(assign_buffers(c, borrow, &p));
  c->borrowed = borrow;
  if (!borrow) STCHK(copy_in(c, c->X, X, (size_t)c->numel_local));
  CUCHK(c, cudaMemsetAsync(c->ws + (borrow ? 0 : align_up(sizeof(double) * c->numel_local)), 0,
                           p.off_stack - (borrow ? 0 : align_up(sizeof(double) * c->numel_local)),
                           c->st));
  CUCHK(c, cudaMallocHost(&c->host_stats, sizeof(double) * (3 * N + 8)));
  CUCHK(c, cudaMallocHost(&c->run_host, sizeof(RunState)));
  CUCHK(c, cudaEventCreate(&c->ev_a));
  CUCHK(c, cudaEventCreate(&c->ev_b));
  {  // the side stream of the Γ factorizations gets the highest priority: its one-CTA kernel is
     // on the critical path whenever M^(n) is cheap (PP sweeps), and must not queue behind the
     // CTAs of the main stream's next kernel
    int lo = 0, hi = 0;
    CUCHK(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUCHK(c, cudaStreamCreateWithPriority(&c->st2, cudaStreamNonBlocking, hi));
  }
  CUCHK(c, cudaStreamCreateWithFlags(&c->st3, cudaStreamNonBlocking));
  CUCHK(c, cudaStreamCreateWithFlags(&c->st4, cudaStreamNonBlocking));
  CUCHK(c, cudaEventCreateWithFlags(&c->ev_pf, cudaEventDisableTiming));
  CUCHK(c, cudaEventCreateWithFlags(&c->ev_pe[0], cudaEventDisableTiming));
  CUCHK(c, cudaEventCreateWithFlags(&c->ev_pe[1], cudaEventDisableTiming));
  CUCHK(c, cudaEventCreateWithFlags(&c->ev_F, cudaEventDisableTiming));
  CUCHK(c, cudaEventCreateWithFlags(&c->ev_T, cudaEventDisableTiming));
  CUCHK(c, cudaEventCreateWithFlags(&c->ev_S, cudaEventDisableTiming));
  CUCHK(c, cudaEventCreateWithFlags(&c->ev_P, cudaEventDisableTiming));
  return tensor_norm(c);
}

cppp_status cp_load_tensor(cppp_ctx* c, const double* X) {
  if (!c) return CPPP_EINVAL;
  if (!X) return fail(c, CPPP_EINVAL, "null tensor");
  STCHK(drain_prefetch(c));
  if (c->borrowed) {
    if (X != c->X)
      return fail(c, CPPP_ESTATE, "borrowed tensor: rewrite the borrowed buffer instead");
  } else {
    STCHK(copy_in(c, c->X, X, (size_t)c->numel_local));
  }
  c->factors_set = false;
  c->ops_valid = false;
  c->op12_fresh = false;
  c->next_phase = CPPP_PHASE_DT;
  return tensor_norm(c);
}

cppp_status cp_set_factors(cppp_ctx* c, const double* const* A) {
  if (!c) return CPPP_EINVAL;
  if (!A) return fail(c, CPPP_EINVAL, "null factor list");
  STCHK(drain_prefetch(c));
  for (int n = 0; n < c->N; ++n) {
    if (!A[n]) return fail(c, CPPP_EINVAL, "null factor %d", n);
    STCHK(copy_in(c, c->A[n], A[n], (size_t)c->s[n] * c->K));
  }
  for (int n = 0; n < c->N; ++n) {
    const int64_t off = (n == c->q) ? c->qoff : 0;
    CUCHK(c, launch_gram(c->A[n] + off * c->K, c->dl[n], c->K, c->S_all + (int64_t)n * c->K * c->K,
                         nullptr, nullptr, nullptr, nullptr, c->gram_scratch, c->gram_counters,
                         c->st));
    if (n == c->q) STCHK(allreduce(c, c->S_all + (int64_t)n * c->K * c->K, (size_t)c->K * c->K));
    CUCHK(c, cudaMemsetAsync(c->dA[n], 0, sizeof(double) * c->s[n] * c->K, c->st));
  }
  CUCHK(c, cudaEventRecord(c->ev_S, c->st));
  c->factors_set = true;
  c->ops_valid = false;
  c->op12_fresh = false;
  c->next_phase = CPPP_PHASE_DT;
  c->sweep = 0;
  c->restarts = 0;
  c->last_fitness = NAN;
  CUCHK(c, cudaStreamSynchronize(c->st));
  return CPPP_OK;
}

cppp_status cp_update_factors(cppp_ctx* c, const double* const* A) {
  if (!c) return CPPP_EINVAL;
  if (!A) return fail(c, CPPP_EINVAL, "null factor list");
  if (!c->factors_set) return fail(c, CPPP_ESTATE, "cp_update_factors before cp_set_factors");
  STCHK(drain_prefetch(c));
  for (int n = 0; n < c->N; ++n) {
    if (!A[n]) return fail(c, CPPP_EINVAL, "null factor %d", n);
    STCHK(copy_in(c, c->A[n], A[n], (size_t)c->s[n] * c->K));
    const int64_t off = (n == c->q) ? c->qoff : 0;
    CUCHK(c, launch_gram(c->A[n] + off * c->K, c->dl[n], c->K, c->S_all + (int64_t)n * c->K * c->K,
                         nullptr, nullptr, nullptr, nullptr, c->gram_scratch, c->gram_counters,
                         c->st));
    if (n == c->q) STCHK(allreduce(c, c->S_all + (int64_t)n * c->K * c->K, (size_t)c->K * c->K));
  }
  // with operators in place the PP state moves with the factors: dA = A - A_p, so a
  // following PP sweep (which reads dA^(i) of the modes it has not updated yet) sees the new A
  if (c->ops_valid)
    for (int n = 0; n < c->N; ++n)
      CUCHK(c, launch_sub(c->A[n], c->Ap[n], c->dA[n], c->s[n] * c->K, c->st));
  CUCHK(c, cudaEventRecord(c->ev_S, c->st));
  CUCHK(c, cudaStreamSynchronize(c->st));
  c->op12_fresh = false;
  return CPPP_OK;
}

cppp_status cp_get_factors(cppp_ctx* c, double* const* A) {
  if (!c) return CPPP_EINVAL;
  if (!A) return fail(c, CPPP_EINVAL, "null output list");
  for (int n = 0; n < c->N; ++n) {
    if (n == c->q) STCHK(gather_rows(c, c->A[n]));
    STCHK(copy_out(c, A[n], c->A[n], (size_t)c->s[n] * c->K));
  }
  CUCHK(c, cudaStreamSynchronize(c->st));
  return CPPP_OK;
}

cppp_status mttkrp_dt(cppp_ctx* c, double* const* M) {
  if (!c) return CPPP_EINVAL;
  if (!c->factors_set) return fail(c, CPPP_ESTATE, "mttkrp_dt before cp_set_factors");
  STCHK(run_dt(c, false, c->M));
  if (M) {
    for (int n = 0; n < c->N; ++n) {
      if (!M[n]) continue;
      STCHK(copy_out(c, M[n], c->M[n], (size_t)c->dl[n] * c->K));
    }
  }
  CUCHK(c, cudaStreamSynchronize(c->st));
  prof_collect(c);
  return CPPP_OK;
}

cppp_status pp_build_operators(cppp_ctx* c) {
  if (!c) return CPPP_EINVAL;
  if (!c->factors_set) return fail(c, CPPP_ESTATE, "pp_build_operators before cp_set_factors");
  STCHK(run_pp_build(c));
  c->op12_fresh = false;
  CUCHK(c, cudaStreamSynchronize(c->st));
  prof_collect(c);
  return CPPP_OK;
}

cppp_status pp_get_operator(cppp_ctx* c, int i, int j, double* out) {
  if (!c) return CPPP_EINVAL;
  if (i < 0 || j >= c->N || i >= j) return fail(c, CPPP_EINVAL, "operator (%d,%d): need 0<=i<j<N", i, j);
  if (!c->ops_valid) return fail(c, CPPP_ESTATE, "no PP operators (call pp_build_operators)");
  if (!out) return fail(c, CPPP_EINVAL, "null output");
  return copy_out(c, out, c->ops[i][j], (size_t)c->dl[i] * c->dl[j] * c->K);
}

cppp_status pp_get_single(cppp_ctx* c, int n, double* out) {
  if (!c) return CPPP_EINVAL;
  if (n < 0 || n >= c->N) return fail(c, CPPP_EINVAL, "mode %d out of range", n);
  if (!c->ops_valid) return fail(c, CPPP_ESTATE, "no PP operators (call pp_build_operators)");
  if (!out) return fail(c, CPPP_EINVAL, "null output");
  return copy_out(c, out, c->Mp[n], (size_t)c->dl[n] * c->K);
}

// M~^(n) at the current factors into `out` (dA = A - A_p already formed)
static cppp_status pp_approx_mode(cppp_ctx* c, int n, double* out) {
  const bool sh = c->q >= 0 && comm_on(c);
  if (sh && n != c->q) {
    // partial term over the local rows of the sharded mode, then all-reduce
    PPUpdateArgs a;
    a.Mp = nullptr;
    a.extra = nullptr;
    a.ny = c->dl[n];
    a.K = c->K;
    a.out = c->T[n];
    a.partial = c->pp_partial;
    a.nterms = 1;
    PPTerm t;
    t.op = c->ops[std::min(c->q, n)][std::max(c->q, n)];
    t.dA = fac_local(c, c->dA, c->q);
    t.nx = c->dl[c->q];
    if (c->q < n) { t.sx = c->dl[n] * c->K; t.sy = c->K; }
    else { t.sx = c->K; t.sy = c->dl[c->q] * c->K; }
    a.t[0] = t;
    CUCHK(c, launch_pp_update(a, c->st));
    STCHK(allreduce(c, c->T[n], (size_t)c->dl[n] * c->K));
    return pp_update_mode(c, n, out, c->T[n], true, c->Mp[n]);
  }
  return pp_update_mode(c, n, out, nullptr, false, c->Mp[n]);
}

cppp_status pp_update(cppp_ctx* c, int n, double* M_tilde) {
  if (!c) return CPPP_EINVAL;
  if (n < 0 || n >= c->N) return fail(c, CPPP_EINVAL, "mode %d out of range", n);
  if (!c->ops_valid) return fail(c, CPPP_ESTATE, "pp_update before pp_build_operators");
  // dA = A - A_p for every mode (the caller may have moved the factors)
  for (int i = 0; i < c->N; ++i)
    CUCHK(c, launch_sub(c->A[i], c->Ap[i], c->dA[i], c->s[i] * c->K, c->st));
  STCHK(pp_approx_mode(c, n, c->M[n]));
  if (M_tilde) STCHK(copy_out(c, M_tilde, c->M[n], (size_t)c->dl[n] * c->K));
  CUCHK(c, cudaStreamSynchronize(c->st));
  prof_collect(c);
  return CPPP_OK;
}

// PP error monitor (Thm 4.1): exact MTTKRPs at the
// current factors (one DT pass, M <- M), each mode's M~ into scratch, column sums of squares,
// then the ratios and the bound certificate (diag.cu), all on the device.
cppp_status pp_error(cppp_ctx* c, double* err, double* eps, double* bound) {
  if (!c) return CPPP_EINVAL;
  if (!c->factors_set) return fail(c, CPPP_ESTATE, "pp_error before cp_set_factors");
  if (!c->ops_valid) return fail(c, CPPP_ESTATE, "pp_error before pp_build_operators");
  const int N = c->N, K = c->K;
  int64_t smax = 0;
  for (int n = 0; n < N; ++n) smax = std::max(smax, c->s[n]);
  double* Mt = c->chk;
  double* msum = Mt + smax * K;          // [N][3][K]
  double* asum = msum + 3 * N * K;       // [N][3][K]
  double* out = asum + 3 * N * K;        // err | eps | bound, each [N][K]
  STCHK(run_dt(c, false, c->M));
  for (int i = 0; i < N; ++i)
    CUCHK(c, launch_sub(c->A[i], c->Ap[i], c->dA[i], c->s[i] * K, c->st));
  for (int n = 0; n < N; ++n) {
    STCHK(pp_approx_mode(c, n, Mt));
    CUCHK(c, launch_colsq(Mt, c->M[n], c->dl[n], K, msum + (int64_t)n * 3 * K, c->st));
    CUCHK(c, launch_colsq(c->Ap[n], c->A[n], c->s[n], K, asum + (int64_t)n * 3 * K, c->st));
  }
  // the sharded mode's M rows are local: its sums are completed across ranks
  if (c->q >= 0 && comm_on(c)) STCHK(allreduce(c, msum + (int64_t)c->q * 3 * K, (size_t)3 * K));
  CUCHK(c, launch_pp_error_final(msum, asum, N, K, std::sqrt(c->normX_sq), out, out + N * K,
                                 out + 2 * N * K, c->st));
  double* dst[3] = {err, eps, bound};
  for (int j = 0; j < 3; ++j)
    if (dst[j]) STCHK(copy_out(c, dst[j], out + (int64_t)j * N * K, (size_t)N * K));
  CUCHK(c, cudaStreamSynchronize(c->st));
  prof_collect(c);
  return CPPP_OK;
}

// Second-order PP term: T2^(n) = Σ_{i<j; i,j≠n} M_p^(i,j,n) ×_i dA^(i)
// ×_j dA^(j).  M_p^(i,j,n) ×_i dA^(i) ×_j dA^(j) is the MTTKRP of mode n with the factor list
// (dA^(i), dA^(j), A_p elsewhere) (Def. 3.1 is multilinear), so one exact pass of the dimension tree
// with that list gives pair (i,j)'s contribution to every mode n ∉ {i,j} at once: C(N,2) passes,
// the contributions added per mode in ascending pair order (the oracle's order).  c->T holds the
// sums (dead between sweeps), c->M is overwritten; factors, operators and the phase state are kept.
cppp_status pp_second_order(cppp_ctx* c, double* const* T2) {
  if (!c) return CPPP_EINVAL;
  if (!c->factors_set) return fail(c, CPPP_ESTATE, "pp_second_order before cp_set_factors");
  if (!c->ops_valid) return fail(c, CPPP_ESTATE, "pp_second_order before pp_build_operators");
  const int N = c->N, K = c->K;
  STCHK(drain_prefetch(c));
  for (int i = 0; i < N; ++i) {
    CUCHK(c, launch_sub(c->A[i], c->Ap[i], c->dA[i], c->s[i] * K, c->st));
    CUCHK(c, cudaMemsetAsync(c->T[i], 0, sizeof(double) * c->dl[i] * K, c->st));
  }
  double* saved[CPPP_MAX_ORDER];
  for (int m = 0; m < N; ++m) saved[m] = c->A[m];
  cppp_status st = CPPP_OK;
  for (int i = 0; i < N && st == CPPP_OK; ++i)
    for (int j = i + 1; j < N && st == CPPP_OK; ++j) {
      for (int m = 0; m < N; ++m) c->A[m] = (m == i || m == j) ? c->dA[m] : c->Ap[m];
      st = run_dt(c, false, c->M);
      for (int n = 0; n < N && st == CPPP_OK; ++n) {
        if (n == i || n == j) continue;
        cudaError_t e = launch_add(c->M[n], c->T[n], c->dl[n] * K, c->st);
        if (e != cudaSuccess) st = fail(c, CPPP_ECUDA, "pp_second_order add: %s", cudaGetErrorString(e));
      }
    }
  for (int m = 0; m < N; ++m) c->A[m] = saved[m];
  STCHK(st);
  if (T2)
    for (int n = 0; n < N; ++n)
      if (T2[n]) STCHK(copy_out(c, T2[n], c->T[n], (size_t)c->dl[n] * K));
  CUCHK(c, cudaStreamSynchronize(c->st));
  prof_collect(c);
  return CPPP_OK;
}

cppp_status cp_set_pp_policy(cppp_ctx* c, int policy, double tol) {
  if (!c) return CPPP_EINVAL;
  if (policy != CPPP_POLICY_EPS_PP && policy != CPPP_POLICY_BOUND)
    return fail(c, CPPP_EINVAL, "unknown PP policy %d", policy);
  if (policy == CPPP_POLICY_BOUND && !(tol > 0.0)) return fail(c, CPPP_EINVAL, "policy tolerance must be > 0");
  if (policy != c->policy) {   // the monitor is part of the PP sweep: recapture the graphs
    STCHK(drain_prefetch(c));
    CUCHK(c, cudaStreamSynchronize(c->st));
    for (auto& g : c->graphs) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      for (auto& p : g.prof) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
      }
      g = cppp_ctx::SweepGraph{};
    }
    if (c->run.exec) cudaGraphExecDestroy(c->run.exec);
    c->run = cppp_ctx::RunGraph{};
  }
  c->policy = policy;
  c->policy_tol = tol;
  return CPPP_OK;
}

cppp_status cp_set_phase_override(cppp_ctx* c, int phase) {
  if (!c) return CPPP_EINVAL;
  if (phase < CPPP_PHASE_AUTO || phase > CPPP_PHASE_PP) return fail(c, CPPP_EINVAL, "bad phase %d", phase);
  c->override_phase = phase;
  return CPPP_OK;
}

cppp_status als_sweep(cppp_ctx* c, double eps, double eps_pp, cppp_sweep_info* info) {
  if (!c) return CPPP_EINVAL;
  if (!c->factors_set) return fail(c, CPPP_ESTATE, "als_sweep before cp_set_factors");
  if (!(eps_pp >= 0.0)) return fail(c, CPPP_EINVAL, "eps_pp must be >= 0");
  const int phase = c->override_phase != CPPP_PHASE_AUTO ? c->override_phase : c->next_phase;
  if (phase == CPPP_PHASE_PP && !c->ops_valid)
    return fail(c, CPPP_ESTATE, "PP sweep requested without operators");
  CUCHK(c, cudaEventRecord(c->ev_a, c->st));
  STCHK(run_phase(c, phase));
  if (phase == CPPP_PHASE_PP_BUILD) c->restarts++;
  CUCHK(c, cudaEventRecord(c->ev_b, c->st));
  const int N = c->N;
  CUCHK(c, cudaMemcpyAsync(c->host_stats, c->stats, sizeof(double) * (3 * N + 7),
                           cudaMemcpyDeviceToHost, c->st));
  CUCHK(c, cudaStreamSynchronize(c->st));
  prof_collect(c);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev_a, c->ev_b);
  const double* hs = c->host_stats;
  double maxrel = 0.0, gsum = 0.0;
  for (int n = 0; n < N; ++n) {
    const double na = hs[3 * n], nd = hs[3 * n + 1], ng = hs[3 * n + 2];
    const double rel = na > 0.0 ? std::sqrt(nd) / std::sqrt(na) : (nd > 0.0 ? INFINITY : 0.0);
    maxrel = std::max(maxrel, rel);
    gsum += std::sqrt(ng);
  }
  const double inner = hs[3 * N], model = hs[3 * N + 1];
  const double r2 = c->normX_sq - 2.0 * inner + model;
  const double fit = 1.0 - std::sqrt(std::max(0.0, r2)) / std::sqrt(c->normX_sq);
  const bool small = maxrel < eps_pp;
  if (phase == CPPP_PHASE_DT) c->next_phase = small ? CPPP_PHASE_PP_BUILD : CPPP_PHASE_DT;
  else c->next_phase = small ? CPPP_PHASE_PP : CPPP_PHASE_DT;
  // CPPP_POLICY_BOUND: a PP phase continues only while the monitor's certificate stays below tol;
  // otherwise it ends like a failed ε_pp test: one regular sweep (exact MTTKRPs) follows, and
  // Alg. 3 decides from there whether to rebuild
  const double bound = (c->policy == CPPP_POLICY_BOUND && phase != CPPP_PHASE_DT) ? hs[3 * N + 6] : NAN;
  if (c->next_phase == CPPP_PHASE_PP && bound >= c->policy_tol) c->next_phase = CPPP_PHASE_DT;
  c->sweep++;
  c->last_fitness = fit;
  if (info) {
    info->sweep = c->sweep;
    info->phase = phase;
    info->fitness = fit;
    info->residual_sq = r2;
    info->grad_norm_sum = gsum;
    info->max_rel_dA = maxrel;
    info->next_phase = c->next_phase;
    info->restarts = c->restarts;
    info->converged = gsum <= eps;
    info->seconds = ms * 1e-3;
    info->approximate = phase != CPPP_PHASE_DT;
    info->pp_bound = bound;
  }
  return CPPP_OK;
}

cppp_status als_run(cppp_ctx* c, double eps, double eps_pp, int max_sweeps, cppp_sweep_info* info,
                    int* done) {
  if (!c) return CPPP_EINVAL;
  if (!c->factors_set) return fail(c, CPPP_ESTATE, "als_run before cp_set_factors");
  if (!(eps_pp >= 0.0)) return fail(c, CPPP_EINVAL, "eps_pp must be >= 0");
  if (max_sweeps < 0 || max_sweeps > RUN_MAX)
    return fail(c, CPPP_EINVAL, "max_sweeps must be in [0, %d]", RUN_MAX);
  if (done) *done = 0;
  if (max_sweeps == 0) return CPPP_OK;
  // the host loop: profiling events, several ranks (collectives stay eager), no graphs, a
  // forced phase, or a GPU/driver that cannot build the conditional graph
  const bool host_loop = (c->flags & (CPPP_FLAG_PROFILE | CPPP_FLAG_NO_GRAPH)) || (comm_on(c) && c->host_ar) ||
                         c->override_phase != CPPP_PHASE_AUTO || c->run.failed ||
                         (c->next_phase == CPPP_PHASE_PP && !c->ops_valid) ||
                         (c->next_phase == CPPP_PHASE_PP_BUILD && reuse12(c) && !c->op12_fresh);
  if (host_loop) {
    for (int i = 0; i < max_sweeps; ++i) {
      cppp_sweep_info one;
      STCHK(als_sweep(c, eps, eps_pp, &one));
      if (info) info[i] = one;
      if (done) *done = i + 1;
      if (one.converged) break;
    }
    return CPPP_OK;
  }
  if (!c->run.exec) {
    cppp_status s = build_run_graph(c);
    if (s != CPPP_OK) {   // fall back for good (recorded in cp_last_error)
      c->run.failed = true;
      return als_run(c, eps, eps_pp, max_sweeps, info, done);
    }
  }
  STCHK(drain_prefetch(c));
  RunState* h = c->run_host;
  h->eps = eps;
  h->eps_pp = eps_pp;
  h->normX_sq = c->normX_sq;
  h->max_sweeps = max_sweeps;
  h->done = 0;
  h->phase = c->next_phase;
  h->restarts = c->restarts;
  h->N = c->N;
  h->policy = c->policy;
  h->policy_tol = c->policy_tol;
  const size_t head = offsetof(RunState, info);
  CUCHK(c, cudaMemcpyAsync(c->run_dev, h, head, cudaMemcpyHostToDevice, c->st));
  CUCHK(c, cudaEventRecord(c->ev_a, c->st));
  CUCHK(c, cudaGraphLaunch(c->run.exec, c->st));
  CUCHK(c, cudaEventRecord(c->ev_b, c->st));
  CUCHK(c, cudaMemcpyAsync(h, c->run_dev, head + sizeof(RunInfo) * max_sweeps,
                           cudaMemcpyDeviceToHost, c->st));
  CUCHK(c, cudaStreamSynchronize(c->st));
  // events recorded inside a capture cannot be waited on outside it: re-arm them eagerly
  CUCHK(c, cudaEventRecord(c->ev_S, c->st));
  CUCHK(c, cudaEventRecord(c->ev_P, c->st));
  c->prefetched = -1;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev_a, c->ev_b);
  const int n = h->done;
  for (int i = 0; i < n; ++i) {
    const RunInfo& r = h->info[i];
    note_launches(c->run.launches_per_sweep[r.phase] + 1);   // + the decision kernel
    if (r.phase == CPPP_PHASE_PP_BUILD) c->ops_valid = true;
    if (reuse12(c)) {
      c->op12_fresh = r.phase == CPPP_PHASE_DT;
      if (r.phase == CPPP_PHASE_DT) c->ops_valid = false;
    }
    c->sweep++;
    if (info) {
      cppp_sweep_info& o = info[i];
      o.sweep = c->sweep;
      o.phase = r.phase;
      o.fitness = r.fitness;
      o.residual_sq = r.residual_sq;
      o.grad_norm_sum = r.gsum;
      o.max_rel_dA = r.maxrel;
      o.next_phase = r.next_phase;
      o.restarts = r.restarts;
      o.converged = r.converged;
      o.seconds = ms * 1e-3 / n;   // the run is one launch: its device time, shared evenly
      o.approximate = r.phase != CPPP_PHASE_DT;
      o.pp_bound = r.bound;
    }
  }
  note_launches(1);   // the prologue
  c->next_phase = h->phase;
  c->restarts = h->restarts;
  if (n > 0) c->last_fitness = h->info[n - 1].fitness;
  if (done) *done = n;
  return CPPP_OK;
}

cppp_status fitness(cppp_ctx* c, double* f) {
  if (!c) return CPPP_EINVAL;
  if (!f) return fail(c, CPPP_EINVAL, "null output");
  if (c->sweep == 0) return fail(c, CPPP_ESTATE, "fitness before any sweep");
  *f = c->last_fitness;
  return CPPP_OK;
}

cppp_status fitness_exact(cppp_ctx* c, double* f, double* residual_sq) {
  if (!c) return CPPP_EINVAL;
  if (!c->factors_set) return fail(c, CPPP_ESTATE, "fitness_exact before cp_set_factors");
  const int N = c->N, K = c->K, n = N - 1;
  STCHK(run_dt(c, false, c->M));   // exact M^(n) at the current factors (no factor update)
  double* fit = c->stats + 3 * N + 4;
  const int64_t off = (n == c->q) ? c->qoff : 0;
  CUCHK(c, launch_fit_terms(c->M[n], c->A[n] + off * K, c->dl[n], K, c->S_all, N, n, fit, c->st));
  if (n == c->q) STCHK(allreduce(c, fit, 1));   // the slab mode's rows are local
  CUCHK(c, cudaMemcpyAsync(c->host_stats, fit, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CUCHK(c, cudaStreamSynchronize(c->st));
  prof_collect(c);
  const double r2 = c->normX_sq - 2.0 * c->host_stats[0] + c->host_stats[1];
  if (residual_sq) *residual_sq = r2;
  if (f) *f = 1.0 - std::sqrt(std::max(0.0, r2)) / std::sqrt(c->normX_sq);
  return CPPP_OK;
}

cppp_status cppp_kernel_stats(cppp_ctx* c, int kclass, cppp_kernel_stat* out) {
  if (!c) return CPPP_EINVAL;
  if (kclass < 0 || kclass >= CPPP_K_COUNT || !out) return fail(c, CPPP_EINVAL, "bad kernel class");
  prof_collect(c);
  *out = c->kstat[kclass];
  return CPPP_OK;
}

cppp_status cppp_reset_kernel_stats(cppp_ctx* c) {
  if (!c) return CPPP_EINVAL;
  prof_collect(c);
  std::memset(c->kstat, 0, sizeof(c->kstat));
  return CPPP_OK;
}

cppp_status cppp_generate(cppp_ctx* c, double* X_dev, int N, const int64_t* s, int K,
                          const double* const* A_true, int noise_kind, double noise, uint64_t seed,
                          int64_t row_lo, int64_t row_hi, void* stream) {
  if (!X_dev || !s || !A_true || N < 2 || N > CPPP_MAX_ORDER || K < 1 || K > CPPP_MAX_RANK)
    return c ? fail(c, CPPP_EINVAL, "cppp_generate: bad arguments") : CPPP_EINVAL;
  if (row_lo < 0 || row_hi > s[0] || row_lo > row_hi)
    return c ? fail(c, CPPP_EINVAL, "cppp_generate: bad row range") : CPPP_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // stage factors on device
  std::vector<double*> Ad(N, nullptr);
  size_t tot = 0;
  for (int n = 0; n < N; ++n) tot += s[n] * K;
  const int64_t nrows = row_hi - row_lo;
  const size_t part = gen_partials_doubles(nrows);
  double* buf = nullptr;
  if (cudaMalloc(&buf, sizeof(double) * (tot + 2 * s[0] + part + 1)) != cudaSuccess)
    return c ? fail(c, CPPP_ENOMEM, "cppp_generate: cudaMalloc") : CPPP_ENOMEM;
  cppp_status rc = CPPP_OK;
  double* p = buf;
  for (int n = 0; n < N && rc == CPPP_OK; ++n) {
    Ad[n] = p;
    if (cudaMemcpyAsync(p, A_true[n], sizeof(double) * s[n] * K, cudaMemcpyDefault, st) != cudaSuccess)
      rc = CPPP_ECUDA;
    p += s[n] * K;
  }
  double* rowsq_x = p;
  double* rowsq_z = p + s[0];
  double* partials = p + 2 * s[0];
  double* scale = partials + part;
  if (rc == CPPP_OK && launch_gen_kruskal(X_dev, N, s, K, Ad.data(), row_lo, row_hi, st) != cudaSuccess)
    rc = CPPP_ECUDA;
  if (rc == CPPP_OK && noise_kind == 1 && noise != 0.0) {
    if (launch_gen_noise_add(X_dev, s, N, seed, row_lo, row_hi, nullptr, noise, st) != cudaSuccess)
      rc = CPPP_ECUDA;
  } else if (rc == CPPP_OK && noise_kind == 2 && noise != 0.0) {
    cudaMemsetAsync(rowsq_x, 0, sizeof(double) * 2 * s[0], st);
    if (launch_gen_noise_rowsq(X_dev, s, N, seed, row_lo, row_hi, rowsq_x, rowsq_z, partials, st) !=
        cudaSuccess)
      rc = CPPP_ECUDA;
    if (rc == CPPP_OK && c && comm_on(c)) {
      cudaStream_t save = c->st;
      c->st = st;
      rc = allreduce(c, rowsq_x, 2 * (size_t)s[0]);
      c->st = save;
    }
    if (rc == CPPP_OK && launch_gen_scale(rowsq_x, rowsq_z, s[0], noise, scale, st) != cudaSuccess)
      rc = CPPP_ECUDA;
    if (rc == CPPP_OK &&
        launch_gen_noise_add(X_dev, s, N, seed, row_lo, row_hi, scale, 0.0, st) != cudaSuccess)
      rc = CPPP_ECUDA;
  }
  cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(buf);
  if (rc == CPPP_OK && e != cudaSuccess) rc = CPPP_ECUDA;
  if (rc != CPPP_OK && c && c->err.empty()) c->err = "cppp_generate: CUDA error";
  return rc;
}

size_t cppp_plan_describe(int N, int shard_mode, char* buf, size_t buflen) {
  // host-only listing of the two trees (no device needed)
  std::string out;
  if (N < 3 || N > CPPP_MAX_ORDER) return 0;
  int64_t s[CPPP_MAX_ORDER];
  for (int n = 0; n < N; ++n) s[n] = 4;
  cppp_opts o;
  cppp_default_opts(&o);
  if (shard_mode >= 0 && shard_mode < N) {
    o.shard_mode = shard_mode;
    o.shard_offset = 0;
    o.shard_extent = 2;
  }
  // PP tree listing (Def. pptree) in tree-mode terms and physical kept sets
  cppp_ctx tmp;
  setup_dims(&tmp, N, s, 1, &o);
  PPTree t{&tmp};
  t.init();
  out += "pptree tau:";
  for (int i = 0; i < N; ++i) out += " " + std::to_string(t.tau[i]);
  out += "\n";
  // BFS over levels
  std::vector<uint32_t> level{0u};
  for (int l = 1; l <= N - 2; ++l) {
    std::vector<uint32_t> next;
    for (uint32_t mu : level) {
      int maxmu = -1;
      for (int q = 0; q < N; ++q)
        if (mu & (1u << q)) maxmu = q;
      for (int w = maxmu + 1; w <= l + 1; ++w) {
        const uint32_t cmu = mu | (1u << w);
        next.push_back(cmu);
        const uint32_t kept = t.kept_of(cmu);
        out += "L" + std::to_string(l) + " kept:";
        for (int v = 0; v < N; ++v)
          if (kept & (1u << v)) out += " " + std::to_string(v);
        out += " contract:" + std::to_string(t.tau[w]) + (l == 1 ? " ttm" : " ttv");
        out += (l == N - 2) ? " leaf\n" : "\n";
      }
    }
    level.swap(next);
  }
  const size_t need = out.size() + 1;
  if (buf && buflen) {
    const size_t n = std::min(buflen - 1, out.size());
    std::memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return need;
}

void cp_destroy(cppp_ctx* c) {
  if (!c) return;
  if (c->st) cudaStreamSynchronize(c->st);
  if (c->st3) cudaStreamSynchronize(c->st3);
  if (c->st4) cudaStreamSynchronize(c->st4);
  if (c->st2) cudaStreamSynchronize(c->st2);
  prof_collect(c);
  for (auto e : c->evpool) cudaEventDestroy(e);
  if (c->ev_a) cudaEventDestroy(c->ev_a);
  if (c->ev_b) cudaEventDestroy(c->ev_b);
  if (c->host_stats) cudaFreeHost(c->host_stats);
  if (c->run_host) cudaFreeHost(c->run_host);
  if (c->run.exec) cudaGraphExecDestroy(c->run.exec);
  if (c->own_ws && c->ws_alloc) cudaFree(c->ws_alloc);
  if (c->comm) g_nccl.commDestroy(c->comm);
  if (c->host_ar_buf) cudaFreeHost(c->host_ar_buf);
  for (auto& g : c->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    for (auto& p : g.prof) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
  }
  if (c->ev_S) cudaEventDestroy(c->ev_S);
  if (c->ev_P) cudaEventDestroy(c->ev_P);
  if (c->st2) cudaStreamDestroy(c->st2);
  if (c->st3) cudaStreamDestroy(c->st3);
  if (c->st4) cudaStreamDestroy(c->st4);
  if (c->ev_pf) cudaEventDestroy(c->ev_pf);
  for (auto& ev : c->ev_pe)
    if (ev) cudaEventDestroy(ev);
  if (c->ev_F) cudaEventDestroy(c->ev_F);
  if (c->ev_T) cudaEventDestroy(c->ev_T);
  if (c->own_stream && c->st) cudaStreamDestroy(c->st);
  delete c;
}

}  // extern "C"
