/*
 * cppp.h — C ABI of libcppp.so: the B200 (sm_100a) hot path of CP-ALS with pairwise
 * perturbation (PP), arXiv 1811.10573.
 *
 * Citations: "P:n" = line n of the paper source, "Lnn" = reading nn of the
 * ambiguity ledger (repeated in DESIGN.md).
 *
 * Conventions (all entry points)
 *   - FP64 only.  All arrays are row-major (last index fastest).  Modes are 0-based
 *     (the paper's mode m is index m-1).
 *   - X is an order-N dense tensor s_0 x ... x s_{N-1}.  A factor A^(n) is s_n x K.
 *   - Every partially contracted intermediate keeps its uncontracted modes in increasing
 *     mode order with the rank index k LAST (Def. 3.1).  A PP operator
 *     M_p^(i,j), i<j, is therefore s_i x s_j x K.
 *   - Pointers may be host or device memory unless stated otherwise; the library asks the
 *     CUDA runtime which one it got (cudaPointerGetAttributes) and copies when needed.
 *   - Calls are ordered on the context's stream.  Only calls that return host values
 *     (getters with host outputs, fitness, als_sweep's info) synchronize that stream.
 *   - Errors: every call returns a cppp_status; nothing aborts.  cp_last_error() gives a
 *     message for the last failing call on that context.  A NULL ctx gives CPPP_EINVAL.
 *   - The context owns no host threads.  A context is bound to one device and must be
 *     used from one host thread at a time.
 */
#ifndef CPPP_H
#define CPPP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CPPP_MAX_ORDER 8          /* N <= 8 */
#define CPPP_MAX_RANK 128         /* K <= 128: the on-device K x K solve keeps Gamma in shared memory */

typedef struct cppp_ctx cppp_ctx;

typedef enum {
  CPPP_OK = 0,
  CPPP_EINVAL = -1,   /* shape / rank / mode mismatch, bad argument */
  CPPP_ENOMEM = -2,   /* workspace too small (message carries the required size) or cudaMalloc failed */
  CPPP_ECUDA = -3,    /* CUDA runtime error (message carries cudaGetErrorString) */
  CPPP_ENCCL = -4,    /* NCCL error or NCCL library not loadable when world > 1 */
  CPPP_ESTATE = -5,   /* call out of order, e.g. pp_update before pp_build_operators */
  CPPP_ENODEV = -6    /* no usable CUDA device */
} cppp_status;

typedef enum {
  CPPP_PHASE_AUTO = -1,     /* let Alg. 3 decide (P:576-598 with L7-L11) */
  CPPP_PHASE_DT = 0,        /* regular dimension-tree ALS sweep (Alg. 1) */
  CPPP_PHASE_PP_BUILD = 1,  /* build PP operators then one PP sweep */
  CPPP_PHASE_PP = 2         /* PP sweep with the existing operators */
} cppp_phase;

/* opts.flags */
#define CPPP_FLAG_BORROW_TENSOR 1u  /* X is a device pointer the caller keeps alive; not copied */
#define CPPP_FLAG_SIMT_TTM      2u  /* force the SIMT (non-tensor-core) TTM kernel (testing) */
#define CPPP_FLAG_PROFILE       4u  /* time each kernel class with CUDA events (cppp_kernel_stats) */
#define CPPP_FLAG_NO_FUSED_TTV  8u  /* order 4: build the PP operators through Def. pptree's level-1
                                        nodes instead of the fused level 1 -> level 2 GEMMs (A/B testing) */
#define CPPP_FLAG_NO_GRAPH     16u  /* run sweeps eagerly instead of replaying captured CUDA graphs */
#define CPPP_FLAG_NO_KRP       32u  /* regular DT sweep: single-mode first-level TTMs instead of one
                                        multi-mode (Khatri-Rao) GEMM per half (testing) */
#define CPPP_FLAG_NO_OVERLAP   64u  /* order-3 DT sweep: run the second first-level TTM after mode 1
                                        instead of beside it (testing) */
#define CPPP_FLAG_FORCE_COMM  128u  /* take the communicating (sharded) code paths even with one
                                        rank: with a one-rank NCCL communicator this runs the
                                        all-reduce transport on a single GPU (testing) */
#define CPPP_FLAG_NO_OP_REUSE 256u /* order 3: PP builds recompute M_p^(1,2) instead of taking the
                                      preceding regular sweep's X x_0 A^(0) (A/B testing) */
#define CPPP_FLAG_NO_FUSED_SOLVE 512u /* K <= 32, modes <= 64 rows: solve each mode through the
                                      factorization + row-solve + Gram kernels instead of the one
                                      fused launch (A/B testing; the two are bit-identical) */

typedef struct {
  int device;               /* CUDA ordinal (default 0) */
  void *stream;             /* cudaStream_t to order all work on; NULL = library-owned stream */
  void *workspace;          /* device buffer of >= cppp_workspace_bytes(); NULL = library cudaMalloc */
  size_t workspace_bytes;
  unsigned flags;           /* CPPP_FLAG_* */
  /* slab sharding of X along one mode (multi-GPU):
   * this process holds rows [shard_offset, shard_offset+shard_extent) of mode shard_mode (any
   * mode 0..N-1; X is then the dense local slab, extent shard_extent in that mode).
   * shard_mode = -1: X is whole.  s[] passed to cp_init are the GLOBAL sizes. */
  int shard_mode;
  int64_t shard_offset, shard_extent;
  /* NCCL bootstrap (world > 1): 128-byte ncclUniqueId created by rank 0 (cppp_nccl_unique_id)
   * and broadcast by the caller, e.g. through torch.distributed. */
  const void *nccl_unique_id;
  int rank, world;
  /* Optional host-side all-reduce (sum) used INSTEAD of NCCL when world > 1: the library copies
   * the device buffer to pinned host memory, calls host_allreduce(buf, count, user) (which must
   * leave the element-wise sum over all ranks in buf and return 0), and copies it back.  Lets
   * several contexts on ONE device (one host thread each) run the sharded algebra in tests. */
  int (*host_allreduce)(double *buf, size_t count, void *user);
  void *host_allreduce_user;
  /* τ of the normal-equation solve (L13): Cholesky of Γ^(n) is accepted iff every
   * pivot > τ·max diag Γ; otherwise the eigen pseudo-inverse drops eigenvalues <= τ·λ_max.
   * 0 = the default 1e-12; must lie in [0, 1). */
  double pinv_rel_tol;
} cppp_opts;

/* Per-sweep record (S:505 trace schema). */
typedef struct {
  int sweep;                 /* 1-based count of sweeps since cp_init / cp_set_factors */
  int phase;                 /* cppp_phase actually run */
  double fitness;            /* 1 - ||X-[[A]]|| / ||X|| by the expansion of S:177 (L17) */
  double residual_sq;        /* the (unclamped) radicand of that expansion */
  double grad_norm_sum;      /* sum_n ||G^(n)||_F (Alg. 1/3 stop metric) */
  double max_rel_dA;         /* max_n ||dA^(n)||_F / ||A^(n)||_F (L7) */
  int next_phase;            /* what CPPP_PHASE_AUTO will run next */
  int restarts;              /* number of PP operator builds so far */
  int converged;             /* grad_norm_sum <= eps */
  double seconds;            /* device time of this sweep (CUDA events) */
  double pp_bound;           /* CPPP_POLICY_BOUND, PP sweeps: the switching monitor's value (the
                                largest certificate bound, see cp_set_pp_policy); NaN otherwise */
  int approximate;           /* 1 when fitness/residual_sq come from the PP-approximated M~^(N)
                                (a PP sweep): then r² is only O(ε²)-accurate and may be
                                negative (clamped in fitness, L17/L27); fitness_exact() gives the
                                exact value.  0 after a regular sweep (exact M^(N)). */
} cppp_sweep_info;

/* Kernel classes for cppp_kernel_stats. */
typedef enum {
  CPPP_K_TTM = 0,       /* first-level TTM X x_m A^(m) (DMMA GEMM) */
  CPPP_K_TTV = 1,       /* multi-TTV (lower tree levels, PP construction tree) */
  CPPP_K_PPUPDATE = 2,  /* fused PP update over all pairs */
  CPPP_K_SOLVE = 3,     /* Gram / Hadamard / Cholesky / row solves / gradient */
  CPPP_K_OTHER = 4,
  CPPP_K_FACTOR = 5,    /* Γ^(n) and its Cholesky factor (side stream, overlapped with M^(n)) */
  CPPP_K_COUNT = 6
} cppp_kernel_class;

typedef struct {
  int64_t launches;
  double total_ms;          /* summed CUDA-event durations on the context stream */
  double flops;             /* algorithmic flops of those launches */
  double bytes;             /* algorithmic HBM bytes of those launches */
} cppp_kernel_stat;

/* Fill *o with defaults (device 0, library stream, library workspace, unsharded, world 1). */
void cppp_default_opts(cppp_opts *o);

/* Bytes of device workspace cp_init needs for this problem (includes a copy of X unless
 * CPPP_FLAG_BORROW_TENSOR): the problem of P:7 / P:572-573 (X, N, s, R) sizes everything -- the
 * factors, the N(N-1)/2 operators of Def. pptree and the tree intermediates, planned by
 * a dry run of one regular sweep and one PP build.  Returns 0 on invalid arguments. */
size_t cppp_workspace_bytes(int N, const int64_t *s, int K, const cppp_opts *o);

/* Create a context for tensor X (order N, GLOBAL sizes s[0..N-1], rank K): the input of CP-ALS
 * with pairwise perturbation, "Input: tensor X, rank R, tolerance" (P:7, Alg. 3).
 *   X: host or device pointer to this rank's slab (whole tensor when unsharded), row-major.
 *   Computes ||X||_F^2 (all-reduced when sharded).  Factors start at zero: call
 *   cp_set_factors before any sweep.  3 <= N <= CPPP_MAX_ORDER, 1 <= K <= CPPP_MAX_RANK. */
cppp_status cp_init(cppp_ctx **ctx, const double *X, int N, const int64_t *s, int K,
                    const cppp_opts *o);

/* Replace the tensor of an existing context with a new one of the same shape (host or device
 * pointer, same slab), recompute ||X||_F^2, and drop the factors and the PP state (call
 * cp_set_factors next).  Keeps the workspace and the captured sweep graphs, so a serving loop
 * can alternate two contexts: the next tensor uploads on one context's stream while the other
 * runs its sweeps.  A context created with CPPP_FLAG_BORROW_TENSOR accepts only its own
 * borrowed pointer (after the caller rewrote that buffer); any other pointer -> CPPP_ESTATE. */
cppp_status cp_load_tensor(cppp_ctx *ctx, const double *X);

/* Set A^(n) for n = 0..N-1 (A[n] is s_n x K, GLOBAL rows even when sharded): the initial
 * factors of Alg. 3 ("initialize A^(1..N)"; L15 for the seeded recipe), and reset the PP
 * state (no operators), the sweep counter and the phase machine (next sweep is DT, L9). */
cppp_status cp_set_factors(cppp_ctx *ctx, const double *const *A);
/* Overwrite the current factors A (and their Grams) WITHOUT resetting the PP snapshot, the
 * operators or the phase machine — e.g. to evaluate pp_update at A = A_p + dA. */
cppp_status cp_update_factors(cppp_ctx *ctx, const double *const *A);
/* Copy the current factors out (GLOBAL rows; sharded runs gather the slab mode's rows). */
cppp_status cp_get_factors(cppp_ctx *ctx, double *const *A);

/* All N MTTKRPs M^(n) = X_(n)(⊙_{m≠n} A^(m)) with the current, fixed factors,
 * computed through the dimension tree (first-level TTMs + multi-TTV).  M[n] is s_n x K.
 * Parity entry for hot-path part (a). */
cppp_status mttkrp_dt(cppp_ctx *ctx, double *const *M);

/* A_p := A, dA := 0, then all N(N-1)/2 operators M_p^(i,j) via the Def. pptree
 * construction tree and M_p^(n) = M_p^(j,n) x_j A_p^(j).
 * Parity entry for hot-path part (b). */
cppp_status pp_build_operators(cppp_ctx *ctx);
/* out (s_i x s_j x K, i<j) := M_p^(i,j).  CPPP_ESTATE before a build. */
cppp_status pp_get_operator(cppp_ctx *ctx, int i, int j, double *out);
/* out (s_n x K) := M_p^(n). */
cppp_status pp_get_single(cppp_ctx *ctx, int n, double *out);

/* M~^(n) = M_p^(n) + Σ_{i≠n} M_p^(i,n) x_i dA^(i) with dA = A - A_p, written to
 * M_tilde (s_n x K).  Parity entry for hot-path part (c).  CPPP_ESTATE before a build. */
cppp_status pp_update(cppp_ctx *ctx, int n, double *M_tilde);

/* PP error monitor (Thm 4.1).  At the current factors A and
 * the operators' A_p (dA = A - A_p), for every mode n and column k (outputs N x K, row n):
 *   err[n][k]   = ||m~_k^(n) - m_k^(n)|| / ||m_k^(n)||      (M~ as pp_update, M the exact MTTKRP)
 *   eps[n][k]   = ||da_k^(n)|| / ||a_k^(n)||                (the ε_k^(n) of Thm 4.1)
 *   bound[n][k] = ||X||_F Σ_{S ⊆ modes≠n, |S|>=2} Π_{i∈S} ||da_k^(i)|| Π_{j∉S} ||a_p,k^(j)||
 *                 / ||m_k^(n)||   — a certificate: err <= bound (the second-and-higher-order terms
 *                 of the P:548 expansion, each bounded with ||X x_S v|| <= ||X||_F Π||v||).
 * A ratio with a zero denominator is 0 when its numerator is 0, else +inf.  Any output may be
 * NULL (host or device pointers).  Costs one DT pass (M is left holding the exact MTTKRPs) and N
 * PP updates; factors, operators and the phase state are unchanged.  CPPP_ESTATE before
 * cp_set_factors or pp_build_operators. */
cppp_status pp_error(cppp_ctx *ctx, double *err, double *eps, double *bound);

/* Second-order PP term (the first term the PP update P:553 drops): at the
 * current factors A and the operators' A_p (dA = A - A_p), for every mode n
 *   T2[n] = Σ_{i<j; i,j≠n} M_p^(i,j,n) ×_i dA^(i) ×_j dA^(j)      (s_n x K, local rows)
 * with M_p^(i,j,n) the Def. 3.1 intermediate at A_p keeping (i,j,n).  M~^(n) + T2[n] is the
 * second-order PP update: exact for N = 3, O(ε³) otherwise.  Computed as C(N,2) exact MTTKRP passes
 * of the dimension tree with the factor lists (dA on {i,j}, A_p elsewhere) -- a diagnostic, each
 * pass costs about a regular sweep's contractions.  T2[n] host or device (NULL entries skipped);
 * factors, operators and the phase state are unchanged.  CPPP_ESTATE before a build. */
cppp_status pp_second_order(cppp_ctx *ctx, double *const *T2);

/* One CP-ALS-PP sweep (Alg. 3, readings L7-L12): phase chosen by the state
 * machine unless cp_set_phase_override forces it.  eps: global stop on Σ||G||;
 * eps_pp: PP tolerance on the relative factor change.  info may be NULL. */
cppp_status als_sweep(cppp_ctx *ctx, double eps, double eps_pp, cppp_sweep_info *info);
/* Up to max_sweeps (<= 1024) sweeps of Alg. 3 in ONE device launch: the phase decisions that
 * als_sweep takes on the host after every sweep (L7-L11) are taken by a kernel on the device, and
 * a CUDA graph with a WHILE node over a SWITCH of the three phase graphs runs the sweeps back to
 * back.  Stops early once grad_norm_sum <= eps.  info[0..*done) (may be NULL) gets the per-sweep
 * records (seconds = the run's device time / *done).  Same results as the same number of
 * als_sweep calls; falls back to those calls with CPPP_FLAG_PROFILE, CPPP_FLAG_NO_GRAPH, several
 * ranks, or a phase override. */
cppp_status als_run(cppp_ctx *ctx, double eps, double eps_pp, int max_sweeps,
                    cppp_sweep_info *info, int *done);
/* PP switching policy (the "alternative schemes for switching" of P:1134).
 *   CPPP_POLICY_EPS_PP (default): Alg. 3 as read in L7-L11 (ε_pp test on max ||dA||/||A||).
 *   CPPP_POLICY_BOUND: the same transitions, and after every PP sweep a monitor evaluates, per mode
 *     n and column k, the certificate of pp_error (||X||_F Σ_{|S|>=2} Π_{i∈S}||da_k^(i)||
 *     Π_{j∉S}||a_p,k^(j)|| / ||m~_k^(n)||, from column norms only: no tensor pass); when its maximum
 *     reaches tol, the PP phase ends as after a failed ε_pp test: the next sweep is a regular one
 *     (exact MTTKRPs), and Alg. 3 decides from there whether to rebuild.  info.pp_bound reports
 *     the value.  tol > 0.
 * Changing the policy drops the captured sweep graphs (recaptured on the next sweeps). */
#define CPPP_POLICY_EPS_PP 0
#define CPPP_POLICY_BOUND 1
cppp_status cp_set_pp_policy(cppp_ctx *ctx, int policy, double tol);

/* Force the phase of the next sweeps (CPPP_PHASE_AUTO to release); used to replay the
 * oracle's phase schedule in parity runs (L12). */
cppp_status cp_set_phase_override(cppp_ctx *ctx, int phase);

/* Fitness of the last sweep (L17): 1 - sqrt(max(0, r²))/||X||, r² by the S:177 expansion with
 * that sweep's last M^(N) (approximate after a PP sweep: see cppp_sweep_info.approximate). */
cppp_status fitness(cppp_ctx *ctx, double *f);
/* Exact fitness at the CURRENT factors (L17): one exact MTTKRP pass through the dimension
 * tree (the cost of a regular sweep without the solves; M^(n) buffers are overwritten, factors,
 * operators and the phase state are not), then r² = ||X||² - 2<M^(N), A^(N)> + 1ᵀ(Γ^(N)∗S^(N))1
 * on the device.  f (may be NULL) = 1 - sqrt(max(0, r²))/||X||; residual_sq (may be NULL) = r²
 * unclamped.  Host outputs; synchronizes.  CPPP_ESTATE before cp_set_factors. */
cppp_status fitness_exact(cppp_ctx *ctx, double *f, double *residual_sq);

/* Per-kernel-class statistics since the last reset (CPPP_FLAG_PROFILE only). */
cppp_status cppp_kernel_stats(cppp_ctx *ctx, int kclass, cppp_kernel_stat *out);
cppp_status cppp_reset_kernel_stats(cppp_ctx *ctx);

/* Device generator (twin of synthgen): writes rows [row_lo,row_hi) of
 * mode 0 of X = [[A_true]] + noise into X_dev (device, (row_hi-row_lo) x prod s[1..]).
 *   A_true: N host or device arrays s_n x K.  noise_kind 0 none, 1 absolute std, 2 relative
 *   eta*||X_true||/||Z||.  For sharded relative noise the per-row squared norms are
 *   all-reduced through ctx's communicator when ctx != NULL and world > 1. */
cppp_status cppp_generate(cppp_ctx *ctx, double *X_dev, int N, const int64_t *s, int K,
                          const double *const *A_true, int noise_kind, double noise,
                          uint64_t seed, int64_t row_lo, int64_t row_hi, void *stream);

/* 128-byte NCCL unique id for a new communicator (rank 0 only). */
cppp_status cppp_nccl_unique_id(void *out128);

/* Host-only helpers (no device needed): the plans the engine executes.
 * cppp_plan_describe writes a human-readable listing of the DT sweep and the PP
 * construction tree (Def. pptree) for N modes with the given sharded mode (-1 none);
 * returns the number of bytes needed (including NUL). */
size_t cppp_plan_describe(int N, int shard_mode, char *buf, size_t buflen);

void cp_destroy(cppp_ctx *ctx);
const char *cp_last_error(const cppp_ctx *ctx);
const char *cppp_status_string(int status);
/* Total kernel launches issued by this library in this process (all contexts). */
uint64_t cppp_launch_count(void);
/* Library build id "cppp <version> sm_100a". */
const char *cppp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CPPP_H */
