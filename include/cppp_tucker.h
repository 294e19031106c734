/*
 * cppp_tucker.h — C ABI of the PP-Tucker contraction path in libcppp.so:
 * the TTMc work of Tucker-ALS (HOOI, Alg. 2) and of pairwise perturbation for Tucker
 * (Def. 3.2, Alg. 4), on the same FP64 tensor-core GEMM as the CP path.
 *
 * A full HOOI / PP-Tucker run (tk_hosvd, tk_sweep) runs on the device as well: the factor
 * update is a Gram matrix, a top-R symmetric eigensolver (Householder tridiagonalization,
 * bisection, inverse iteration) and a sign fix.
 *
 * Conventions (in addition to cppp.h's: FP64, row-major, 0-based modes, host or device pointers,
 * stream ordering, status codes):
 *   - X is s_0 x ... x s_{N-1} (3 <= N <= 8); factor A^(n) is s_n x R_n (R_n <= s_n), used as
 *     X x_n A^(n)T: the rank index z_n takes mode n's place.
 *   - Results are returned in the CANONICAL layout: modes in their original order, x_m at a kept
 *     mode, z_m at a contracted one.  Y^(n) is R_0 x .. x s_n x .. x R_{N-1}; the operator
 *     Y_p^(i,j) (i < j) has s_i at position i, s_j at j and R_m elsewhere.
 *   - The context copies X to device memory unless CPPP_FLAG_BORROW_TENSOR (then X must be a
 *     device pointer the caller keeps alive); CPPP_FLAG_SIMT_TTM forces the SIMT contraction
 *     kernel (testing).  Device memory is allocated by the library (cudaMalloc).
 */
#ifndef CPPP_TUCKER_H
#define CPPP_TUCKER_H

#include "cppp.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tk_ctx tk_ctx;

typedef struct {
  int sweep;            /* 1-based count since tk_set_factors / tk_hosvd */
  int phase;            /* cppp_phase actually run */
  int next_phase;       /* what the Alg. 4 state machine picks next (readings T4) */
  int converged;        /* core_change <= eps (T5) */
  double core_change;   /* ||G_new - G||_F (Alg. 2 F) */
  double core_norm;     /* ||G||_F */
  double residual;      /* sqrt(max(0, ||X||^2 - ||G||^2)) / ||X|| (orthonormal factors) */
  double max_rel_dA;    /* max_n ||dA^(n)||_F / ||A^(n)||_F (the eps_pp test, T4) */
} tk_sweep_info;

/* New context on the current device; stream = cudaStream_t (NULL = legacy default).
 * CPPP_EINVAL for N outside [3, 8], a dimension < 1, or R_n outside [1, s_n]. */
cppp_status tk_init(tk_ctx **ctx, const double *X, int N, const int64_t *s, const int *R,
                    void *stream, unsigned flags);
/* A[n]: s_n x R_n.  Drops the PP operators. */
cppp_status tk_set_factors(tk_ctx *ctx, const double *const *A);
/* Moves the factors, keeping the operators (dA = A - A_p for tk_pp_update). */
cppp_status tk_update_factors(tk_ctx *ctx, const double *const *A);
/* All N TTMcs Y^(n) = X x_{m != n} A^(m)T at the current factors, through the binary
 * dimension tree (each edge one TTM on the DMMA GEMM).  Y[n] may be NULL. */
cppp_status tk_ttmc(tk_ctx *ctx, double *const *Y);
/* A_p := A, dA := 0, the N(N-1)/2 operators Y_p^(i,j) = X x_{m not in {i,j}} A_p^(m)T via the
 * Def. pptree construction tree (Ttmc_Map_PP), and Y_p^(n) = Y_p^(j,n) x_j A_p^(j)T,
 * j = min{j != n} (reading T3). */
cppp_status tk_pp_build(tk_ctx *ctx);
/* out := Y_p^(i,j), i < j (canonical layout).  CPPP_ESTATE before a build. */
cppp_status tk_pp_get_operator(tk_ctx *ctx, int i, int j, double *out);
/* out := Y_p^(n) (canonical layout).  CPPP_ESTATE before a build. */
cppp_status tk_pp_get_single(tk_ctx *ctx, int n, double *out);
/* Y~^(n) = Y_p^(n) + sum_{i != n} Y_p^(i,n) x_i dA^(i)T with dA = A - A_p, terms in
 * ascending i.  CPPP_ESTATE before a build. */
cppp_status tk_pp_update(tk_ctx *ctx, int n, double *Y_tilde);
/* HOSVD initialization: A^(n) = the R_n leading left singular vectors of X_(n) from
 * the Gram matrix X_(n) X_(n)^T (sign: largest-magnitude entry positive, T2), core
 * G = X x_1 A^(1)T .. x_N A^(N)T.  Needs every s_n <= 128 (one-CTA eigensolver); else
 * CPPP_EINVAL (set the factors instead). */
cppp_status tk_hosvd(tk_ctx *ctx);
/* One sweep of PP-Tucker-ALS (Alg. 4; plain Alg. 2 when eps_pp = 0): regular sweeps
 * update A^(n) from the exact Y^(n) through the dimension tree (Gauss-Seidel order), PP sweeps
 * from Y~^(n) of the operators (built first in a pp-build sweep); the core G = Y^(N) x_N A^(N)T
 * from the last mode's Y (T1).  Every step on the device: TTMc GEMMs, the smaller Gram of Y_(n)
 * (s_n or prod of the other ranks; must be <= 128, else CPPP_EINVAL), top-R eigensolver,
 * selection and sign fix.  info may be NULL. */
cppp_status tk_sweep(tk_ctx *ctx, double eps, double eps_pp, tk_sweep_info *info);
/* Force the next sweeps' phase (CPPP_PHASE_AUTO to release), as cp_set_phase_override. */
cppp_status tk_set_phase_override(tk_ctx *ctx, int phase);
cppp_status tk_get_factors(tk_ctx *ctx, double *const *A);
/* G (R_0 x .. x R_{N-1}) of the last sweep (or of the initial factors). */
cppp_status tk_get_core(tk_ctx *ctx, double *G);
const char *tk_last_error(const tk_ctx *ctx);
void tk_destroy(tk_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* CPPP_TUCKER_H */
