/*
 * cppp_tucker.h — C ABI of the PP-Tucker contraction path in libcppp.so:
 * the TTMc work of Tucker-ALS (HOOI, Alg. 2) and of pairwise perturbation for Tucker
 * (Def. 3.2, Alg. 4), on the same FP64 tensor-core GEMM as the CP path.
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
const char *tk_last_error(const tk_ctx *ctx);
void tk_destroy(tk_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* CPPP_TUCKER_H */
