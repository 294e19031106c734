// internal.h — shared declarations of the libcppp.so translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#define CPPP_MAX_TERMS_ 8
#define CPPP_MAX_ORDER_ 8

#include <utility>

// Programmatic dependent launch: kernels started with launch_pdl may be scheduled while the
// previous kernel on the stream drains (its launch latency and prologue overlap the tail); each
// of them calls pdl_wait() before touching anything an earlier kernel wrote.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Let the next kernel on the stream launch before this one ends (its CTAs run up to their own
// pdl_wait).  Called after pdl_wait by the kernels that feed the fused small-mode solve, whose
// pre-wait part (Γ and its factorization) reads only data of kernels two or more launches back.
#ifndef CPPP_NO_TRIGGER   // A/B builds
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#else
__device__ __forceinline__ void pdl_trigger() {}
#endif
#endif
namespace cppp {
bool pdl_enabled();   // false when CPPP_NO_PDL is set (A/B measurements) or suppressed
void pdl_suppress(bool on);   // this thread: plain launches (graph bodies that reject PDL edges)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
}  // namespace cppp

namespace cppp {

struct Dims {
  int64_t s[8];
};

// Count of kernel launches issued by this library (all contexts), for the bench's
// gpu_launches claim.  note_launch() follows every <<<>>> in the library.
void note_launch();
void note_launches(uint64_t n);   // n may be a wrapped negative (two's complement)
uint64_t launch_count();

// ---------------------------------------------------------------- kernel launchers
// All launchers enqueue on `st` and return the launch's cudaError_t.

// TTM (first tree level, P:78-80 / P:408-414): out[b][r][n] = Σ_x X[b][x][r] * F[x][n]
// X viewed as [B][S][R] (row-major), F is S x K (ld K), out is [B][R][K].
// R == 1 is the natural mode-(N-1) unfolding X(BxS)·F; R > 1 contracts a middle/first mode.
// Uses the DMMA (FP64 tensor core) kernel with TMA staging when the shape allows it (even
// S and R, K <= 128), else the SIMT FP64 kernel.  `Fpad` is scratch of ttm_scratch_doubles(S)
// doubles (padded factor, the persistent kernel's tile counter and tail tickets, tail partials;
// zeroed once, left zeroed).
cudaError_t launch_ttm(const double* X, int64_t B, int64_t S, int64_t R,
                       const double* F, int K, double* out, double* Fpad,
                       bool force_simt, cudaStream_t st);
// The two halves of launch_ttm, so the engine can time the GEMM alone: ttm_prepare pads F
// into Fpad (no-op for the SIMT path); launch_ttm_core runs the GEMM.
bool ttm_uses_dmma(int64_t B, int64_t S, int64_t R, int K, bool force_simt);
cudaError_t ttm_prepare(int64_t S, const double* F, int K, double* Fpad, cudaStream_t st);
// doubles of TTM scratch (`Fpad`) for a contracted extent S (padded factor + scheduler + tail)
size_t ttm_scratch_doubles(int64_t S);
// Multi-mode first level: KR = A^(m_0) ⊙ ... ⊙ A^(m_{h-1}) (consecutive modes, row-major over
// (x_0..x_{h-1})) into the padded-factor area of Fpad; then launch_ttm_padded contracts X viewed
// as [B][S = Π s_{m_j}][R] with it (DMMA path only: ttm_uses_dmma must hold).
struct KrpArgs {
  const double* F[CPPP_MAX_ORDER_];
  int64_t dims[CPPP_MAX_ORDER_];
  int nm;
  int K;
  int ld;          // set by ttm_prepare_krp
  int64_t rows;    // set by ttm_prepare_krp
};
cudaError_t ttm_prepare_krp(const KrpArgs& a, double* Fpad, cudaStream_t st);
// Tucker's multi-mode contraction: the Kronecker product F_0 ⊗ ... ⊗ F_{h-1} (F_j: dims[j] x
// ranks[j]; rows (x_0..x_{h-1}) and columns (z_0..z_{h-1}) row-major, Π ranks <= 128) into the
// padded-factor area of Fpad, for launch_ttm_padded with K = Π ranks.
struct KronArgs {
  const double* F[CPPP_MAX_ORDER_];
  int64_t dims[CPPP_MAX_ORDER_];
  int ranks[CPPP_MAX_ORDER_];
  int nm;
  int cols;        // set by ttm_prepare_kron
  int ld;          // set by ttm_prepare_kron
  int64_t rows;    // set by ttm_prepare_kron
};
cudaError_t ttm_prepare_kron(const KronArgs& a, double* Fpad, cudaStream_t st);
cudaError_t launch_ttm_padded(const double* X, int64_t B, int64_t S, int64_t R, int K, double* out,
                              const double* Fpad, cudaStream_t st);
// Scheduling of one GEMM beside other streams' work: reserve_sms SMs get no (persistent) CTA;
// max_stages (>= 2) caps the shared-memory ring so small kernels can share the SMs.
struct TtmOpts {
  int reserve_sms = 0;
  int max_stages = 0;
  // DMMA path: read the factor F (S x K, K even, 16-byte aligned) in place instead of the padded
  // copy ttm_prepare makes; the last row's last box reads up to ttm_ld(K) - K doubles past
  // F + S*K (only into discarded columns), so F must sit inside a larger allocation
  bool direct_factor = false;
};
// whether launch_ttm_core can take F in place (TtmOpts::direct_factor)
bool ttm_direct_ok(const double* F, int K);
// padded column count of the GEMM's factor tiles (a multiple of 16 >= K)
int ttm_ld(int K);
cudaError_t launch_ttm_core(const double* X, int64_t B, int64_t S, int64_t R, const double* F,
                            int K, double* out, const double* Fpad, bool force_simt,
                            cudaStream_t st, TtmOpts topt = TtmOpts{});
// Fused PP-construction level 1 -> level 2 (order 4): the m-contiguous GEMM
// T = X ×_a F (F padded in Fpad, as ttm_prepare leaves it) whose epilogue contracts every tile of T
// into two leaves -- the fast leaf over the last kept mode f (s_f % 128 == 0; nh = s_f / 128
// block partials) and the loop leaf over mode l (nP x_l-chunk partials); T itself is never
// written.  Then launch_sum_parts adds the partials in order.
struct TtmFused {
  int64_t o_str, l_str;    // tile strides (flattened kept index / 128) of x_o, x_l
  int64_t n_o, n_l, sf;    // extents of modes o, l, f
  int64_t nP;              // x_l chunks (loop-leaf partials)
  const double* Af;        // s_f x K
  const double* Al;        // s_l x K
  double* fast;            // [s_f / 128][n_o n_l][K]
  int64_t fl_o, fl_l;      // fast-leaf row strides of x_o, x_l
  double* loop;            // [nP][n_o s_f][K]
};
bool ttm_fused_ok(int64_t B, int64_t S, int64_t R, int K, int64_t sf);
cudaError_t launch_ttm_fused(const double* X, int64_t B, int64_t S, int64_t R, int K, const double* Fpad,
                             const TtmFused& f, cudaStream_t st);
// out[e] = Σ_{q < np} part[q n + e] (q ascending)
cudaError_t launch_sum_parts(const double* part, int np, int64_t n, double* out, cudaStream_t st);
cudaError_t launch_ttm_simt(const double* X, int64_t B, int64_t S, int64_t R,
                            const double* F, int K, double* out, cudaStream_t st);
bool ttm_dmma_supported(int64_t B, int64_t S, int64_t R, int K);

// Multi-TTV: rank-diagonal contraction of one mode of a parent intermediate,
// out[b][r][k] = Σ_x P[b][x][r][k] * F[x][k];  parent viewed as [B][S][R][K].
// Small outputs split x over a (1, xs, 1) cluster reduced over DSMEM; `scratch` is unused.
cudaError_t launch_ttv(const double* P, int64_t B, int64_t S, int64_t R, int K,
                       const double* F, double* out, double* scratch, cudaStream_t st);
size_t ttv_scratch_doubles();
cudaError_t launch_ttv_cfg(const double* P, int64_t B, int64_t S, int64_t R, int K,
                           const double* F, double* out, int V, int U, int xs, cudaStream_t st);

// Batched multi-TTV (ttv.cu): job j views its parent as [Bo][Sa][Sb][IN] (IN includes K) and
// writes outB[bo][xa][t] = Σ_xb P·Fb[xb][k]; a PAIR job (Fa != null, Sb <= TTV_PAIR_MAXSB) also writes
// outA[bo][xb][t] = Σ_xa P·Fa[xa][k] from the same pass over the parent (Sb <= TTV_PAIR_MAXSB).
// Single jobs: Sa = 1.
struct TtvJob {
  const double* P = nullptr;
  const double* Fa = nullptr;
  const double* Fb = nullptr;
  double* outA = nullptr;
  double* outB = nullptr;
  int64_t Bo = 1, IN = 1;
  int Sa = 1, Sb = 1;
  int64_t nvec = 0;   // set by the launcher
  int cta0 = 0;       // set by the launcher
  int stream = 0;     // parent read with evict-first loads (large parents)
};
constexpr int TTV_MAX_JOBS = 24;
constexpr int TTV_PAIR_MAXSB = 24;   // inner extent of a one-pass pair (register-resident sums)
struct TtvBatch {
  TtvJob j[TTV_MAX_JOBS];
  int njobs;
  int K;
};
cudaError_t launch_ttv_batch(const TtvJob* jobs, int n, int K, cudaStream_t st);


// PP update (Alg. 3): Mt[y][k] = Mp[y][k] + extra[y][k]
//   + Σ_t Σ_x Op_t(x, y, k) * dA_t[x][k], Op_t(x,y,k) at Op_t + x*sx_t + y*sy_t + k.
struct PPTerm {
  const double* op;
  const double* dA;
  int64_t sx, sy;   // strides (doubles) of the contracted index x and of the output row y
  int64_t nx;       // extent of x
};
struct PPUpdateArgs {
  const double* Mp;       // s_n x K
  const double* extra;    // optional additive s_n x K term (sharded runs), may be null
  int nterms;
  PPTerm t[CPPP_MAX_TERMS_];
  int64_t ny;             // s_n (local)
  int K;
  double* out;            // s_n x K
  double* partial;        // scratch for split-x partial sums (>= xsplit * ny * K doubles)
};
cudaError_t launch_pp_update(const PPUpdateArgs& a, cudaStream_t st);
// the two halves of a split update: partial sums of a term subset into `partial` (*xs_used parts;
// grid_cap > 0 caps the CTAs), then out = (Mp [+ extra]) + (Σ pE parts + Σ pL parts)
cudaError_t launch_pp_partial(const PPUpdateArgs& a, double* partial, int grid_cap, int* xs_used,
                              cudaStream_t st);
cudaError_t launch_pp_combine2(const PPUpdateArgs& a, const double* pE, int xsE, const double* pL,
                               int xsL, cudaStream_t st);
size_t pp_update_scratch_doubles(int64_t ny, int K, int64_t max_nx);


// ---------------------------------------------------------------- small dense ops (K <= 128)
// Γ^(n) = Hadamard of S[m], m != n -> Gamma (ld x ld, ld = solve_ld(K), zero padding);
// Cholesky factor (L13 pivot rule) packed into Tp (ld x ld: diag 1/L[j][j], upper = Lᵀ,
// lower = L, zero padding with a unit diagonal) with
// *mode = 0, else the eigen pseudo-inverse P -> Tp with *mode = 1.  One CTA per kernel.
// Vscratch: K*K doubles (Jacobi V).
int solve_ld(int K);
cudaError_t launch_gamma_factor(const double* S_all /* N x K x K */, int N, int n, int K,
                                double* Gamma, double* Tp, int* mode, double* Vscratch,
                                cudaStream_t st, double tau = 1e-12);
// Row solves: A_new = M Γ^† (substitution with the packed factor, or M P) ; G = (A_old - A_new) Γ ;
// dA = A_new - ref ; per-row statistics -> rowstat (rows x 4: ‖a_new‖², ‖dA‖², ‖g‖², Σ m∘a_new).
// A is updated in place; ref may alias A.
cudaError_t launch_solve_rows(const double* M, double* A, const double* ref, double* dA,
                              int64_t rows, int K, const double* Gamma, const double* Tp,
                              const int* mode, double* rowstat, cudaStream_t st);
// S = AᵀA (fixed order).  With nrm: nrm[0..2] = Σ_rows rowstat[.][0..2]; with Gamma_model also
// fit[0] = Σ_rows rowstat[.][3] and fit[1] = Σ Γ∘S.  scratch: gram_scratch_doubles() doubles;
// counters: 64 zeroed device words the kernel leaves zeroed (K <= 128).
int gram_tiles(int K);
size_t gram_scratch_doubles();
cudaError_t launch_gram(const double* A, int64_t rows, int K, double* S, const double* rowstat,
                        double* nrm, const double* Gamma_model, double* fit, double* scratch,
                        unsigned int* counters, cudaStream_t st);
// One small mode (K <= 32, rows <= 64) in ONE CTA: Γ^(n) from S_all, its factorization (L13;
// the pseudo-inverse fallback through Gamma / Tp / Vscratch), A_new, G, dA, S^(n) -> Sn, and the
// statistics gram_kernel leaves (nrm[0..2]; fit[0..1] when fit != null, Γ^(n)'s S:177 terms) —
// bit-identical to launch_gamma_factor + launch_solve_rows + launch_gram.
bool mode_small_ok(int K, int64_t rows);
cudaError_t launch_mode_small(const double* S_all, int N, int n, int K, const double* M, double* A,
                              const double* ref, double* dA, int64_t rows, double* Sn, double* nrm,
                              double* fit, double* Gamma, double* Tp, double* Vscratch,
                              cudaStream_t st, double tau);
// ||x||² with a fixed reduction tree: partial[nblk] then out[0]
cudaError_t launch_sqnorm(const double* x, int64_t n, double* partial, int nblk, double* out,
                          cudaStream_t st);
int sqnorm_blocks(int64_t n);
// a one-thread ~3 µs kernel (stream-order spacer)
cudaError_t launch_stagger(cudaStream_t st);
// y = a - b (elementwise)
cudaError_t launch_sub(const double* a, const double* b, double* y, int64_t n, cudaStream_t st);
// y = y + x (elementwise)
cudaError_t launch_add(const double* x, double* y, int64_t n, cudaStream_t st);

// PP error monitor (diag.cu).  colsq: sums[0..K) = Σ_y (a−b)², [K..2K) = Σ_y b², [2K..3K) = Σ_y a²
// over a rows x K row-major pair.  pp_error_final: per (n, k) the error ratio, ε and bound
// certificate from the [N][3][K] sums of (M~, M) and (A_p, A).
cudaError_t launch_colsq(const double* a, const double* b, int64_t rows, int K, double* sums,
                         cudaStream_t st);
cudaError_t launch_pp_error_final(const double* msum, const double* asum, int N, int K,
                                  double normX, double* err, double* eps, double* bound,
                                  cudaStream_t st);
// max over (n, k) of the PP certificate bound with ||m_k|| from M~ (msum: colsq of (M~, M~))
cudaError_t launch_pp_bound_max(const double* msum, const double* asum, int N, int K,
                                const double* normX_sq, double* out, cudaStream_t st);
// fit[0] = Σ M∘A over rows x K, fit[1] = Σ (Hadamard_{m≠n} S^(m)) ∘ S^(n) (S:177 terms; one CTA)
cudaError_t launch_fit_terms(const double* M, const double* A, int64_t rows, int K,
                             const double* S_all, int N, int n, double* fit, cudaStream_t st);
// Fp[x][n] = F[x][n] for n < K, 0 for K <= n < ld (TMA-aligned copy of a factor)
cudaError_t launch_pad_rows(const double* F, int64_t S, int K, double* Fp, int ld, cudaStream_t st);

// ---------------------------------------------------------------- generator (twin of synthgen)
cudaError_t launch_gen_kruskal(double* X, int N, const int64_t* s, int K, const double* const* A_dev,
                               int64_t row_lo, int64_t row_hi, cudaStream_t st);
// per-row Σ X_true² and Σ Z² into rowsq_x/z[row_lo..row_hi) (partials: gen_partials_doubles)
cudaError_t launch_gen_noise_rowsq(double* X, const int64_t* s, int N, uint64_t seed,
                                   int64_t row_lo, int64_t row_hi, double* rowsq_x, double* rowsq_z,
                                   double* partials, cudaStream_t st);
size_t gen_partials_doubles(int64_t nrows);
cudaError_t launch_gen_noise_add(double* X, const int64_t* s, int N, uint64_t seed, int64_t row_lo,
                                 int64_t row_hi, const double* scale_dev, double abs_scale,
                                 cudaStream_t st);
cudaError_t launch_gen_scale(const double* rowsq_x, const double* rowsq_z, int64_t s0, double eta,
                             double* scale_dev, cudaStream_t st);

}  // namespace cppp
