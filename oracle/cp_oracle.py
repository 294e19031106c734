"""ORACLE for CP-ALS with pairwise perturbation (arXiv 1811.10573) — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct FP64 CPU implementation written from PAPER.md.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  It shares no code with the CUDA path
(``paper_1811_10573_b200``) and never imports it.

Citations: ``P:n`` = line n of PAPER.md (the LaTeX source); ``L<n>`` = reading n of the
ambiguity ledger in SURVEY.md §8(c), repeated in DESIGN.md.

Conventions
  * Tensors are numpy arrays, row-major (last mode fastest).  Modes are 0-based here;
    the paper's mode m is index m-1.
  * Factor A[n] is s_n x K.  Rank index k is always the LAST index of an intermediate
    (Def. 3.1).

What is the plain definition and what follows an algorithm
  * MTTKRP and the partially contracted intermediates / PP operators (Def. 3.1,
    P:524-535) have plain definitions; they are computed as written: generalized
    unfolding times the explicit Khatri-Rao product.
  * The PP tree (Def. pptree) is built literally from its definition.
  * The PP update, the normal-equation solve, Alg. 1
    and Alg. 3 follow the paper step by step in its order.
  * Fitness (not defined by the paper, L17) is the expansion of S:177.

Error analysis: Alg. 5's pushed updates (cp_als_pushed) and the
column-wise PP error monitor with its certificate (pp_error_monitor, Thm 4.1).

Pins: every function here is pinned by tests in tests/test_oracle_*.py against closed
forms, brute-force index loops, invariants and printed examples — see DESIGN.md
"Oracle pins".  Parity unpinned: none of the functions below (the whole-trajectory
values on C2-C5 have no printed reference; they are pinned only through the pinned
building blocks and exact recovery).
"""
from __future__ import annotations

import math
import time
from itertools import combinations
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

PIVOT_TAU = 1e-12   # L13 / S:201: Cholesky accepted iff every pivot > tau * max diag(Gamma)
PINV_TAU = 1e-12    # L13: eigenvalues <= tau * lambda_max treated as zero in the pseudo-inverse


# --------------------------------------------------------------------------------------
# §2.1 notation
# --------------------------------------------------------------------------------------
def khatri_rao(mats: Sequence[np.ndarray]) -> np.ndarray:
    """A ⊙ B = [a_1⊗b_1, ..., a_K⊗b_K]; for a list, left to right, so the
    LAST factor's row index varies fastest (Kronecker order, pairs with row-major unfolding)."""
    K = mats[0].shape[1]
    out = np.asarray(mats[0], dtype=np.float64)
    for B in mats[1:]:
        out = (out[:, None, :] * np.asarray(B)[None, :, :]).reshape(-1, K)
    return out


def unfold_multi(X: np.ndarray, kept: Sequence[int]) -> np.ndarray:
    """Generalized unfolding X_(i1..im): kept modes first (in the given order), the
    remaining modes flattened into the last index in increasing mode order, last fastest."""
    rest = [m for m in range(X.ndim) if m not in kept]
    Y = np.transpose(X, list(kept) + rest)
    return Y.reshape([X.shape[m] for m in kept] + [-1])


def unfold(X: np.ndarray, n: int) -> np.ndarray:
    """Mode-n matricization X_(n), columns in row-major order of the other modes."""
    return unfold_multi(X, [n])


# --------------------------------------------------------------------------------------
# MTTKRP and Definition 3.1
# --------------------------------------------------------------------------------------
def partial_mttkrp(X: np.ndarray, A: Sequence[np.ndarray], kept: Sequence[int]) -> np.ndarray:
    """M^(i1..im) = X_(i1..im) ⊙_{j ∉ kept} A^(j)   (Def. 3.1).

    Elementwise M(x_kept, k) = Σ_{other x} X(x) Π_{r ∉ kept} A^(r)(x_r, k).  ``kept`` is
    given in increasing mode order; the result has shape (s_kept..., K)."""
    kept = list(kept)
    assert kept == sorted(kept)
    rest = [m for m in range(X.ndim) if m not in kept]
    K = A[0].shape[1]
    # empty product over no contracted modes = 1 for every k
    P = khatri_rao([A[m] for m in rest]) if rest else np.ones((1, K))   # (Π s_rest) x K
    Xu = unfold_multi(X, kept)                             # (s_kept...) x (Π s_rest)
    M = Xu.reshape(-1, Xu.shape[-1]) @ P
    return M.reshape([X.shape[m] for m in kept] + [K])


def mttkrp(X: np.ndarray, A: Sequence[np.ndarray], n: int) -> np.ndarray:
    """M^(n) = X_(n) (A^(1)⊙…⊙A^(n-1)⊙A^(n+1)⊙…⊙A^(N))."""
    P = khatri_rao([A[m] for m in range(X.ndim) if m != n])
    return unfold(X, n) @ P


def pp_operator(X: np.ndarray, A: Sequence[np.ndarray], i: int, j: int) -> np.ndarray:
    """M_p^(i,j) for i<j: Def. 3.1 with kept = (i, j), shape (s_i, s_j, K)."""
    assert i < j
    return partial_mttkrp(X, A, [i, j])


def pp_operators(X: np.ndarray, A_p: Sequence[np.ndarray]) -> Dict[Tuple[int, int], np.ndarray]:
    """All N(N-1)/2 unordered-pair operators (L5: stored once, (n,i) read as a transpose)."""
    N = X.ndim
    return {(i, j): pp_operator(X, A_p, i, j) for i, j in combinations(range(N), 2)}


def op_pair(ops: Dict[Tuple[int, int], np.ndarray], i: int, n: int) -> np.ndarray:
    """M_p^(i,n)(x, y, k) for any i != n, using M_p^(i,n) = M_p^(n,i)^T."""
    if i < n:
        return ops[(i, n)]
    return np.transpose(ops[(n, i)], (1, 0, 2))


def pp_single(ops, A_p: Sequence[np.ndarray], n: int, N: int, j: Optional[int] = None) -> np.ndarray:
    """M_p^(n) = M_p^(j,n) ×_j A_p^(j) for j = min{j != n} (reading L6)."""
    if j is None:
        j = min(m for m in range(N) if m != n)
    Op = op_pair(ops, j, n)                                 # (s_j, s_n, K)
    return np.einsum("xyk,xk->yk", Op, A_p[j])


# --------------------------------------------------------------------------------------
# Definition pptree and its cost
# --------------------------------------------------------------------------------------
def pp_tree(N: int):
    """The PP construction tree of Def. pptree, 1-based modes as in the paper.

    Returns {level l: [(kept tuple, mu frozenset, parent kept tuple)]} for l = 1..N-2.
    Level l holds T_(i,j,l+3,...,N) for i<j in [1,l+2]; mu is the contracted set
    N_N \\ kept; the parent is T_(s,t,v,l+3,..,N) with
    {s,t,v} = {i,j} ∪ {max_{w ∈ {l,l+1,l+2} \\ {i,j}} w}; level-1 parents are the root."""
    allm = frozenset(range(1, N + 1))
    levels = {}
    for l in range(1, N - 1):
        nodes = []
        for i, j in combinations(range(1, l + 3), 2):
            kept = (i, j) + tuple(range(l + 3, N + 1))
            mu = allm - set(kept)
            if l == 1:
                parent = tuple(range(1, N + 1))
            else:
                w = max(set(range(l, l + 3)) - {i, j})
                parent = tuple(sorted({i, j, w})) + tuple(range(l + 3, N + 1))
            nodes.append((kept, mu, parent))
        levels[l] = nodes
    return levels


def pp_build_flops_formula(N: int, s: int, R: int) -> int:
    """2R Σ_{l=2}^{N-1} C(l+1,2) s^{N-l+2}."""
    return 2 * R * sum(math.comb(l + 1, 2) * s ** (N - l + 2) for l in range(2, N))


def pp_tree_flops(N: int, s: int, R: int) -> int:
    """Flops of Tree_Map_PP on the tree: a level-1 node is a TTM X ×_i A^(i)
    (2 s^N R flops); a deeper node contracts one mode of its parent rank-diagonally
    (2 |parent| flops)."""
    total = 0
    for l, nodes in pp_tree(N).items():
        for kept, mu, parent in nodes:
            total += 2 * R * s ** len(parent)
    return total


# --------------------------------------------------------------------------------------
# PP update (Alg. 3 line P:586-587)
# --------------------------------------------------------------------------------------
def pp_update(Mp_n: np.ndarray, ops, dA: Sequence[np.ndarray], n: int) -> np.ndarray:
    """M~^(n)(y,k) = M_p^(n)(y,k) + Σ_{i≠n} Σ_x M_p^(i,n)(x,y,k) dA^(i)(x,k).
    Sum over i ascending (L: O8)."""
    N = len(dA)
    out = np.array(Mp_n, dtype=np.float64, copy=True)
    for i in range(N):
        if i == n:
            continue
        out = out + np.einsum("xyk,xk->yk", op_pair(ops, i, n), dA[i])
    return out


def second_order_term(X, A_p, dA, n):
    """Σ_{i<j; i,j≠n} Σ_{x,z} M_p^(i,j,n)(x,z,y,k) dA^(i)(x,k) dA^(j)(z,k) — the first term
    dropped by the PP truncation.  Used by tests only."""
    N = X.ndim
    out = 0.0
    for i, j in combinations([m for m in range(N) if m != n], 2):
        kept = sorted([i, j, n])
        T = partial_mttkrp(X, A_p, kept)
        # move (i, j, n) into that order
        perm = [kept.index(i), kept.index(j), kept.index(n), 3]
        T = np.transpose(T, perm)
        out = out + np.einsum("xzyk,xk,zk->yk", T, dA[i], dA[j])
    return out


# --------------------------------------------------------------------------------------
# Normal equations (Alg. 1 lines P:393-399)
# --------------------------------------------------------------------------------------
def gram(A: np.ndarray) -> np.ndarray:
    """S = A^T A."""
    return A.T @ A


def gamma(S: Sequence[np.ndarray], n: int) -> np.ndarray:
    """Γ^(n) = S^(1) ∗ … ∗ S^(n-1) ∗ S^(n+1) ∗ … ∗ S^(N), Hadamard in ascending m."""
    out = None
    for m, Sm in enumerate(S):
        if m == n:
            continue
        out = np.array(Sm, copy=True) if out is None else out * Sm
    return out


def cholesky_pivots(G: np.ndarray, tau: float = PIVOT_TAU):
    """Textbook column Cholesky Γ = L L^T.  Returns (L, ok) where ok is False as soon as a
    pivot d_j = Γ_jj - Σ_{p<j} L_jp^2 is <= tau * max diag(Γ) (L13, default τ = PIVOT_TAU)."""
    K = G.shape[0]
    L = np.zeros_like(G)
    thresh = tau * max(float(np.max(np.diag(G))), 0.0)
    for j in range(K):
        d = G[j, j] - float(np.dot(L[j, :j], L[j, :j]))
        if not d > thresh:
            return L, False
        L[j, j] = math.sqrt(d)
        L[j + 1:, j] = (G[j + 1:, j] - L[j + 1:, :j] @ L[j, :j]) / L[j, j]
    return L, True


def solve_normal(M: np.ndarray, G: np.ndarray, tau: Optional[float] = None) -> np.ndarray:
    """A_new = M Γ^†.  Cholesky path when Γ is numerically PD (L13); otherwise the
    eigen pseudo-inverse with cutoff τ * λ_max.  Γ = 0 gives 0.
    τ defaults to PIVOT_TAU for the pivot rule and PINV_TAU for the cutoff (both 1e-12); a given
    τ is used for both (the library's cppp_opts.pinv_rel_tol)."""
    L, ok = cholesky_pivots(G, PIVOT_TAU if tau is None else tau)
    if ok:
        # Γ a^T = m^T per row:  L z = m^T (forward), L^T a^T = z (back)
        Z = np.zeros_like(M.T)
        Mt = M.T
        K = G.shape[0]
        for j in range(K):
            Z[j] = (Mt[j] - L[j, :j] @ Z[:j]) / L[j, j]
        At = np.zeros_like(Z)
        for j in range(K - 1, -1, -1):
            At[j] = (Z[j] - L[j + 1:, j] @ At[j + 1:]) / L[j, j]
        return At.T.copy()
    lam, V = np.linalg.eigh(G)
    lmax = float(np.max(lam)) if lam.size else 0.0
    cut = PINV_TAU if tau is None else tau
    inv = np.where(lam > cut * lmax, 1.0 / np.where(lam > 0, lam, 1.0), 0.0) if lmax > 0 else np.zeros_like(lam)
    Gp = (V * inv) @ V.T
    return M @ Gp


def gradient(A_old: np.ndarray, A_new: np.ndarray, G: np.ndarray) -> np.ndarray:
    """G^(n) = (A^(n) - A_new^(n)) Γ^(n)."""
    return (A_old - A_new) @ G


# --------------------------------------------------------------------------------------
# Fitness (L17)
# --------------------------------------------------------------------------------------
def residual_sq_expansion(normX_sq: float, M_last: np.ndarray, A_last: np.ndarray,
                          Gamma_last: np.ndarray, S_last: np.ndarray) -> float:
    """‖X - [[A]]‖² = ‖X‖² - 2 Σ_k ⟨M^(N)_k, A^(N)_k⟩ + 1^T (Γ^(N) ∗ S^(N)) 1."""
    inner = math.fsum((M_last * A_last).ravel().tolist())
    model = math.fsum((Gamma_last * S_last).ravel().tolist())
    return normX_sq - 2.0 * inner + model


def fitness_from(normX_sq, M_last, A_last, Gamma_last, S_last) -> float:
    """fitness = 1 - sqrt(max(0, r²)) / ‖X‖  (L17; radicand clamped at 0)."""
    r2 = residual_sq_expansion(normX_sq, M_last, A_last, Gamma_last, S_last)
    return 1.0 - math.sqrt(max(0.0, r2)) / math.sqrt(normX_sq)


def kruskal_full(A: Sequence[np.ndarray]) -> np.ndarray:
    """[[A^(1),…,A^(N)]] = Σ_r a_r^(1) ∘ … ∘ a_r^(N) — tests only (tiny sizes)."""
    N = len(A)
    P = khatri_rao(list(A[1:]))
    return (A[0] @ P.T).reshape([a.shape[0] for a in A])


# --------------------------------------------------------------------------------------
# Sweeps: Alg. 1 (regular) and Alg. 3 (PP)
# --------------------------------------------------------------------------------------
class State:
    """CP-ALS(-PP) state: factors, Grams, perturbations, PP snapshot and operators."""

    def __init__(self, X: np.ndarray, A0: Sequence[np.ndarray], tau: Optional[float] = None):
        self.tau = tau   # L13's τ (None: the defaults)
        self.X = np.asarray(X, dtype=np.float64)
        self.N = self.X.ndim
        self.A = [np.array(a, dtype=np.float64, copy=True) for a in A0]
        self.S = [gram(a) for a in self.A]
        self.dA = [None] * self.N
        self.A_p = None
        self.ops = None
        self.Mp = None
        self.normX_sq = float(np.dot(self.X.ravel(), self.X.ravel()))
        self.G_norms = [math.inf] * self.N
        self.M_last = None
        self.Gamma_last = None

    def _update_mode(self, n: int, M: np.ndarray, dA_ref: np.ndarray):
        Gm = gamma(self.S, n)
        A_new = solve_normal(M, Gm, self.tau)
        Gr = gradient(self.A[n], A_new, Gm)
        self.G_norms[n] = float(np.linalg.norm(Gr))
        self.A[n] = A_new
        self.S[n] = gram(A_new)
        self.dA[n] = A_new - dA_ref
        if n == self.N - 1:
            self.M_last, self.Gamma_last = M, Gm

    def dt_sweep(self):
        """Regular ALS sweep (Alg. 1) with dA = A_new - A_old."""
        for n in range(self.N):
            M = mttkrp(self.X, self.A, n)          # exact MTTKRP with current factors
            self._update_mode(n, M, self.A[n])

    def pp_build(self):
        """A_p := A, dA := 0, operators M_p^(i,j) and M_p^(n) (Alg. 3)."""
        self.A_p = [a.copy() for a in self.A]
        self.dA = [np.zeros_like(a) for a in self.A]
        self.ops = pp_operators(self.X, self.A_p)
        self.Mp = [pp_single(self.ops, self.A_p, n, self.N) for n in range(self.N)]

    def pp_sweep(self):
        """PP sweep (Alg. 3): M~ from the operators, dA = A_new - A_p (L8)."""
        for n in range(self.N):
            M = pp_update(self.Mp[n], self.ops, self.dA, n)
            self._update_mode(n, M, self.A_p[n])

    def rel_dA(self) -> List[float]:
        """‖dA^(i)‖_F / ‖A^(i)‖_F with the current A (L7)."""
        return [float(np.linalg.norm(d) / np.linalg.norm(a)) for d, a in zip(self.dA, self.A)]

    def residual_sq(self) -> float:
        """The unclamped radicand r² of the S:177 expansion with the last computed M^(N) (L17,
        L27): exact ‖X − [[A]]‖² after a regular sweep, O(ε²)-approximate after a PP sweep."""
        return residual_sq_expansion(self.normX_sq, self.M_last, self.A[-1], self.Gamma_last, self.S[-1])

    def fitness(self) -> float:
        return fitness_from(self.normX_sq, self.M_last, self.A[-1], self.Gamma_last, self.S[-1])


def cp_als(X, A0, sweeps: int):
    """Plain CP-ALS (Alg. 1) for a fixed number of sweeps; returns (factors, fitness trace)."""
    st = State(X, A0)
    trace = []
    for _ in range(sweeps):
        st.dt_sweep()
        trace.append(st.fitness())
    return st.A, trace


def pp_cp_als(X, A0, eps: float, eps_pp: float, max_sweeps: int,
              phase_override: Optional[Sequence[str]] = None, deadline: Optional[float] = None,
              tau: Optional[float] = None):
    """PP-CP-ALS, Alg. 3 with readings L7-L12:
      * the first sweep is regular (L9);
      * after each complete regular sweep, if max_i ‖dA^(i)‖/‖A^(i)‖ < ε_pp the next sweep
        builds the operators and runs a PP sweep (tagged 'pp-build');
      * after each PP sweep, if the test still holds (dA against A_p) the next sweep is a PP
        sweep ('pp-approx'), otherwise exactly one regular sweep follows;
      * stop when Σ‖G^(i)‖_F <= ε or after max_sweeps sweeps (L11).
    ``phase_override`` (L12) forces the phase of each sweep (used to replay a schedule).
    ``deadline`` (a time.perf_counter() value; bench.py's bounded CPU sample only) stops after
    the sweep during which it passed — control flow only, the arithmetic is unchanged.
    ``tau`` is L13's τ (None: the defaults).
    Returns (factors, trace) with one dict per sweep."""
    st = State(X, A0, tau)
    trace = []
    next_phase = "dt"
    for sw in range(max_sweeps):
        phase = phase_override[sw] if phase_override is not None else next_phase
        if phase == "dt":
            st.dt_sweep()
        elif phase == "pp-build":
            st.pp_build()
            st.pp_sweep()
        elif phase == "pp-approx":
            st.pp_sweep()
        else:
            raise ValueError(phase)
        rel = st.rel_dA()
        small = max(rel) < eps_pp
        if phase == "dt":
            next_phase = "pp-build" if small else "dt"
        else:
            next_phase = "pp-approx" if small else "dt"
        gsum = float(sum(st.G_norms))
        trace.append(dict(sweep=sw + 1, phase=phase, fitness=st.fitness(), residual_sq=st.residual_sq(),
                          grad_norm_sum=gsum, max_rel_dA=max(rel), margin=abs(max(rel) - eps_pp),
                          normX_sq=st.normX_sq))
        if gsum <= eps:
            break
        if deadline is not None and time.perf_counter() >= deadline:
            break
    return st.A, trace


# --------------------------------------------------------------------------------------
# Error analysis (§4.1)
# --------------------------------------------------------------------------------------
def cp_als_pushed(X, A0, sweeps: int):
    """Alg. 5, the reinterpreted ALS: every M^(n) formed once from the initial
    factors; then, per mode n in order, Γ^(n), A_new = M^(n) Γ^(n)†,
    δA^(n) = A_new - A^(n), A^(n) <- A_new, S^(n) <- A^T A, and the update
    is pushed to every other right-hand side:
        M^(m)(x,k) += Σ_y M^(m,n)(x,y,k) δA^(n)(y,k)   (= H^(m,n))
    with M^(m,n) (Def. 3.1) at the current factors — the oracle-like use P:779 names.  Runs a
    fixed number of sweeps (the while test of P:756 left to the caller); returns (factors,
    fitness trace) like cp_als."""
    X = np.asarray(X, dtype=np.float64)
    N = X.ndim
    A = [np.array(a, dtype=np.float64, copy=True) for a in A0]
    S = [gram(a) for a in A]
    M = [mttkrp(X, A, n) for n in range(N)]
    normX_sq = float(np.dot(X.ravel(), X.ravel()))
    trace = []
    for _ in range(sweeps):
        for n in range(N):
            Gm = gamma(S, n)
            A_new = solve_normal(M[n], Gm)
            dA = A_new - A[n]
            A[n] = A_new
            S[n] = gram(A_new)
            if n == N - 1:
                M_last, Gamma_last = M[n], Gm
            for m in range(N):
                if m == n:
                    continue
                lo, hi = min(m, n), max(m, n)
                Mmn = partial_mttkrp(X, A, [lo, hi])          # M^(lo,hi), current factors
                Mmn = Mmn if m < n else np.transpose(Mmn, (1, 0, 2))   # index (x_m, y_n, k)
                M[m] = M[m] + np.einsum("xyk,yk->xk", Mmn, dA)
        trace.append(fitness_from(normX_sq, M_last, A[N - 1], Gamma_last, S[N - 1]))
    return A, trace


def pp_error_monitor(X, A, A_p):
    """Column-wise error of the PP approximation at factors A with operators built at A_p.

    For every mode n and column k, with dA = A - A_p:
      err[n][k]   = ||m~_k - m_k|| / ||m_k||: M~ the first two terms of the P:548 expansion
                    (P:553), M the exact MTTKRP at A;
      eps[n][k]   = ||da_k^(n)|| / ||a_k^(n)|| (the ε_k^(n) of Thm 4.1);
      bound[n][k] = ||X||_F Σ_{S ⊆ {i≠n}, |S| >= 2} Π_{i∈S} ||da_k^(i)|| Π_{j∉S} ||a_p,k^(j)||
                    / ||m_k||: every dropped term of P:548 contracts X with the vectors da
                    (i ∈ S) and a_p (j ∉ S), and ||X ×_S v|| <= ||X||_F Π ||v|| — the
                    expansion of the proof of Thm 4.1 applied to M.
    A ratio with zero denominator is 0 for a zero numerator, else inf.  Returns three N x K
    arrays."""
    X = np.asarray(X, dtype=np.float64)
    N = X.ndim
    K = A[0].shape[1]
    ops = pp_operators(X, A_p)
    dA = [a - ap for a, ap in zip(A, A_p)]
    normX = math.sqrt(float(np.dot(X.ravel(), X.ravel())))

    def ratio(num, den):
        if num == 0.0:
            return 0.0
        return num / den if den > 0.0 else math.inf

    err = np.zeros((N, K))
    eps = np.zeros((N, K))
    bound = np.zeros((N, K))
    for n in range(N):
        M = mttkrp(X, A, n)
        Mt = pp_update(pp_single(ops, A_p, n, N), ops, dA, n)
        others = [i for i in range(N) if i != n]
        for k in range(K):
            mk = float(np.linalg.norm(M[:, k]))
            err[n, k] = ratio(float(np.linalg.norm(Mt[:, k] - M[:, k])), mk)
            eps[n, k] = ratio(float(np.linalg.norm(dA[n][:, k])), float(np.linalg.norm(A[n][:, k])))
            d = {i: float(np.linalg.norm(dA[i][:, k])) for i in others}
            p = {i: float(np.linalg.norm(A_p[i][:, k])) for i in others}
            tot = 0.0
            for size in range(2, len(others) + 1):
                for Sset in combinations(others, size):
                    tot += math.prod(d[i] if i in Sset else p[i] for i in others)
            bound[n, k] = ratio(normX * tot, mk)
    return err, eps, bound
