"""ORACLE for Tucker-ALS (HOOI) with pairwise perturbation (arXiv 1811.10573) —
TEST INFRASTRUCTURE ONLY.

Plain FP64 numpy written from PAPER.md; only ``tests/`` may import it.  It shares no code with
the CUDA path (``paper_1811_10573_b200``) and never imports it.

Citations: ``P:n`` = line n of PAPER.md; ``S:n`` = line n of SPEC.md (interfaces and examples);
``T<n>`` = Tucker reading n in DESIGN.md.

Conventions
  * Tensors are row-major numpy arrays, modes 0-based.  Factor A[n] is s_n x R_n with
    orthonormal columns.
  * ``X ×_n A^T`` contracts mode n of X with the ROWS of A; the rank index z_n
    takes mode n's position (the mode-n product of P:282 with the matrix A^T).  Every Y here
    therefore keeps the original mode order: x at the kept positions, z elsewhere ("canonical
    layout"; the GPU path's results are compared in this layout).

Plain definitions computed as written: the mode product, TTMc Y^(n), Def. 3.2
operators, the PP approximation.  Algorithms followed step by step:
HOSVD, Alg. 2, Alg. 4 with the readings in DESIGN.md.

Pins: tests/test_oracle_tucker.py (brute-force loops, SPEC S:231-262 examples, exact Tucker
recovery, residual identity, core-norm monotonicity (Lemma 4.7), PP exactness and quadratic
error).  Parity unpinned: none.
"""
from __future__ import annotations

import math
from itertools import combinations
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np


# --------------------------------------------------------------------------------------
# Contractions (Def. 3.2)
# --------------------------------------------------------------------------------------
def mode_product_t(X: np.ndarray, A: np.ndarray, n: int) -> np.ndarray:
    """X ×_n A^T: Y(.., z, ..) = Σ_{x_n} X(.., x_n, ..) A(x_n, z), z at position n."""
    Y = np.tensordot(X, A, axes=([n], [0]))        # z appended last
    return np.moveaxis(Y, -1, n)


def ttmc(X: np.ndarray, A: Sequence[np.ndarray], skip: Optional[int] = None) -> np.ndarray:
    """Y^(n) = X ×_1 A^(1)T ⋯ ×_{n-1} A^(n-1)T ×_{n+1} ⋯ ×_N A^(N)T; skip=None gives
    the core X ×_1 A^(1)T ⋯ ×_N A^(N)T.  Modes contracted in ascending order."""
    Y = np.asarray(X, dtype=np.float64)
    for m in range(Y.ndim):
        if m != skip:
            Y = mode_product_t(Y, A[m], m)
    return Y


def partial_ttmc(X: np.ndarray, A: Sequence[np.ndarray], kept: Sequence[int]) -> np.ndarray:
    """Y^(i_1..i_m) = X ×_{j ∉ kept} A^(j)T (Def. 3.2), canonical layout."""
    Y = np.asarray(X, dtype=np.float64)
    for m in range(Y.ndim):
        if m not in kept:
            Y = mode_product_t(Y, A[m], m)
    return Y


def unfold(Y: np.ndarray, n: int) -> np.ndarray:
    """Y_(n): mode n as rows, the other modes flattened row-major."""
    return np.moveaxis(Y, n, 0).reshape(Y.shape[n], -1)


# --------------------------------------------------------------------------------------
# Factor update: leading left singular vectors from the Gram matrix
# --------------------------------------------------------------------------------------
def leading_left_singvecs(Y: np.ndarray, n: int, R: int) -> np.ndarray:
    """The R leading eigenvectors of W = Y_(n) Y_(n)^T, eigenvalues descending, each
    column's sign fixed so that its largest-magnitude entry (first one on a tie) is positive
    (reading T2)."""
    Yn = unfold(Y, n)
    if R > Yn.shape[0]:
        raise ValueError("rank exceeds the mode dimension")
    W = Yn @ Yn.T
    lam, V = np.linalg.eigh(W)
    order = np.argsort(-lam, kind="stable")[:R]
    U = V[:, order].copy()
    for j in range(R):
        i = int(np.argmax(np.abs(U[:, j])))
        if U[i, j] < 0:
            U[:, j] = -U[:, j]
    return U


def hosvd(X: np.ndarray, ranks: Sequence[int]):
    """Classical HOSVD: A^(n) = leading left singular vectors of X_(n); core
    G = X ×_1 A^(1)T ⋯ ×_N A^(N)T."""
    A = [leading_left_singvecs(X, n, ranks[n]) for n in range(X.ndim)]
    return ttmc(X, A), A


# --------------------------------------------------------------------------------------
# PP operators and update (Alg. 4)
# --------------------------------------------------------------------------------------
def pp_operators(X: np.ndarray, A_p: Sequence[np.ndarray]) -> Dict[Tuple[int, int], np.ndarray]:
    """Y_p^(i,j) for i < j (Def. 3.2 at A_p), canonical layout."""
    return {(i, j): partial_ttmc(X, A_p, [i, j]) for i, j in combinations(range(X.ndim), 2)}


def pp_single(ops, A_p: Sequence[np.ndarray], n: int, N: int) -> np.ndarray:
    """Y_p^(n) = Y_p^(j,n) ×_j A_p^(j)T with j = min{j ≠ n} (draft P:139; reading T3)."""
    j = min(m for m in range(N) if m != n)
    return mode_product_t(ops[(min(j, n), max(j, n))], A_p[j], j)


def pp_update(Yp_n: np.ndarray, ops, dA: Sequence[np.ndarray], n: int) -> np.ndarray:
    """Ỹ^(n) = Y_p^(n) + Σ_{i≠n} Y_p^(i,n) ×_i dA^(i)T, i ascending."""
    out = np.array(Yp_n, dtype=np.float64, copy=True)
    for i in range(len(dA)):
        if i != n:
            out = out + mode_product_t(ops[(min(i, n), max(i, n))], dA[i], i)
    return out


# --------------------------------------------------------------------------------------
# Sweeps: Alg. 2 (regular) and Alg. 4 (PP), with readings T1-T5
# --------------------------------------------------------------------------------------
class TuckerState:
    def __init__(self, X: np.ndarray, ranks: Sequence[int], A0=None):
        self.X = np.asarray(X, dtype=np.float64)
        self.N = self.X.ndim
        self.ranks = list(ranks)
        if A0 is None:
            self.G, self.A = hosvd(self.X, ranks)
        else:
            self.A = [np.array(a, dtype=np.float64, copy=True) for a in A0]
            self.G = ttmc(self.X, self.A)
        self.dA = [np.zeros_like(a) for a in self.A]
        self.A_p = None
        self.ops = None
        self.Yp = None
        self.normX_sq = float(np.dot(self.X.ravel(), self.X.ravel()))
        self.F_norm = math.inf

    def _finish(self, Y_last: np.ndarray):
        """Core from the last mode's Y (T1): G_new = Y^(N) ×_N A^(N)T, F = G_new - G."""
        n = self.N - 1
        G_new = mode_product_t(Y_last, self.A[n], n)
        self.F_norm = float(np.linalg.norm(G_new - self.G))
        self.G = G_new

    def dt_sweep(self):
        """Alg. 2 body, dA = A_new - A_old."""
        Y = None
        for n in range(self.N):
            Y = ttmc(self.X, self.A, skip=n)
            A_new = leading_left_singvecs(Y, n, self.ranks[n])
            self.dA[n] = A_new - self.A[n]
            self.A[n] = A_new
        self._finish(Y)

    def pp_build(self):
        """A_p := A, dA := 0, operators Y_p^(i,j) and Y_p^(n) (Alg. 4)."""
        self.A_p = [a.copy() for a in self.A]
        self.dA = [np.zeros_like(a) for a in self.A]
        self.ops = pp_operators(self.X, self.A_p)
        self.Yp = [pp_single(self.ops, self.A_p, n, self.N) for n in range(self.N)]

    def pp_sweep(self):
        """Alg. 4: Ỹ^(n) from the operators, A^(n) its leading left singular vectors,
        dA^(n) = A^(n) - A_p^(n)."""
        Y = None
        for n in range(self.N):
            Y = pp_update(self.Yp[n], self.ops, self.dA, n)
            self.A[n] = leading_left_singvecs(Y, n, self.ranks[n])
            self.dA[n] = self.A[n] - self.A_p[n]
        self._finish(Y)

    def rel_dA(self) -> List[float]:
        return [float(np.linalg.norm(d) / np.linalg.norm(a)) for d, a in zip(self.dA, self.A)]

    def residual(self) -> float:
        """||X - [[G; A]]|| / ||X|| = sqrt(max(0, ||X||² - ||G||²)) / ||X|| (orthonormal factors,
        S:258)."""
        g2 = float(np.dot(self.G.ravel(), self.G.ravel()))
        return math.sqrt(max(0.0, self.normX_sq - g2)) / math.sqrt(self.normX_sq)


def pp_tucker_als(X, ranks, eps: float, eps_pp: float, max_sweeps: int, A0=None,
                  phase_override: Optional[Sequence[str]] = None):
    """PP-Tucker-ALS, Alg. 4, HOSVD initialization unless A0 is given, with the CP
    phase machine readings (L7-L11 applied to Tucker: T4): the first sweep is regular; after
    a regular sweep with max_i ||dA^(i)||_F/||A^(i)||_F < ε_pp the next sweep builds the
    operators and runs a PP sweep; PP sweeps continue while the test holds, else exactly one
    regular sweep; stop when ||F||_F <= ε (T5) or after max_sweeps.  ε_pp = 0 is plain
    Tucker-ALS (Alg. 2).  Returns (state, trace)."""
    st = TuckerState(X, ranks, A0)
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
        next_phase = ("pp-build" if small else "dt") if phase == "dt" else ("pp-approx" if small else "dt")
        trace.append(dict(sweep=sw + 1, phase=phase, core_change=st.F_norm,
                          core_norm=float(np.linalg.norm(st.G)), residual=st.residual(),
                          max_rel_dA=max(rel)))
        if st.F_norm <= eps:
            break
    return st, trace
