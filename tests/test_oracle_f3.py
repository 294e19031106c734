"""Pins for the error-analysis oracle: Alg. 5's pushed updates and the
column-wise PP error monitor with its certificate (oracle/cp_oracle.py).  CPU only."""
import math

import numpy as np
import pytest

import oracle.cp_oracle as O


def rng(seed):
    return np.random.default_rng(seed)


def rand_state(dims, K, seed, t):
    """Random X, A_p and A = A_p + dA with ||da_k|| = t ||a_p,k|| per column."""
    r = rng(seed)
    X = r.standard_normal(dims)
    Ap = [r.standard_normal((s, K)) for s in dims]
    dA = []
    for a in Ap:
        d = r.standard_normal(a.shape)
        d *= t * np.linalg.norm(a, axis=0) / np.linalg.norm(d, axis=0)
        dA.append(d)
    return X, Ap, [a + d for a, d in zip(Ap, dA)]


# ---------------------------------------------------------------- Alg. 5
@pytest.mark.parametrize("dims,K,seed", [((6, 5, 7), 3, 1), ((4, 5, 3, 4), 2, 2)])
def test_pushed_updates_equal_alg1(dims, K, seed):
    """Alg. 5 is algebraically equivalent to Alg. 1: same factors and fitness trace
    (up to rounding) as plain CP-ALS, which forms every M^(n) afresh."""
    r = rng(seed)
    X = r.uniform(size=dims)
    A0 = [r.uniform(size=(s, K)) for s in dims]
    A1, tr1 = O.cp_als(X, A0, 4)
    A5, tr5 = O.cp_als_pushed(X, A0, 4)
    for a, b in zip(A1, A5):
        assert np.linalg.norm(a - b) / np.linalg.norm(a) < 1e-9
    assert max(abs(x - y) for x, y in zip(tr1, tr5)) < 1e-10


# ---------------------------------------------------------------- Cor. 4.2
def test_cor42_bound_N3():
    """N = 3 (0-based modes): the PP update H~^(0,2) (operator M_p^(0,2) at A_p) and the exact
    H^(0,2) (M^(0,2) at A) differ per column by at most ||T̂||_2 ||a_k^(1)|| ε_k^(1), and by at
    most κ(T̂) ε_k^(1) relative to ||h_k||, with T̂ = X ×_2 δa_k^(2)."""
    X, Ap, A = rand_state((9, 6, 5), 3, 4, 0.05)
    dN = 0.1 * rng(5).standard_normal((5, 3))                 # δA^(2) of an ALS step
    Mp02 = O.pp_operator(X, Ap, 0, 2)
    M02 = O.pp_operator(X, A, 0, 2)
    Ht = np.einsum("xyk,yk->xk", Mp02, dN)
    H = np.einsum("xyk,yk->xk", M02, dN)
    for k in range(3):
        T = np.einsum("abc,c->ab", X, dN[:, k])              # s0 x s1
        eps1 = np.linalg.norm(A[1][:, k] - Ap[1][:, k]) / np.linalg.norm(A[1][:, k])
        e = np.linalg.norm(Ht[:, k] - H[:, k])
        sv = np.linalg.svd(T, compute_uv=False)
        assert e <= sv[0] * np.linalg.norm(A[1][:, k]) * eps1 * (1 + 1e-12)
        assert e / np.linalg.norm(H[:, k]) <= sv[0] / sv[-1] * eps1 * (1 + 1e-12)
        # the error is exactly T̂ da_k^(1) (P:803 with S = {1})
        assert np.linalg.norm((Ht[:, k] - H[:, k]) + T @ (A[1][:, k] - Ap[1][:, k])) < 1e-12 * max(e, 1e-300)


# ---------------------------------------------------------------- the error monitor
@pytest.mark.parametrize("dims,K", [((7, 6, 5), 3), ((5, 4, 6, 3), 2), ((3, 4, 3, 2, 3), 2)])
@pytest.mark.parametrize("t", [0.3, 1e-2])
def test_monitor_certificate_holds(dims, K, t):
    """err <= bound for every (n, k): the certificate is a proven upper bound."""
    X, Ap, A = rand_state(dims, K, 6, t)
    err, eps, bound = O.pp_error_monitor(X, A, Ap)
    assert np.all(err <= bound * (1 + 1e-10))
    assert np.all(err > 0)


def test_monitor_eps_closed_form():
    """dA = t A_p column-wise scaled: ε = t / (1 + t) exactly."""
    r = rng(7)
    dims, K, t = (4, 5, 3), 3, 0.07
    X = r.standard_normal(dims)
    Ap = [r.standard_normal((s, K)) for s in dims]
    A = [(1 + t) * a for a in Ap]
    _, eps, _ = O.pp_error_monitor(X, A, Ap)
    assert np.allclose(eps, t / (1 + t), rtol=1e-13, atol=0)


def test_monitor_rank1_tight():
    """Rank-1 X = u∘v∘w, K = 1, da^(0) ∥ u, da^(1) ∥ v, no change in mode 2: mode 2's dropped
    term is (u·da0)(v·da1) w with norm ||X||_F d0 d1 — the certificate is attained."""
    r = rng(8)
    u, v, w = r.standard_normal(5), r.standard_normal(4), r.standard_normal(6)
    X = np.einsum("a,b,c->abc", u, v, w)
    Ap = [r.standard_normal((s, 1)) for s in (5, 4, 6)]
    d0, d1 = 0.02, 0.03
    A = [Ap[0] + d0 * u[:, None] / np.linalg.norm(u), Ap[1] + d1 * v[:, None] / np.linalg.norm(v),
         Ap[2].copy()]
    err, _, bound = O.pp_error_monitor(X, A, Ap)
    assert abs(err[2, 0] - bound[2, 0]) <= 1e-9 * bound[2, 0]
    m2 = np.linalg.norm(O.mttkrp(X, A, 2))
    assert abs(bound[2, 0] - np.linalg.norm(X) * d0 * d1 / m2) <= 1e-12 * bound[2, 0]


def test_monitor_quadratic_and_zero():
    """err(t/10) ≈ err(t)/100 (second order) and no perturbation gives err at rounding
    level and bound = 0."""
    e = []
    for t in (1e-2, 1e-3):
        X, Ap, A = rand_state((6, 5, 4, 5), 2, 9, t)
        err, _, bound = O.pp_error_monitor(X, A, Ap)
        e.append(err)
    ratio = e[0] / e[1]
    assert np.all(np.abs(ratio / 100 - 1) < 0.05)
    X, Ap, _ = rand_state((6, 5, 4), 2, 10, 0.0)
    err, eps, bound = O.pp_error_monitor(X, Ap, Ap)
    assert np.all(err < 1e-13) and np.all(eps == 0) and np.all(bound == 0)
