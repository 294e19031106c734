"""Pins for the Tucker / PP-Tucker oracle (oracle/tucker_oracle.py), CPU only:
brute-force index loops, SPEC's worked examples, exact recovery of Tucker tensors,
the residual identity, core-norm monotonicity (Lemma 4.7) and the PP expansion
(P:630-646)."""
import itertools
import math

import numpy as np
import pytest

import oracle.tucker_oracle as T


def rng(seed):
    return np.random.default_rng(seed)


def orth(r, s, R):
    q, _ = np.linalg.qr(r.standard_normal((s, R)))
    return q


def tucker_tensor(dims, ranks, seed, noise=0.0):
    r = rng(seed)
    G = r.standard_normal(ranks)
    A = [orth(r, s, R) for s, R in zip(dims, ranks)]
    X = G
    for m, a in enumerate(A):
        X = np.moveaxis(np.tensordot(X, a, axes=([m], [1])), -1, m)
    if noise:
        Z = r.standard_normal(dims)
        X = X + noise * np.linalg.norm(X) / np.linalg.norm(Z) * Z
    return X, G, A


# ---------------------------------------------------------------- contractions
def test_mode_product_brute_force():
    r = rng(1)
    X = r.standard_normal((3, 4, 5))
    A = r.standard_normal((4, 2))
    Y = T.mode_product_t(X, A, 1)
    assert Y.shape == (3, 2, 5)
    for a, z, c in itertools.product(range(3), range(2), range(5)):
        assert abs(Y[a, z, c] - sum(X[a, b, c] * A[b, z] for b in range(4))) < 1e-13


def test_ttmc_identity_and_matrix_case():
    """identity factors give X; N = 2, skip 0: X · A^(1)."""
    r = rng(2)
    X = r.standard_normal((3, 4, 2))
    I = [np.eye(s) for s in X.shape]
    for n in range(3):
        assert np.array_equal(T.ttmc(X, I, n), X)
    M = r.standard_normal((5, 6))
    B = r.standard_normal((6, 3))
    assert np.allclose(T.ttmc(M, [None, B], 0), M @ B, rtol=0, atol=1e-13)


def test_ttmc_and_partial_brute_force():
    r = rng(3)
    dims, ranks = (3, 4, 2, 3), (2, 3, 2, 2)
    X = r.standard_normal(dims)
    A = [r.standard_normal((s, R)) for s, R in zip(dims, ranks)]
    Y = T.ttmc(X, A, 2)          # keep mode 2
    for z0, z1, x2, z3 in itertools.product(range(2), range(3), range(2), range(2)):
        v = sum(X[a, b, x2, d] * A[0][a, z0] * A[1][b, z1] * A[3][d, z3]
                for a in range(3) for b in range(4) for d in range(3))
        assert abs(Y[z0, z1, x2, z3] - v) < 1e-12
    P = T.partial_ttmc(X, A, [1, 3])
    for z0, x1, z2, x3 in itertools.product(range(2), range(4), range(2), range(3)):
        v = sum(X[a, x1, c, x3] * A[0][a, z0] * A[2][c, z2] for a in range(3) for c in range(2))
        assert abs(P[z0, x1, z2, x3] - v) < 1e-12


# ---------------------------------------------------------------- factor update / HOSVD
def test_leading_singvecs_examples():
    """Y_(n) = diag(3, 1), R = 1 -> e1; against a dense SVD (projectors) on random Y;
    sign rule: largest-magnitude entry positive."""
    Y = np.diag([3.0, 1.0])
    U = T.leading_left_singvecs(Y, 0, 1)
    assert np.allclose(U[:, 0], [1.0, 0.0])
    Y = -np.diag([3.0, 1.0])
    assert np.allclose(T.leading_left_singvecs(Y, 0, 1)[:, 0], [1.0, 0.0])
    r = rng(4)
    Y = r.standard_normal((6, 4, 5))
    for n in range(3):
        U = T.leading_left_singvecs(Y, n, 3)
        Us = np.linalg.svd(T.unfold(Y, n), full_matrices=False)[0][:, :3]
        assert np.allclose(U @ U.T, Us @ Us.T, atol=1e-12)
        assert np.allclose(U.T @ U, np.eye(3), atol=1e-13)
        for j in range(3):
            i = int(np.argmax(np.abs(U[:, j])))
            assert U[i, j] > 0
    with pytest.raises(ValueError):
        T.leading_left_singvecs(Y, 2, 6)


def test_hosvd_examples():
    """superdiagonal 2x2x2 (3, 1), ranks 1 -> e1 factors, core 3; full ranks ->
    exact reconstruction."""
    X = np.zeros((2, 2, 2))
    X[0, 0, 0], X[1, 1, 1] = 3.0, 1.0
    G, A = T.hosvd(X, (1, 1, 1))
    for a in A:
        assert np.allclose(a[:, 0], [1.0, 0.0])
    assert abs(G.ravel()[0] - 3.0) < 1e-14
    r = rng(5)
    X = r.standard_normal((3, 4, 2))
    G, A = T.hosvd(X, X.shape)
    Xr = G
    for m, a in enumerate(A):
        Xr = np.moveaxis(np.tensordot(Xr, a, axes=([m], [1])), -1, m)
    assert np.linalg.norm(Xr - X) <= 1e-12 * np.linalg.norm(X)


# ---------------------------------------------------------------- Alg. 2
def test_exact_tucker_recovered_and_residual_identity():
    """An exact multilinear-rank tensor is recovered by HOSVD + HOOI (residual < 1e-10,
    S:253); ||X - model||² = ||X||² - ||G||²."""
    X, _, _ = tucker_tensor((8, 7, 6), (3, 2, 2), 6)
    st, tr = T.pp_tucker_als(X, (3, 2, 2), 0.0, 0.0, 3)
    Xr = st.G
    for m, a in enumerate(st.A):
        Xr = np.moveaxis(np.tensordot(Xr, a, axes=([m], [1])), -1, m)
    assert np.linalg.norm(X - Xr) < 1e-12 * np.linalg.norm(X)
    assert tr[-1]["residual"] < 1e-7      # the expansion's sqrt of a cancellation
    X, _, _ = tucker_tensor((8, 7, 6, 5), (3, 2, 2, 2), 7, noise=0.05)
    st, tr = T.pp_tucker_als(X, (3, 2, 2, 2), 0.0, 0.0, 2)
    Xr = st.G
    for m, a in enumerate(st.A):
        Xr = np.moveaxis(np.tensordot(Xr, a, axes=([m], [1])), -1, m)
    lhs = np.linalg.norm(X - Xr) ** 2
    rhs = np.linalg.norm(X) ** 2 - np.linalg.norm(st.G) ** 2
    assert abs(lhs - rhs) <= 1e-9 * np.linalg.norm(X) ** 2
    for a in st.A:
        assert np.linalg.norm(a.T @ a - np.eye(a.shape[1])) < 1e-10


def test_core_norm_monotone():
    """Lemma 4.7: ||G||_F is non-decreasing over Tucker-ALS sweeps."""
    X, _, _ = tucker_tensor((9, 8, 7), (3, 3, 2), 8, noise=0.3)
    _, tr = T.pp_tucker_als(X, (3, 3, 2), 0.0, 0.0, 8)
    g = [t["core_norm"] for t in tr]
    assert all(b >= a * (1 - 1e-10) for a, b in zip(g, g[1:]))


# ---------------------------------------------------------------- PP (Alg. 4)
def pp_setup(dims, ranks, seed, t):
    r = rng(seed)
    X = r.standard_normal(dims)
    Ap = [orth(r, s, R) for s, R in zip(dims, ranks)]
    dA = [t * r.standard_normal(a.shape) for a in Ap]
    ops = T.pp_operators(X, Ap)
    Yp = [T.pp_single(ops, Ap, n, len(dims)) for n in range(len(dims))]
    return X, Ap, dA, ops, Yp


def test_pp_operators_definition_and_count():
    """C(N,2) operators; each equals Def. 3.2 built by explicit loops (N = 3)."""
    X, Ap, _, ops, Yp = pp_setup((3, 4, 2), (2, 2, 2), 9, 0.0)
    assert len(ops) == 3
    Y02 = ops[(0, 2)]
    for x0, z1, x2 in itertools.product(range(3), range(2), range(2)):
        v = sum(X[x0, b, x2] * Ap[1][b, z1] for b in range(4))
        assert abs(Y02[x0, z1, x2] - v) < 1e-13
    for n in range(3):
        assert np.allclose(Yp[n], T.ttmc(X, Ap, n), atol=1e-12)


@pytest.mark.parametrize("dims,ranks", [((5, 4, 6), (2, 3, 2)), ((4, 3, 5, 4), (2, 2, 3, 2))])
def test_pp_update_exactness(dims, ranks):
    """dA = 0 -> Ỹ = Y_p exactly; one perturbed mode m -> Ỹ^(n) = Y^(n) at A_p + dA for n ≠ m
    (multilinearity)."""
    X, Ap, dA, ops, Yp = pp_setup(dims, ranks, 10, 0.3)
    N = len(dims)
    zero = [np.zeros_like(a) for a in Ap]
    for n in range(N):
        assert np.array_equal(T.pp_update(Yp[n], ops, zero, n), Yp[n])
    for m in range(N):
        d = [np.zeros_like(a) for a in Ap]
        d[m] = dA[m]
        A = [a + x for a, x in zip(Ap, d)]
        for n in range(N):
            if n != m:
                ref = T.ttmc(X, A, n)
                assert np.linalg.norm(T.pp_update(Yp[n], ops, d, n) - ref) <= 1e-12 * np.linalg.norm(ref)


def test_pp_update_quadratic_error():
    """||Ỹ^(n) - Y^(n)|| falls quadratically in ||dA|| (the dropped terms of P:636 are second
    order): err(t/10) ≈ err(t)/100."""
    e = []
    for t in (1e-2, 1e-3):
        X, Ap, dA, ops, Yp = pp_setup((6, 5, 4, 5), (2, 2, 2, 2), 11, t)
        A = [a + d for a, d in zip(Ap, dA)]
        e.append(max(np.linalg.norm(T.pp_update(Yp[n], ops, dA, n) - T.ttmc(X, A, n)) for n in range(4)))
    assert abs(e[0] / e[1] / 100 - 1) < 0.05


def test_pp_tucker_runs():
    """ε_pp = 0 is Alg. 2 exactly; on a noisy multilinear-rank tensor PP phases are entered and
    the final residual matches Alg. 2's within 1e-6 (S:...pp_tucker_run examples)."""
    X, _, _ = tucker_tensor((12, 10, 9), (3, 3, 3), 12, noise=0.1)
    ranks = (3, 3, 3)
    _, tr0 = T.pp_tucker_als(X, ranks, 0.0, 0.0, 12)
    assert all(t["phase"] == "dt" for t in tr0)
    _, tr1 = T.pp_tucker_als(X, ranks, 0.0, 0.2, 12)
    assert any(t["phase"] != "dt" for t in tr1)
    assert abs(tr1[-1]["residual"] - tr0[-1]["residual"]) < 1e-6
