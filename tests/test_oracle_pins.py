"""Pins for the oracle (oracle/cp_oracle.py) against what the paper and mathematics fix.

Each test checks an oracle function against something OTHER than itself: printed worked
examples (tests/golden, with citations), brute-force index loops on tiny inputs, closed
forms (Kruskal / rank-1), invariants of the definitions, or an independently constructed
answer.  CPU only (`-m "not gpu"`).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle.cp_oracle as O
import synthgen as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def rng(seed=0):
    return np.random.default_rng(seed)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


# ---------------------------------------------------------------- notation
def test_khatri_rao_spec_examples():
    g = gold("spec_examples.json")
    for key in ("khatri_rao_identity", "khatri_rao_general"):
        e = g[key]
        got = O.khatri_rao([np.array(e["A"], float), np.array(e["B"], float)])
        assert np.array_equal(got, np.array(e["expected"], float)), e["cite"]


def test_khatri_rao_columns_are_kronecker():
    """Column k of A⊙B is a_k ⊗ b_k — checked with np.kron per column."""
    r = rng(1)
    A, B, C = r.random((3, 4)), r.random((5, 4)), r.random((2, 4))
    P = O.khatri_rao([A, B, C])
    for k in range(4):
        assert np.array_equal(P[:, k], np.kron(np.kron(A[:, k], B[:, k]), C[:, k]))


def test_generalized_unfolding_row_major_reading_of_P287():
    """P:287 X(j,k,l,m) = X_(1,3)(j,l,k+(m-1)s_2) in Kolda order; our row-major reading (L22)
    is X_(1,3)(j,l, k*s_4 + m) (0-based).  Checked element by element."""
    r = rng(2)
    X = r.random((2, 3, 4, 5))
    U = O.unfold_multi(X, [0, 2])
    for j, k, l, m in itertools.product(*map(range, X.shape)):
        assert U[j, l, k * 5 + m] == X[j, k, l, m]


def test_mttkrp_matches_kolda_convention():
    """L22: MTTKRP does not depend on the unfolding convention.  Kolda: X_(n) column-major
    over the other modes with P = A^(N)⊙…⊙A^(1) (reverse order).  Built independently here."""
    r = rng(3)
    X = r.random((3, 4, 5, 2))
    A = [r.random((d, 3)) for d in X.shape]
    for n in range(4):
        others = [m for m in range(4) if m != n]
        Xk = np.moveaxis(X, n, 0).reshape(X.shape[n], -1, order="F")
        P = A[others[-1]]
        for m in reversed(others[:-1]):
            P = (P[:, None, :] * A[m][None, :, :]).reshape(-1, 3)
        assert rel(O.mttkrp(X, A, n), Xk @ P) < 1e-14


# ---------------------------------------------------------------- MTTKRP
def brute_mttkrp(X, A, n):
    N = X.ndim
    K = A[0].shape[1]
    M = np.zeros((X.shape[n], K))
    for idx in itertools.product(*map(range, X.shape)):
        for k in range(K):
            p = X[idx]
            for m in range(N):
                if m != n:
                    p *= A[m][idx[m], k]
            M[idx[n], k] += p
    return M


@pytest.mark.parametrize("dims,K", [((3, 4, 5), 2), ((2, 3, 2, 3), 3), ((2, 2, 3, 2, 2), 2)])
def test_mttkrp_brute_force(dims, K):
    r = rng(4)
    X = r.standard_normal(dims)
    A = [r.standard_normal((d, K)) for d in dims]
    for n in range(len(dims)):
        assert rel(O.mttkrp(X, A, n), brute_mttkrp(X, A, n)) < 1e-13


def test_mttkrp_all_ones_spec_example():
    e = gold("spec_examples.json")["mttkrp_all_ones"]
    X = np.ones(e["dims"])
    A = [np.array([[7.0], [-3.0]]), np.array(e["A2"], float), np.array(e["A3"], float)]
    assert np.array_equal(O.mttkrp(X, A, 0), np.array(e["expected_M1"], float)), e["cite"]


def test_mttkrp_rank1_closed_form():
    """X = a∘b∘c with unit b, c ⇒ M^(1) with factors (·, b, c) equals a."""
    r = rng(5)
    a, b, c = r.standard_normal(4), r.standard_normal(5), r.standard_normal(6)
    b /= np.linalg.norm(b)
    c /= np.linalg.norm(c)
    X = np.multiply.outer(np.multiply.outer(a, b), c)
    M = O.mttkrp(X, [np.zeros((4, 1)), b[:, None], c[:, None]], 0)
    assert rel(M[:, 0], a) < 1e-14


def test_mttkrp_matrix_case():
    """N=2 ⇒ M^(1) = X A^(2), M^(2) = X^T A^(1)."""
    r = rng(6)
    X = r.standard_normal((5, 7))
    A = [r.standard_normal((5, 3)), r.standard_normal((7, 3))]
    assert rel(O.mttkrp(X, A, 0), X @ A[1]) < 1e-14
    assert rel(O.mttkrp(X, A, 1), X.T @ A[0]) < 1e-14


def kruskal_closed_form(B, A, kept):
    """For X = [[B]], T_U(x_U,k) = Σ_r Π_{u∈U} B^(u)(x_u,r) Π_{m∉U} (B^(m)ᵀA^(m))(r,k)."""
    N = len(B)
    R = B[0].shape[1]
    K = A[0].shape[1]
    W = np.ones((R, K))
    for m in range(N):
        if m not in kept:
            W = W * (B[m].T @ A[m])
    # outer over kept modes of B columns, contracted with W over r
    T = B[kept[0]]
    for u in kept[1:]:
        T = (T[..., None, :] * B[u].reshape((1,) * (T.ndim - 1) + B[u].shape))
    return np.tensordot(T, W, axes=([T.ndim - 1], [0]))


@pytest.mark.parametrize("N,s,R,K", [(3, 6, 2, 3), (4, 5, 3, 2), (5, 3, 2, 4)])
def test_partial_mttkrp_kruskal_closed_form(N, s, R, K):
    r = rng(7)
    B = [r.standard_normal((s, R)) for _ in range(N)]
    A = [r.standard_normal((s, K)) for _ in range(N)]
    X = G.kruskal_slab(B)
    for m in range(1, N):
        for kept in itertools.combinations(range(N), m):
            kept = list(kept)
            assert rel(O.partial_mttkrp(X, A, kept), kruskal_closed_form(B, A, kept)) < 1e-12


# ---------------------------------------------------------------- Def. 3.1 operators
def brute_operator(X, A, i, n):
    """M^(i,n)(x,y,k) = Σ_{others} X Π_{r∉{i,n}} A^(r)(x_r,k) — any i≠n order (Def. 3.1)."""
    N = X.ndim
    K = A[0].shape[1]
    M = np.zeros((X.shape[i], X.shape[n], K))
    for idx in itertools.product(*map(range, X.shape)):
        for k in range(K):
            p = X[idx]
            for m in range(N):
                if m not in (i, n):
                    p *= A[m][idx[m], k]
            M[idx[i], idx[n], k] += p
    return M


def test_operators_brute_force_and_symmetry():
    r = rng(8)
    dims = (3, 4, 2, 3)
    X = r.standard_normal(dims)
    A = [r.standard_normal((d, 2)) for d in dims]
    ops = O.pp_operators(X, A)
    assert len(ops) == 6
    for i in range(4):
        for n in range(4):
            if i != n:
                assert rel(O.op_pair(ops, i, n), brute_operator(X, A, i, n)) < 1e-13


def test_single_mode_terms_consistent_for_every_pair():
    """M_p^(n) = M_p^(j,n) ×_j A_p^(j) for EVERY j ≠ n and = MTTKRP(A_p)."""
    r = rng(9)
    dims = (4, 3, 5, 2)
    X = r.standard_normal(dims)
    A = [r.standard_normal((d, 3)) for d in dims]
    ops = O.pp_operators(X, A)
    for n in range(4):
        ref = O.mttkrp(X, A, n)
        for j in range(4):
            if j != n:
                assert rel(O.pp_single(ops, A, n, 4, j=j), ref) < 1e-13


# ---------------------------------------------------------------- Def. pptree
def test_pptree_N4_golden():
    g = gold("pptree_N4.json")
    tree = O.pp_tree(4)
    for l, nodes in g["levels"].items():
        got = sorted((tuple(k), tuple(sorted(mu)), tuple(p)) for k, mu, p in tree[int(l)])
        want = sorted((tuple(n["kept"]), tuple(n["mu"]), tuple(n["parent"])) for n in nodes)
        assert got == want


@pytest.mark.parametrize("N", range(3, 9))
def test_pptree_structure(N):
    tree = O.pp_tree(N)
    assert sorted(tree) == list(range(1, N - 1))
    allm = set(range(1, N + 1))
    for l, nodes in tree.items():
        assert len(nodes) == math.comb(l + 2, 2)                    # Lemma cost
        for kept, mu, parent in nodes:
            assert set(kept) | set(mu) == allm and len(mu) == l
            if l == 1:
                assert parent == tuple(range(1, N + 1))
            else:
                # the child contracts i = max μ(t) from its parent
                pmu = allm - set(parent)
                assert pmu == set(mu) - {max(mu)}
                assert parent in [k for k, _, _ in tree[l - 1]]
    leaves = tree[N - 2]
    assert sorted(tuple(k) for k, _, _ in leaves) == sorted(itertools.combinations(range(1, N + 1), 2))


@pytest.mark.parametrize("N", range(3, 9))
@pytest.mark.parametrize("s,R", [(2, 1), (5, 3), (20, 30)])
def test_pptree_cost_matches_P718(N, s, R):
    assert O.pp_tree_flops(N, s, R) == O.pp_build_flops_formula(N, s, R)
    if N >= 4:
        lead = 6 * s ** N * R + 12 * s ** (N - 1) * R
        rest = 2 * R * sum(math.comb(l + 1, 2) * s ** (N - l + 2) for l in range(4, N))
        assert O.pp_build_flops_formula(N, s, R) == lead + rest


# ---------------------------------------------------------------- PP update
def setup_pp(dims, K, seed):
    r = rng(seed)
    X = r.standard_normal(dims)
    Ap = [r.standard_normal((d, K)) for d in dims]
    ops = O.pp_operators(X, Ap)
    Mp = [O.pp_single(ops, Ap, n, len(dims)) for n in range(len(dims))]
    return r, X, Ap, ops, Mp


def test_pp_update_zero_perturbation_is_exact_bitwise():
    r, X, Ap, ops, Mp = setup_pp((4, 3, 5), 3, 10)
    dA = [np.zeros_like(a) for a in Ap]
    for n in range(3):
        assert np.array_equal(O.pp_update(Mp[n], ops, dA, n), Mp[n])


@pytest.mark.parametrize("dims", [(4, 3, 5), (3, 4, 2, 3), (2, 3, 2, 2, 3)])
def test_pp_update_single_mode_perturbation_is_exact(dims):
    """Only dA^(m) ≠ 0 ⇒ M~^(n) = exact MTTKRP at A_p + dA for n ≠ m (multilinearity)."""
    r, X, Ap, ops, Mp = setup_pp(dims, 2, 11)
    N = len(dims)
    for m in range(N):
        dA = [np.zeros_like(a) for a in Ap]
        dA[m] = 0.3 * r.standard_normal(Ap[m].shape)
        A = [a + d for a, d in zip(Ap, dA)]
        for n in range(N):
            if n != m:
                assert rel(O.pp_update(Mp[n], ops, dA, n), O.mttkrp(X, A, n)) < 1e-13


def test_pp_update_N3_closed_form_error_term():
    """N=3: M^(n) - M~^(n) = X ×_i dA^(i)(:,k) ×_j dA^(j)(:,k) exactly, computed
    here straight from X with einsum (no operators)."""
    r, X, Ap, ops, Mp = setup_pp((5, 4, 6), 3, 12)
    dA = [0.1 * r.standard_normal(a.shape) for a in Ap]
    A = [a + d for a, d in zip(Ap, dA)]
    specs = {0: "abc,bk,ck->ak", 1: "abc,ak,ck->bk", 2: "abc,ak,bk->ck"}
    for n in range(3):
        others = [dA[m] for m in range(3) if m != n]
        err = O.mttkrp(X, A, n) - O.pp_update(Mp[n], ops, dA, n)
        want = np.einsum(specs[n], X, *others)
        assert rel(err, want) < 1e-11
        # and the oracle's own second-order term agrees
        assert rel(O.second_order_term(X, Ap, dA, n), want) < 1e-12


def test_pp_update_quadratic_error_scaling():
    """err(ε/10) <= err(ε)/30 for ε in {1e-2,1e-3,1e-4} (Thm 4.1 / S:559), N=4, s=8, R=3."""
    r, X, Ap, ops, Mp = setup_pp((8, 8, 8, 8), 3, 13)
    D = [r.standard_normal(a.shape) for a in Ap]
    errs = []
    for eps in (1e-2, 1e-3, 1e-4):
        dA = [eps * np.linalg.norm(a) * d / np.linalg.norm(d) for a, d in zip(Ap, D)]
        A = [a + d for a, d in zip(Ap, dA)]
        errs.append(max(np.linalg.norm(O.mttkrp(X, A, n) - O.pp_update(Mp[n], ops, dA, n))
                        for n in range(4)))
    assert errs[1] <= errs[0] / 30 and errs[2] <= errs[1] / 30


# ---------------------------------------------------------------- normal equations
def test_gamma_and_solve_spec_examples():
    g = gold("spec_examples.json")
    e = g["gamma_scalar"]
    S = [np.array([[99.0]]), np.array(e["S2"], float), np.array(e["S3"], float)]
    assert np.array_equal(O.gamma(S, e["n"]), np.array(e["expected"], float))
    for key in ("solve_scalar", "solve_zero_gamma"):
        e = g[key]
        got = O.solve_normal(np.array(e["M"], float), np.array(e["Gamma"], float))
        assert np.allclose(got, np.array(e["expected"], float), rtol=0, atol=1e-15), e["cite"]


def test_gamma_identity_and_hadamard():
    r = rng(14)
    I = np.eye(4)
    assert np.array_equal(O.gamma([I, I, I, I], 2), I)
    S = [r.random((3, 3)) for _ in range(4)]
    assert np.array_equal(O.gamma(S, 1), S[0] * S[2] * S[3])


def test_cholesky_reconstructs_and_solve_residual():
    r = rng(15)
    B = r.standard_normal((40, 12))
    Gm = B.T @ B
    L, ok = O.cholesky_pivots(Gm)
    assert ok and rel(L @ L.T, Gm) < 1e-14 and np.allclose(np.triu(L, 1), 0)
    M = r.standard_normal((9, 12))
    An = O.solve_normal(M, Gm)
    assert np.linalg.norm(An @ Gm - M) <= 1e-12 * np.linalg.norm(M) * np.linalg.cond(Gm)


def test_solve_singular_gamma_pseudo_inverse_closed_form():
    """Γ = V diag(λ) Vᵀ with λ having exact zeros ⇒ A_new = M V diag(λ⁺) Vᵀ."""
    r = rng(16)
    V, _ = np.linalg.qr(r.standard_normal((6, 6)))
    lam = np.array([5.0, 3.0, 1.0, 0.5, 0.0, 0.0])
    Gm = (V * lam) @ V.T
    Gm = 0.5 * (Gm + Gm.T)
    M = r.standard_normal((7, 6))
    want = M @ ((V * np.array([1 / 5, 1 / 3, 1.0, 2.0, 0.0, 0.0])) @ V.T)
    assert rel(O.solve_normal(M, Gm), want) < 1e-12


def test_gradient_examples():
    r = rng(17)
    A, An = r.random((5, 3)), r.random((5, 3))
    assert np.array_equal(O.gradient(A, A, r.random((3, 3))), np.zeros((5, 3)))
    assert np.array_equal(O.gradient(A, An, np.eye(3)), A - An)


# ---------------------------------------------------------------- fitness
def test_residual_expansion_vs_explicit_reconstruction():
    r = rng(18)
    dims = (4, 5, 3, 4)
    X = r.standard_normal(dims)
    A = [r.standard_normal((d, 3)) for d in dims]
    S = [a.T @ a for a in A]
    M = O.mttkrp(X, A, 3)
    r2 = O.residual_sq_expansion(float(np.sum(X * X)), M, A[3], O.gamma(S, 3), S[3])
    explicit = float(np.sum((X - O.kruskal_full(A)) ** 2))
    assert abs(r2 - explicit) <= 1e-10 * np.sum(X * X)


def test_kruskal_full_matches_generator_materialization():
    """Oracle [[A]] (KRP matmul) vs synthgen's fixed-order elementwise loop — two codes."""
    r = rng(19)
    A = [r.standard_normal((d, 4)) for d in (3, 5, 4)]
    assert rel(O.kruskal_full(A), G.kruskal_slab(A)) < 1e-14


# ---------------------------------------------------------------- sweeps (Alg. 1 / Alg. 3)
def small_problem(noise=0.0, seed=20, dims=(8, 9, 7), R=3):
    r = rng(seed)
    B = [r.random((d, R)) for d in dims]
    X = G.kruskal_slab(B) + noise * r.standard_normal(dims)
    A0 = [r.random((d, R)) for d in dims]
    return X, B, A0


def test_true_factors_give_zero_gradient_and_unit_fitness():
    X, B, _ = small_problem()
    st = O.State(X, B)
    st.dt_sweep()
    assert max(st.G_norms) < 1e-9 * np.linalg.norm(X)
    assert st.fitness() > 1 - 1e-6
    assert all(rel(a, b) < 1e-9 for a, b in zip(st.A, B))


def test_eps_pp_zero_is_plain_als():
    X, _, A0 = small_problem(noise=1e-2)
    A_als, tr_als = O.cp_als(X, A0, 12)
    A_pp, tr_pp = O.pp_cp_als(X, A0, 0.0, 0.0, 12)
    assert all(t["phase"] == "dt" for t in tr_pp)
    assert all(np.array_equal(a, b) for a, b in zip(A_als, A_pp))
    assert [t["fitness"] for t in tr_pp] == tr_als


def test_exact_als_residual_monotone():
    X, _, A0 = small_problem(noise=5e-2, seed=21)
    _, tr = O.cp_als(X, A0, 40)
    res = [1 - f for f in tr]
    nx = 1.0
    assert all(res[i + 1] <= res[i] + 1e-10 * nx for i in range(len(res) - 1))


def test_first_pp_sweep_exact_for_modes_1_and_2():
    """After a build, M~^(1) uses dA=0 and M~^(2) only dA^(1): both equal the exact MTTKRP."""
    X, _, A0 = small_problem(noise=1e-2, seed=22, dims=(6, 7, 5, 6))
    st = O.State(X, A0)
    for _ in range(3):
        st.dt_sweep()
    st.pp_build()
    for n in (0, 1):
        M_pp = O.pp_update(st.Mp[n], st.ops, st.dA, n)
        assert rel(M_pp, O.mttkrp(X, st.A, n)) < 1e-12
        st._update_mode(n, M_pp, st.A_p[n])


def test_exact_recovery_noise_free():
    """Noise-free rank-R input ⇒ fitness → 1 (north_star).  Exact ALS reaches fitness 1 - 1e-6;
    PP-ALS (ε_pp = 0.1, PP phases entered) reaches a true relative residual (explicit
    reconstruction) below 1e-4 — its expansion fitness is only O(ε²)-accurate (L17, L27)."""
    r = rng(23)
    B = [r.standard_normal((10, 3)) for _ in range(3)]
    X = G.kruskal_slab(B)
    r = rng(123)
    A0 = [b + 0.05 * r.standard_normal(b.shape) for b in B]
    A, tr = O.cp_als(X, A0, 30)
    assert tr[-1] > 1 - 1e-6
    assert np.linalg.norm(X - O.kruskal_full(A)) / np.linalg.norm(X) < 1e-6
    A, tr = O.pp_cp_als(X, A0, 0.0, 0.1, 30)
    assert any(t["phase"] == "pp-approx" for t in tr)
    assert np.linalg.norm(X - O.kruskal_full(A)) / np.linalg.norm(X) < 1e-4


def test_pp_phase_machine_readings():
    """L9-L11: first sweep dt; pp-build only right after a dt sweep with small change; after a
    PP sweep that fails the test exactly one dt sweep follows."""
    X, _, A0 = small_problem(noise=1e-2, seed=24)
    _, tr = O.pp_cp_als(X, A0, 0.0, 0.2, 40)
    ph = [t["phase"] for t in tr]
    assert ph[0] == "dt"
    for a, b, t in zip(ph, ph[1:], tr):
        if b == "pp-build":
            assert a == "dt" and t["max_rel_dA"] < 0.2
        if b == "pp-approx":
            assert a in ("pp-build", "pp-approx") and t["max_rel_dA"] < 0.2
        if a in ("pp-build", "pp-approx") and t["max_rel_dA"] >= 0.2:
            assert b == "dt"


def test_phase_override_replays_schedule():
    X, _, A0 = small_problem(noise=1e-2, seed=25)
    _, tr = O.pp_cp_als(X, A0, 0.0, 0.2, 25)
    sched = [t["phase"] for t in tr]
    _, tr2 = O.pp_cp_als(X, A0, 0.0, 0.2, 25, phase_override=sched)
    assert [t["fitness"] for t in tr2] == [t["fitness"] for t in tr]


# ---------------------------------------------------------------- the ε_pp metric (L7) and r² (L17)
@pytest.mark.parametrize("t", [0.05, 0.5])
@pytest.mark.parametrize("phase", ["dt", "pp-build"])
def test_rel_dA_closed_form_scaled_update(t, phase):
    """X = (1+t)[[A]]: one sweep from A moves A^(1) to (1+t)A^(1) and leaves the others (mode 0's
    least-squares solution absorbs the scale; with dA^(2..N) = 0 the PP update is exact too,
    P:553-557).  So dA^(1) = t A^(1) (L8) and the relative metric of L7, ‖dA‖/‖A‖ with the
    CURRENT A, is exactly t/(1+t) -- an absolute norm would give t‖A‖, a metric normalised by
    A_prev or A_p would give t."""
    r = rng(40)
    dims = (7, 6, 8, 5)
    A = [r.random((d, 3)) + 0.1 for d in dims]
    X = (1.0 + t) * O.kruskal_full(A)
    _, tr = O.pp_cp_als(X, A, 0.0, 0.1, 1, phase_override=[phase])
    assert abs(tr[0]["max_rel_dA"] - t / (1.0 + t)) < 1e-10
    st = O.State(X, A)
    st.pp_build() if phase != "dt" else None
    st.pp_sweep() if phase != "dt" else st.dt_sweep()
    rels = st.rel_dA()
    assert abs(rels[0] - t / (1.0 + t)) < 1e-10 and max(rels[1:]) < 1e-10
    # the new factor itself: exactly (1+t) A^(1) up to rounding
    assert rel(st.A[0], (1.0 + t) * A[0]) < 1e-10


def test_phase_sequence_invariant_under_tensor_scaling():
    """Scaling X and A^(1) by c = 1e6 scales every later A^(1) by c and leaves A^(2..N) unchanged
    (the normal equations are homogeneous), so a RELATIVE ε_pp metric (L7) sees the same numbers
    and Alg. 3 takes the same phases; an absolute ‖dA‖ test would not."""
    X, _, A0 = small_problem(noise=1e-2, seed=24)
    c = 1e6
    A1 = [a.copy() for a in A0]
    A1[0] = c * A1[0]
    _, tr = O.pp_cp_als(X, A0, 0.0, 0.2, 30)
    _, tr_c = O.pp_cp_als(c * X, A1, 0.0, 0.2, 30)
    assert any(t["phase"] != "dt" for t in tr)
    assert [t["phase"] for t in tr] == [t["phase"] for t in tr_c]
    for a, b in zip(tr, tr_c):
        assert abs(a["max_rel_dA"] - b["max_rel_dA"]) <= 1e-9 * a["max_rel_dA"]
        assert abs(a["fitness"] - b["fitness"]) <= 1e-9


def test_trace_residual_sq_is_explicit_residual_after_regular_sweeps():
    """The trace's unclamped r² (S:177 with the sweep's last M^(N)) equals ‖X - [[A]]‖² computed
    by explicit reconstruction after every regular sweep (L17)."""
    X, _, A0 = small_problem(noise=1e-2, seed=26)
    nx2 = float(np.sum(X * X))
    st = O.State(X, A0)
    for _ in range(5):
        st.dt_sweep()
        explicit = float(np.sum((X - O.kruskal_full(st.A)) ** 2))
        assert abs(st.residual_sq() - explicit) <= 1e-12 * nx2


@pytest.mark.parametrize("dims", [(5, 4, 6, 3), (4, 3, 5, 3, 4)])
def test_second_order_term_multilinear_remainder(dims):
    """Multilinearity of M^(n) in the factors: with A = A_p + dA,
    M^(n)(A) = Σ_{S ⊆ modes≠n} M^(n)(dA on S, A_p elsewhere).  |S| = 0, 1 are the PP update
    (P:553), |S| = 2 is second_order_term; the rest (|S| >= 3) is computed here by plain MTTKRPs
    with mixed factor lists, so M - M~ - T2 must equal that remainder."""
    from itertools import combinations as comb
    N = len(dims)
    r, X, Ap, ops, Mp = setup_pp(dims, 3, 31)
    dA = [0.2 * r.standard_normal(a.shape) for a in Ap]
    A = [a + d for a, d in zip(Ap, dA)]
    for n in range(N):
        others = [m for m in range(N) if m != n]
        rem = np.zeros_like(Mp[n])
        for size in range(3, N):
            for S in comb(others, size):
                F = [dA[m] if m in S else Ap[m] for m in range(N)]
                rem = rem + O.mttkrp(X, F, n)
        got = O.mttkrp(X, A, n) - O.pp_update(Mp[n], ops, dA, n) - O.second_order_term(X, Ap, dA, n)
        assert rel(got, rem) < 1e-10, n


def test_solve_tau_selects_the_branch():
    """L13's τ: a Γ with a pivot ratio of ~1e-3 is solved by Cholesky at τ = 1e-12 and by the
    eigen pseudo-inverse at τ = 1e-2, which then drops the eigenvalues below τ λ_max -- the
    minimum-norm solution on the remaining eigenspace, built here from numpy's eigh."""
    r = rng(41)
    Q = np.linalg.qr(r.standard_normal((5, 5)))[0]
    lam = np.array([1.0, 0.5, 0.2, 4e-3, 1e-3])
    G = (Q * lam) @ Q.T
    M = r.standard_normal((7, 5))
    assert O.cholesky_pivots(G)[1] and not O.cholesky_pivots(G, 1e-2)[1]
    assert rel(O.solve_normal(M, G), M @ np.linalg.inv(G)) < 1e-10
    keep = lam > 1e-2 * lam.max()
    want = M @ ((Q[:, keep] / lam[keep]) @ Q[:, keep].T)
    assert rel(O.solve_normal(M, G, 1e-2), want) < 1e-10
