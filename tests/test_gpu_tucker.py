"""GPU parity of the PP-Tucker contraction path (include/cppp_tucker.h) against
oracle/tucker_oracle.py on identical seeded inputs: TTMc Y^(n) through the dimension tree, the
Def. 3.2 operators Y_p^(i,j) through the construction tree, Y_p^(n), and the PP update
Y~^(n) — relative Frobenius 1e-11 (the CP path's kernel tolerance; every result is a chain of
FP64 GEMMs)."""
import numpy as np
import pytest

import oracle.tucker_oracle as T

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1811_10573_b200.cppp as cp  # noqa: E402

TOL = 1e-11
SHAPES = [((40, 36, 34), (10, 8, 6)),           # DMMA path (even extents)
          ((7, 9, 5), (3, 2, 4)),               # odd extents: SIMT path
          ((20, 18, 16, 14), (4, 4, 3, 3)),
          ((6, 5, 4, 6, 5), (2, 3, 2, 2, 3)),
          ((12, 12, 12, 12, 12, 12), (3, 3, 3, 3, 3, 3))]   # the paper's N = 6 shape, reduced


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def problem(dims, ranks, seed):
    r = np.random.default_rng(seed)
    X = r.standard_normal(dims)
    A = [np.linalg.qr(r.standard_normal((s, R)))[0].copy() for s, R in zip(dims, ranks)]
    return X, A


@pytest.mark.parametrize("dims,ranks", SHAPES)
@pytest.mark.parametrize("simt", [False, True])
def test_ttmc_matches_oracle(dims, ranks, simt):
    X, A = problem(dims, ranks, 1)
    ctx = cp.tk_init(X, dims, ranks, flags=cp.FLAG_SIMT_TTM if simt else 0)
    cp.tk_set_factors(ctx, A)
    Y = cp.tk_ttmc(ctx)
    for n in range(len(dims)):
        assert rel(Y[n], T.ttmc(X, A, n)) < TOL, n
    cp.tk_destroy(ctx)


@pytest.mark.parametrize("flags", [0, cp.FLAG_NO_KRP])
@pytest.mark.parametrize("dims,ranks", [((20, 18, 16, 14), (4, 4, 3, 3)), ((40, 36, 34), (4, 2, 6)),
                                        ((12, 12, 12, 12, 12, 12), (3, 3, 3, 3, 3, 3)),
                                        ((8, 6, 10, 6, 8, 4, 6), (2, 3, 2, 2, 3, 2, 2))])
def test_kronecker_first_level_and_pair_tree(dims, ranks, flags):
    """Halves of the regular tree with Π R <= 16 contracted from X in one Kronecker GEMM each, and
    (order >= 6) the PP operators built below the neighbour pairs (0,1), (2,3), ... (default) --
    or one mode at a time through Def. pptree (FLAG_NO_KRP): TTMc and operators against the
    oracle."""
    X, A = problem(dims, ranks, 7)
    ctx = cp.tk_init(X, dims, ranks, flags=flags)
    cp.tk_set_factors(ctx, A)
    Y = cp.tk_ttmc(ctx)
    for n in range(len(dims)):
        assert rel(Y[n], T.ttmc(X, A, n)) < TOL, n
    cp.tk_pp_build(ctx)
    for (i, j), ref in T.pp_operators(X, A).items():
        assert rel(cp.tk_pp_get_operator(ctx, i, j), ref) < TOL, (i, j)
    cp.tk_destroy(ctx)


@pytest.mark.parametrize("dims,ranks", SHAPES)
def test_pp_operators_and_update_match_oracle(dims, ranks):
    X, Ap = problem(dims, ranks, 2)
    N = len(dims)
    ctx = cp.tk_init(X, dims, ranks)
    cp.tk_set_factors(ctx, Ap)
    cp.tk_pp_build(ctx)
    ops = T.pp_operators(X, Ap)
    for (i, j), ref in ops.items():
        assert rel(cp.tk_pp_get_operator(ctx, i, j), ref) < TOL, (i, j)
    Yp = [T.pp_single(ops, Ap, n, N) for n in range(N)]
    for n in range(N):
        assert rel(cp.tk_pp_get_single(ctx, n), Yp[n]) < TOL, n
    r = np.random.default_rng(3)
    dA = [0.01 * r.standard_normal(a.shape) for a in Ap]
    cp.tk_update_factors(ctx, [a + d for a, d in zip(Ap, dA)])
    for n in range(N):
        assert rel(cp.tk_pp_update(ctx, n), T.pp_update(Yp[n], ops, dA, n)) < TOL, n
    cp.tk_destroy(ctx)


def test_tucker_errors_and_device_tensor():
    X, A = problem((8, 6, 4), (2, 3, 2), 4)
    with pytest.raises(cp.CpppError):
        cp.tk_init(X, (8, 6, 4), (9, 3, 2))          # R_0 > s_0
    ctx = cp.tk_init(X, (8, 6, 4), (2, 3, 2))
    with pytest.raises(cp.CpppError):
        cp.tk_ttmc(ctx)                              # before tk_set_factors
    cp.tk_set_factors(ctx, A)
    with pytest.raises(cp.CpppError):
        cp.tk_pp_update(ctx, 0)                      # before tk_pp_build
    cp.tk_destroy(ctx)
    Xd = torch.from_numpy(X).cuda()
    ctx = cp.tk_init(Xd, (8, 6, 4), (2, 3, 2), flags=cp.FLAG_BORROW_TENSOR)
    cp.tk_set_factors(ctx, A)
    Y = cp.tk_ttmc(ctx)
    assert rel(Y[1], T.ttmc(X, A, 1)) < TOL
    cp.tk_destroy(ctx)


# ---------------------------------------------------------------- the HOOI / PP-Tucker driver
def tucker_tensor(dims, ranks, seed, noise):
    r = np.random.default_rng(seed)
    X = r.standard_normal(ranks)
    for m, (s, R) in enumerate(zip(dims, ranks)):
        a = np.linalg.qr(r.standard_normal((s, R)))[0]
        X = np.moveaxis(np.tensordot(X, a, axes=([m], [1])), -1, m)
    Z = r.standard_normal(dims)
    return X + noise * np.linalg.norm(X) / np.linalg.norm(Z) * Z


def check_trace(ctx, X, tr, A_ref):
    for t in tr:
        cp.tk_set_phase_override(ctx, t["phase"])
        g = cp.tk_sweep(ctx, 0.0, 0.2)
        assert g["phase"] == t["phase"]
        assert abs(g["core_norm"] - t["core_norm"]) <= 1e-10 * t["core_norm"], (g, t)
        assert abs(g["core_change"] - t["core_change"]) <= 1e-8 * t["core_norm"], (g, t)
        assert abs(g["residual"] - t["residual"]) <= 1e-8, (g, t)
        assert abs(g["max_rel_dA"] - t["max_rel_dA"]) <= 1e-8, (g, t)
    A = cp.tk_get_factors(ctx)
    for a, b in zip(A, A_ref):
        assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b)


@pytest.mark.parametrize("dims,ranks", [((40, 36, 34), (5, 4, 3)), ((20, 18, 16, 14), (3, 3, 2, 2))])
def test_hosvd_and_pp_tucker_trace_match_oracle(dims, ranks):
    """tk_hosvd = oracle HOSVD (factors, core); then 12 sweeps of Alg. 4 (ε_pp = 0.2, the oracle's
    phase schedule replayed) match per sweep: core norm, core change, residual, max ||dA||/||A||;
    final factors within 1e-8 (eigenvectors of well-separated Gram spectra)."""
    X = tucker_tensor(dims, ranks, 5, 0.1)
    G0, A0 = T.hosvd(X, ranks)
    ctx = cp.tk_init(X, dims, ranks)
    cp.tk_hosvd(ctx)
    for a, b in zip(cp.tk_get_factors(ctx), A0):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
    assert rel(cp.tk_get_core(ctx), G0) < 1e-10
    st, tr = T.pp_tucker_als(X, ranks, 0.0, 0.2, 12)
    assert any(t["phase"] != "dt" for t in tr)
    check_trace(ctx, X, tr, st.A)
    cp.tk_destroy(ctx)


def test_pp_tucker_large_mode_uses_the_rank_side_gram():
    """s_0 = 200 > 128: the factor update takes the Gram of Y_(n)^T (R^(N-1) = 20 <= 128) and maps
    the eigenvectors back (Y v / sqrt(λ)); factors given (the oracle's HOSVD)."""
    dims, ranks = (200, 40, 36), (5, 5, 4)
    X = tucker_tensor(dims, ranks, 6, 0.1)
    _, A0 = T.hosvd(X, ranks)
    ctx = cp.tk_init(X, dims, ranks)
    with pytest.raises(cp.CpppError):
        cp.tk_hosvd(ctx)
    cp.tk_set_factors(ctx, A0)
    st, tr = T.pp_tucker_als(X, ranks, 0.0, 0.2, 8, A0=A0)
    check_trace(ctx, X, tr, st.A)
    cp.tk_destroy(ctx)


@pytest.mark.parametrize("dims,ranks", [((5, 4, 6), (1, 1, 1)),                 # rank 1
                                        ((4, 3, 5), (4, 3, 5)),                 # full ranks
                                        ((3, 2, 2, 3, 2, 2, 3, 2), (2, 1, 2, 2, 1, 2, 2, 1))])  # N = 8
def test_tucker_edge_shapes(dims, ranks):
    """Degenerate ranks and the maximum order: contractions, operators, updates and 4 sweeps of
    Alg. 4 from HOSVD against the oracle."""
    X, Ap = problem(dims, ranks, 12)
    N = len(dims)
    ctx = cp.tk_init(X, dims, ranks)
    cp.tk_set_factors(ctx, Ap)
    Y = cp.tk_ttmc(ctx)
    for n in range(N):
        assert rel(Y[n], T.ttmc(X, Ap, n)) < TOL, n
    cp.tk_pp_build(ctx)
    ops = T.pp_operators(X, Ap)
    for (i, j), ref in ops.items():
        assert rel(cp.tk_pp_get_operator(ctx, i, j), ref) < TOL, (i, j)
    st, tr = T.pp_tucker_als(X, ranks, 0.0, 0.2, 4)
    cp.tk_hosvd(ctx)
    for t in tr:
        cp.tk_set_phase_override(ctx, t["phase"])
        g = cp.tk_sweep(ctx, 0.0, 0.2)
        assert abs(g["core_norm"] - t["core_norm"]) <= 1e-9 * t["core_norm"], (g, t)
    cp.tk_destroy(ctx)


def test_tucker_gram_too_large_rejected():
    """Both sides of Y_(n) above 128 (s_0 = 200, prod of the other ranks = 11 x 13 = 143): the
    problem is refused at tk_init with CPPP_EINVAL instead of running out of the one-CTA solver."""
    dims, ranks = (200, 12, 14), (3, 11, 13)
    X, A = problem(dims, ranks, 13)
    with pytest.raises(cp.CpppError) as e:
        cp.tk_init(X, dims, ranks)
    assert e.value.status == -1


def lowrank_tensor(dims, core_ranks, seed, equal=True):
    """X = G ×_1 U1 ×_2 U2 ... with orthonormal U_n (s_n x r_n) and a super-diagonal core of
    ones (equal=True): every Gram of Y_(n) = X_(n) X_(n)ᵀ then has the eigenvalue 1 repeated."""
    r = np.random.default_rng(seed)
    U = [np.linalg.qr(r.standard_normal((s, q)))[0] for s, q in zip(dims, core_ranks)]
    q = min(core_ranks)
    G = np.zeros(core_ranks)
    for i in range(q):
        G[(i,) * len(dims)] = 1.0 if equal else 1.0 + i
    X = G
    for n, u in enumerate(U):
        X = np.moveaxis(np.tensordot(u, np.moveaxis(X, n, 0), axes=(1, 0)), 0, n)
    return np.ascontiguousarray(X), U


def check_orthonormal_and_span(A, U):
    for a, u in zip(A, U):
        assert np.all(np.isfinite(a))
        assert np.abs(a.T @ a - np.eye(a.shape[1])).max() < 1e-10
        assert np.linalg.norm(u - a @ (a.T @ u)) < 1e-8 * np.linalg.norm(u)


def test_tucker_repeated_eigenvalues_stay_orthonormal():
    """equal (and zero) eigenvalues among the R_n leading ones -- a super-diagonal core
    of ones gives the eigenvalue 1 three times and R_n = 4 adds a zero one.  The factors must stay
    finite and orthonormal and span the true subspaces (the top-R solver's clusters get distinct
    start vectors; an unseparated cluster falls back to the Jacobi solver)."""
    dims = (20, 18, 16)
    X, U = lowrank_tensor(dims, (3, 3, 3), 21)
    ctx = cp.tk_init(X, dims, (4, 4, 4))
    cp.tk_hosvd(ctx)
    check_orthonormal_and_span(cp.tk_get_factors(ctx), U)
    for _ in range(3):
        cp.tk_sweep(ctx, 0.0, 0.1)
    check_orthonormal_and_span(cp.tk_get_factors(ctx), U)
    cp.tk_destroy(ctx)


def test_tucker_rank_side_null_directions_completed():
    """s_0 = 200 > 128: mode 0's factor comes from the rank-side Gram (R_1 R_2 = 4 x 4), which has
    rank 2 here (multilinear rank 2): two null directions.  They are completed to an orthonormal
    basis (no division by sqrt(0)); a rank that exceeds the rank side is rejected at tk_init."""
    dims = (200, 6, 5)
    X, U = lowrank_tensor(dims, (2, 2, 2), 22, equal=False)
    ctx = cp.tk_init(X, dims, (4, 2, 2))
    r = np.random.default_rng(23)
    A0 = [np.linalg.qr(r.standard_normal((s, q)))[0].copy() for s, q in zip(dims, (4, 2, 2))]
    cp.tk_set_factors(ctx, A0)
    for _ in range(3):
        cp.tk_sweep(ctx, 0.0, 0.1)
    A = cp.tk_get_factors(ctx)
    check_orthonormal_and_span(A, U)
    cp.tk_destroy(ctx)
    with pytest.raises(cp.CpppError):
        cp.tk_init(X, dims, (5, 2, 2))   # R_0 = 5 > R_1 R_2 = 4 with s_0 > 128
