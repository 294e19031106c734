"""GPU parity: the CUDA path (through the C ABI) against the oracle on identical seeded inputs.

Tolerances (BASELINE.json north_star): MTTKRP, PP operators and PP updates within relative
Frobenius 1e-11 given identical factors; per-sweep fitness traces within 1e-8 over 20 sweeps
(phase schedule replayed, L12), applied while the relative residual ρ >= 1e-6 (L27).
"""
import numpy as np
import pytest

import oracle.cp_oracle as O
import synthgen as G
from trace_check import check, conditioning, golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1811_10573_b200.cppp as cp  # noqa: E402

TOL = 1e-11


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def problem(cfg_name, seed=0):
    cfg = G.CONFIGS[cfg_name]
    X = G.make_tensor(cfg, seed)
    A0 = G.initial_factors(cfg, seed)
    return cfg, X, A0


def random_problem(dims, K, seed):
    r = np.random.default_rng(seed)
    X = r.standard_normal(dims)
    A = [r.standard_normal((d, K)) for d in dims]
    return X, A


SMALL = ["C1", "C2mini", "C3mini", "C4mini", "C5mini"]
RAGGED = [((7, 9, 5), 3), ((6, 10, 12), 17), ((130, 4, 6), 5), ((8, 6, 4, 10), 7),
          ((3, 4, 2, 3, 2), 2), ((40, 36, 34), 128), ((34, 18, 10, 6), 100),
          # trailing extents that are multiples of 128: the one-load 4-D TMA path of the
          # m-contiguous GEMM (B = 1 and flattened B > 1)
          ((20, 16, 8), 12), ((6, 10, 256), 24), ((4, 128, 130), 20),
          # multiples of 16 only: the 4-D load for tiles inside one batch, 16-row boxes for the rest
          ((6, 10, 400), 16), ((3, 20, 48, 16), 8)]


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("simt", [False, True])
def test_mttkrp_dt_matches_oracle(name, simt):
    cfg, X, A0 = problem(name)
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K, flags=cp.FLAG_SIMT_TTM if simt else 0)
    cp.cp_set_factors(ctx, A0)
    M = cp.mttkrp_dt(ctx)
    for n in range(cfg.N):
        assert rel(M[n], O.mttkrp(X, A0, n)) < TOL, (name, n)


@pytest.mark.parametrize("dims,K", RAGGED)
def test_mttkrp_ragged_and_general_dims(dims, K):
    X, A = random_problem(dims, K, 1)
    ctx = cp.cp_init(X, len(dims), dims, K)
    cp.cp_set_factors(ctx, A)
    M = cp.mttkrp_dt(ctx)
    for n in range(len(dims)):
        assert rel(M[n], O.mttkrp(X, A, n)) < TOL, (dims, K, n)


@pytest.mark.parametrize("name", SMALL)
def test_pp_operators_and_singles_match_oracle(name):
    cfg, X, A0 = problem(name)
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    cp.cp_set_factors(ctx, A0)
    cp.pp_build_operators(ctx)
    ops = O.pp_operators(X, A0)
    for (i, j), ref in ops.items():
        assert rel(cp.pp_get_operator(ctx, i, j), ref) < TOL, (name, i, j)
    for n in range(cfg.N):
        assert rel(cp.pp_get_single(ctx, n), O.mttkrp(X, A0, n)) < TOL, (name, n)


@pytest.mark.parametrize("dims,K", RAGGED + [((7, 30, 64), 20), ((3, 64, 5, 48), 24),
                                            ((9, 400, 16), 8)])
def test_pp_operators_ragged(dims, K):
    # the last three contract a middle mode with R % 16 == 0: tiles over the flattened (b, r)
    X, A = random_problem(dims, K, 2)
    ctx = cp.cp_init(X, len(dims), dims, K)
    cp.cp_set_factors(ctx, A)
    cp.pp_build_operators(ctx)
    for (i, j), ref in O.pp_operators(X, A).items():
        assert rel(cp.pp_get_operator(ctx, i, j), ref) < TOL, (dims, K, i, j)


@pytest.mark.parametrize("flags", [0, cp.FLAG_NO_KRP])
@pytest.mark.parametrize("dims,K", [((6, 7, 8, 9), 12), ((5, 6, 4, 7, 3), 9), ((4, 5, 3, 4, 3, 4), 10),
                                    ((12, 10, 11, 9, 8), 33), ((4, 6, 4, 2, 6, 4), 10),
                                    ((6, 4, 2, 4, 6, 2, 4), 7), ((4, 4, 6, 4, 4, 6), 40)])
def test_pp_level2_from_x(dims, K, flags):
    """Order >= 4: the last level-1 node's only child {2, 3} comes straight from X in one
    Khatri-Rao GEMM when its two modes are neighbours; order >= 6 (even extents): the whole tree
    hangs from the neighbour pairs (0,1), (2,3), ... contracted from X (default) -- or Def. pptree
    with its level-1 nodes (FLAG_NO_KRP); both against the oracle's operators and single-mode
    MTTKRPs."""
    X, A = random_problem(dims, K, 41)
    ctx = cp.cp_init(X, len(dims), dims, K, flags=flags)
    cp.cp_set_factors(ctx, A)
    cp.pp_build_operators(ctx)
    for (i, j), ref in O.pp_operators(X, A).items():
        assert rel(cp.pp_get_operator(ctx, i, j), ref) < TOL, (dims, K, i, j)
    for n in range(len(dims)):
        assert rel(cp.pp_get_single(ctx, n), O.mttkrp(X, A, n)) < TOL, (dims, n)


@pytest.mark.parametrize("name", SMALL)
def test_pp_update_matches_oracle(name):
    cfg, X, Ap = problem(name)
    r = np.random.default_rng(3)
    dA = [0.01 * r.standard_normal(a.shape) for a in Ap]
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    cp.cp_set_factors(ctx, Ap)
    cp.pp_build_operators(ctx)
    ops = O.pp_operators(X, Ap)
    Mp = [O.pp_single(ops, Ap, n, cfg.N) for n in range(cfg.N)]
    # move the factors without dropping the operators: pp_update reads dA = A - A_p
    cp.cp_update_factors(ctx, [a + d for a, d in zip(Ap, dA)])
    for n in range(cfg.N):
        ref = O.pp_update(Mp[n], ops, dA, n)
        assert rel(cp.pp_update(ctx, n), ref) < TOL, (name, n)


@pytest.mark.parametrize("name,sweeps", [("C1", 20), ("C2mini", 20), ("C3mini", 20), ("C4mini", 20),
                                         ("C5mini", 20), ("LAPmini", 20)])
def test_sweep_trace_matches_oracle(name, sweeps):
    """Every sweep of the replayed 20-sweep trace (tests/trace_check.py): fitness (north_star
    1e-8), the unclamped r², Σ‖G‖, max ‖dA‖/‖A‖ and the final factors -- including the PP sweeps
    whose radicand is negative (fitness clamped)."""
    cfg, X, A0 = problem(name)
    A_or, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, sweeps)
    cond = golden(name, X, A0, cfg.eps_pp, tr, A_or)
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    cp.cp_set_factors(ctx, A0)
    infos = []
    for t in tr:
        cp.cp_set_phase_override(ctx, t["phase"])
        infos.append(cp.als_sweep(ctx, 0.0, cfg.eps_pp))
    check(tr, infos, cond, A_or, cp.cp_get_factors(ctx), tag=name)
    assert any(i["phase"] != "dt" for i in infos) or cfg.name in ("C4mini", "LAPmini")
    cp.cp_destroy(ctx)


def test_fitness_exact_matches_explicit_residual():
    """fitness_exact: one exact MTTKRP at the current factors (L17); after a PP sweep it differs
    from the sweep's approximate value and equals the oracle's explicit ‖X − [[A]]‖."""
    cfg, X, A0 = problem("C2mini")
    _, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, 20)
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    cp.cp_set_factors(ctx, A0)
    nx2 = float(np.sum(X * X))
    seen_pp = False
    for t in tr:
        cp.cp_set_phase_override(ctx, t["phase"])
        info = cp.als_sweep(ctx, 0.0, cfg.eps_pp)
        f, r2 = cp.fitness_exact(ctx)
        A = cp.cp_get_factors(ctx)
        explicit = float(np.sum((X - O.kruskal_full(A)) ** 2))
        assert abs(r2 - explicit) <= 1e-11 * nx2, (t["sweep"], r2, explicit)
        assert abs(f - (1 - np.sqrt(max(explicit, 0.0) / nx2))) < 1e-9
        if t["phase"] == "dt":
            assert info["approximate"] is False and abs(info["residual_sq"] - r2) <= 1e-11 * nx2
        else:
            assert info["approximate"] is True
            seen_pp = True
    assert seen_pp
    cp.cp_destroy(ctx)


def test_free_running_phase_machine_matches_oracle_schedule():
    cfg, X, A0 = problem("C1")
    _, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, 20)
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    cp.cp_set_factors(ctx, A0)
    for t in tr:
        info = cp.als_sweep(ctx, 0.0, cfg.eps_pp)
        if t["margin"] > 1e-6:
            assert info["phase"] == t["phase"]


def test_device_generator_matches_synthgen():
    for name in ["C1", "C2mini", "C5mini", "C4mini"]:
        cfg = G.CONFIGS[name]
        A = G.true_factors(cfg)
        Xh = G.make_tensor(cfg, A_true=A)
        Xd = torch.empty(cfg.numel, dtype=torch.float64, device="cuda")
        kind = {"none": 0, "abs": 1, "rel": 2}[cfg.noise_kind]
        cp.cppp_generate(Xd, cfg.dims, cfg.K, A, kind, cfg.noise)
        Xg = Xd.cpu().numpy().reshape(cfg.dims)
        assert np.max(np.abs(Xg - Xh)) <= 1e-13 * np.max(np.abs(Xh)), name


def test_error_paths():
    cfg, X, A0 = problem("C1")
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    with pytest.raises(cp.CpppError) as e:
        cp.als_sweep(ctx, 0.0, 0.1)
    assert e.value.status == -5
    cp.cp_set_factors(ctx, A0)
    with pytest.raises(cp.CpppError) as e:
        cp.pp_update(ctx, 0)
    assert e.value.status == -5
    with pytest.raises(cp.CpppError) as e:
        cp.pp_get_operator(ctx, 2, 1)
    assert e.value.status == -1
    with pytest.raises(cp.CpppError):
        cp.cp_init(X, 3, (40, 40, 40), 129)


def test_singular_gamma_uses_pseudo_inverse():
    """Duplicate factor columns make every Γ singular: both sides must take the eigen
    pseudo-inverse branch of L13 and agree on the minimum-norm solution."""
    cfg, X, A0 = problem("C1")
    A = [a.copy() for a in A0]
    for a in A:
        a[:, 1] = a[:, 0]
    st = O.State(X, A)
    st.dt_sweep()
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    cp.cp_set_factors(ctx, A)
    cp.cp_set_phase_override(ctx, "dt")
    cp.als_sweep(ctx, 0.0, cfg.eps_pp)
    got = cp.cp_get_factors(ctx)
    for n in range(cfg.N):
        assert rel(got[n], st.A[n]) < 1e-8, n


@pytest.mark.parametrize("unfused", [False, True])
@pytest.mark.parametrize("K", [5, 16, 30, 40])
def test_singular_gamma_each_factorization_kernel(K, unfused):
    """The same L13 branch on every factorization kernel: the fused small-mode kernel and (with
    FLAG_NO_FUSED_SOLVE) the one-warp kernel at K <= 8, 16 and 32 (K = 5, 16, 30), and the
    CTA-wide Cholesky chain (K = 40); duplicate columns make Γ singular, distinct ones keep it
    regular -- both sweeps against the oracle."""
    if unfused and K > 32:
        pytest.skip("K > 32 always takes the factorization chain")
    dims = (30, 28, 26, 24)   # the fused small-mode kernel runs for K <= 32
    X, _ = random_problem(dims, K, 21)
    r = np.random.default_rng(22)
    for dup in (False, True):
        A = [r.standard_normal((d, K)) for d in dims]
        if dup:
            for a in A:
                a[:, 1] = a[:, 0]
        st = O.State(X, [a.copy() for a in A])
        st.dt_sweep()
        ctx = cp.cp_init(X, 4, dims, K, flags=cp.FLAG_NO_FUSED_SOLVE if unfused else 0)
        cp.cp_set_factors(ctx, A)
        cp.cp_set_phase_override(ctx, "dt")
        cp.als_sweep(ctx, 0.0, 0.1)
        got = cp.cp_get_factors(ctx)
        for n in range(4):
            assert rel(got[n], st.A[n]) < 1e-8, (dup, n)


# fused small-mode solve (K <= 32, modes <= 64 rows): one launch per mode, the same IEEE
# operations in the same order as the factorization + row-solve + Gram chain
FUSED_CASES = [("C1", None), ("C3mini", None), ("C4mini", None), ("C5mini", None), ("LAPmini", None),
               (None, ((7, 9, 5), 3)), (None, ((40, 36, 34), 32)),
               (None, ((7, 9, 5, 4), 3)), (None, ((40, 36, 34, 2), 32)), (None, ((64, 6, 9, 5), 17)),
               (None, ((60, 62, 64, 3), 32)), (None, ((12, 3, 10, 4, 2), 8)), (None, ((20, 21, 22, 23), 16))]


@pytest.mark.parametrize("name,shape", FUSED_CASES)
def test_fused_small_mode_is_bit_identical(name, shape):
    """20 free-running sweeps (every phase: DT, PP build, PP) through the fused small-mode kernel
    and through the three-kernel chain give bit-identical sweep records and factors; the same
    run through als_run (the graph device loop) too."""
    if name is not None:
        cfg, X, A0 = problem(name)
        N, dims, K, epp = cfg.N, cfg.dims, cfg.K, cfg.eps_pp
    else:
        dims, K = shape
        X, _ = random_problem(dims, K, 31)
        r = np.random.default_rng(32)
        A0 = [r.random((d, K)) for d in dims]
        N, epp = len(dims), 0.5
    a = cp.cp_init(X, N, dims, K)
    b = cp.cp_init(X, N, dims, K, flags=cp.FLAG_NO_FUSED_SOLVE)
    c = cp.cp_init(X, N, dims, K)
    cp.cp_set_factors(a, A0)
    cp.cp_set_factors(b, A0)
    cp.cp_set_factors(c, A0)
    fa = [cp.als_sweep(a, 0.0, epp) for _ in range(20)]
    fb = [cp.als_sweep(b, 0.0, epp) for _ in range(20)]
    fc = cp.als_run(c, 0.0, epp, 20)
    assert {x["phase"] for x in fa} >= {"dt"}
    for x, y, z in zip(fa, fb, fc):
        for key in ("phase", "fitness", "residual_sq", "grad_norm_sum", "max_rel_dA"):
            assert x[key] == y[key] == z[key], (key, x, y, z)
    for x, y, z in zip(cp.cp_get_factors(a), cp.cp_get_factors(b), cp.cp_get_factors(c)):
        assert np.array_equal(x, y) and np.array_equal(x, z)


@pytest.mark.parametrize("dims,K", [((160, 150, 140), 128), ((30, 28, 26, 24), 64)])
def test_sweeps_large_rank(dims, K):
    X, _ = random_problem(dims, K, 5)
    r = np.random.default_rng(6)
    A0 = [r.random((d, K)) for d in dims]
    A_or, tr = O.pp_cp_als(X, A0, 0.0, 0.5, 6)
    cond = conditioning(X, A0, 0.5, 6, tr, A_or)
    ctx = cp.cp_init(X, len(dims), dims, K)
    cp.cp_set_factors(ctx, A0)
    infos = []
    for t in tr:
        cp.cp_set_phase_override(ctx, t["phase"])
        infos.append(cp.als_sweep(ctx, 0.0, 0.5))
    check(tr, infos, cond, A_or, cp.cp_get_factors(ctx), tag=str(dims))


# ---- scheduling paths of the GEMM / TTV kernels: each shape is chosen to hit one
# ---- path; the values must not depend on the path (parity with the oracle either way)
@pytest.mark.parametrize("krp", [True, False])
@pytest.mark.parametrize("dims,K", [((6, 7, 40, 42), 30), ((8, 6, 5, 4, 6, 5), 16),
                                    ((12, 10, 9, 11, 8), 33)])
def test_multimode_first_level_matches_single_mode_chain(dims, K, krp):
    """Order >= 4: each DT half is contracted from X in one Khatri-Rao GEMM (default) or by a
    single-mode TTM followed by multi-TTVs (CPPP_FLAG_NO_KRP); both equal the oracle MTTKRP."""
    X, A = random_problem(dims, K, 11)
    ctx = cp.cp_init(X, len(dims), dims, K, flags=0 if krp else cp.FLAG_NO_KRP)
    cp.cp_set_factors(ctx, A)
    M = cp.mttkrp_dt(ctx)
    for n in range(len(dims)):
        assert rel(M[n], O.mttkrp(X, A, n)) < TOL, (dims, K, n, krp)


@pytest.mark.parametrize("dims,K", [
    ((120, 160, 64), 24),      # 19200 / 128 = 150 output tiles: half-empty last wave -> k halves
    ((100, 190, 64), 8),       # 148 tiles + 1 -> tail split with NT = 1
    ((4, 4, 60, 64), 16),      # multi-mode GEMM, 1 tile, S = 3840: every tile in k chunks
    ((6, 6, 50, 50), 100),     # 1 tile of 36 rows, S = 2500, NT = 13
    ((44, 44, 40, 30), 20),    # X_(01) GEMM: 10 tiles (ragged), 121 k slices -> stream-K ranges
])
def test_ttm_split_units_match_oracle(dims, K):
    X, A = random_problem(dims, K, 12)
    ctx = cp.cp_init(X, len(dims), dims, K)
    cp.cp_set_factors(ctx, A)
    M = cp.mttkrp_dt(ctx)
    for n in range(len(dims)):
        assert rel(M[n], O.mttkrp(X, A, n)) < TOL, (dims, K, n)
    # and the same factors twice: the split tickets must be left reset by the first run
    M2 = cp.mttkrp_dt(ctx)
    for n in range(len(dims)):
        assert np.array_equal(M[n], M2[n]), n


@pytest.mark.parametrize("dims,K", [((300, 64, 64), 2), ((64, 256, 3), 9), ((17, 33, 400), 11)])
def test_ttv_cluster_split_matches_oracle(dims, K):
    """Small level-2 outputs split the contracted range over a (1, xs, 1) cluster reduced over
    DSMEM (odd K exercises the 8-byte path)."""
    X, A = random_problem(dims, K, 13)
    ctx = cp.cp_init(X, len(dims), dims, K)
    cp.cp_set_factors(ctx, A)
    M = cp.mttkrp_dt(ctx)
    for n in range(len(dims)):
        assert rel(M[n], O.mttkrp(X, A, n)) < TOL, (dims, K, n)


def test_load_tensor_replaces_the_tensor():
    """cp_load_tensor: a second tensor of the same shape in an existing context (host and device
    sources) gives the oracle's MTTKRP and sweep trace for that tensor; the graphs captured for
    the first tensor keep working."""
    cfg = G.CONFIGS["C2mini"]
    X1, A0 = G.make_tensor(cfg, 0), G.initial_factors(cfg, 0)
    X2 = G.make_tensor(cfg, 1)
    ctx = cp.cp_init(X1, cfg.N, cfg.dims, cfg.K)
    cp.cp_set_factors(ctx, A0)
    for _ in range(4):
        cp.als_sweep(ctx, 0.0, cfg.eps_pp)
    for src in (X2, torch.from_numpy(X2.ravel().copy()).cuda()):
        cp.cp_load_tensor(ctx, src)
        cp.cp_set_factors(ctx, A0)
        M = cp.mttkrp_dt(ctx)
        for n in range(cfg.N):
            assert rel(M[n], O.mttkrp(X2, A0, n)) < TOL, n
        cp.cp_set_factors(ctx, A0)
        A_or, tr = O.pp_cp_als(X2, A0, 0.0, cfg.eps_pp, 8)
        cond = conditioning(X2, A0, cfg.eps_pp, 8, tr, A_or)
        infos = []
        for t in tr:
            cp.cp_set_phase_override(ctx, t["phase"])
            infos.append(cp.als_sweep(ctx, 0.0, cfg.eps_pp))
        check(tr, infos, cond, A_or, cp.cp_get_factors(ctx), tag="load_tensor")
    b = cp.cp_init(torch.from_numpy(X1.ravel().copy()).cuda(), cfg.N, cfg.dims, cfg.K,
                   flags=cp.FLAG_BORROW_TENSOR)
    with pytest.raises(cp.CpppError):
        cp.cp_load_tensor(b, X2)


@pytest.mark.parametrize("name", ["C1", "C2mini"])
def test_order3_overlapped_schedule_is_bit_identical(name):
    """Order 3: the second first-level TTM runs beside mode 1's work (default) or after it
    (CPPP_FLAG_NO_OVERLAP); same contractions in the same order -> identical sweeps."""
    cfg, X, A0 = problem(name)
    a = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    b = cp.cp_init(X, cfg.N, cfg.dims, cfg.K, flags=cp.FLAG_NO_OVERLAP)
    for c in (a, b):
        cp.cp_set_factors(c, A0)
    for _ in range(12):
        ia, ib = cp.als_sweep(a, 0.0, cfg.eps_pp), cp.als_sweep(b, 0.0, cfg.eps_pp)
        assert ia["fitness"] == ib["fitness"] and ia["phase"] == ib["phase"], (ia, ib)
    for x, y in zip(cp.cp_get_factors(a), cp.cp_get_factors(b)):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("name", ["C1", "C2mini", "C4mini"])
def test_als_run_device_loop_matches_host_loop(name):
    """als_run (one launch: device-side Alg. 3 decisions, WHILE over a SWITCH of the phase
    graphs) gives bit-identical sweeps to the same number of als_sweep calls, and follows the
    oracle's free-running schedule."""
    cfg, X, A0 = problem(name)
    a = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    b = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    for rep in range(2):   # the second run replays the instantiated run graph
        cp.cp_set_factors(a, A0)
        cp.cp_set_factors(b, A0)
        host = [cp.als_sweep(a, 0.0, cfg.eps_pp) for _ in range(20)]
        dev = cp.als_run(b, 0.0, cfg.eps_pp, 20)
        assert len(dev) == 20
        # one launch for the whole run: the device time is shared evenly (the host loop would
        # report per-sweep times) -- i.e. the device loop ran, not the fallback
        assert len({d["seconds"] for d in dev}) == 1, cp.lib().cp_last_error(b.h)
        for h, d in zip(host, dev):
            for key in ("sweep", "phase", "next_phase", "restarts", "converged"):
                assert h[key] == d[key], (rep, key, h, d)
            for key in ("fitness", "residual_sq", "grad_norm_sum", "max_rel_dA"):
                assert h[key] == d[key], (rep, key, h, d)
        for x, y in zip(cp.cp_get_factors(a), cp.cp_get_factors(b)):
            assert np.array_equal(x, y)
    _, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, 20)
    margin_ok = all(t["margin"] > 1e-6 for t in tr)
    if margin_ok:
        assert [t["phase"] for t in tr] == [d["phase"] for d in dev]
    # a stop on the gradient norm ends the run early, like als_sweep's converged flag
    cp.cp_set_factors(b, A0)
    big = cp.als_run(b, 1e300, cfg.eps_pp, 20)
    assert len(big) == 1 and big[0]["converged"] == 1


def moved_factors(Ap, t, seed):
    """A = A_p + dA with ||da_k|| = t ||a_p,k|| per column."""
    r = np.random.default_rng(seed)
    out = []
    for a in Ap:
        d = r.standard_normal(a.shape)
        d *= t * np.linalg.norm(a, axis=0) / np.linalg.norm(d, axis=0)
        out.append(a + d)
    return out


@pytest.mark.parametrize("name", SMALL + ["LAPmini"])
@pytest.mark.parametrize("t", [1e-1, 1e-2])
def test_pp_error_monitor_matches_oracle(name, t):
    """pp_error against oracle.pp_error_monitor at the same (A, A_p): ε and the
    certificate to 1e-12 relative; err = ||M~ - M|| / ||M|| is a difference of two FP64
    results of size ~t²||M||, so it carries their rounding (~1e-15 ||M||) amplified by 1/t²:
    1e-8 relative plus 1e-13 absolute."""
    cfg, X, Ap = problem(name)
    A = moved_factors(Ap, t, 5)
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    cp.cp_set_factors(ctx, Ap)
    cp.pp_build_operators(ctx)
    cp.cp_update_factors(ctx, A)
    err, eps, bound = cp.pp_error(ctx)
    e_ref, eps_ref, b_ref = O.pp_error_monitor(X, A, Ap)
    assert np.allclose(eps, eps_ref, rtol=1e-12, atol=0)
    assert np.allclose(bound, b_ref, rtol=1e-12, atol=0)
    assert np.all(np.abs(err - e_ref) <= 1e-8 * e_ref + 1e-13), (err, e_ref)
    assert np.all(err <= bound * (1 + 1e-9))
    cp.cp_destroy(ctx)


def test_pp_error_quadratic_and_run_unchanged():
    """Device monitor: err(t/10) ≈ err(t)/100, and calling it between sweeps leaves a
    CP-ALS-PP run bit-identical."""
    cfg, X, Ap = problem("C3mini")
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    e = []
    for t in (1e-2, 1e-3):
        cp.cp_set_factors(ctx, Ap)
        cp.pp_build_operators(ctx)
        cp.cp_update_factors(ctx, moved_factors(Ap, t, 6))
        e.append(cp.pp_error(ctx)[0])
    assert np.all(np.abs(e[0] / e[1] / 100 - 1) < 0.05)
    cp.cp_destroy(ctx)
    cfg, X, A0 = problem("C2mini")
    _, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, 12)
    a, b = (cp.cp_init(X, cfg.N, cfg.dims, cfg.K) for _ in range(2))
    for c in (a, b):
        cp.cp_set_factors(c, A0)
    seen = 0
    for t in tr:
        for c in (a, b):
            cp.cp_set_phase_override(c, t["phase"])
        ia, ib = cp.als_sweep(a, 0.0, cfg.eps_pp), cp.als_sweep(b, 0.0, cfg.eps_pp)
        assert ia["fitness"] == ib["fitness"], (t, ia, ib)
        if t["phase"] != "dt":
            err, eps, bound = cp.pp_error(b)
            assert np.all(err <= bound * (1 + 1e-9))
            seen += 1
    assert seen > 0
    assert all(np.array_equal(x, y) for x, y in zip(cp.cp_get_factors(a), cp.cp_get_factors(b)))
    cp.cp_destroy(a)
    cp.cp_destroy(b)


@pytest.mark.parametrize("name", ["C1", "C2mini"])
def test_order3_operator_reuse_is_bit_identical(name):
    """Order 3: the PP build takes M_p^(1,2) from the preceding regular sweep's X ×_0 A^(0)
    (same kernel, same shape).  Replayed schedule, a forced second build in a row (recomputed),
    and als_run all match a context that recomputes it (CPPP_FLAG_NO_OP_REUSE) bit for bit."""
    cfg, X, A0 = problem(name)
    _, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, 20)
    assert any(t["phase"] == "pp-build" for t in tr)
    a = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    b = cp.cp_init(X, cfg.N, cfg.dims, cfg.K, flags=cp.FLAG_NO_OP_REUSE)
    for c in (a, b):
        cp.cp_set_factors(c, A0)
    sched = [t["phase"] for t in tr] + ["pp-build", "pp-build", "pp-approx", "dt", "pp-build"]
    for ph in sched:
        ia, ib = [], []
        for c, out in ((a, ia), (b, ib)):
            cp.cp_set_phase_override(c, ph)
            out.append(cp.als_sweep(c, 0.0, cfg.eps_pp))
        assert ia[0]["fitness"] == ib[0]["fitness"], (ph, ia, ib)
    for n in range(cfg.N):
        for i in range(n + 1, cfg.N):
            assert np.array_equal(cp.pp_get_operator(a, n, i), cp.pp_get_operator(b, n, i))
    for c in (a, b):
        cp.cp_set_phase_override(c, cp.PHASE_AUTO)
        cp.cp_set_factors(c, A0)
    ra = cp.als_run(a, 0.0, cfg.eps_pp, 20)
    rb = cp.als_run(b, 0.0, cfg.eps_pp, 20)
    assert [r["fitness"] for r in ra] == [r["fitness"] for r in rb]
    assert [r["phase"] for r in ra] == [t["phase"] for t in tr]
    cp.cp_destroy(a)
    cp.cp_destroy(b)


@pytest.mark.parametrize("dims,K", [((6, 5, 7), 1),                      # rank 1
                                    ((2, 3, 2, 2, 3, 2, 2, 3), 3),       # maximum order N = 8
                                    ((5, 1, 4), 2), ((1, 6, 1, 5), 2)])  # unit extents
def test_edge_shapes(dims, K):
    """Degenerate and extreme shapes: MTTKRP, every PP operator and update, and 6 replayed sweeps
    against the oracle."""
    X, A = random_problem(dims, K, 11)
    A = [np.abs(a) + 0.1 for a in A]
    N = len(dims)
    ctx = cp.cp_init(X, N, dims, K)
    cp.cp_set_factors(ctx, A)
    M = cp.mttkrp_dt(ctx)
    for n in range(N):
        assert rel(M[n], O.mttkrp(X, A, n)) < TOL, n
    cp.pp_build_operators(ctx)
    ops = O.pp_operators(X, A)
    for (i, j), ref in ops.items():
        assert rel(cp.pp_get_operator(ctx, i, j), ref) < TOL, (i, j)
    r = np.random.default_rng(2)
    dA = [0.01 * r.standard_normal(a.shape) for a in A]
    cp.cp_update_factors(ctx, [a + d for a, d in zip(A, dA)])
    Mp = [O.pp_single(ops, A, n, N) for n in range(N)]
    for n in range(N):
        assert rel(cp.pp_update(ctx, n), O.pp_update(Mp[n], ops, dA, n)) < TOL, n
    A_or, tr = O.pp_cp_als(X, A, 0.0, 0.1, 6)
    cond = conditioning(X, A, 0.1, 6, tr, A_or)
    cp.cp_set_factors(ctx, A)
    infos = []
    for t in tr:
        cp.cp_set_phase_override(ctx, t["phase"])
        infos.append(cp.als_sweep(ctx, 0.0, 0.1))
    check(tr, infos, cond, A_or, cp.cp_get_factors(ctx), tag=str(dims))
    cp.cp_destroy(ctx)


def test_empty_and_oversized_inputs_rejected():
    X = np.zeros((4, 0, 3))
    with pytest.raises(cp.CpppError):
        cp.cp_init(X, 3, (4, 0, 3), 2)
    X = np.zeros((2,) * 9)
    with pytest.raises(cp.CpppError):
        cp.cp_init(X, 9, (2,) * 9, 2)


@pytest.mark.parametrize("name", ["C1", "C2mini", "C3mini", "C4mini", "C5mini"])
def test_pp_second_order_matches_oracle(name):
    """pp_second_order (f3): T2^(n) = Σ_{i<j≠n} M_p^(i,j,n) ×_i dA ×_j dA against the
    oracle's second_order_term; for N = 3 M~ + T2 is the exact MTTKRP (the expansion ends there)."""
    cfg, X, Ap = problem(name)
    A = moved_factors(Ap, 0.05, 9)
    dA = [a - ap for a, ap in zip(A, Ap)]
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    cp.cp_set_factors(ctx, Ap)
    cp.pp_build_operators(ctx)
    cp.cp_update_factors(ctx, A)
    T2 = cp.pp_second_order(ctx)
    for n in range(cfg.N):
        ref = O.second_order_term(X, Ap, dA, n)
        assert rel(T2[n], ref) < 1e-11, (name, n)
        if cfg.N == 3:
            Mt = cp.pp_update(ctx, n)
            assert rel(Mt + T2[n], O.mttkrp(X, A, n)) < 1e-11, (name, n)
    # the state is untouched: a PP sweep afterwards equals one on a fresh context
    b = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    cp.cp_set_factors(b, Ap)
    cp.pp_build_operators(b)
    cp.cp_update_factors(b, A)
    for c in (ctx, b):
        cp.cp_set_phase_override(c, "pp-approx")
    ia, ib = cp.als_sweep(ctx, 0.0, 1.0), cp.als_sweep(b, 0.0, 1.0)
    assert ia["residual_sq"] == ib["residual_sq"]
    cp.cp_destroy(ctx)
    cp.cp_destroy(b)


def monitor_bound(A, Ap, Mt_colnorms, normX):
    """max_{n,k} ||X||_F Σ_{S ⊆ others, |S|>=2} Π_{i∈S}||da_k^(i)|| Π_{j∉S}||a_p,k^(j)|| / ||m~_k^(n)||
    (the certificate of oracle.pp_error_monitor with ||m~|| in the denominator)."""
    from itertools import combinations as comb
    N, K = len(A), A[0].shape[1]
    best = 0.0
    for n in range(N):
        others = [i for i in range(N) if i != n]
        for k in range(K):
            d = {i: np.linalg.norm(A[i][:, k] - Ap[i][:, k]) for i in others}
            p = {i: np.linalg.norm(Ap[i][:, k]) for i in others}
            tot = sum(np.prod([d[i] if i in S else p[i] for i in others])
                      for size in range(2, len(others) + 1) for S in comb(others, size))
            best = max(best, normX * tot / Mt_colnorms[n][k])
    return best


@pytest.mark.parametrize("name", ["C1", "C3mini"])
def test_pp_policy_bound_monitor_and_switch(name):
    """CPPP_POLICY_BOUND (f3 switching policy): the monitor value after a PP sweep equals the
    certificate from the oracle's own sweep (||m~|| from its M~); with tol = 1e300 the run is
    bit-identical to the default policy; with a tol below every monitor value no pp-approx sweep
    is left (every PP phase ends after its build sweep, a regular sweep follows)."""
    cfg, X, Ap = problem(name)
    A = moved_factors(Ap, 0.02, 10)
    st = O.State(X, Ap)
    st.pp_build()
    st.A = [a.copy() for a in A]
    st.S = [O.gram(a) for a in st.A]
    st.dA = [a - ap for a, ap in zip(A, Ap)]
    norms = []
    for n in range(cfg.N):
        M = O.pp_update(st.Mp[n], st.ops, st.dA, n)
        norms.append(np.linalg.norm(M, axis=0))
        st._update_mode(n, M, st.A_p[n])
    want = monitor_bound(st.A, st.A_p, norms, np.sqrt(st.normX_sq))
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    cp.cp_set_pp_policy(ctx, cp.POLICY_BOUND, 1e300)
    cp.cp_set_factors(ctx, Ap)
    cp.pp_build_operators(ctx)
    cp.cp_update_factors(ctx, A)
    cp.cp_set_phase_override(ctx, "pp-approx")
    info = cp.als_sweep(ctx, 0.0, cfg.eps_pp)
    assert abs(info["pp_bound"] - want) <= 1e-9 * want, (info["pp_bound"], want)
    cp.cp_destroy(ctx)
    # whole runs: default vs tol = 1e300 (identical) vs a tiny tol (no pp-approx left)
    runs = {}
    for key, pol, tol in (("default", cp.POLICY_EPS_PP, 0.0), ("loose", cp.POLICY_BOUND, 1e300),
                          ("tight", cp.POLICY_BOUND, 1e-300)):
        c = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
        cp.cp_set_pp_policy(c, pol, tol)
        cp.cp_set_factors(c, Ap)
        runs[key] = (cp.als_run(c, 0.0, cfg.eps_pp, 20),
                     [cp.als_sweep(c, 0.0, cfg.eps_pp) for _ in range(0)])
        cp.cp_set_factors(c, Ap)
        host = [cp.als_sweep(c, 0.0, cfg.eps_pp) for _ in range(20)]
        # the device loop (als_run) and the host loop take the same decisions
        assert [h["phase"] for h in host] == [d["phase"] for d in runs[key][0]], key
        assert [h["residual_sq"] for h in host] == [d["residual_sq"] for d in runs[key][0]], key
        cp.cp_destroy(c)
    dflt, loose, tight = (runs[k][0] for k in ("default", "loose", "tight"))
    assert [d["residual_sq"] for d in dflt] == [d["residual_sq"] for d in loose]
    assert any(d["phase"] == "pp-approx" for d in dflt)
    assert not any(d["phase"] == "pp-approx" for d in tight)
    assert any(d["phase"] == "pp-build" for d in tight)
    ph = [d["phase"] for d in tight]
    assert all(b == "dt" for a, b in zip(ph, ph[1:]) if a == "pp-build")
    assert all(np.isnan(d["pp_bound"]) for d in dflt)


@pytest.mark.parametrize("dims,K", [((6, 4, 10, 128), 16), ((4, 6, 8, 256), 40), ((2, 130, 4, 128), 8),
                                    ((8, 8, 6, 384), 100), ((4, 4, 4, 128), 1)])
def test_fused_level1_build_matches_oracle(dims, K):
    """Order 4 with s_4 % 128 == 0: the operators come from three GEMMs whose
    epilogues contract each level-1 tile into two leaves (no level-1 node in memory).  Every
    operator and M_p^(n) against the oracle, and the plain Def. pptree build (NO_FUSED_TTV)."""
    X, A = random_problem(dims, K, 14)
    ops = O.pp_operators(X, A)
    res = []
    for flags in (0, cp.FLAG_NO_FUSED_TTV):
        ctx = cp.cp_init(X, 4, dims, K, flags=flags)
        cp.cp_set_factors(ctx, A)
        cp.pp_build_operators(ctx)
        got = {(i, j): cp.pp_get_operator(ctx, i, j) for (i, j) in ops}
        for (i, j), ref in ops.items():
            assert rel(got[(i, j)], ref) < TOL, (dims, K, flags, i, j)
        for n in range(4):
            assert rel(cp.pp_get_single(ctx, n), O.mttkrp(X, A, n)) < TOL, (dims, K, flags, n)
        res.append(got)
        cp.cp_destroy(ctx)


@pytest.mark.parametrize("dims,K", [((25, 25, 25, 25), 2), ((31, 17, 9), 5), ((5, 3, 7, 9, 11, 3), 16),
                                    ((9, 9, 9, 9, 9, 9), 1), ((3, 101, 7), 8),
                                    ((13, 97, 23), 4), ((7, 1031, 3), 2), ((3, 5, 2053), 3)])
def test_skinny_odd_extent_contractions(dims, K):
    """Odd extents (no 16-byte TMA strides: the compact Laplacian's s = 25) with K <= 16:
    the bandwidth-shaped kernels (bulk-copied chunks of rows or of r blocks, ragged last chunks by
    plain loads; thread per (b, r) for short m-contiguous rows, shared-memory rows or warp per row
    for the natural unfolding) -- MTTKRP, every operator and a PP update."""
    X, A = random_problem(dims, K, 15)
    N = len(dims)
    ctx = cp.cp_init(X, N, dims, K)
    cp.cp_set_factors(ctx, A)
    M = cp.mttkrp_dt(ctx)
    for n in range(N):
        assert rel(M[n], O.mttkrp(X, A, n)) < TOL, (dims, K, n)
    cp.pp_build_operators(ctx)
    ops = O.pp_operators(X, A)
    for (i, j), ref in ops.items():
        assert rel(cp.pp_get_operator(ctx, i, j), ref) < TOL, (dims, K, i, j)
    r = np.random.default_rng(16)
    dA = [0.01 * r.standard_normal(a.shape) for a in A]
    cp.cp_update_factors(ctx, [a + d for a, d in zip(A, dA)])
    Mp = [O.pp_single(ops, A, n, N) for n in range(N)]
    for n in range(N):
        assert rel(cp.pp_update(ctx, n), O.pp_update(Mp[n], ops, dA, n)) < TOL, (dims, K, n)
    cp.cp_destroy(ctx)


@pytest.mark.parametrize("K", [10, 40])
def test_pinv_rel_tol_option(K):
    """cppp_opts.pinv_rel_tol (L13's τ): τ = 0.05 sends ill-conditioned Γ down the
    eigen pseudo-inverse branch on both sides (one-warp kernel at K = 10, the CTA kernel at 40);
    three replayed sweeps against the oracle run with the same τ."""
    dims = (30, 28, 26)
    X, _ = random_problem(dims, K, 31)
    r = np.random.default_rng(32)
    A0 = [r.random((d, K)) for d in dims]
    for a in A0:   # two nearly parallel columns: Γ's pivot ratio ~1e-4, well below τ
        a[:, 1] = a[:, 0] + 1e-2 * r.standard_normal(a.shape[0])
    tau = 0.05
    A_or, tr = O.pp_cp_als(X, A0, 0.0, 0.1, 3, phase_override=["dt"] * 3, tau=tau)
    st = O.State(X, A0, tau)
    assert not all(O.cholesky_pivots(O.gamma(st.S, n), tau)[1] for n in range(3))
    ctx = cp.cp_init(X, 3, dims, K, pinv_rel_tol=tau)
    cp.cp_set_factors(ctx, A0)
    for t in tr:
        cp.cp_set_phase_override(ctx, "dt")
        info = cp.als_sweep(ctx, 0.0, 0.1)
        assert abs(info["residual_sq"] - t["residual_sq"]) <= 1e-9 * t["normX_sq"], (t, info)
    for a, b in zip(cp.cp_get_factors(ctx), A_or):
        assert rel(a, b) < 1e-8
    with pytest.raises(cp.CpppError):
        cp.cp_init(X, 3, dims, K, pinv_rel_tol=1.5)
    cp.cp_destroy(ctx)


def test_fused_build_inside_sweeps_and_graphs():
    """An order-4 problem whose PP builds take the fused level-1 GEMMs (s_4 = 128): the 20-sweep
    trace replayed through als_sweep (eager first uses, then captured phase graphs) against the
    oracle, and als_run (one device launch, the fused build inside the SWITCH body) bit-identical
    to the host loop and following the oracle's free-running schedule."""
    import synthgen as Gs
    r = np.random.default_rng(41)
    dims, K = (6, 8, 6, 128), 16
    B = [r.random((d, K)) for d in dims]
    X = np.ascontiguousarray(Gs.kruskal_slab(B) + 0.01 * r.standard_normal(dims))
    A0 = [r.random((d, K)) for d in dims]
    A_or, tr = O.pp_cp_als(X, A0, 0.0, 0.1, 20)
    assert sum(t["phase"] == "pp-build" for t in tr) >= 2
    cond = conditioning(X, A0, 0.1, 20, tr, A_or)
    ctx = cp.cp_init(X, 4, dims, K)
    cp.cp_set_factors(ctx, A0)
    infos = []
    for t in tr:
        cp.cp_set_phase_override(ctx, t["phase"])
        infos.append(cp.als_sweep(ctx, 0.0, 0.1))
    check(tr, infos, cond, A_or, cp.cp_get_factors(ctx), tag="fused-build trace")
    cp.cp_set_phase_override(ctx, cp.PHASE_AUTO)
    b = cp.cp_init(X, 4, dims, K)
    for rep in range(2):
        cp.cp_set_factors(ctx, A0)
        cp.cp_set_factors(b, A0)
        host = [cp.als_sweep(ctx, 0.0, 0.1) for _ in range(20)]
        dev = cp.als_run(b, 0.0, 0.1, 20)
        assert len({d["seconds"] for d in dev}) == 1
        assert [h["residual_sq"] for h in host] == [d["residual_sq"] for d in dev], rep
    if all(t["margin"] > 1e-6 for t in tr):
        assert [d["phase"] for d in dev] == [t["phase"] for t in tr]
    cp.cp_destroy(ctx)
    cp.cp_destroy(b)


def test_fused_build_uneven_x_l_chunks():
    """The fused build cuts the loop mode's range into chunks (one partial each); with 6 values and
    a wish for 4 chunks (300 units of the other modes) the chunks are 2, 2, 2 -- none empty (a
    fourth, empty chunk would leave its partial unwritten)."""
    dims, K = (2, 6, 300, 128), 4
    X, A = random_problem(dims, K, 17)
    ctx = cp.cp_init(X, 4, dims, K)
    cp.cp_set_factors(ctx, A)
    cp.pp_build_operators(ctx)
    for (i, j), ref in O.pp_operators(X, A).items():
        assert rel(cp.pp_get_operator(ctx, i, j), ref) < TOL, (i, j)
    cp.cp_destroy(ctx)


_BULK_AB = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1811_10573_b200.cppp as cp
r = np.random.default_rng(41)
dims, K = {dims!r}, {K}
X = r.standard_normal(dims)
A = [r.standard_normal((d, K)) for d in dims]
ctx = cp.cp_init(X, len(dims), dims, K)
cp.cp_set_factors(ctx, A)
M = list(cp.mttkrp_dt(ctx))
cp.pp_build_operators(ctx)
N = len(dims)
M += [cp.pp_get_operator(ctx, i, j) for i in range(N) for j in range(i + 1, N)]
M += [cp.pp_get_single(ctx, n) for n in range(N)]
np.savez({out!r}, *M)
"""


@pytest.mark.parametrize("env,dims,K", [("CPPP_NO_SKINNY_BULK", (25, 25, 25, 25), 2),
                                         ("CPPP_NO_SKINNY_BULK", (13, 97, 23), 4),
                                         ("CPPP_NO_SKINNY_BULK", (7, 1031, 3), 2),
                                         ("CPPP_NO_TTV_PIPE", (40, 64, 50), 24),
                                         ("CPPP_NO_TTV_PIPE", (72, 130, 66, 4), 20),
                                         ("CPPP_NO_TTV_PIPE", (9, 9, 9, 9, 9, 9), 2),
                                         ("CPPP_NO_TTV_PIPE", (12, 10, 9, 11, 8, 7), 16)])
def test_kernel_variants_bit_identical(env, dims, K, tmp_path):
    """Kernels that replace another one without changing any output's fma order:
    the bulk-copy skinny kernels (CPPP_NO_SKINNY_BULK: the register-load kernels) and the
    software-pipelined multi-TTVs (CPPP_NO_TTV_PIPE: ttv_kernel and the 256-thread batched
    kernel) -- the MTTKRPs, PP operators and single-mode operators of one process with the
    switch set and of one without are equal bit for bit."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for off in (False, True):
        out = str(tmp_path / f"m{int(off)}.npz")
        penv = dict(os.environ)
        penv.pop(env, None)
        if off:
            penv[env] = "1"
        code = _BULK_AB.format(root=root, dims=tuple(dims), K=K, out=out)
        subprocess.run([sys.executable, "-c", code], check=True, env=penv, timeout=300)
        with np.load(out) as z:
            outs.append([z[k] for k in sorted(z.files, key=lambda f: int(f.split("_")[1]))])
    assert len(outs[0]) == len(outs[1]) > len(dims)
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
