"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

C2, C3, C4: the whole tensor goes to the oracle (seconds), every MTTKRP, PP operator, M_p^(n) and
PP update is compared element by element, and each 20-sweep trace is replayed and compared on
every sweep.
C5 (32 GiB): too large for the oracle; the kernels are pinned by the Kruskal closed form on the
noise-free variant X = [[B]] generated on the device — for kept modes U,
    T_U(x_U, k) = Σ_r Π_{u∈U} B^(u)(x_u, r) · Π_{m∉U} (B^(m)ᵀ A^(m))(r, k)      (Def. 3.1 on P:343)
computed from the generating factors only (O(s² R K)), so no expected value comes from the GPU.
"""
import itertools

import numpy as np
import pytest

import oracle.cp_oracle as O
import synthgen as G
from trace_check import check, golden

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1811_10573_b200.cppp as cp  # noqa: E402

TOL = 1e-11


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def device_ctx(cfg, X=None, A_true=None, noise=True):
    """Context exactly as bench.py builds it: device-resident X (borrowed), library flags."""
    if X is None:
        Xd = torch.empty(cfg.numel, dtype=torch.float64, device="cuda")
        kind = {"none": 0, "abs": 1, "rel": 2}[cfg.noise_kind] if noise else 0
        cp.cppp_generate(Xd, cfg.dims, cfg.K, A_true, kind, cfg.noise)
    else:
        Xd = torch.from_numpy(np.ascontiguousarray(X).reshape(-1)).cuda()
    stream = torch.cuda.current_stream()
    ctx = cp.cp_init(Xd, cfg.N, cfg.dims, cfg.K, stream=stream,
                     flags=cp.FLAG_BORROW_TENSOR | cp.FLAG_PROFILE)
    return ctx, Xd


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_fullsize_kernels_match_oracle(name):
    cfg = G.CONFIGS[name]
    X = G.make_tensor(cfg)
    A0 = G.initial_factors(cfg)
    ctx, _ = device_ctx(cfg, X=X)
    cp.cp_set_factors(ctx, A0)
    M = cp.mttkrp_dt(ctx)
    for n in range(cfg.N):
        assert rel(M[n], O.mttkrp(X, A0, n)) < TOL, (name, n)
    cp.pp_build_operators(ctx)
    ops = O.pp_operators(X, A0)
    for (i, j), ref in ops.items():
        got = cp.pp_get_operator(ctx, i, j)
        assert rel(got, ref) < TOL, (name, i, j)
    Mp = [O.pp_single(ops, A0, n, cfg.N) for n in range(cfg.N)]
    for n in range(cfg.N):
        assert rel(cp.pp_get_single(ctx, n), Mp[n]) < TOL, (name, n)
    r = np.random.default_rng(11)
    dA = [0.01 * np.linalg.norm(a) / np.sqrt(a.size) * r.standard_normal(a.shape) for a in A0]
    cp.cp_update_factors(ctx, [a + d for a, d in zip(A0, dA)])
    for n in range(cfg.N):
        assert rel(cp.pp_update(ctx, n), O.pp_update(Mp[n], ops, dA, n)) < TOL, (name, n)


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_fullsize_trace_matches_oracle(name):
    """The full-size 20-sweep run in the bench's launch configuration, every sweep compared
    (tests/trace_check.py: fitness, unclamped r², Σ‖G‖, max ‖dA‖/‖A‖, final factors)."""
    cfg = G.CONFIGS[name]
    X = G.make_tensor(cfg)
    A0 = G.initial_factors(cfg)
    A_or, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, cfg.sweeps)
    cond = golden(name, X, A0, cfg.eps_pp, tr, A_or)
    ctx, _ = device_ctx(cfg, X=X)
    cp.cp_set_factors(ctx, A0)
    infos = []
    for t in tr:
        cp.cp_set_phase_override(ctx, t["phase"])
        infos.append(cp.als_sweep(ctx, 0.0, cfg.eps_pp))
    check(tr, infos, cond, A_or, cp.cp_get_factors(ctx), tag=name)
    cp.cp_destroy(ctx)


def kruskal_node(B, A, kept):
    W = np.ones((B[0].shape[1], A[0].shape[1]))
    for m in range(len(B)):
        if m not in kept:
            W = W * (B[m].T @ A[m])
    T = B[kept[0]]
    for u in kept[1:]:
        T = T[..., None, :] * B[u].reshape((1,) * (T.ndim - 1) + B[u].shape)
    return np.tensordot(T, W, axes=([T.ndim - 1], [0]))


def test_fullsize_C5_kernels_kruskal_closed_form():
    cfg = G.CONFIGS["C5"]
    if torch.cuda.get_device_properties(0).total_memory < 120 * 2**30:
        pytest.skip("needs ~85 GiB of device memory")
    B = G.true_factors(cfg)
    A0 = G.initial_factors(cfg)
    ctx, Xd = device_ctx(cfg, A_true=B, noise=False)
    cp.cp_set_factors(ctx, A0)
    M = cp.mttkrp_dt(ctx)
    for n in range(cfg.N):
        assert rel(M[n], kruskal_node(B, A0, [n])) < TOL, n
    cp.pp_build_operators(ctx)
    for i, j in itertools.combinations(range(cfg.N), 2):
        assert rel(cp.pp_get_operator(ctx, i, j), kruskal_node(B, A0, [i, j])) < TOL, (i, j)
    # PP update: exact expansion on a Kruskal tensor is also closed form —
    # M~^(n) = M_p^(n) + Σ_i T_{(i,n)}(A_p) ×_i dA^(i)
    r = np.random.default_rng(12)
    dA = [1e-3 * r.standard_normal(a.shape) for a in A0]
    cp.cp_update_factors(ctx, [a + d for a, d in zip(A0, dA)])
    for n in range(cfg.N):
        ref = kruskal_node(B, A0, [n]).copy()
        for i in range(cfg.N):
            if i == n:
                continue
            lo, hi = min(i, n), max(i, n)
            T = kruskal_node(B, A0, [lo, hi])
            ref += np.einsum("xyk,xk->yk", T, dA[i]) if i < n else np.einsum("yxk,xk->yk", T, dA[i])
        assert rel(cp.pp_update(ctx, n), ref) < TOL, n
    cp.cp_destroy(ctx)
    del Xd
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_fullsize_als_run_free_running_matches_oracle(name):
    """The benchmarked call itself: one als_run (20 sweeps, device-side Alg. 3 decisions, one graph
    launch) on the full-size tensor, free-running, against the oracle's free-running run: the same
    phase schedule wherever the oracle's ε_pp margins are clear of rounding, and then every sweep
    within the trace tolerances (tests/trace_check.py)."""
    cfg = G.CONFIGS[name]
    X = G.make_tensor(cfg)
    A0 = G.initial_factors(cfg)
    A_or, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, cfg.sweeps)
    ctx, _ = device_ctx(cfg, X=X)
    # (device_ctx profiles every kernel class, which sends als_run to the host loop: use a plain one)
    cp.cp_destroy(ctx)
    Xd = torch.from_numpy(np.ascontiguousarray(X).reshape(-1)).cuda()
    ctx = cp.cp_init(Xd, cfg.N, cfg.dims, cfg.K, stream=torch.cuda.current_stream(), flags=cp.FLAG_BORROW_TENSOR)
    cp.cp_set_factors(ctx, A0)
    cp.als_run(ctx, 0.0, cfg.eps_pp, cfg.sweeps)          # first run: captures the graphs
    cp.cp_set_factors(ctx, A0)
    infos = cp.als_run(ctx, 0.0, cfg.eps_pp, cfg.sweeps)
    assert len({i["seconds"] for i in infos}) == 1          # one device launch
    if all(t["margin"] > 1e-6 for t in tr):
        assert [i["phase"] for i in infos] == [t["phase"] for t in tr]
        check(tr, infos, golden(name, X, A0, cfg.eps_pp, tr, A_or), A_or, cp.cp_get_factors(ctx), tag=name)
    cp.cp_destroy(ctx)
