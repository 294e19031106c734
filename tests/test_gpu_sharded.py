"""The sharded (multi-GPU) code path of libcppp on ONE device: P contexts, one host thread each,
each holding a mode-0 slab, with the library's all-reduce routed through a host-side reducer
(cppp_opts.host_allreduce) instead of NCCL.  No kernel waits on another context, so this is safe
on a single GPU; it exercises every sharded branch of the engine (partial leaves, local solves of
the sharded mode, the PP-sweep exchange) against the unsharded oracle."""
import threading

import numpy as np
import pytest

import oracle.cp_oracle as O
import synthgen as G
from trace_check import check, golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1811_10573_b200.cppp as cp  # noqa: E402


class HostReducer:
    """Sum over P participants in rank order (deterministic)."""

    def __init__(self, P):
        self.P = P
        self.bar = threading.Barrier(P)
        self.slots = [None] * P
        self.total = None

    def fn(self, rank):
        def reduce(buf):
            self.slots[rank] = buf.copy()
            self.bar.wait()
            if rank == 0:
                tot = self.slots[0].copy()
                for r in range(1, self.P):
                    tot += self.slots[r]
                self.total = tot
            self.bar.wait()
            buf[:] = self.total
            self.bar.wait()
        return reduce


def slab(s0, rank, world):
    return rank * s0 // world, (rank + 1) * s0 // world


def run_sharded(P, X, dims, K, body, q=0):
    """Run body(rank, ctx, lo, hi) on P threads with contexts sharded along mode q; returns
    per-rank results."""
    red = HostReducer(P)
    out = [None] * P
    err = [None] * P

    def work(rank):
        try:
            lo, hi = slab(dims[q], rank, P)
            Xs = np.ascontiguousarray(np.take(X, np.arange(lo, hi), axis=q))
            ctx = cp.cp_init(Xs, len(dims), dims, K, shard_offset=lo, shard_extent=hi - lo, rank=rank,
                             world=P, torch_workspace=False, host_allreduce=red.fn(rank), shard_mode=q)
            out[rank] = body(rank, ctx, lo, hi)
            cp.cp_destroy(ctx)
        except Exception as e:  # noqa: BLE001
            err[rank] = e
            try:
                red.bar.abort()
            except Exception:
                pass

    ths = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    return out


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("name", ["C1", "C3mini", "C5mini"])
def test_sharded_kernels_match_oracle(P, name):
    cfg = G.CONFIGS[name]
    X = G.make_tensor(cfg)
    A0 = G.initial_factors(cfg)
    r = np.random.default_rng(4)
    dA = [0.01 * r.standard_normal(a.shape) for a in A0]

    def body(rank, ctx, lo, hi):
        cp.cp_set_factors(ctx, A0)
        M = cp.mttkrp_dt(ctx)
        cp.pp_build_operators(ctx)
        ops = {(i, j): cp.pp_get_operator(ctx, i, j) for i in range(cfg.N) for j in range(i + 1, cfg.N)}
        singles = [cp.pp_get_single(ctx, n) for n in range(cfg.N)]
        cp.cp_update_factors(ctx, [a + d for a, d in zip(A0, dA)])
        upd = [cp.pp_update(ctx, n) for n in range(cfg.N)]
        return M, ops, singles, upd

    res = run_sharded(P, X, cfg.dims, cfg.K, body)
    ops_ref = O.pp_operators(X, A0)
    Mp_ref = [O.pp_single(ops_ref, A0, n, cfg.N) for n in range(cfg.N)]
    for rank, (M, ops, singles, upd) in enumerate(res):
        lo, hi = slab(cfg.s, rank, P)
        for n in range(cfg.N):
            ref = O.mttkrp(X, A0, n)
            ref = ref[lo:hi] if n == 0 else ref
            assert rel(M[n], ref) < 1e-11, (rank, n)
            sref = Mp_ref[n][lo:hi] if n == 0 else Mp_ref[n]
            assert rel(singles[n], sref) < 1e-11, (rank, n)
            uref = O.pp_update(Mp_ref[n], ops_ref, dA, n)
            uref = uref[lo:hi] if n == 0 else uref
            assert rel(upd[n], uref) < 1e-11, (rank, n)
        for (i, j), ref in ops_ref.items():
            ref = ref[lo:hi] if i == 0 else ref
            assert rel(ops[(i, j)], ref) < 1e-11, (rank, i, j)


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("name", ["C1", "C3mini", "C5mini", "C4mini"])
def test_sharded_trace_matches_oracle(P, name):
    cfg = G.CONFIGS[name]
    X = G.make_tensor(cfg)
    A0 = G.initial_factors(cfg)
    A_fin, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, 20)

    def body(rank, ctx, lo, hi):
        cp.cp_set_factors(ctx, A0)
        infos = []
        for t in tr:
            cp.cp_set_phase_override(ctx, t["phase"])
            infos.append(cp.als_sweep(ctx, 0.0, cfg.eps_pp))
        return infos, cp.cp_get_factors(ctx)

    res = run_sharded(P, X, cfg.dims, cfg.K, body)
    cond = golden(name, X, A0, cfg.eps_pp, tr, A_fin)
    for rank, (infos, A) in enumerate(res):
        check(tr, infos, cond, A_fin, A, tag=(name, P, rank))
    # replicas agree bit for bit on the replicated factors (deterministic reductions)
    for n in range(1, cfg.N):
        for rank in range(1, P):
            assert np.array_equal(res[rank][1][n], res[0][1][n])


@pytest.mark.parametrize("name", ["C1", "C2mini", "C5mini"])
def test_nccl_transport_single_rank(name):
    """The NCCL transport itself on one GPU: a one-rank communicator (ncclCommInitRank with
    nranks = 1) and CPPP_FLAG_FORCE_COMM, so every sharded branch runs and every all-reduce is a
    real ncclAllReduce on the library stream.  The trace must match the oracle, and an unsharded
    context to rounding (the sharded schedule keeps the slab mode out of the multi-mode first
    level and contracts it last, so the operation order differs)."""
    cfg = G.CONFIGS[name]
    X = G.make_tensor(cfg)
    A0 = G.initial_factors(cfg)
    _, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, 12)
    uid = cp.cppp_nccl_unique_id()
    nc = cp.cp_init(X, cfg.N, cfg.dims, cfg.K, shard_offset=0, shard_extent=cfg.dims[0],
                    rank=0, world=1, nccl_unique_id=uid, flags=cp.FLAG_FORCE_COMM)
    plain = cp.cp_init(X, cfg.N, cfg.dims, cfg.K, flags=cp.FLAG_NO_OVERLAP)
    for c in (nc, plain):
        cp.cp_set_factors(c, A0)
    cond = golden(name, X, A0, cfg.eps_pp, tr)
    infos = []
    for t in tr:
        for c in (nc, plain):
            cp.cp_set_phase_override(c, t["phase"])
        a, b = cp.als_sweep(nc, 0.0, cfg.eps_pp), cp.als_sweep(plain, 0.0, cfg.eps_pp)
        infos.append(a)
        assert abs(a["fitness"] - b["fitness"]) < 1e-9, (a, b)
    check(tr, infos, cond, tag=(name, "nccl1"))
    M = cp.mttkrp_dt(nc)
    A = cp.cp_get_factors(nc)
    for n in range(cfg.N):
        assert rel(M[n], O.mttkrp(X, A, n)) < 1e-11, n
    # the sharded path with NCCL runs its sweeps from captured graphs, and als_run as ONE device
    # launch (the collectives inside the WHILE/SWITCH body): the same sweeps, bit for bit, as the
    # host loop of als_sweep calls, with no host round trip per sweep
    cp.cp_set_phase_override(nc, cp.PHASE_AUTO)
    cp.cp_set_factors(nc, A0)
    host = [cp.als_sweep(nc, 0.0, cfg.eps_pp) for _ in range(12)]
    for rep in range(2):
        cp.cp_set_factors(nc, A0)
        dev = cp.als_run(nc, 0.0, cfg.eps_pp, 12)
        assert len({d["seconds"] for d in dev}) == 1, cp.lib().cp_last_error(nc.h)
        for h, d in zip(host, dev):
            for key in ("phase", "residual_sq", "grad_norm_sum", "max_rel_dA"):
                assert h[key] == d[key], (rep, key, h, d)
    cp.cp_destroy(nc)
    cp.cp_destroy(plain)


def test_pp_error_sharded_single_rank():
    """pp_error through the sharded branches (one-rank NCCL communicator, FORCE_COMM): the
    slab mode's column sums go through the all-reduce; values match the oracle."""
    cfg = G.CONFIGS["C3mini"]
    X = G.make_tensor(cfg)
    Ap = G.initial_factors(cfg)
    r = np.random.default_rng(7)
    A = [a + 0.02 * r.standard_normal(a.shape) * np.linalg.norm(a, axis=0) / np.sqrt(a.shape[0])
         for a in Ap]
    uid = cp.cppp_nccl_unique_id()
    nc = cp.cp_init(X, cfg.N, cfg.dims, cfg.K, shard_offset=0, shard_extent=cfg.dims[0],
                    rank=0, world=1, nccl_unique_id=uid, flags=cp.FLAG_FORCE_COMM)
    cp.cp_set_factors(nc, Ap)
    cp.pp_build_operators(nc)
    cp.cp_update_factors(nc, A)
    err, eps, bound = cp.pp_error(nc)
    e_ref, eps_ref, b_ref = O.pp_error_monitor(X, A, Ap)
    assert np.allclose(eps, eps_ref, rtol=1e-12, atol=0)
    assert np.allclose(bound, b_ref, rtol=1e-12, atol=0)
    assert np.all(np.abs(err - e_ref) <= 1e-8 * e_ref + 1e-13)
    cp.cp_destroy(nc)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_als_run_free_running(P):
    """A whole free-running run through als_run on P slab contexts (C5mini): the phase decisions
    are taken from the all-reduced statistics, so every replica follows the oracle's schedule
    (where its ε_pp margins are clear) and ends with bit-identical replicated factors."""
    cfg = G.CONFIGS["C5mini"]
    X = G.make_tensor(cfg)
    A0 = G.initial_factors(cfg)
    A_fin, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, 20)

    def body(rank, ctx, lo, hi):
        cp.cp_set_factors(ctx, A0)
        return cp.als_run(ctx, 0.0, cfg.eps_pp, 20), cp.cp_get_factors(ctx)

    res = run_sharded(P, X, cfg.dims, cfg.K, body)
    if all(t["margin"] > 1e-6 for t in tr):
        for infos, _ in res:
            assert [i["phase"] for i in infos] == [t["phase"] for t in tr]
    for infos, _ in res[1:]:
        assert [i["residual_sq"] for i in infos] == [i["residual_sq"] for i in res[0][0]]
    for n in range(cfg.N):
        for rank in range(1, P):
            assert np.array_equal(res[rank][1][n], res[0][1][n])
    cond = golden("C5mini", X, A0, cfg.eps_pp, tr, A_fin)
    if [i["phase"] for i in res[0][0]] == [t["phase"] for t in tr]:
        check(tr, res[0][0], cond, A_fin, res[0][1], tag=("als_run", P))


@pytest.mark.parametrize("q", [1, "last"])
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("name", ["C1", "C3mini", "C4mini"])
def test_sharded_along_other_modes(q, P, name):
    """Slabs of a middle or of the LAST mode (BASELINE C5 names mode-4 slabs): MTTKRP, every
    operator and a replayed 12-sweep trace against the unsharded oracle, replicas bit-identical."""
    cfg = G.CONFIGS[name]
    q = cfg.N - 1 if q == "last" else q
    X = G.make_tensor(cfg)
    A0 = G.initial_factors(cfg)
    A_fin, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, 12)

    def body(rank, ctx, lo, hi):
        cp.cp_set_factors(ctx, A0)
        M = cp.mttkrp_dt(ctx)
        cp.pp_build_operators(ctx)
        ops = {(i, j): cp.pp_get_operator(ctx, i, j) for i in range(cfg.N) for j in range(i + 1, cfg.N)}
        cp.cp_set_factors(ctx, A0)
        infos = []
        for t in tr:
            cp.cp_set_phase_override(ctx, t["phase"])
            infos.append(cp.als_sweep(ctx, 0.0, cfg.eps_pp))
        return M, ops, infos, cp.cp_get_factors(ctx)

    res = run_sharded(P, X, cfg.dims, cfg.K, body, q=q)
    ops_ref = O.pp_operators(X, A0)
    cond = golden(name, X, A0, cfg.eps_pp, tr, A_fin)
    for rank, (M, ops, infos, A) in enumerate(res):
        lo, hi = slab(cfg.s, rank, P)
        for n in range(cfg.N):
            ref = O.mttkrp(X, A0, n)
            assert rel(M[n], ref[lo:hi] if n == q else ref) < 1e-11, (rank, n)
        for (i, j), ref in ops_ref.items():
            if i == q:
                ref = ref[lo:hi]
            elif j == q:
                ref = ref[:, lo:hi]
            assert rel(ops[(i, j)], ref) < 1e-11, (rank, i, j)
        check(tr, infos, cond, A_fin, A, tag=(name, q, P, rank))
    for n in range(cfg.N):
        if n != q:
            for rank in range(1, P):
                assert np.array_equal(res[rank][3][n], res[0][3][n])
