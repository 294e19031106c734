"""Multi-process (gloo, world size 2, CPU) checks of the mode-0 slab sharding algebra that the
multi-GPU path implements: every contraction is linear in X, so partial results
computed on the slabs and all-reduced equal the whole-tensor results (oracle arithmetic on the
slabs), and the seeded generator is shard-invariant under a real all-reduce."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def slab(s0, rank, world):
    """The bench's partition of mode 0 (bench.py): rows [rank*s0//world, (rank+1)*s0//world)."""
    return rank * s0 // world, (rank + 1) * s0 // world


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle.cp_oracle as O
    import synthgen as G
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def allreduce(v):
            t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
            dist.all_reduce(t)
            return t.numpy()

        cfg = G.CONFIGS["C5mini"]             # N=4, s=64, K=32, gaussian + 1% noise
        lo, hi = slab(cfg.s, rank, world)
        A_true = G.true_factors(cfg)
        Xs = G.make_tensor(cfg, row_lo=lo, row_hi=hi, A_true=A_true, reduce=allreduce)
        X = G.make_tensor(cfg, A_true=A_true)
        assert np.array_equal(Xs, X[lo:hi]), "generator not shard-invariant"

        r = np.random.default_rng(7)
        A = [r.standard_normal((cfg.s, cfg.K)) for _ in range(cfg.N)]
        As = [A[0][lo:hi]] + A[1:]
        # DT: M^(n), n != 0 — partial over local rows of mode 0, all-reduced
        for n in range(1, cfg.N):
            part = O.mttkrp(Xs, As, n)
            full = allreduce(part)
            assert np.linalg.norm(full - O.mttkrp(X, A, n)) <= 1e-12 * np.linalg.norm(full)
        # M^(0): exact for the local rows, no communication
        assert np.allclose(O.mttkrp(Xs, As, 0), O.mttkrp(X, A, 0)[lo:hi], rtol=1e-13, atol=0)
        # ||X||² all-reduced
        assert abs(allreduce(np.array([np.sum(Xs * Xs)]))[0] - np.sum(X * X)) <= 1e-12 * np.sum(X * X)
        # PP operators: pairs without mode 0 are all-reduced partials; pairs (0, j) stay local
        ops_full = O.pp_operators(X, A)
        for (i, j), ref in ops_full.items():
            loc = O.pp_operator(Xs, As, i, j)
            if i == 0:
                assert np.allclose(loc, ref[lo:hi], rtol=1e-12, atol=1e-12 * np.abs(ref).max())
            else:
                red = allreduce(loc)
                assert np.linalg.norm(red - ref) <= 1e-12 * np.linalg.norm(ref)
        # PP sweep exchange: T_m = M_p^(0,m) x_0 dA^(0) over local rows, all-reduced (SURVEY C-c)
        dA0 = 0.01 * r.standard_normal((cfg.s, cfg.K))
        for m in range(1, cfg.N):
            loc = np.einsum("xyk,xk->yk", O.pp_operator(Xs, As, 0, m), dA0[lo:hi])
            ref = np.einsum("xyk,xk->yk", ops_full[(0, m)], dA0)
            assert np.linalg.norm(allreduce(loc) - ref) <= 1e-12 * np.linalg.norm(ref)
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_slab_partition_covers_mode_exactly():
    for s0 in (7, 64, 256, 400):
        for world in (1, 2, 3, 4, 8):
            rows = []
            for r in range(world):
                lo, hi = slab(s0, r, world)
                rows += list(range(lo, hi))
            assert rows == list(range(s0))


@pytest.mark.timeout(300)
def test_sharded_algebra_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=280) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_plan_puts_sharded_mode_last_in_pptree():
    import paper_1811_10573_b200.cppp as cp
    for N in (3, 4, 6):
        first = cp.cppp_plan_describe(N, 0).splitlines()[0].split(":")[1].split()
        assert first[-1] == "0" and sorted(first) == [str(i) for i in range(N)]
        lines = [l for l in cp.cppp_plan_describe(N, 0).splitlines() if l.startswith("L")]
        # the sharded mode is contracted only at the leaves (Def. pptree: tree mode N)
        for l in lines:
            if "contract:0 " in l or l.endswith("contract:0"):
                assert "leaf" in l
