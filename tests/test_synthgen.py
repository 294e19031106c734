"""Pins for the shared input generator (synthgen) — CPU only."""
import json
import os

import numpy as np

import synthgen as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_known_answers():
    cases = json.load(open(os.path.join(GOLD, "spec_examples.json")))["philox4x32_10_kat"]["cases"]
    for c in cases:
        ctr = [np.uint64(int(x, 16)) for x in c["ctr"]]
        key = [int(x, 16) for x in c["key"]]
        out = G.philox4x32_10_raw(*ctr, *key)
        assert [int(x) for x in out] == [int(x, 16) for x in c["out"]]


def test_uniform_and_normal_moments():
    idx = np.arange(200000, dtype=np.uint64)
    u = G.uniform(idx, 3)
    z = G.normal(idx, 4)
    assert 0.0 <= u.min() and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 5e-3 and abs(u.var() - 1 / 12) < 2e-3
    assert abs(z.mean()) < 1e-2 and abs(z.var() - 1) < 2e-2


def test_streams_are_distinct_and_deterministic():
    idx = np.arange(64, dtype=np.uint64)
    assert np.array_equal(G.uniform(idx, 1), G.uniform(idx, 1))
    assert not np.array_equal(G.uniform(idx, 1), G.uniform(idx, 2))
    assert not np.array_equal(G.uniform(idx, 1, seed=0), G.uniform(idx, 1, seed=1))


def test_slab_generation_is_shard_invariant():
    cfg = G.CONFIGS["C5mini"]
    full = G.make_tensor(cfg)
    parts = []

    def reduce_all(v):   # emulate an all-reduce over 4 ranks holding disjoint rows
        return v
    # emulate: each rank computes rows; the reduce sums the rank vectors
    bounds = [(0, 16), (16, 32), (32, 48), (48, 64)]
    A_true = G.true_factors(cfg)
    vecs = {}
    import synthgen as _g
    # collect per-rank vectors through a recording reducer, then replay with the true sum
    for lo, hi in bounds:
        rec = []
        _g.make_tensor(cfg, row_lo=lo, row_hi=hi, A_true=A_true, reduce=lambda v: (rec.append(v.copy()), v)[1])
        vecs[(lo, hi)] = rec
    tot = [sum(vecs[b][i] for b in bounds) for i in range(2)]
    for lo, hi in bounds:
        it = iter(tot)
        parts.append(_g.make_tensor(cfg, row_lo=lo, row_hi=hi, A_true=A_true, reduce=lambda v: next(it)))
    assert np.array_equal(np.concatenate(parts, axis=0), full)


def test_collinear_factors_cosines():
    """L18: unit columns; cosines concentrate near c_n in [c_lo, c_hi]."""
    cfg = G.CONFIGS["C2"]
    A = G.true_factors(cfg)
    for n, a in enumerate(A):
        C = a.T @ a
        assert np.allclose(np.diag(C), 1.0, atol=1e-14)
        off = C[~np.eye(cfg.K, dtype=bool)]
        c = G.collinearity_c(cfg, n)
        assert cfg.c_lo <= c <= cfg.c_hi
        assert abs(off.mean() - c) < 0.02


def test_relative_noise_level():
    cfg = G.CONFIGS["C3mini"]
    A = G.true_factors(cfg)
    Xt = G.kruskal_slab(A)
    X = G.make_tensor(cfg, A_true=A)
    assert abs(np.linalg.norm(X - Xt) / np.linalg.norm(Xt) - 0.01) < 1e-12


def test_laplacian_tensor_is_the_papers_sum_of_outer_products():
    """Tensor 2: X = sum_k vec(I) o ... o vec(D) o ... o vec(I), D in position k,
    written out directly with the 1-D second-difference matrix D = tridiag(-1, 2, -1)."""
    cfg = G.CONFIGS["LAPmini"]          # order 4, n = 3 (s = 9), CP rank 4
    n = 3
    D = 2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    vI, vD = np.eye(n).ravel(), D.ravel()
    ref = np.zeros(cfg.dims)
    for k in range(cfg.N):
        vecs = [vD if m == k else vI for m in range(cfg.N)]
        ref += np.einsum("a,b,c,d->abcd", *vecs)
    X = G.make_tensor(cfg)
    assert np.array_equal(X, ref) or np.allclose(X, ref, rtol=0, atol=1e-15)
    # it is the d-dimensional Laplacian operator, entry (i, j) of sum_k I x .. x D x .. x I,
    # with the row and column indices of each factor interleaved into one mode of size n^2
    A = G.true_factors(cfg)
    assert all(a.shape == (9, 4) for a in A)
    assert cfg.rank_true == 4 and cfg.K == 2


def test_paper_scaling_shapes():
    """f4 shapes: weak scaling at p = 1 and the strong-scaling tensor."""
    w, s = G.CONFIGS["P6W"], G.CONFIGS["P6S"]
    assert (w.N, w.s, w.K) == (6, int(32 * 1 ** (1 / 6)), int(4 * 1 ** (1 / 6)))
    assert (s.N, s.s, s.K) == (6, 50, 6)
    assert s.numel * 8 == 125 * 10 ** 9
