"""synthgen — seeded, counter-based synthetic inputs shared by the oracle tests and the GPU path.

This module holds NONE of the method's arithmetic (no MTTKRP, no PP operator, no ALS
step).  It only draws random numbers and materialises the generating CP model
X_true = [[A_true]] (the model of PAPER.md P:336-345) plus noise, so that
the oracle (``oracle/``) and the CUDA path (``paper_1811_10573_b200``) can be fed the
same bytes.  The CUDA library has a device twin of this generator (``gen.cu``) that
implements the same counter-based Philox4x32-10 stream and the same per-element
formula; tests compare the two.

Counter-based random numbers
-------------------------------------------------
Every random number is a pure function of (seed, stream, element index):
    counter = (lo32(idx), hi32(idx), stream, 0),   key = (lo32(seed), hi32(seed))
    (x0, x1, x2, x3) = Philox4x32-10(counter, key)
    uniform(idx) = res53(x0, x1)                      in [0, 1)
    normal(idx)  = sqrt(-2 log(1 - res53(x0,x1))) * cos(2 pi res53(x2,x3))   (Box-Muller)
Streams: 0..N-1 true factors, N noise, N+1..2N initial factors, 2N+1 collinearity draws.
Because the element index is the GLOBAL linear index, any slab of the tensor can be
generated independently (shard invariance for the multi-GPU path).

Config readings (BASELINE.json configs[0..4]) are in
``CONFIGS``; DESIGN.md lists them.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np

__all__ = [
    "philox4x32_10", "philox4x32_10_raw", "uniform", "normal", "Config", "CONFIGS", "get_config",
    "true_factors", "initial_factors", "kruskal_slab", "make_tensor", "collinearity_c", "laplacian_1d",
]

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = 0x9E3779B9
_W1 = 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10_raw(c0, c1, c2, c3, k0: int, k1: int):
    """Philox4x32-10 (Salmon et al., SC'11) on arbitrary 32-bit counter words (uint64 arrays)."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) for c in (c0, c1, c2, c3))
    for r in range(10):
        if r:
            k0 = (k0 + _W0) & 0xFFFFFFFF
            k1 = (k1 + _W1) & 0xFFFFFFFF
        p0 = _M0 * c0              # < 2^64, exact in uint64
        p1 = _M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0)), lo1, (hi0 ^ c3 ^ np.uint64(k1)), lo0
    return c0, c1, c2, c3


def philox4x32_10(idx: np.ndarray, stream: int, seed: int):
    """Philox4x32-10 on counters (lo(idx), hi(idx), stream, 0), key (lo(seed), hi(seed)).

    Returns four uint64 arrays holding 32-bit values.  Vectorised over ``idx``.
    """
    idx = np.asarray(idx, dtype=np.uint64)
    c0 = idx & _MASK32
    c1 = idx >> np.uint64(32)
    c2 = np.full_like(c0, np.uint64(stream & 0xFFFFFFFF))
    c3 = np.zeros_like(c0)
    return philox4x32_10_raw(c0, c1, c2, c3, seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)


def _res53(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """53-bit uniform in [0,1) from two 32-bit words (a: 27 high bits, b: 26 low bits)."""
    hi = (a >> np.uint64(5)).astype(np.float64)
    lo = (b >> np.uint64(6)).astype(np.float64)
    return (hi * 67108864.0 + lo) * (1.0 / 9007199254740992.0)


_CHUNK = 1 << 18


def _chunked(fn, idx):
    idx = np.asarray(idx, dtype=np.uint64)
    if idx.size <= _CHUNK:
        return fn(idx)
    out = np.empty(idx.shape, dtype=np.float64)
    flat_i, flat_o = idx.reshape(-1), out.reshape(-1)

    def work(a):
        flat_o[a:a + _CHUNK] = fn(flat_i[a:a + _CHUNK])

    # numpy ufuncs release the GIL: chunks run in parallel; each element's value is unchanged
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(work, range(0, flat_i.size, _CHUNK)))
    return out


def uniform(idx, stream: int, seed: int = 0) -> np.ndarray:
    def f(i):
        x0, x1, _, _ = philox4x32_10(i, stream, seed)
        return _res53(x0, x1)
    return _chunked(f, idx)


def normal(idx, stream: int, seed: int = 0) -> np.ndarray:
    def f(i):
        x0, x1, x2, x3 = philox4x32_10(i, stream, seed)
        u1 = _res53(x0, x1)
        u2 = _res53(x2, x3)
        return np.sqrt(-2.0 * np.log(1.0 - u1)) * np.cos(2.0 * math.pi * u2)
    return _chunked(f, idx)


@dataclass(frozen=True)
class Config:
    """One synthetic workload (BASELINE.json configs; readings SURVEY.md §8(c))."""
    name: str
    N: int
    s: int
    K: int
    family: str                 # "uniform" | "collinear" | "gaussian" | "laplacian"
    noise_kind: str             # "none" | "abs" (std) | "rel" (eta * ||X_true|| / ||noise||)
    noise: float = 0.0
    c_lo: float = 0.0
    c_hi: float = 0.0
    sweeps: int = 20
    eps_pp: float = 0.1
    R_true: int = 0             # rank of the generating CP model (0: the decomposition rank K)

    @property
    def dims(self):
        return (self.s,) * self.N

    @property
    def rank_true(self):
        return self.R_true if self.R_true > 0 else self.K

    @property
    def numel(self):
        return self.s ** self.N


CONFIGS = {
    # configs[0]: s=40, K=10, U[0,1) factors, seed 0, Gaussian noise std 1e-3, 20 sweeps, eps_pp=0.1
    "C1": Config("C1", 3, 40, 10, "uniform", "abs", 1e-3),
    # configs[1]: s=400, K=100 collinear (cosines in [0.6,0.8], Cholesky mixing), 1% noise
    "C2": Config("C2", 3, 400, 100, "collinear", "rel", 0.01, 0.6, 0.8),
    # configs[2]: s=100, K=50 U[0,1) factors + 1% noise
    "C3": Config("C3", 4, 100, 50, "uniform", "rel", 0.01),
    # configs[3]: s=20, K=30 collinear cosines in [0.5,0.9]; no noise stated (L19: eta=0)
    "C4": Config("C4", 6, 20, 30, "collinear", "none", 0.0, 0.5, 0.9),
    # configs[4]: s=256, K=128 N(0,1) factors + 1% noise (sharded config)
    "C5": Config("C5", 4, 256, 128, "gaussian", "rel", 0.01),
    # reduced-size stand-ins with the same families (parity helpers)
    "C5mini": Config("C5mini", 4, 64, 32, "gaussian", "rel", 0.01),
    "C2mini": Config("C2mini", 3, 72, 24, "collinear", "rel", 0.01, 0.6, 0.8),
    "C3mini": Config("C3mini", 4, 20, 12, "uniform", "rel", 0.01),
    "C4mini": Config("C4mini", 6, 8, 10, "collinear", "none", 0.0, 0.5, 0.9),
    # the paper's own workloads, synthetic:
    # weak-scaling shape at p = 1 (N = 6, s = floor(32 p^(1/6)), R = floor(4 p^(1/6))); the paper
    # does not say what those tensors hold: reading, Tensor 3 (U[0,1) factors, R = K) + 1% noise
    "P6W": Config("P6W", 6, 32, 4, "uniform", "rel", 0.01),
    # strong-scaling shape (N = 6, s = 50, R = 6): 1.56e10 entries, 125 GB -- fits one B200
    "P6S": Config("P6S", 6, 50, 6, "uniform", "rel", 0.01),
    # compact Laplacian tensor (Tensor 2) of order 6 with n = 5 (s = n^2 = 25),
    # CP rank 6, approximated with rank 2 as in the paper
    "LAP": Config("LAP", 6, 25, 2, "laplacian", "none", 0.0, R_true=6),
    "LAPmini": Config("LAPmini", 4, 9, 2, "laplacian", "none", 0.0, R_true=4),
}


def get_config(name: str) -> Config:
    return CONFIGS[name]


def collinearity_c(cfg: Config, n: int, seed: int = 0) -> float:
    """Per-factor equicorrelation c_n ~ U[c_lo, c_hi] (L18), stream 2N+1, element n."""
    u = uniform(np.array([n], dtype=np.uint64), 2 * cfg.N + 1, seed)[0]
    return cfg.c_lo + (cfg.c_hi - cfg.c_lo) * u


def _factor_draw(cfg: Config, n: int, stream: int, kind: str, seed: int, R: int = 0) -> np.ndarray:
    R = R or cfg.K
    idx = np.arange(cfg.s * R, dtype=np.uint64)
    v = uniform(idx, stream, seed) if kind == "uniform" else normal(idx, stream, seed)
    return v.reshape(cfg.s, R)


def laplacian_1d(n: int) -> np.ndarray:
    """The 1-D second-difference matrix tridiag(-1, 2, -1) (reading of the paper's D)."""
    return 2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)


def true_factors(cfg: Config, seed: int = 0):
    """Generating factors A_true^(n) (s x K, row-major).

    uniform  : i.i.d. U[0,1)  (Tensor 3)
    gaussian : i.i.d. N(0,1)  (BASELINE configs[4])
    collinear: Cholesky mixing (L18): A = normalize_columns(G L^T), C_n = (1-c)I + c 11^T = L L^T
    laplacian: Tensor 2, X = sum_k vec(I) o ... o vec(D) o ... o vec(I) (D in
               position k): A^(n)[:, k] = vec(D) if k == n else vec(I); s = n_D^2, rank N.
    Columns: cfg.rank_true.
    """
    out = []
    R = cfg.rank_true
    for n in range(cfg.N):
        if cfg.family == "uniform":
            out.append(_factor_draw(cfg, n, n, "uniform", seed, R))
        elif cfg.family == "gaussian":
            out.append(_factor_draw(cfg, n, n, "normal", seed, R))
        elif cfg.family == "laplacian":
            nd = int(round(math.sqrt(cfg.s)))
            assert nd * nd == cfg.s and R == cfg.N, "laplacian: s = n^2 and rank N"
            A = np.empty((cfg.s, R))
            for k in range(R):
                A[:, k] = (laplacian_1d(nd) if k == n else np.eye(nd)).ravel()
            out.append(A)
        elif cfg.family == "collinear":
            G = _factor_draw(cfg, n, n, "normal", seed, R)
            c = collinearity_c(cfg, n, seed)
            C = (1.0 - c) * np.eye(R) + c * np.ones((R, R))
            L = np.linalg.cholesky(C)
            A = G @ L.T
            A = A / np.linalg.norm(A, axis=0, keepdims=True)
            out.append(np.ascontiguousarray(A))
        else:
            raise ValueError(cfg.family)
    return out


def initial_factors(cfg: Config, seed: int = 0):
    """ALS initial guess: i.i.d. U[0,1) on streams N+1..2N (L15)."""
    return [_factor_draw(cfg, n, cfg.N + 1 + n, "uniform", seed) for n in range(cfg.N)]


def kruskal_slab(A: Sequence[np.ndarray], row_lo: int = 0, row_hi: Optional[int] = None) -> np.ndarray:
    """Rows [row_lo,row_hi) of mode 1 of [[A^(1),...,A^(N)]].

    Fixed arithmetic order (the device twin uses the same): for each element,
    p_r = ((A1(i1,r)*A2(i2,r))*A3(i3,r))*...,  x = ((0 + p_0) + p_1) + ... + p_{K-1}.
    Rows are processed in cache-sized blocks; the per-element order is unchanged.
    """
    N = len(A)
    K = A[0].shape[1]
    row_hi = A[0].shape[0] if row_hi is None else row_hi
    dims = [row_hi - row_lo] + [a.shape[0] for a in A[1:]]
    X = np.zeros(dims, dtype=np.float64)
    row_elems = int(np.prod(dims[1:])) if N > 1 else 1
    blk = max(1, (1 << 19) // max(row_elems, 1))

    def work(r0):
        r1 = min(row_hi, r0 + blk)
        Xb = X[r0 - row_lo:r1 - row_lo]
        for r in range(K):
            p = A[0][r0:r1, r]
            for n in range(1, N):
                p = np.multiply.outer(p, A[n][:, r])
            Xb += p

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(work, range(row_lo, row_hi, blk)))
    return X


def make_tensor(cfg: Config, seed: int = 0, row_lo: int = 0, row_hi: Optional[int] = None,
                reduce: Optional[Callable[[np.ndarray], np.ndarray]] = None,
                A_true: Optional[Sequence[np.ndarray]] = None) -> np.ndarray:
    """X = X_true + noise (P:1040-1048 with the readings L19), rows [row_lo,row_hi) of mode 1.

    The noise element at global linear index e is normal(e, stream=N).  For "rel" noise the
    scale eta*||X_true||_F/||noise||_F needs global norms: per-row partial sums are placed in a
    length-s vector, ``reduce`` (e.g. an all-reduce over ranks) sums the vectors, then the
    total is summed in a fixed order — so every shard count gives the same X.
    """
    s = cfg.s
    row_hi = s if row_hi is None else row_hi
    if A_true is None:
        A_true = true_factors(cfg, seed)
    X = kruskal_slab(A_true, row_lo, row_hi)
    if cfg.noise_kind == "none" or cfg.noise == 0.0:
        return X
    row_elems = s ** (cfg.N - 1)
    idx = np.arange(row_lo * row_elems, row_hi * row_elems, dtype=np.uint64)
    Z = normal(idx, cfg.N, seed).reshape(X.shape)
    if cfg.noise_kind == "abs":
        return X + cfg.noise * Z
    vx = np.zeros(s)
    vz = np.zeros(s)
    vx[row_lo:row_hi] = np.einsum("ij,ij->i", X.reshape(X.shape[0], -1), X.reshape(X.shape[0], -1))
    vz[row_lo:row_hi] = np.einsum("ij,ij->i", Z.reshape(Z.shape[0], -1), Z.reshape(Z.shape[0], -1))
    if reduce is not None:
        vx = reduce(vx)
        vz = reduce(vz)
    nx = math.sqrt(math.fsum(vx.tolist()))
    nz = math.sqrt(math.fsum(vz.tolist()))
    scale = cfg.noise * nx / nz
    return X + scale * Z
