"""Thin ctypes binding of libcppp.so (include/cppp.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only converts
numpy arrays / torch tensors to pointers, allocates the device workspace through PyTorch
(device memory and streams are PyTorch's; the library never owns a torch object), and turns
status codes into exceptions.  There is no CPU fallback: if the library or a CUDA device is
missing, every call raises.

Function names mirror the C ABI: cp_init, cp_set_factors, cp_get_factors, mttkrp_dt,
pp_build_operators, pp_get_operator, pp_get_single, pp_update, pp_error, als_sweep,
cp_set_phase_override, fitness, cppp_generate, cp_destroy.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CPPP_LIB") or os.path.join(_HERE, "libcppp.so")   # CPPP_LIB: A/B builds

PHASE_AUTO, PHASE_DT, PHASE_PP_BUILD, PHASE_PP = -1, 0, 1, 2
PHASE_NAMES = {PHASE_DT: "dt", PHASE_PP_BUILD: "pp-build", PHASE_PP: "pp-approx"}
PHASE_BY_NAME = {v: k for k, v in PHASE_NAMES.items()}
FLAG_BORROW_TENSOR, FLAG_SIMT_TTM, FLAG_PROFILE, FLAG_NO_FUSED_TTV, FLAG_NO_GRAPH = 1, 2, 4, 8, 16
FLAG_NO_KRP = 32
FLAG_NO_OVERLAP = 64
FLAG_FORCE_COMM = 128
FLAG_NO_OP_REUSE = 256
FLAG_NO_FUSED_SOLVE = 512
K_TTM, K_TTV, K_PPUPDATE, K_SOLVE, K_OTHER = range(5)
KCLASS_NAMES = ["ttm", "ttv", "pp_update", "solve", "other", "factor"]


class CpppError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"cppp status {status}: {msg}")
        self.status = status


HOST_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_size_t, C.c_void_p)


class Opts(C.Structure):
    _fields_ = [("device", C.c_int), ("stream", C.c_void_p), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("flags", C.c_uint), ("shard_mode", C.c_int),
                ("shard_offset", C.c_int64), ("shard_extent", C.c_int64),
                ("nccl_unique_id", C.c_void_p), ("rank", C.c_int), ("world", C.c_int),
                ("host_allreduce", HOST_ALLREDUCE), ("host_allreduce_user", C.c_void_p),
                ("pinv_rel_tol", C.c_double)]


class TkSweepInfo(C.Structure):
    _fields_ = [("sweep", C.c_int), ("phase", C.c_int), ("next_phase", C.c_int), ("converged", C.c_int),
                ("core_change", C.c_double), ("core_norm", C.c_double), ("residual", C.c_double),
                ("max_rel_dA", C.c_double)]

    def as_dict(self):
        return dict(sweep=self.sweep, phase=PHASE_NAMES[self.phase], next_phase=PHASE_NAMES[self.next_phase],
                    converged=bool(self.converged), core_change=self.core_change, core_norm=self.core_norm,
                    residual=self.residual, max_rel_dA=self.max_rel_dA)


class SweepInfo(C.Structure):
    _fields_ = [("sweep", C.c_int), ("phase", C.c_int), ("fitness", C.c_double),
                ("residual_sq", C.c_double), ("grad_norm_sum", C.c_double),
                ("max_rel_dA", C.c_double), ("next_phase", C.c_int), ("restarts", C.c_int),
                ("converged", C.c_int), ("seconds", C.c_double), ("pp_bound", C.c_double),
                ("approximate", C.c_int)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["approximate"] = bool(self.approximate)
        d["phase"] = PHASE_NAMES.get(self.phase, str(self.phase))
        d["next_phase"] = PHASE_NAMES.get(self.next_phase, str(self.next_phase))
        return d


class KernelStat(C.Structure):
    _fields_ = [("launches", C.c_int64), ("total_ms", C.c_double), ("flops", C.c_double),
                ("bytes", C.c_double)]


_lib = None


def lib():
    """Load libcppp.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1811_10573_b200.build`")
    L = C.CDLL(LIB_PATH)
    P, I, D, V = C.c_void_p, C.c_int, C.c_double, None
    sig = {
        "cppp_default_opts": (V, [C.POINTER(Opts)]),
        "cppp_workspace_bytes": (C.c_size_t, [I, C.POINTER(C.c_int64), I, C.POINTER(Opts)]),
        "cp_init": (I, [C.POINTER(P), P, I, C.POINTER(C.c_int64), I, C.POINTER(Opts)]),
        "cp_load_tensor": (I, [P, P]),
        "cp_set_factors": (I, [P, C.POINTER(P)]),
        "cp_get_factors": (I, [P, C.POINTER(P)]),
        "cp_update_factors": (I, [P, C.POINTER(P)]),
        "mttkrp_dt": (I, [P, C.POINTER(P)]),
        "pp_build_operators": (I, [P]),
        "pp_get_operator": (I, [P, I, I, P]),
        "pp_get_single": (I, [P, I, P]),
        "pp_update": (I, [P, I, P]),
        "pp_error": (I, [P, P, P, P]),
        "pp_second_order": (I, [P, C.POINTER(P)]),
        "als_sweep": (I, [P, D, D, C.POINTER(SweepInfo)]),
        "als_run": (I, [P, D, D, I, C.POINTER(SweepInfo), C.POINTER(I)]),
        "cp_set_phase_override": (I, [P, I]),
        "cp_set_pp_policy": (I, [P, I, D]),
        "fitness": (I, [P, C.POINTER(D)]),
        "fitness_exact": (I, [P, C.POINTER(D), C.POINTER(D)]),
        "cppp_kernel_stats": (I, [P, I, C.POINTER(KernelStat)]),
        "cppp_reset_kernel_stats": (I, [P]),
        "cppp_generate": (I, [P, P, I, C.POINTER(C.c_int64), I, C.POINTER(P), I, D, C.c_uint64,
                              C.c_int64, C.c_int64, P]),
        "cppp_nccl_unique_id": (I, [P]),
        "cppp_plan_describe": (C.c_size_t, [I, I, C.c_char_p, C.c_size_t]),
        "cp_destroy": (V, [P]),
        "cp_last_error": (C.c_char_p, [P]),
        "cppp_status_string": (C.c_char_p, [I]),
        "cppp_version": (C.c_char_p, []),
        "cppp_launch_count": (C.c_uint64, []),
        "tk_init": (I, [C.POINTER(P), P, I, C.POINTER(C.c_int64), C.POINTER(I), P, C.c_uint]),
        "tk_set_factors": (I, [P, C.POINTER(P)]),
        "tk_update_factors": (I, [P, C.POINTER(P)]),
        "tk_ttmc": (I, [P, C.POINTER(P)]),
        "tk_pp_build": (I, [P]),
        "tk_pp_get_operator": (I, [P, I, I, P]),
        "tk_pp_get_single": (I, [P, I, P]),
        "tk_pp_update": (I, [P, I, P]),
        "tk_hosvd": (I, [P]),
        "tk_sweep": (I, [P, D, D, C.POINTER(TkSweepInfo)]),
        "tk_set_phase_override": (I, [P, I]),
        "tk_get_factors": (I, [P, C.POINTER(P)]),
        "tk_get_core": (I, [P, P]),
        "tk_last_error": (C.c_char_p, [P]),
        "tk_destroy": (V, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTED = ["cppp_default_opts", "cppp_workspace_bytes", "cp_init", "cp_load_tensor", "cp_set_factors",
            "cp_update_factors",
            "cp_get_factors", "mttkrp_dt", "pp_build_operators", "pp_get_operator",
            "pp_get_single", "pp_update", "pp_error", "pp_second_order", "als_sweep", "als_run", "cp_set_phase_override", "cp_set_pp_policy", "fitness",
            "fitness_exact", "cppp_kernel_stats", "cppp_reset_kernel_stats", "cppp_generate",
            "cppp_nccl_unique_id", "cppp_plan_describe", "cp_destroy", "cp_last_error",
            "cppp_status_string", "cppp_version", "cppp_launch_count",
            "tk_init", "tk_set_factors", "tk_update_factors", "tk_ttmc", "tk_pp_build",
            "tk_pp_get_operator", "tk_pp_get_single", "tk_pp_update", "tk_hosvd", "tk_sweep",
            "tk_set_phase_override", "tk_get_factors", "tk_get_core", "tk_last_error", "tk_destroy"]


# ------------------------------------------------------------------ marshalling helpers
def _ptr(a) -> int:
    """Data pointer of a C-contiguous float64 numpy array or torch tensor."""
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    if not (isinstance(a, np.ndarray) and a.flags.c_contiguous and a.dtype == np.float64):
        raise ValueError("expected a C-contiguous float64 numpy array or torch tensor")
    return a.ctypes.data


def _ptrs(arrs) -> C.Array:
    return (C.c_void_p * len(arrs))(*[_ptr(a) for a in arrs])


def _check(ctx, status: int):
    if status != 0:
        msg = lib().cp_last_error(ctx.h if ctx is not None else None)
        raise CpppError(status, (msg or b"").decode() or lib().cppp_status_string(status).decode())


class Ctx:
    """Handle returned by cp_init: owns the C context and keeps the torch workspace alive."""

    def __init__(self):
        self.h = C.c_void_p()
        self.N = 0
        self.K = 0
        self.s: List[int] = []
        self.local_rows: List[int] = []
        self.keep = []

    def __del__(self):
        try:
            cp_destroy(self)
        except Exception:
            pass


def _torch_workspace(nbytes: int, device: int):
    import torch
    return torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")


def cp_init(X, N: int, s: Sequence[int], K: int, *, device: int = 0, stream=None,
            flags: int = 0, shard_offset: Optional[int] = None, shard_extent: Optional[int] = None,
            nccl_unique_id: Optional[bytes] = None, rank: int = 0, world: int = 1,
            torch_workspace: bool = True, host_allreduce=None, pinv_rel_tol: float = 0.0,
            shard_mode: int = 0) -> Ctx:
    """cp_init (include/cppp.h).  X: numpy array (host) or torch CUDA tensor (device; borrowed
    with FLAG_BORROW_TENSOR); sharded (shard_extent given): this rank's slab of mode shard_mode.  The device workspace is a torch uint8 tensor unless
    torch_workspace=False (then the library cudaMallocs it).  stream: a torch.cuda.Stream or
    None (library-owned stream)."""
    L = lib()
    ctx = Ctx()
    ctx.N, ctx.K, ctx.s = N, K, list(s)
    o = Opts()
    L.cppp_default_opts(C.byref(o))
    o.device = device
    o.flags = flags
    if stream is not None:
        o.stream = stream.cuda_stream
    if shard_extent is not None:
        o.shard_mode = int(shard_mode)
        o.shard_offset = int(shard_offset)
        o.shard_extent = int(shard_extent)
    o.rank, o.world = rank, world
    o.pinv_rel_tol = pinv_rel_tol
    if host_allreduce is not None:
        # host_allreduce(np.ndarray view of the staged buffer) -> None, sums in place
        def _cb(buf, count, _user, _fn=host_allreduce):
            try:
                _fn(np.ctypeslib.as_array(buf, shape=(count,)))
                return 0
            except Exception:  # noqa: BLE001 - reported as a status by the library
                return 1
        cb = HOST_ALLREDUCE(_cb)
        ctx.keep.append(cb)
        o.host_allreduce = cb
    if nccl_unique_id is not None:
        idbuf = C.create_string_buffer(bytes(nccl_unique_id), 128)
        ctx.keep.append(idbuf)
        o.nccl_unique_id = C.cast(idbuf, C.c_void_p)
    dims = (C.c_int64 * N)(*s)
    if torch_workspace:
        nbytes = L.cppp_workspace_bytes(N, dims, K, C.byref(o))
        if nbytes == 0:
            raise CpppError(-1, "invalid problem for cppp_workspace_bytes")
        ws = _torch_workspace(nbytes, device)
        ctx.keep.append(ws)
        o.workspace = ws.data_ptr()
        o.workspace_bytes = nbytes
    if hasattr(X, "data_ptr"):
        ctx.keep.append(X)
    st = L.cp_init(C.byref(ctx.h), _ptr(X), N, dims, K, C.byref(o))
    _check(ctx, st)
    ctx.local_rows = list(s)
    if shard_extent is not None:
        ctx.local_rows[int(shard_mode)] = int(shard_extent)
    return ctx


def cp_load_tensor(ctx: Ctx, X) -> None:
    """cp_load_tensor (include/cppp.h): a new tensor of the same shape (numpy host array or torch
    CUDA tensor) into an existing context; call cp_set_factors next."""
    if hasattr(X, "data_ptr"):
        ctx.keep.append(X)
    _check(ctx, lib().cp_load_tensor(ctx.h, _ptr(X)))


def cp_set_factors(ctx: Ctx, A: Sequence) -> None:
    arrs = [np.ascontiguousarray(a, dtype=np.float64) if isinstance(a, np.ndarray) else a for a in A]
    _check(ctx, lib().cp_set_factors(ctx.h, _ptrs(arrs)))


def cp_update_factors(ctx: Ctx, A: Sequence) -> None:
    arrs = [np.ascontiguousarray(a, dtype=np.float64) if isinstance(a, np.ndarray) else a for a in A]
    _check(ctx, lib().cp_update_factors(ctx.h, _ptrs(arrs)))


def cp_get_factors(ctx: Ctx, out=None) -> List:
    if out is None:
        out = [np.empty((ctx.s[n], ctx.K)) for n in range(ctx.N)]
    _check(ctx, lib().cp_get_factors(ctx.h, _ptrs(out)))
    return out


def mttkrp_dt(ctx: Ctx) -> List[np.ndarray]:
    out = [np.empty((ctx.local_rows[n], ctx.K)) for n in range(ctx.N)]
    _check(ctx, lib().mttkrp_dt(ctx.h, _ptrs(out)))
    return out


def pp_build_operators(ctx: Ctx) -> None:
    _check(ctx, lib().pp_build_operators(ctx.h))


def pp_get_operator(ctx: Ctx, i: int, j: int, out=None) -> np.ndarray:
    if out is None:
        out = np.empty((ctx.local_rows[i], ctx.local_rows[j], ctx.K))
    _check(ctx, lib().pp_get_operator(ctx.h, i, j, _ptr(out)))
    return out


def pp_get_single(ctx: Ctx, n: int) -> np.ndarray:
    out = np.empty((ctx.local_rows[n], ctx.K))
    _check(ctx, lib().pp_get_single(ctx.h, n, _ptr(out)))
    return out


def pp_update(ctx: Ctx, n: int, out=None) -> np.ndarray:
    if out is None:
        out = np.empty((ctx.local_rows[n], ctx.K))
    _check(ctx, lib().pp_update(ctx.h, n, _ptr(out)))
    return out


def pp_error(ctx: Ctx):
    """pp_error (include/cppp.h): (err, eps, bound), each N x K — the column-wise relative error
    of the PP approximation M~ against the exact MTTKRP, ε_k^(n), and the error certificate."""
    err, eps, bound = (np.empty((ctx.N, ctx.K)) for _ in range(3))
    _check(ctx, lib().pp_error(ctx.h, _ptr(err), _ptr(eps), _ptr(bound)))
    return err, eps, bound


def pp_second_order(ctx: Ctx) -> List[np.ndarray]:
    """pp_second_order (include/cppp.h): T2^(n) = Σ_{i<j≠n} M_p^(i,j,n) ×_i dA^(i) ×_j dA^(j)."""
    out = [np.empty((ctx.local_rows[n], ctx.K)) for n in range(ctx.N)]
    _check(ctx, lib().pp_second_order(ctx.h, _ptrs(out)))
    return out


def als_sweep(ctx: Ctx, eps: float, eps_pp: float) -> dict:
    info = SweepInfo()
    _check(ctx, lib().als_sweep(ctx.h, eps, eps_pp, C.byref(info)))
    return info.as_dict()


def als_run(ctx: Ctx, eps: float, eps_pp: float, max_sweeps: int) -> list:
    """als_run (include/cppp.h): up to max_sweeps sweeps in one device launch; per-sweep dicts."""
    infos = (SweepInfo * max(max_sweeps, 1))()
    done = C.c_int(0)
    _check(ctx, lib().als_run(ctx.h, eps, eps_pp, max_sweeps, infos, C.byref(done)))
    return [infos[i].as_dict() for i in range(done.value)]


POLICY_EPS_PP, POLICY_BOUND = 0, 1


def cp_set_pp_policy(ctx: Ctx, policy: int, tol: float = 0.0) -> None:
    """cp_set_pp_policy (include/cppp.h): POLICY_EPS_PP (Alg. 3) or POLICY_BOUND (rebuild when the
    switching monitor's certificate reaches tol)."""
    _check(ctx, lib().cp_set_pp_policy(ctx.h, int(policy), float(tol)))


def cp_set_phase_override(ctx: Ctx, phase) -> None:
    if isinstance(phase, str):
        phase = PHASE_BY_NAME[phase]
    _check(ctx, lib().cp_set_phase_override(ctx.h, int(phase)))


def fitness(ctx: Ctx) -> float:
    f = C.c_double()
    _check(ctx, lib().fitness(ctx.h, C.byref(f)))
    return f.value


def fitness_exact(ctx: Ctx):
    """fitness_exact (include/cppp.h): (fitness, unclamped r²) at the current factors from one
    exact MTTKRP pass."""
    f, r2 = C.c_double(), C.c_double()
    _check(ctx, lib().fitness_exact(ctx.h, C.byref(f), C.byref(r2)))
    return f.value, r2.value


def kernel_stats(ctx: Ctx) -> dict:
    out = {}
    for k, name in enumerate(KCLASS_NAMES):
        st = KernelStat()
        _check(ctx, lib().cppp_kernel_stats(ctx.h, k, C.byref(st)))
        out[name] = dict(launches=st.launches, total_ms=st.total_ms, flops=st.flops, bytes=st.bytes)
    return out


def reset_kernel_stats(ctx: Ctx) -> None:
    _check(ctx, lib().cppp_reset_kernel_stats(ctx.h))


def cppp_generate(X_dev, s: Sequence[int], K: int, A_true: Sequence, noise_kind: int, noise: float,
                  seed: int = 0, row_lo: int = 0, row_hi: Optional[int] = None, stream=None,
                  ctx: Optional[Ctx] = None) -> None:
    """Device twin of synthgen.make_tensor: X_dev (torch CUDA tensor) := rows [row_lo,row_hi)."""
    N = len(s)
    row_hi = s[0] if row_hi is None else row_hi
    arrs = [np.ascontiguousarray(a, dtype=np.float64) if isinstance(a, np.ndarray) else a for a in A_true]
    dims = (C.c_int64 * N)(*s)
    st = lib().cppp_generate(ctx.h if ctx else None, _ptr(X_dev), N, dims, K, _ptrs(arrs), noise_kind,
                             noise, seed, row_lo, row_hi, stream.cuda_stream if stream is not None else None)
    _check(ctx, st)


def cppp_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = lib().cppp_nccl_unique_id(C.cast(buf, C.c_void_p))
    if st != 0:
        raise CpppError(st, "ncclGetUniqueId failed")
    return buf.raw


def cppp_plan_describe(N: int, shard_mode: int = -1) -> str:
    need = lib().cppp_plan_describe(N, shard_mode, None, 0)
    buf = C.create_string_buffer(need)
    lib().cppp_plan_describe(N, shard_mode, buf, need)
    return buf.value.decode()


def cp_destroy(ctx: Ctx) -> None:
    if ctx is not None and ctx.h:
        lib().cp_destroy(ctx.h)
        ctx.h = C.c_void_p()
        ctx.keep.clear()   # the borrowed tensor and the torch workspace can go now


def cppp_launch_count() -> int:
    return int(lib().cppp_launch_count())


def cppp_version() -> str:
    return lib().cppp_version().decode()


# ------------------------------------------------------------------ PP-Tucker (cppp_tucker.h)
class TkCtx:
    """Handle returned by tk_init (include/cppp_tucker.h)."""

    def __init__(self, N, s, R):
        self.h = C.c_void_p()
        self.N, self.s, self.R = N, list(s), list(R)
        self.keep = []

    def canon_shape(self, kept):
        return tuple(self.s[m] if m in kept else self.R[m] for m in range(self.N))

    def __del__(self):
        try:
            tk_destroy(self)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def _tk_check(ctx, status: int):
    if status != 0:
        msg = lib().tk_last_error(ctx.h if ctx is not None else None)
        raise CpppError(status, (msg or b"").decode() or lib().cppp_status_string(status).decode())


def tk_init(X, s: Sequence[int], R: Sequence[int], *, stream=None, flags: int = 0) -> TkCtx:
    """tk_init: X numpy (host) or torch CUDA tensor; ranks R[n] <= s[n]."""
    N = len(s)
    ctx = TkCtx(N, s, R)
    dims = (C.c_int64 * N)(*s)
    ranks = (C.c_int * N)(*R)
    st = C.c_void_p(stream.cuda_stream) if stream is not None else None
    if flags & FLAG_BORROW_TENSOR:
        ctx.keep.append(X)
    _tk_check(None, lib().tk_init(C.byref(ctx.h), _ptr(X), N, dims, ranks, st, flags))
    return ctx


def tk_set_factors(ctx: TkCtx, A) -> None:
    _tk_check(ctx, lib().tk_set_factors(ctx.h, _ptrs([np.ascontiguousarray(a) if isinstance(a, np.ndarray) else a for a in A])))


def tk_update_factors(ctx: TkCtx, A) -> None:
    _tk_check(ctx, lib().tk_update_factors(ctx.h, _ptrs([np.ascontiguousarray(a) if isinstance(a, np.ndarray) else a for a in A])))


def tk_ttmc(ctx: TkCtx):
    """All N TTMcs Y^(n), canonical layout (numpy)."""
    out = [np.empty(ctx.canon_shape({n})) for n in range(ctx.N)]
    _tk_check(ctx, lib().tk_ttmc(ctx.h, _ptrs(out)))
    return out


def tk_pp_build(ctx: TkCtx) -> None:
    _tk_check(ctx, lib().tk_pp_build(ctx.h))


def tk_pp_get_operator(ctx: TkCtx, i: int, j: int) -> np.ndarray:
    out = np.empty(ctx.canon_shape({i, j}))
    _tk_check(ctx, lib().tk_pp_get_operator(ctx.h, i, j, _ptr(out)))
    return out


def tk_pp_get_single(ctx: TkCtx, n: int) -> np.ndarray:
    out = np.empty(ctx.canon_shape({n}))
    _tk_check(ctx, lib().tk_pp_get_single(ctx.h, n, _ptr(out)))
    return out


def tk_pp_update(ctx: TkCtx, n: int) -> np.ndarray:
    out = np.empty(ctx.canon_shape({n}))
    _tk_check(ctx, lib().tk_pp_update(ctx.h, n, _ptr(out)))
    return out


def tk_hosvd(ctx: TkCtx) -> None:
    _tk_check(ctx, lib().tk_hosvd(ctx.h))


def tk_sweep(ctx: TkCtx, eps: float, eps_pp: float) -> dict:
    info = TkSweepInfo()
    _tk_check(ctx, lib().tk_sweep(ctx.h, eps, eps_pp, C.byref(info)))
    return info.as_dict()


def tk_set_phase_override(ctx: TkCtx, phase) -> None:
    if isinstance(phase, str):
        phase = PHASE_BY_NAME[phase]
    _tk_check(ctx, lib().tk_set_phase_override(ctx.h, phase))


def tk_get_factors(ctx: TkCtx):
    out = [np.empty((ctx.s[n], ctx.R[n])) for n in range(ctx.N)]
    _tk_check(ctx, lib().tk_get_factors(ctx.h, _ptrs(out)))
    return out


def tk_get_core(ctx: TkCtx) -> np.ndarray:
    out = np.empty(tuple(ctx.R))
    _tk_check(ctx, lib().tk_get_core(ctx.h, _ptr(out)))
    return out


def tk_destroy(ctx: TkCtx) -> None:
    if ctx is not None and ctx.h:
        lib().tk_destroy(ctx.h)
        ctx.h = C.c_void_p()
        ctx.keep.clear()
