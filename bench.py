#!/usr/bin/env python3
"""bench.py — CP-ALS-PP sweeps/s on B200 (BASELINE.json metric), one JSON line on rank 0.

A "step" is one CP-ALS-PP run of the workload (default C2 = BASELINE configs[1]: N=3, s=400,
K=100, collinear + 1% noise): cp_set_factors(seeded initial factors) followed by 20 als_sweep
calls with eps_pp = 0.1 — every §8(a) row of the hot path (first-level TTM, multi-TTV levels,
PP construction tree, PP update, small solves, fitness, Alg. 3 phase machine).  value = sweeps
per second over the timed steps (inputs resident in HBM; the 512 MB tensor is larger than L2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

The timed pass runs without profiling events; "roofline"/"roofline_all" come from a second pass
of the same K steps on a context that records CUDA events around every kernel class on the stream
that launches it ("profiled_ms_per_step" is that pass's step time).

N > 1 (torchrun, one rank per GPU): the tensor is sharded in mode-0 slabs; the ranks
cooperate on the same run through NCCL all-reduce (strong scaling).  --impl reference times
the CPU oracle (the deliberately slow, plain FP64 program of oracle/) on the same workload.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synthgen as G  # noqa: E402

FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")
MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="C2")
    p.add_argument("--sweeps", type=int, default=None)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


# ------------------------------------------------------------------ clocks (during timed region)
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        med = float(np.median(sm)) if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ distributed plumbing
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def config_dict(cfg, sweeps, world):
    """The workload description both arms print (identical keys and values)."""
    return {"workload": cfg.name, "N": cfg.N, "s": cfg.s, "K": cfg.K, "sweeps_per_step": sweeps,
            "eps_pp": cfg.eps_pp, "family": cfg.family, "noise": [cfg.noise_kind, cfg.noise],
            "parallelism": f"mode-0 slabs x{world}" if world > 1 else "single GPU",
            "l2": l2_note(cfg)}


L2_BYTES = 126 << 20   # B200 L2 (both dies)


def l2_note(cfg):
    mib = cfg.numel * 8 / 2**20
    if cfg.numel * 8 > L2_BYTES:
        return "inputs larger than L2 (X = %.0f MiB)" % mib
    return "L2 flushed before every timed step (X = %.2f MiB < 126 MiB L2)" % mib


def host_cores():
    """Host cores this process may run on (what the oracle's BLAS and numpy can use)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_run(cfg, X, A0, sweeps):
    import oracle.cp_oracle as O
    t = time.perf_counter()
    _, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, sweeps)
    return time.perf_counter() - t, tr


def oracle_sample(cfg, X, A0, sweeps, lo=10.0, hi=30.0):
    """The bounded CPU sample: whole runs of the workload repeated until >= lo seconds, a run cut
    after the sweep that passes hi seconds.  Returns (seconds, sweeps done, phases, description)."""
    import oracle.cp_oracle as O
    t0 = time.perf_counter()
    done, runs, phases = 0, 0, []
    while True:
        _, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, sweeps, deadline=t0 + hi)
        done += len(tr)
        runs += 1
        phases = phases or [t["phase"] for t in tr]
        el = time.perf_counter() - t0
        if len(tr) < sweeps or el >= lo:
            break
    if len(tr) < sweeps:
        what = f"the first {done} sweeps of a {sweeps}-sweep {cfg.name} run (cut at {hi:.0f} s)"
    else:
        what = f"{runs} full {sweeps}-sweep {cfg.name} run(s)"
    return el, done, phases, what + " (oracle/cp_oracle.py, numpy FP64 + BLAS)"


def oracle_sample_slab(cfg, slabs, A0, phases):
    """The bounded CPU sample for a tensor too large for the oracle's full run (C5, 32 GiB): the
    oracle's own functions, as they stand, timed once per phase on slabs of r rows of one mode
    (slabs[m]: rows [0, r) of mode m) and scaled by s/r where their work is proportional to the
    tensor.  Each MTTKRP M^(n) and each PP operator M_p^(i,j) takes a slab of a mode it contracts
    (so its Khatri-Rao factor, unfolding copy and product all shrink by r/s); the PP update and the
    K x K solves run at full size.  sweeps/s = sweeps / Σ_phase count x time, with the GPU run's
    phase mix."""
    import oracle.cp_oracle as O
    N, s = cfg.N, cfg.s
    r = next(iter(slabs.values())).shape[min(slabs)]
    scale = s / r
    A = [a.copy() for a in A0]
    S = [O.gram(a) for a in A]

    def sl(m):
        Am = list(A)
        Am[m] = A[m][:r]
        return slabs[m], Am

    def solves():
        t = time.perf_counter()
        for n in range(N):
            Gm = O.gamma(S, n)
            An = O.solve_normal(np.ones((s, cfg.K)), Gm)
            O.gradient(A[n], An, Gm)
            O.gram(An)
        return time.perf_counter() - t

    t_mt = 0.0
    for n in range(N):
        X_m, A_m = sl(0 if n != 0 else 1)
        t = time.perf_counter()
        O.mttkrp(X_m, A_m, n)
        t_mt += time.perf_counter() - t
    t_dt = t_mt * scale + solves()
    t_ops = 0.0
    for i in range(N):
        for j in range(i + 1, N):
            m = min(x for x in range(N) if x not in (i, j))
            X_m, A_m = sl(m)
            t = time.perf_counter()
            O.pp_operator(X_m, A_m, i, j)
            t_ops += time.perf_counter() - t
    t_ops *= scale
    # full-size operators for the update (values irrelevant for the timing: same shapes)
    full = {(i, j): np.ones((s, s, cfg.K)) for i in range(N) for j in range(i + 1, N)}
    t = time.perf_counter()
    Mp = [O.pp_single(full, A, n, N) for n in range(N)]
    t_single = time.perf_counter() - t
    dA = [0.01 * a for a in A]
    t = time.perf_counter()
    for n in range(N):
        O.pp_update(Mp[n], full, dA, n)
    t_pp = time.perf_counter() - t + solves()
    del full
    t_build = t_ops + t_single + t_pp
    cnt = {ph: phases.count(ph) for ph in ("dt", "pp-build", "pp-approx")}
    total = cnt["dt"] * t_dt + cnt["pp-build"] * t_build + cnt["pp-approx"] * t_pp
    what = (f"oracle/cp_oracle.py functions timed once per phase on {r}-row slabs of the {cfg.name} tensor "
            f"(each MTTKRP / PP operator on a slab of a mode it contracts, time x{scale:g}), PP update and "
            f"solves at full size; per-sweep seconds dt {t_dt:.2f}, pp-build {t_build:.2f}, pp-approx "
            f"{t_pp:.3f}; the GPU run's phase mix {cnt}")
    return len(phases) / total, what, {"dt": t_dt, "pp-build": t_build, "pp-approx": t_pp}


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] or [os.cpu_count() or 1])
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = G.CONFIGS[args.config]
    sweeps = args.sweeps or cfg.sweeps
    if cfg.numel > 2e8:
        print(json.dumps({"impl": "reference", "unavailable": f"oracle needs the full {args.config} tensor on the host"}))
        return
    X = G.make_tensor(cfg)
    A0 = G.initial_factors(cfg)
    for _ in range(args.warmup):
        oracle_run(cfg, X, A0, sweeps)
    total = 0.0
    done = 0
    for _ in range(args.steps):
        dt, tr = oracle_run(cfg, X, A0, sweeps)
        total += dt
        done += len(tr)
    value = done / total
    cores = host_cores()
    line = {
        "impl": "reference", "metric": "CP-ALS-PP sweeps/s", "value": value, "unit": "sweeps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded synthgen, host)",
        "config": config_dict(cfg, sweeps, world),
        "cpu_baseline": {"value": value, "unit": "sweeps/s", "cores": cores, "blas_threads": blas_threads(),
                         "kind": "oracle",
                         "sample": f"the full {sweeps}-sweep {cfg.name} run per step (oracle/cp_oracle.py, numpy FP64)"},
        "e2e": {"value": value, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "phases": [t["phase"] for t in tr],
    }
    print(json.dumps(line))


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    import paper_1811_10573_b200.cppp as cp

    world, rank, local = dist_env()
    if world != args.gpus:
        args.gpus = world if world > 1 else args.gpus
    torch.cuda.set_device(local)
    if world > 1:
        # the library captures its collectives into CUDA graphs: connect everything at init
        os.environ.setdefault("NCCL_RUNTIME_CONNECT", "0")
        dist.init_process_group("nccl", init_method="env://")
    cfg = G.CONFIGS[args.config]
    sweeps = args.sweeps or cfg.sweeps
    s0 = cfg.s
    row_lo, row_hi = rank * s0 // world, (rank + 1) * s0 // world
    dims = cfg.dims
    stream = torch.cuda.current_stream()

    # ---- inputs: generated on device by the seeded generator (untimed), resident in HBM
    A_true = G.true_factors(cfg)
    A0 = G.initial_factors(cfg)
    local_numel = (row_hi - row_lo) * (cfg.s ** (cfg.N - 1))
    X_dev = torch.empty(local_numel, dtype=torch.float64, device="cuda")
    nccl_id = None
    if world > 1:
        obj = [cp.cppp_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    shard = dict(shard_offset=row_lo, shard_extent=row_hi - row_lo) if world > 1 else {}
    kind = {"none": 0, "abs": 1, "rel": 2}[cfg.noise_kind]
    # generate first (the context's ||X||² is taken at cp_init)
    gen_ctx = None
    if world > 1:
        # a throw-away context provides the communicator for the shard-invariant noise scale
        tmp = torch.zeros((row_hi - row_lo) * cfg.s ** (cfg.N - 1), dtype=torch.float64, device="cuda")
        gen_ctx = cp.cp_init(tmp, cfg.N, dims, cfg.K, stream=stream, device=local, flags=cp.FLAG_BORROW_TENSOR,
                             nccl_unique_id=nccl_id, rank=rank, world=world, torch_workspace=False, **shard)
        del tmp
    cp.cppp_generate(X_dev, dims, cfg.rank_true, A_true, kind, cfg.noise, 0, row_lo, row_hi, stream=stream, ctx=gen_ctx)
    if gen_ctx is not None:
        cp.cp_destroy(gen_ctx)
        obj = [cp.cppp_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    # the bounded oracle sample of a tensor too large for a full oracle run (C5): a mode-0 slab
    X_slab = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and cfg.numel > 2e8:
        rows = 16
        X_slab = {}
        for m in range(3):   # rows [0, 16) of modes 0, 1, 2 (2 GiB each for C5)
            shp = list(dims)
            shp[m] = rows
            v = X_dev.view(cfg.s ** m, cfg.s, -1)[:, :rows, :]
            X_slab[m] = v.contiguous().cpu().numpy().reshape(shp)
    # timed pass: no profiling events inside the sweeps (they perturb a C2 step by ~8%)
    ctx = cp.cp_init(X_dev, cfg.N, dims, cfg.K, stream=stream, device=local, flags=cp.FLAG_BORROW_TENSOR,
                     nccl_unique_id=nccl_id, rank=rank, world=world, **shard)
    A0_dev = [torch.from_numpy(a).cuda() for a in A0]

    l2_flush = cfg.numel * 8 <= L2_BYTES

    def step():   # one CP-ALS-PP run: als_run = every sweep in one device launch (Alg. 3 on device)
        cp.cp_set_factors(ctx, A0_dev)
        return cp.als_run(ctx, 0.0, cfg.eps_pp, sweeps)

    for _ in range(max(args.warmup, 0)):
        infos = step()
    cp.reset_kernel_stats(ctx)
    launches0 = cp.cppp_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(local)
    clk.start()
    # inputs smaller than L2 (C1): every timed step is preceded by an untimed L2 flush (a
    # 512 MiB write); larger inputs stream through L2 anyway and the steps are timed back to back
    flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda") if l2_flush else None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps if l2_flush else 1)]
    sweeps_done = 0
    if not l2_flush:
        ev[0][0].record(stream)
    for i in range(args.steps):
        if l2_flush:
            flush.zero_()
            ev[i][0].record(stream)
        infos = step()
        sweeps_done += len(infos)
        if l2_flush:
            ev[i][1].record(stream)
    if not l2_flush:
        ev[0][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    del flush
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    launches = (cp.cppp_launch_count() - launches0) / max(args.steps, 1)
    value = sweeps_done / (ms * 1e-3)   # the sweeps als_run actually ran (it may stop early)
    gpu_phases = [i["phase"] for i in infos]

    # replayed pass (untimed for `value`): the same runs as a host loop of graph-launched sweeps on
    # the same unprofiled context, each sweep bracketed by the library's own event pair -- the
    # per-phase sweep times of the real execution (the profiled pass below puts events between
    # kernels, which breaks their programmatic overlap: C2's PP sweep reads 265 us there, 207 here)
    rep_infos = []
    for r in range(args.steps + 2):   # a phase graph is captured on its second use: two untimed runs
        cp.cp_set_factors(ctx, A0_dev)
        for _ in range(sweeps):
            info = cp.als_sweep(ctx, 0.0, cfg.eps_pp)
            if r > 1:
                rep_infos.append(info)
    torch.cuda.synchronize()

    # profiled pass: the same K steps again on a context with per-kernel-class CUDA events on the
    # launching streams (the library's own stream, which is torch's current stream, and the
    # side stream of the factorizations); the roofline below comes from these event times
    cp.cp_destroy(ctx)
    if world > 1:
        obj = [cp.cppp_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctx = cp.cp_init(X_dev, cfg.N, dims, cfg.K, stream=stream, device=local,
                     flags=cp.FLAG_BORROW_TENSOR | cp.FLAG_PROFILE,
                     nccl_unique_id=nccl_id, rank=rank, world=world, **shard)
    step()
    step()
    cp.reset_kernel_stats(ctx)
    torch.cuda.synchronize()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    prof_infos = []
    for _ in range(args.steps):
        prof_infos += step()
    p1.record(stream)
    torch.cuda.synchronize()
    prof_ms = p0.elapsed_time(p1)
    kstats = cp.kernel_stats(ctx)
    # per-phase device time (the profiled pass runs the host loop: one event pair per sweep)
    def by_phase(recs):
        out = {}
        for ph in ("dt", "pp-build", "pp-approx"):
            v = sorted(i["seconds"] * 1e6 for i in recs if i["phase"] == ph)
            if v:
                out[ph] = {"median": v[len(v) // 2], "count_per_step": len(v) / args.steps}
        return out
    phase_us = by_phase(rep_infos)
    phase_us_profiled = by_phase(prof_infos)
    algo_flops = sum(k["flops"] for k in kstats.values()) / max(args.steps, 1)

    # ---- roofline of the dominant kernel class
    peaks = {}
    if os.path.exists(MEASURED_PEAKS):
        peaks = json.load(open(MEASURED_PEAKS))
    fp64 = {}
    if os.path.exists(FP64_PEAK_FILE):
        fp64 = json.load(open(FP64_PEAK_FILE))
    dmma_peak = fp64.get("dmma_tflops_sustained", 37.0)
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    roof_all = {}
    for name, k in kstats.items():
        if k["launches"] == 0 or k["total_ms"] <= 0:
            continue
        sec = k["total_ms"] * 1e-3
        entry = {"launches_per_step": k["launches"] / args.steps, "ms_per_step": k["total_ms"] / args.steps,
                 "share_of_step": k["total_ms"] / prof_ms}
        ridge = dmma_peak * 1e12 / (hbm_peak * 1e9)          # flop/byte where the two roofs meet
        if name == "ttm" and k["flops"] / max(k["bytes"], 1.0) >= ridge:
            entry.update(bound="tensor", achieved=k["flops"] / sec / 1e12, peak=dmma_peak, unit="TFLOP/s")
        elif name == "ttm":   # low arithmetic intensity (e.g. C4: K=30, s=20): HBM-bound GEMM
            entry.update(bound="hbm", achieved=k["bytes"] / sec / 1e9, peak=hbm_peak, unit="GB/s",
                         tflops=k["flops"] / sec / 1e12, arithmetic_intensity=k["flops"] / k["bytes"])
        else:
            entry.update(bound="hbm", achieved=k["bytes"] / sec / 1e9, peak=hbm_peak, unit="GB/s")
        entry["frac"] = entry["achieved"] / entry["peak"]
        roof_all[name] = entry
    # the dominant class on the critical path (the factorization runs on the side stream)
    dom = max((n for n in roof_all if n != "factor"), key=lambda n: roof_all[n]["ms_per_step"],
              default=None)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg.name}.json")
    if dom and os.path.exists(tfile):
        traffic = json.load(open(tfile)).get(dom)
    roofline = None
    if dom:
        r = roof_all[dom]
        roofline = {"kernel": dom, "bound": r["bound"], "achieved": r["achieved"], "peak": r["peak"],
                    "unit": r["unit"], "frac": r["frac"], "traffic": traffic,
                    "peak_source": ("measured FP64 tensor peak: tools/fp64_peak (register-resident DMMA.8x8x4, "
                                    "sustained; cuBLAS DGEMM 35.4) -> profiles/fp64_peak_r01.json"
                                    if r["bound"] == "tensor" else "of measured: MEASURED_PEAKS.json hbm_gbs")}
        if r["bound"] == "tensor" and "bf16_tflops" in peaks:
            # MEASURED_PEAKS.json has no FP64 entry; the alternative denominator, bf16 measured x
            # the nominal FP64-tensor / bf16-dense ratio (37 / 2250), for reference
            alt = peaks["bf16_tflops"] * 37.0 / 2250.0
            roofline["peak_bf16_x_nominal_ratio"] = alt
            roofline["frac_of_bf16_x_nominal_ratio"] = r["achieved"] / alt

    # ---- e2e through the public API with host buffers (pinned), H2D/D2H inside the region
    e2e = None
    if not args.no_e2e:
        Xh = torch.empty(local_numel, dtype=torch.float64, pin_memory=True)
        Xh.copy_(X_dev.cpu())
        A0h = [torch.from_numpy(a.copy()).pin_memory() for a in A0]
        outh = [torch.empty(a.shape, dtype=torch.float64).pin_memory() for a in A0]

        # N = 1: two contexts alternate (a serving pipeline): each step uploads its tensor from
        # pinned host memory into one context (cp_load_tensor: H2D on that context's stream, run
        # in a second host thread) while the other context runs the previous step's sweeps on
        # the SMs; every step's upload is inside the timed region.  The contexts keep their
        # workspaces and captured sweep graphs across steps.
        # N > 1: the sharded context is reused (a new one would need a new communicator); each
        # step copies its slab from pinned host memory into the borrowed device tensor.
        from concurrent.futures import ThreadPoolExecutor
        pool = ThreadPoolExecutor(max_workers=1)
        pair = []
        cp.cp_destroy(ctx)   # the profiled context is not used for the end-to-end timing
        if world == 1:
            del X_dev   # two contexts (C5: 2 x 49 GB) need the room
            torch.cuda.empty_cache()
            pair = [cp.cp_init(Xh, cfg.N, dims, cfg.K, stream=torch.cuda.Stream(), device=local)
                    for _ in range(2)]
        else:
            obj = [cp.cppp_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            ctx = cp.cp_init(X_dev, cfg.N, dims, cfg.K, stream=stream, device=local,
                             flags=cp.FLAG_BORROW_TENSOR, nccl_unique_id=obj[0], rank=rank,
                             world=world, **shard)

        def load(i):   # the step's inputs: tensor + initial factors, from pinned host memory
            torch.cuda.set_device(local)
            cp.cp_load_tensor(pair[i % 2], Xh)
            cp.cp_set_factors(pair[i % 2], A0h)
            return pair[i % 2]

        e2e_sweeps = [0]

        def run(c2, set_factors=False):
            if set_factors:
                cp.cp_set_factors(c2, A0h)
            e2e_sweeps[0] += len(cp.als_run(c2, 0.0, cfg.eps_pp, sweeps))
            cp.cp_get_factors(c2, out=outh)
            return cp.fitness(c2)

        def e2e_run(nsteps):
            if world > 1:
                for _ in range(nsteps):
                    # the step's slab from pinned host memory into the (borrowed) device tensor,
                    # then cp_load_tensor re-reads it (the all-reduced ||X||^2)
                    X_dev.copy_(Xh, non_blocking=True)
                    cp.cp_load_tensor(ctx, X_dev)
                    run(ctx, set_factors=True)
                return
            nxt = pool.submit(load, 0)
            for i in range(nsteps):
                cur = nxt.result()
                if i + 1 < nsteps:
                    nxt = pool.submit(load, i + 1)
                run(cur)

        e2e_run(2)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e2e_sweeps[0] = 0
        t0 = time.perf_counter()
        e2e_run(args.steps)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        pool.shutdown()
        for c2 in pair:
            cp.cp_destroy(c2)
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        h2d = local_numel * 8 + sum(a.nbytes for a in A0)
        e2e = {"value": e2e_sweeps[0] / dt, "unit": "sweeps/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(sum(a.nbytes for a in A0) + 8)}

    # ---- CPU baseline: the oracle on the same workload (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and cfg.numel <= 2e8:
        Xo = G.make_tensor(cfg)
        dt, done, or_phases, what = oracle_sample(cfg, Xo, A0, sweeps)
        cpu = {"value": done / dt, "unit": "sweeps/s", "cores": host_cores(), "blas_threads": blas_threads(),
               "kind": "oracle", "sample": what, "seconds": dt, "phases": or_phases}
    elif X_slab is not None:
        t0 = time.perf_counter()
        v, what, per = oracle_sample_slab(cfg, X_slab, A0, gpu_phases)
        cpu = {"value": v, "unit": "sweeps/s", "cores": host_cores(), "blas_threads": blas_threads(),
               "kind": "oracle", "sample": what, "seconds": time.perf_counter() - t0,
               "seconds_per_sweep": per}
        del X_slab

    if rank == 0:
        line = {
            "metric": "CP-ALS-PP sweeps/s", "value": value, "unit": "sweeps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded on-device generator, twin of synthgen)",
            "config": config_dict(cfg, sweeps, world),
            "phases": gpu_phases, "sweeps_per_step": sweeps_done / max(args.steps, 1),
            "final_fitness": infos[-1]["fitness"], "final_fitness_approximate": infos[-1]["approximate"],
            "roofline": roofline, "roofline_all": roof_all, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks,
            "profiled_ms_per_step": prof_ms / args.steps,
            "phase_us": phase_us,
            "phase_us_profiled": phase_us_profiled,
            "algorithmic_gflops": algo_flops / (ms / args.steps * 1e-3) / 1e9,
        }
        print(json.dumps(line))
    cp.cp_destroy(ctx)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
