#!/usr/bin/env python3
"""PP-Tucker on one B200: device time of a regular HOOI sweep (Alg. 2 through the
dimension tree), a PP-build sweep (operators + PP sweep) and a PP sweep (Alg. 4 middle step), on
synthetic tensors of the paper's Tucker shapes.  One JSON line per workload.

  python tools/tucker_bench.py [--workloads T6W,T4,T3] [--reps 3]

Workloads (input: a seeded CP tensor of rank 2R + 1% Gaussian noise from the device generator,
content not stated by the paper):
  T6W  N = 6, s = 32, R = 4: the weak-scaling shape at p = 1
  T4   N = 4, s = 100, R = 10
  T3   N = 3, s = 400, R = 10 (mode sizes > 128: random orthonormal start, rank-side Gram)
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1811_10573_b200.cppp as cp  # noqa: E402

WORKLOADS = {"T6W": (6, 32, 4), "T4": (4, 100, 10), "T3": (3, 400, 10)}


def timed(stream, fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), out


def run(name, reps):
    N, s, R = WORKLOADS[name]
    dims, ranks = [s] * N, [R] * N
    stream = torch.cuda.current_stream()
    X = torch.empty(s ** N, dtype=torch.float64, device="cuda")
    r = np.random.default_rng(0)
    Kt = 2 * R
    cp.cppp_generate(X, dims, Kt, [r.uniform(size=(s, Kt)) for _ in range(N)], 2, 0.01, 0, stream=stream)
    ctx = cp.tk_init(X, dims, ranks, stream=stream, flags=cp.FLAG_BORROW_TENSOR)
    if s <= 128:
        init_ms, _ = timed(stream, lambda: cp.tk_hosvd(ctx))
    else:
        cp.tk_set_factors(ctx, [np.linalg.qr(r.standard_normal((s, R)))[0].copy() for _ in range(N)])
        init_ms = None
    times = {"dt": [], "pp-build": [], "pp-approx": []}
    info = {}
    for phase in ["dt", "dt", "pp-build"] + ["pp-approx"] * reps + ["dt"] * reps + ["pp-build"] * (reps - 1):
        cp.tk_set_phase_override(ctx, phase)
        ms, info = timed(stream, lambda: cp.tk_sweep(ctx, 0.0, 0.2))
        times[phase].append(ms)
    med = {k: float(np.median(v[1:] if len(v) > 1 else v)) for k, v in times.items()}
    flops_dt = 4.0 * s ** N * R   # leading order of a regular sweep
    print(json.dumps({"workload": name, "N": N, "s": s, "R": R, "tensor_GB": 8 * s ** N / 1e9,
                      "hosvd_ms": init_ms, "dt_ms": med["dt"], "pp_build_ms": med["pp-build"],
                      "pp_ms": med["pp-approx"], "dt_over_pp": med["dt"] / med["pp-approx"],
                      "dt_leading_gflops": flops_dt / (med["dt"] * 1e-3) / 1e9,
                      "last_residual": info.get("residual")}))
    cp.tk_destroy(ctx)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="T6W,T4,T3")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    for w in a.workloads.split(","):
        run(w, a.reps)


if __name__ == "__main__":
    main()
