#!/usr/bin/env python3
"""Where does a bench step go?  Per-sweep device time (the library's ev_a..ev_b) against the
host wall clock, with and without FLAG_PROFILE, for one config.

  python tools/timeline.py [--config C2] [--reps 3]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthgen as G  # noqa: E402
import paper_1811_10573_b200.cppp as cp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--flags", type=int, default=0, help="extra CPPP_FLAG_* bits")
    ap.add_argument("--run", action="store_true", help="also time als_run (one launch per run)")
    a = ap.parse_args()
    cfg = G.CONFIGS[a.config]
    stream = torch.cuda.current_stream()
    X = torch.empty(cfg.s ** cfg.N, dtype=torch.float64, device="cuda")
    kind = {"none": 0, "abs": 1, "rel": 2}[cfg.noise_kind]
    cp.cppp_generate(X, cfg.dims, cfg.rank_true, G.true_factors(cfg), kind, cfg.noise, 0, stream=stream)
    A0 = [torch.from_numpy(x).cuda() for x in G.initial_factors(cfg)]
    for flags, name in ((cp.FLAG_BORROW_TENSOR | a.flags, "plain"),
                        (cp.FLAG_BORROW_TENSOR | cp.FLAG_PROFILE | a.flags, "profile")):
        ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K, stream=stream, flags=flags)
        for r in range(a.reps + 2):
            cp.cp_set_factors(ctx, A0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            t0 = time.perf_counter()
            infos, walls = [], []
            for _ in range(cfg.sweeps):
                t = time.perf_counter()
                infos.append(cp.als_sweep(ctx, 0.0, cfg.eps_pp))
                walls.append(time.perf_counter() - t)
            e1.record(stream)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            ms = e0.elapsed_time(e1)
            if r < 2:
                continue
            dev = [i["seconds"] * 1e3 for i in infos]
            by = {}
            for i, d, w in zip(infos, dev, walls):
                b = by.setdefault(i["phase"], [0, 0.0, 0.0])
                b[0] += 1
                b[1] += d
                b[2] += w * 1e3
            print(f"[{name}] {a.config} step {ms:.3f} ms (wall {wall * 1e3:.3f}); device in sweeps "
                  f"{sum(dev):.3f} ms; gaps {ms - sum(dev):.3f} ms")
            for ph, (n, d, w) in by.items():
                print(f"    {ph:10s} x{n:2d}  device per sweep {1e3 * d / n:9.1f} us"
                      f"  wall per sweep {1e3 * w / n:9.1f} us")
        cp.cp_destroy(ctx)
    if a.run:
        ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K, stream=stream, flags=cp.FLAG_BORROW_TENSOR | a.flags)
        for r in range(a.reps + 2):
            cp.cp_set_factors(ctx, A0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            infos = cp.als_run(ctx, 0.0, cfg.eps_pp, cfg.sweeps)
            e1.record(stream)
            torch.cuda.synchronize()
            if r >= 2:
                print(f"[als_run] {a.config} step {e0.elapsed_time(e1):.3f} ms "
                      f"({len(infos)} sweeps, one launch)")
        cp.cp_destroy(ctx)


if __name__ == "__main__":
    main()
