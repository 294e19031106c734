#!/usr/bin/env python3
"""Overlap check for the pipelined e2e loop: upload alone, sweeps alone, both concurrently."""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synthgen as G  # noqa: E402
import paper_1811_10573_b200.cppp as cp  # noqa: E402

cfg = G.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
X = torch.empty(cfg.s ** cfg.N, dtype=torch.float64, device="cuda")
kind = {"none": 0, "abs": 1, "rel": 2}[cfg.noise_kind]
cp.cppp_generate(X, cfg.dims, cfg.rank_true, G.true_factors(cfg), kind, cfg.noise, 0)
Xh = torch.empty(X.numel(), dtype=torch.float64, pin_memory=True)
Xh.copy_(X.cpu())
A0 = [torch.from_numpy(a).pin_memory() for a in G.initial_factors(cfg)]
a, b = (cp.cp_init(Xh, cfg.N, cfg.dims, cfg.K, stream=torch.cuda.Stream()) for _ in range(2))


def run(c):
    cp.cp_set_factors(c, A0)
    for _ in range(cfg.sweeps):
        cp.als_sweep(c, 0.0, cfg.eps_pp)


for _ in range(2):
    run(a)
    cp.cp_load_tensor(b, Xh)
torch.cuda.synchronize()
t = time.perf_counter(); cp.cp_load_tensor(b, Xh); t_load = time.perf_counter() - t
t = time.perf_counter(); run(a); t_run = time.perf_counter() - t
th = threading.Thread(target=lambda: (cp.cp_load_tensor(b, Xh), cp.cp_set_factors(b, A0)))
t = time.perf_counter(); th.start(); run(a); th.join(); t_both = time.perf_counter() - t
print(f"{cfg.name}: load {t_load * 1e3:.2f} ms ({Xh.numel() * 8 / t_load / 1e9:.1f} GB/s), "
      f"run {t_run * 1e3:.2f} ms, both {t_both * 1e3:.2f} ms")

# where does the concurrent run lose time? per-sweep wall / device time with a load in flight
cp.cp_set_factors(a, A0)
torch.cuda.synchronize()
th = threading.Thread(target=lambda: cp.cp_load_tensor(b, Xh))
th.start()
rows = []
for i in range(cfg.sweeps):
    t = time.perf_counter()
    info = cp.als_sweep(a, 0.0, cfg.eps_pp)
    rows.append((i, info["phase"], (time.perf_counter() - t) * 1e3, info["seconds"] * 1e3))
th.join()
print("  sweep phase wall_ms device_ms:", " ".join(f"{i}:{p[:3]}:{w:.2f}/{d:.2f}" for i, p, w, d in rows))
