#!/usr/bin/env python3
"""Per-scope device timeline of one CP-ALS-PP run (CPPP_TRACE=1 + FLAG_PROFILE): for the chosen
sweeps, every profiled kernel class with start/end (us from the sweep's first event).

  python tools/trace.py [--config C2] [--sweeps 0,7,8]
"""
import argparse
import os
import sys

os.environ["CPPP_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synthgen as G  # noqa: E402
import paper_1811_10573_b200.cppp as cp  # noqa: E402

NAMES = cp.KCLASS_NAMES


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--sweeps", default="1,7,8")
    ap.add_argument("--flags", type=int, default=0, help="extra CPPP_FLAG_* bits")
    a = ap.parse_args()
    want = {int(x) for x in a.sweeps.split(",")}
    cfg = G.CONFIGS[a.config]
    stream = torch.cuda.current_stream()
    X = torch.empty(cfg.s ** cfg.N, dtype=torch.float64, device="cuda")
    kind = {"none": 0, "abs": 1, "rel": 2}[cfg.noise_kind]
    cp.cppp_generate(X, cfg.dims, cfg.rank_true, G.true_factors(cfg), kind, cfg.noise, 0, stream=stream)
    A0 = [torch.from_numpy(x).cuda() for x in G.initial_factors(cfg)]
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K, stream=stream,
                     flags=cp.FLAG_BORROW_TENSOR | cp.FLAG_PROFILE | a.flags)
    for _ in range(2):   # warm (graphs captured)
        cp.cp_set_factors(ctx, A0)
        for _ in range(cfg.sweeps):
            cp.als_sweep(ctx, 0.0, cfg.eps_pp)
    torch.cuda.synchronize()
    cp.cp_set_factors(ctx, A0)
    r, w = os.pipe()
    saved = os.dup(2)
    for i in range(cfg.sweeps):
        os.dup2(w, 2)
        info = cp.als_sweep(ctx, 0.0, cfg.eps_pp)
        os.dup2(saved, 2)
        os.write(w, b"end\n")
        data = b""
        while not data.endswith(b"end\n"):
            data += os.read(r, 1 << 20)
        if i not in want:
            continue
        print(f"sweep {i} phase {info['phase']} device {info['seconds'] * 1e6:.1f} us")
        rows = []
        for line in data.decode().splitlines():
            p = line.split()
            if len(p) == 5 and p[0] == "trace":
                rows.append((float(p[3]), float(p[4]), NAMES[int(p[2])]))
        for t0, t1, nm in sorted(rows):
            print(f"   {t0:9.1f} {t1:9.1f} {t1 - t0:8.1f}  {nm}")
    cp.cp_destroy(ctx)


if __name__ == "__main__":
    main()
