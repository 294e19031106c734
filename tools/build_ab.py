"""A/B of the PP build on a config: the fused level-1 -> level-2 build (default) against the plain
Def. pptree build (CPPP_FLAG_NO_FUSED_TTV) -- device time of pp_build_operators (CUDA events, best
of 3) and the largest relative difference between the two builds' operators.

  python tools/build_ab.py [C5] [reps]
"""
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
    name = sys.argv[1] if len(sys.argv) > 1 else "C5"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cfg = G.CONFIGS[name]
    st = torch.cuda.current_stream()
    X = torch.empty(cfg.numel, dtype=torch.float64, device="cuda")
    kind = {"none": 0, "abs": 1, "rel": 2}[cfg.noise_kind]
    cp.cppp_generate(X, cfg.dims, cfg.rank_true, G.true_factors(cfg), kind, cfg.noise, 0, stream=st)
    A0 = [torch.from_numpy(a).cuda() for a in G.initial_factors(cfg)]
    out = {}
    for label, flags in (("fused", 0), ("pptree", cp.FLAG_NO_FUSED_TTV)):
        ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K, stream=st, flags=cp.FLAG_BORROW_TENSOR | flags)
        cp.cp_set_factors(ctx, A0)
        cp.pp_build_operators(ctx)
        best = 1e30
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            cp.pp_build_operators(ctx)
            b.record(st)
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        ops = {(i, j): cp.pp_get_operator(ctx, i, j) for i in range(cfg.N) for j in range(i + 1, cfg.N)}
        out[label] = (best, ops)
        cp.cp_destroy(ctx)
        torch.cuda.empty_cache()
    d = max(float(np.linalg.norm(out["fused"][1][k] - out["pptree"][1][k]) / np.linalg.norm(out["pptree"][1][k]))
            for k in out["fused"][1])
    print({"config": name, "fused_ms": out["fused"][0], "pptree_ms": out["pptree"][0], "max_rel_diff": d})


if __name__ == "__main__":
    main()
