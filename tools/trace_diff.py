"""Diagnostic: per-sweep differences between the CUDA path and the oracle on a replayed phase
schedule (the quantities tests/test_gpu_*.py compare), one JSON line per config.

  python tools/trace_diff.py C1 C2mini C3mini ... [--sweeps 20] [--perturb]

--perturb also runs the oracle from initial factors perturbed by one ulp (np.nextafter), which
measures how far two correct FP64 evaluations of the same trajectory drift apart (the
conditioning of the trace) -- the yardstick for the trace tolerances in DESIGN.md §3.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle.cp_oracle as O  # noqa: E402
import synthgen as G  # noqa: E402


def diffs(tr_a, tr_b, Aa, Ab):
    out = []
    for a, b in zip(tr_a, tr_b):
        nx2 = a["normX_sq"]
        rho = max(0.0, a["residual_sq"]) ** 0.5 / nx2 ** 0.5
        out.append(dict(
            sweep=a["sweep"], phase=a["phase"], rho=rho,
            dfit=abs(a["fitness"] - b["fitness"]),
            dr2=abs(a["residual_sq"] - b["residual_sq"]) / nx2,
            r2=a["residual_sq"] / nx2,
            dgn=abs(a["grad_norm_sum"] - b["grad_norm_sum"]) / max(abs(a["grad_norm_sum"]), 1e-300),
            dmr=abs(a["max_rel_dA"] - b["max_rel_dA"]) / max(abs(a["max_rel_dA"]), 1e-300),
            mr=a["max_rel_dA"]))
    fac = [float(np.linalg.norm(x - y) / np.linalg.norm(x)) for x, y in zip(Aa, Ab)]
    return out, fac


def main():
    names = [a for a in sys.argv[1:] if not a.startswith("--")]
    sweeps = 20
    if "--sweeps" in sys.argv:
        sweeps = int(sys.argv[sys.argv.index("--sweeps") + 1])
    perturb = "--perturb" in sys.argv
    gpu = "--no-gpu" not in sys.argv
    if gpu:
        import torch
        import paper_1811_10573_b200.cppp as cp
    for name in names:
        cfg = G.CONFIGS[name]
        X = G.make_tensor(cfg)
        A0 = G.initial_factors(cfg)
        t0 = time.time()
        Aor, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, sweeps)
        t_or = time.time() - t0
        rec = {"config": name, "oracle_s": t_or, "phases": [t["phase"] for t in tr]}
        if gpu:
            Xd = torch.from_numpy(np.ascontiguousarray(X).reshape(-1)).cuda()
            ctx = cp.cp_init(Xd, cfg.N, cfg.dims, cfg.K, stream=torch.cuda.current_stream(),
                             flags=cp.FLAG_BORROW_TENSOR)
            cp.cp_set_factors(ctx, A0)
            gt = []
            for t in tr:
                cp.cp_set_phase_override(ctx, t["phase"])
                i = cp.als_sweep(ctx, 0.0, cfg.eps_pp)
                i["normX_sq"] = t["normX_sq"]
                gt.append(i)
            Ag = cp.cp_get_factors(ctx)
            d, fac = diffs(tr, gt, Aor, Ag)
            rec["gpu"] = d
            rec["gpu_factors_rel"] = fac
            cp.cp_destroy(ctx)
        if perturb:
            A1 = [np.nextafter(a, np.inf) for a in A0]
            Ap, trp = O.pp_cp_als(X, A1, 0.0, cfg.eps_pp, sweeps, phase_override=[t["phase"] for t in tr])
            d, fac = diffs(tr, trp, Aor, Ap)
            rec["ulp"] = d
            rec["ulp_factors_rel"] = fac
        for key in ("gpu", "ulp"):
            if key in rec:
                m = {q: max(x[q] for x in rec[key]) for q in ("dfit", "dr2", "dgn", "dmr")}
                rec[key + "_max"] = m
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
