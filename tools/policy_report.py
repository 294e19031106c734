"""f3 switching-policy report: for each config, one 20-sweep run with Alg. 3's ε_pp test alone and
with CPPP_POLICY_BOUND at a few tolerances; prints the phase mix, the device time of the run and
the exact final residual (fitness_exact: one exact MTTKRP pass at the final factors).

  python tools/policy_report.py [C1 C2 C3 C4] [--tols 1,0.3,0.1]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synthgen as G  # noqa: E402
import paper_1811_10573_b200.cppp as cp  # noqa: E402


def main():
    names = [a for a in sys.argv[1:] if not a.startswith("--") and not a[0].isdigit()] or ["C1", "C2", "C3", "C4"]
    tols = [1e3, 1e2, 10.0, 1.0]
    if "--tols" in sys.argv:
        tols = [float(x) for x in sys.argv[sys.argv.index("--tols") + 1].split(",")]
    st = torch.cuda.current_stream()
    for name in names:
        cfg = G.CONFIGS[name]
        X = torch.empty(cfg.numel, dtype=torch.float64, device="cuda")
        kind = {"none": 0, "abs": 1, "rel": 2}[cfg.noise_kind]
        cp.cppp_generate(X, cfg.dims, cfg.rank_true, G.true_factors(cfg), kind, cfg.noise, 0, stream=st)
        A0 = [torch.from_numpy(a).cuda() for a in G.initial_factors(cfg)]
        rows = []
        for pol, tol in [(cp.POLICY_EPS_PP, 0.0)] + [(cp.POLICY_BOUND, t) for t in tols]:
            ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K, stream=st, flags=cp.FLAG_BORROW_TENSOR)
            cp.cp_set_pp_policy(ctx, pol, tol)
            for _ in range(2):   # warm (graphs), then the measured run
                cp.cp_set_factors(ctx, A0)
                infos = cp.als_run(ctx, 0.0, cfg.eps_pp, cfg.sweeps)
            f, r2 = cp.fitness_exact(ctx)
            ph = [i["phase"] for i in infos]
            bounds = [i["pp_bound"] for i in infos if i["phase"] != "dt"]
            rows.append({"policy": "eps_pp" if pol == cp.POLICY_EPS_PP else f"bound<{tol:g}",
                         "dt": ph.count("dt"), "pp_build": ph.count("pp-build"),
                         "pp_approx": ph.count("pp-approx"), "run_ms": 1e3 * sum(i["seconds"] for i in infos),
                         "final_rel_residual": (max(r2, 0.0) / float((X * X).sum())) ** 0.5,
                         "monitor_max": max(bounds) if bounds else None,
                         "worst_max_rel_dA": max(i["max_rel_dA"] for i in infos),
                         "last_phase": ph[-1]})
            cp.cp_destroy(ctx)
        print(json.dumps({"config": name, "runs": rows}), flush=True)
        del X
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
