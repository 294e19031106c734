"""A minimal driver for ncu captures of single kernels at a config's full size: one exact MTTKRP
pass (the first-level GEMMs, the multi-TTVs), one PP build and one PP update of every mode.

  ncu --set full -k regex:ttm_dmma -c 1 python tools/ncu_target.py C2
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthgen as G  # noqa: E402
import paper_1811_10573_b200.cppp as cp  # noqa: E402


def main():
    cfg = G.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
    st = torch.cuda.current_stream()
    X = torch.empty(cfg.numel, dtype=torch.float64, device="cuda")
    kind = {"none": 0, "abs": 1, "rel": 2}[cfg.noise_kind]
    cp.cppp_generate(X, cfg.dims, cfg.rank_true, G.true_factors(cfg), kind, cfg.noise, 0, stream=st)
    A0 = G.initial_factors(cfg)
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K, stream=st, flags=cp.FLAG_BORROW_TENSOR)
    cp.cp_set_factors(ctx, A0)
    cp.mttkrp_dt(ctx)
    cp.pp_build_operators(ctx)
    r = np.random.default_rng(1)
    cp.cp_update_factors(ctx, [a * (1 + 0.01 * r.standard_normal(a.shape)) for a in A0])
    for n in range(cfg.N):
        cp.pp_update(ctx, n)
    torch.cuda.synchronize()
    cp.cp_destroy(ctx)


if __name__ == "__main__":
    main()
