"""Prints the bit patterns of a replayed-schedule trace and of the final factors (one JSON line),
so two library configurations (e.g. CPPP_OLD_CHOL=1 vs the default) can be compared bit for bit
from separate processes (the A/B environment switches are read once per process).

  python tools/trace_bits.py C2mini [sweeps]
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle.cp_oracle as O  # noqa: E402
import synthgen as G  # noqa: E402
import paper_1811_10573_b200.cppp as cp  # noqa: E402


def main():
    name = sys.argv[1]
    sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    cfg = G.CONFIGS[name]
    X = G.make_tensor(cfg)
    A0 = G.initial_factors(cfg)
    _, tr = O.pp_cp_als(X, A0, 0.0, cfg.eps_pp, sweeps)
    ctx = cp.cp_init(X, cfg.N, cfg.dims, cfg.K)
    cp.cp_set_factors(ctx, A0)
    fits = []
    for t in tr:
        cp.cp_set_phase_override(ctx, t["phase"])
        i = cp.als_sweep(ctx, 0.0, cfg.eps_pp)
        fits.append(float(i["residual_sq"]).hex())
    h = hashlib.sha256()
    for a in cp.cp_get_factors(ctx):
        h.update(np.ascontiguousarray(a).tobytes())
    print(json.dumps({"config": name, "r2": fits, "factors_sha256": h.hexdigest()}))


if __name__ == "__main__":
    main()
