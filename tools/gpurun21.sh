#!/bin/bash
python -m pytest tests/test_gpu_tucker.py -x -q 2>&1 | tail -3
timeout 600 python tools/tucker_bench.py 2>&1 | tail -4
python - <<'PY'
import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1811_10573_b200.cppp as cp
s, R, N = 400, 10, 3
r = np.random.default_rng(0)
X = r.standard_normal((s,)*N)
ctx = cp.tk_init(X, [s]*N, [R]*N)
cp.tk_set_factors(ctx, [np.linalg.qr(r.standard_normal((s, R)))[0].copy() for _ in range(N)])
for ph in ["dt", "pp-build", "pp-approx", "pp-approx"]:
    cp.tk_set_phase_override(ctx, ph); t = time.perf_counter(); cp.tk_sweep(ctx, 0, 0.2); print(ph, round((time.perf_counter()-t)*1e3, 2), "ms")
for n in range(3):
    t = time.perf_counter(); cp.tk_pp_update(ctx, n); print("pp_update", n, round((time.perf_counter()-t)*1e3, 2), "ms")
PY
