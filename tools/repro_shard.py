"""Single-thread reproduction of the sharded path: rank 0 of world 2 with a fake host all-reduce
(doubles the buffer).  Numbers are meaningless; used under compute-sanitizer to find faults."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synthgen as G
import paper_1811_10573_b200.cppp as cp
cfg = G.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
X = G.make_tensor(cfg); A0 = G.initial_factors(cfg)
lo, hi = 0, cfg.s // 2
def red(buf):
    buf *= 2.0
ctx = cp.cp_init(np.ascontiguousarray(X[lo:hi]), cfg.N, cfg.dims, cfg.K, shard_offset=lo, shard_extent=hi - lo,
                 rank=0, world=2, torch_workspace=False, host_allreduce=red)
print("init ok", flush=True)
cp.cp_set_factors(ctx, A0); print("set ok", flush=True)
cp.mttkrp_dt(ctx); print("mttkrp ok", flush=True)
cp.pp_build_operators(ctx); print("build ok", flush=True)
for n in range(cfg.N): cp.pp_update(ctx, n)
print("update ok", flush=True)
cp.cp_set_factors(ctx, A0)
for ph in ["dt", "dt", "pp-build", "pp-approx", "dt"]:
    cp.cp_set_phase_override(ctx, ph); cp.als_sweep(ctx, 0.0, 0.1)
print("sweeps ok", flush=True)
cp.cp_get_factors(ctx); print("all ok")
