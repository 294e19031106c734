#!/bin/bash
# spacer gated on operator size: C1 should match CPPP_NO_STAGGER, C2 keep the spacer
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for rep in 1 2; do
  for cfg in C1 C2 C4; do
    timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_${rep}.json 2>gpurun_out/ab_err.log
    python -c "import json,sys;d=json.loads(open('gpurun_out/ab_${cfg}_${rep}.json').read().strip().splitlines()[-1]);print('$cfg',$rep,round(d['value'],2),round(d['ms_per_step'],3),d['gpu_launches'])"
  done
done
