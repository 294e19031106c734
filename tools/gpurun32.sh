#!/bin/bash
# two-warp factorization for 32 < K <= 64 (default) vs the CTA-wide chain (CPPP_NO_SMALL_FACTOR=1)
mkdir -p gpurun_out
./tools/probe_solve 50; ./tools/probe_solve 30 | tail -1; ./tools/probe_solve 10 | tail -1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for rep in 1 2; do
  for cfg in C3 C1 C4; do
    for v in small old; do
      if [ $v = old ]; then export CPPP_NO_SMALL_FACTOR=1; else unset CPPP_NO_SMALL_FACTOR; fi
      timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_${v}_${rep}.json 2>gpurun_out/ab_err.log
      python -c "import json,sys;d=json.loads(open('gpurun_out/ab_${cfg}_${v}_${rep}.json').read().strip().splitlines()[-1]);print('$cfg','$v',$rep,round(d['value'],2),round(d['ms_per_step'],3),d['gpu_launches'])"
    done
  done
done
