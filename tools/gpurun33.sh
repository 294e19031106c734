#!/bin/bash
# stream-K over 146 CTAs (two SMs free) vs the uniform split (CPPP_NO_STREAMK=1)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
CPPP_DEBUG_TTM=1 ./tools/probe_ttm 1 10000 10000 50 2>&1 | head -3
for rep in 1 2; do
  for v in sk uni; do
    if [ $v = uni ]; then export CPPP_NO_STREAMK=1; else unset CPPP_NO_STREAMK; fi
    timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_C3_${v}_${rep}.json 2>gpurun_out/ab_err.log
    python -c "import json,sys;d=json.loads(open('gpurun_out/ab_C3_${v}_${rep}.json').read().strip().splitlines()[-1]);print('C3','$v',$rep,round(d['value'],2),round(d['ms_per_step'],3),round(d['roofline']['frac'],3))"
  done
done
