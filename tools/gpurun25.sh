#!/bin/bash
# in-place factor read (default) vs padded copy (CPPP_PAD_FACTOR=1): GPU parity, then alternating bench lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2; do
  for cfg in C1 C2 C4 C3; do
    for v in direct pad; do
      if [ $v = pad ]; then export CPPP_PAD_FACTOR=1; else unset CPPP_PAD_FACTOR; fi
      timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${cfg}_${v}_${rep}.json 2>gpurun_out/ab_err.log
      python -c "import json,sys;d=json.loads(open('gpurun_out/ab_${cfg}_${v}_${rep}.json').read().strip().splitlines()[-1]);print('$cfg','$v',$rep,round(d['value'],1),round(d['ms_per_step'],3),d['e2e']['value'] if d.get('e2e') else None,d['gpu_launches'],d['roofline']['frac'])"
    done
  done
done
