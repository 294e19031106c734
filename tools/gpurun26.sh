#!/bin/bash
# in-place factor read except on the side stream, vs padded copy (CPPP_PAD_FACTOR=1)
mkdir -p gpurun_out
for rep in 1 2 3; do
  for cfg in C2 C1; do
    for v in direct pad; do
      if [ $v = pad ]; then export CPPP_PAD_FACTOR=1; else unset CPPP_PAD_FACTOR; fi
      timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${cfg}_${v}_${rep}.json 2>gpurun_out/ab_err.log
      python -c "import json,sys;d=json.loads(open('gpurun_out/ab_${cfg}_${v}_${rep}.json').read().strip().splitlines()[-1]);print('$cfg','$v',$rep,round(d['value'],1),round(d['ms_per_step'],3),d['e2e']['value'] if d.get('e2e') else None,d['gpu_launches'],d['roofline']['frac'])"
    done
  done
done
