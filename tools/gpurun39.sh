#!/bin/bash
# PP-sweep spacer kernel on/off (CPPP_NO_STAGGER=1) across configs
mkdir -p gpurun_out
for rep in 1 2; do
  for cfg in C1 C2 C3 C4; do
    for v in on off; do
      if [ $v = off ]; then export CPPP_NO_STAGGER=1; else unset CPPP_NO_STAGGER; fi
      timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_${v}_${rep}.json 2>gpurun_out/ab_err.log
      python -c "import json,sys;d=json.loads(open('gpurun_out/ab_${cfg}_${v}_${rep}.json').read().strip().splitlines()[-1]);print('$cfg','$v',$rep,round(d['value'],2),round(d['ms_per_step'],3))"
    done
  done
done
