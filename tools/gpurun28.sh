#!/bin/bash
# stream-K only for splits whose last wave is < 95% full; A/B vs CPPP_NO_STREAMK=1 on C3, C4, P6W, LAP and the Tucker shapes
mkdir -p gpurun_out
for rep in 1 2; do
  for cfg in C3 C4 P6W LAP; do
    for v in sk uni; do
      if [ $v = uni ]; then export CPPP_NO_STREAMK=1; else unset CPPP_NO_STREAMK; fi
      timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_${v}_${rep}.json 2>gpurun_out/ab_err.log
      python -c "import json,sys;d=json.loads(open('gpurun_out/ab_${cfg}_${v}_${rep}.json').read().strip().splitlines()[-1]);print('$cfg','$v',$rep,round(d['value'],2),round(d['ms_per_step'],3),d['gpu_launches'],d['roofline']['frac'])"
    done
  done
done
for v in sk uni; do
  if [ $v = uni ]; then export CPPP_NO_STREAMK=1; else unset CPPP_NO_STREAMK; fi
  echo "tucker $v"; timeout 300 python tools/tucker_bench.py --reps 3 2>&1 | tail -3
done
