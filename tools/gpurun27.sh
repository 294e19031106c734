#!/bin/bash
# stream-K split of the multi-mode first level (default) vs the uniform k split (CPPP_NO_STREAMK=1)
mkdir -p gpurun_out
for a in "1 10000 10000 50" "10000 10000 1 50" "1 8000 8000 30" "8000 8000 1 30" "1 65536 65536 128"; do
  for v in 1 0; do
    if [ $v = 1 ]; then export CPPP_NO_STREAMK=1; else unset CPPP_NO_STREAMK; fi
    echo "== $a no_sk=$v"; CPPP_DEBUG_TTM=1 timeout 120 ./tools/probe_ttm $a 2>&1 | grep -v "no error\|first-wave" | tail -4
  done
done
unset CPPP_NO_STREAMK
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2; do
  for cfg in C3 C4; do
    for v in sk uni; do
      if [ $v = uni ]; then export CPPP_NO_STREAMK=1; else unset CPPP_NO_STREAMK; fi
      timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_${v}_${rep}.json 2>gpurun_out/ab_err.log
      python -c "import json,sys;d=json.loads(open('gpurun_out/ab_${cfg}_${v}_${rep}.json').read().strip().splitlines()[-1]);print('$cfg','$v',$rep,round(d['value'],1),round(d['ms_per_step'],3),d['gpu_launches'],d['roofline']['frac'])"
    done
  done
done
for v in sk uni; do
  if [ $v = uni ]; then export CPPP_NO_STREAMK=1; else unset CPPP_NO_STREAMK; fi
  timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_C5_${v}.json 2>gpurun_out/ab_err.log
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab_C5_${v}.json').read().strip().splitlines()[-1]);print('C5','$v',round(d['value'],2),round(d['ms_per_step'],3),d['roofline']['frac'])"
done
