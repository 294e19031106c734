#!/bin/bash
# Gram: single-CTA fast path + fused last-tile statistics (in-tree) vs HEAD (tools/ab/libcppp_base.so)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for rep in 1 2; do
  for cfg in C4 C2 C1; do
    for v in new base; do
      if [ $v = base ]; then export CPPP_LIB=$PWD/tools/ab/libcppp_base.so; else unset CPPP_LIB; fi
      timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_${v}_${rep}.json 2>gpurun_out/ab_err.log
      python -c "import json,sys;d=json.loads(open('gpurun_out/ab_${cfg}_${v}_${rep}.json').read().strip().splitlines()[-1]);print('$cfg','$v',$rep,round(d['value'],2),round(d['ms_per_step'],3))"
    done
  done
done
