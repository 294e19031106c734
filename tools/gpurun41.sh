#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --config C1 --steps 5 --warmup 3 > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err
timeout 900 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for c in C1 C2; do python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'e2e', d['e2e'] and round(d['e2e']['value'],1), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value'],3), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'], 'launches', d['gpu_launches'])"; done
