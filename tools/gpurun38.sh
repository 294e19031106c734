#!/bin/bash
# final bench lines C1-C4 (+ reference arm) and smoke after the Gram change
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for c in C1 C3 C4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
for c in C1 C2 C3 C4; do python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'e2e', d['e2e'] and round(d['e2e']['value'],1), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value'],3), 'roof', round(d['roofline']['achieved'],2), round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'], 'launches', d['gpu_launches'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C1.csv python bench.py --config C1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l1.log 2>&1; tail -1 gpurun_out/ncu_l1.log | cut -c1-60
