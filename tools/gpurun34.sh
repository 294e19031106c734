#!/bin/bash
# final check: GPU suite, smoke, C3 bench line (stream-K on 146 CTAs), C2 default line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --config C3 --steps 5 --warmup 3 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
timeout 900 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for c in C2 C3; do python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'e2e', d['e2e'] and round(d['e2e']['value'],1), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value'],3), 'roof', round(d['roofline']['achieved'],2), round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
