mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; tail -2 gpurun_out/bench_C2.err
for c in C1 C3 C4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; done
timeout 1200 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; tail -2 gpurun_out/bench_C5.err
for c in C1 C2 C3 C4 C5; do python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'e2e', d['e2e'] and round(d['e2e']['value'],1), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value'],3), 'roof', d['roofline']['kernel'], round(d['roofline']['achieved'],2), d['roofline']['unit'], round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_C2.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref_C2.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; tail -1 gpurun_out/ncu_launches.log | cut -c1-100
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ttm_dmma|pp_update_partial|ttv_kernel|solve_rows|gram_kernel" -s 12 -c 10 -o gpurun_out/prof_C2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
