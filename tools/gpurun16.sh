mkdir -p gpurun_out
timeout 300 python tools/timeline.py --config C2 > gpurun_out/timeline_C2.log 2>&1; cat gpurun_out/timeline_C2.log
timeout 300 python tools/timeline.py --config C1 > gpurun_out/timeline_C1.log 2>&1; cat gpurun_out/timeline_C1.log
for c in C2 C3 C4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench16_$c.json 2> gpurun_out/bench16_$c.err; python -c "
import json; d=json.load(open('gpurun_out/bench16_$c.json')); print('$c', d['value'], {k:(round(v['ms_per_step'],2), round(v['frac'],3)) for k,v in d['roofline_all'].items()})"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gamma_chol|solve_rows|gram_reduce|ttv_split" -s 40 -c 8 -o gpurun_out/prof_solve python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_solve.log 2>&1; tail -1 gpurun_out/ncu_solve.log
