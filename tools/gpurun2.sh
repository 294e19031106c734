set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; tail -5 gpurun_out/bench_C2.err; cat gpurun_out/bench_C2.json
for c in C1 C3 C4; do python bench.py --config $c --steps 3 --warmup 2 --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; cat gpurun_out/bench_$c.json; done
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; tail -3 gpurun_out/ncu_launches.log
ncu --set full --clock-control none --import-source on -k regex:ttm_dmma -s 2 -c 2 -o gpurun_out/prof_ttm_C2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ttm.log 2>&1; tail -3 gpurun_out/ncu_ttm.log
ncu --set full --clock-control none --import-source on -k regex:pp_update_partial -s 3 -c 2 -o gpurun_out/prof_pp_C2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pp.log 2>&1; tail -3 gpurun_out/ncu_pp.log
ls -la gpurun_out
