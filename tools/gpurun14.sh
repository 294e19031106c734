timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; tail -3 gpurun_out/bench_C2.err
for c in C1 C3 C4; do python bench.py --config $c --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_C2.json 2> gpurun_out/bench_ref.err; tail -2 gpurun_out/bench_ref.err
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; tail -1 gpurun_out/ncu_launches.log
ncu --set full --clock-control none --import-source on -k regex:"ttm_dmma|pp_update_partial" -s 6 -c 4 -o gpurun_out/prof_C2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
