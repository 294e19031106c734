./tools/probe_solve
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
./tools/probe_solve > /dev/null && ncu --set full --clock-control none --import-source on -k regex:"solve_rows" -s 82 -c 1 -o gpurun_out/prof_rows3 ./tools/probe_solve > gpurun_out/ncu_rows.log 2>&1; tail -1 gpurun_out/ncu_rows.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; tail -3 gpurun_out/bench_C2.err
