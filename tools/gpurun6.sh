set -x
./tools/probe_solve
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; tail -3 gpurun_out/bench_C2.err
for c in C1 C3 C4; do python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; done
./tools/probe_solve > /dev/null && ncu --set full --clock-control none --import-source on -k regex:"solve_rows|gamma_inverse" -s 60 -c 2 -o gpurun_out/prof_solve2 ./tools/probe_solve > gpurun_out/ncu_solve.log 2>&1; tail -2 gpurun_out/ncu_solve.log
