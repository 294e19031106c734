timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; tail -3 gpurun_out/bench_C2.err
for c in C1 C3 C4; do python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; done
