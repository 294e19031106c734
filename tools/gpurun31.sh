#!/bin/bash
# round-end refresh: GPU suite, bench lines C1-C5 + f4 workloads + reference arm, Tucker bench,
# ncu launch list and --set full capture of C2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
bash tools/gpurun18.sh
for c in P6W LAP; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -1 gpurun_out/bench_$c.json | cut -c1-160; done
timeout 600 python tools/tucker_bench.py --reps 3 > gpurun_out/tucker_bench.jsonl 2> gpurun_out/tucker.err; wc -l gpurun_out/tucker_bench.jsonl
