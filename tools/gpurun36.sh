#!/bin/bash
# ncu --set full of the C3 stream-K multi-mode GEMM and of C1's one-warp factorization
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ttm_dmma -s 3 -c 1 -o gpurun_out/prof_C3_sk ./tools/probe_ttm 1 10000 10000 50 > gpurun_out/ncu_c3.log 2>&1; tail -1 gpurun_out/ncu_c3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gamma_small -s 20 -c 2 -o gpurun_out/prof_C1_factor python bench.py --config C1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1; tail -1 gpurun_out/ncu_c1.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C1.csv python bench.py --config C1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l1.log 2>&1; tail -1 gpurun_out/ncu_l1.log | cut -c1-80
