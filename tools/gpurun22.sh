#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tk_T3.csv python tools/tucker_bench.py --workloads T3 --reps 2 > gpurun_out/tk_ncu.log 2>&1
python tools/ncu_summary.py launches gpurun_out/tk_T3.csv | head -20
