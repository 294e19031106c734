#!/bin/bash
mkdir -p gpurun_out
./tools/probe_ttm 50 20 64000 30 | head -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ttm_dmma -s 3 -c 1 -o gpurun_out/prof_ttm_s20 ./tools/probe_ttm 50 20 64000 30 > gpurun_out/ncu_s20.log 2>&1; tail -2 gpurun_out/ncu_s20.log
