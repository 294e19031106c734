#!/bin/bash
# reserve-SM sweep for the order-3 overlapped TTM
for r in 0 2 4; do
  echo "reserve $r"; CPPP_TTM_RESERVE=$r python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
done
CPPP_TTM_RESERVE=2 python tools/trace.py --config C2 --sweeps 1,17 2>&1 | grep -v "^trace" | tail -40
