#!/bin/bash
# MR=1 vs MR=2 on the TTM shapes of C3/C4/P6W/LAP (KRP GEMMs) and C2, C3 middle modes
for mr in 1 2; do
  echo "== MR $mr"
  for shape in "10000 10000 1 50" "8000 8000 1 30" "32768 32768 1 4" "15625 15625 1 2" "160000 400 1 100" "100 100 10000 50" "400 400 400 100" "1 100 1000000 50" "50 20 64000 30"; do
    CPPP_TTM_MR=$mr ./tools/probe_ttm $shape | head -1
  done
done
