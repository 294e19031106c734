#!/usr/bin/env bash
# measure_round.sh OUTDIR — the round's measurement set on one B200 (run under gpurun from the
# repo root): bench lines of every config (value, roofline, cpu_baseline, e2e, clocks), the
# reference arm on C2, ncu launch lists of C2 and C4 (cold-cache, serialised: shares only) and
# `ncu --set full` captures of the top kernels, summarised by tools/ncu_summary.py.
set -x
O=${1:-gpurun_out/measure}; mkdir -p "$O"
(nproc; free -g; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv) > "$O/host.txt" 2>&1
for c in C2 C1 C3 C4 LAP P6W; do
  python bench.py --config $c --steps 5 --warmup 3 > "$O/bench_$c.json" 2> "$O/bench_$c.err"
done
python bench.py --config C5 --steps 2 --warmup 3 > "$O/bench_C5.json" 2> "$O/bench_C5.err"
# the paper's strong-scaling tensor (125 GB): device-resident only (its upload alone is ~2.3 s)
python bench.py --config P6S --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > "$O/bench_P6S.json" 2> "$O/bench_P6S.err"
python bench.py --impl reference --steps 2 --warmup 1 > "$O/bench_ref_C2.json" 2> "$O/bench_ref_C2.err"
for c in C2 C4 LAP; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$O/launches_$c.csv" \
    python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > "$O/ncu_l_$c.log" 2>&1
  python tools/ncu_summary.py launches "$O/launches_$c.csv" > "$O/launches_$c.md"
done
DM=sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_dmma.sum
ncu --set full --metrics $DM --clock-control none --import-source on -k regex:"ttm_dmma|pp_update_partial|ttv_pipe|ttv_kernel" -c 5 \
  -o "$O/full_C2" python tools/ncu_target.py C2 > "$O/ncu_full_C2.log" 2>&1
ncu --set full --metrics $DM --clock-control none --import-source on -k regex:"ttv_pair|ttm_dmma" -c 3 \
  -o "$O/full_C4" python tools/ncu_target.py C4 > "$O/ncu_full_C4.log" 2>&1
ncu --set full --clock-control none --import-source on -k regex:"skinny" -c 2 \
  -o "$O/full_LAP" python tools/ncu_target.py LAP > "$O/ncu_full_LAP.log" 2>&1
python tools/ncu_summary.py full "$O/full_LAP.ncu-rep" > "$O/ncu_full_LAP.json" 2>&1
python tools/ncu_summary.py full "$O/full_C2.ncu-rep" > "$O/ncu_full_C2.json" 2>&1
python tools/ncu_summary.py full "$O/full_C4.ncu-rep" > "$O/ncu_full_C4.json" 2>&1
ls -la "$O"
