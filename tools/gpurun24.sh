#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tk_T6W.csv python tools/tucker_bench.py --workloads T6W --reps 2 > gpurun_out/tk6.log 2>&1
python tools/ncu_summary.py launches gpurun_out/tk_T6W.csv | head -16
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/tk_T6W.csv')))
h=None
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=r; start=i; break
ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size') if 'Grid Size' in h else None
agg=collections.defaultdict(list)
for r in rows[start+1:]:
    if len(r)==len(h) and r[ki].startswith('ttm_dmma'):
        agg[(r[ki], r[gi] if gi is not None else '')].append(float(r[vi].replace(',','')))
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1]))[:10]: print(k, len(v), round(sum(v)/len(v),1))
PY
