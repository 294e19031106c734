mkdir -p gpurun_out

timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in C2 C1 C3 C4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b17_$c.json 2> gpurun_out/b17_$c.err; tail -2 gpurun_out/b17_$c.err; python -c "
import json; d=json.load(open('gpurun_out/b17_$c.json')); print('$c', round(d['value'],1), round(d['ms_per_step'],3), 'prof', round(d['profiled_ms_per_step'],3), {k:(round(v['ms_per_step'],3), v['launches_per_step'], round(v['frac'],3)) for k,v in d['roofline_all'].items()})"; done
