set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1; cat gpurun_out/fp64_peak.json
python - <<'PY' > gpurun_out/dgemm.json 2>&1
import torch, time, json
a=torch.randn(8192,8192,dtype=torch.float64,device='cuda'); b=torch.randn_like(a)
for _ in range(2): torch.matmul(a,b)
torch.cuda.synchronize(); best=0
for _ in range(5):
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); torch.matmul(a,b); e.record(); torch.cuda.synchronize()
    best=max(best, 2*8192**3/(s.elapsed_time(e)*1e-3)/1e12)
print(json.dumps({"cublas_dgemm_8192_tflops_burst": best}))
PY
cat gpurun_out/dgemm.json
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
