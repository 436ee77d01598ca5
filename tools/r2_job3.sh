# round 2, job 3: planner pins (new planner kernels), Alg. 3 cross-check on the GPU, plan time
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu_planner.py tests/test_alg3_crosscheck.py tests/test_gpu_parity.py tests/test_gpu_configs.py -q -rf -s --durations=10 > gpurun_out/pytest3.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest3.log
python - <<'PY' > gpurun_out/plan_time.txt 2>&1
import torch, time
from paper_2411_00033_b200 import Plan
for n, V in ((1_000_000, 1), (1 << 20, 1), (10_000_000, 1), (4096, 4096), (8192, 8192)):
    for d in ("leg2cheb", "cheb2leg"):
        ts = []
        for _ in range(3):
            torch.cuda.synchronize(); t = time.perf_counter(); p = Plan(n, d, batch=V); w = (time.perf_counter() - t) * 1e3
            ts.append((p.plan_device_ms, w)); p.close()
        print(n, V, d, "device_ms", [round(a, 3) for a, _ in ts], "wall_ms", [round(b, 1) for _, b in ts])
PY
cat gpurun_out/plan_time.txt
