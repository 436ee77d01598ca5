mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/timeline.py 1000000 leg2cheb > gpurun_out/tl_cfg2.txt 2>&1; echo tl rc=$?
timeout 300 python tools/timeline.py 4096 leg2cheb batch=4096 > gpurun_out/tl_cfg3.txt 2>&1; echo tl3 rc=$?
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.txt
