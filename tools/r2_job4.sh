mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu_planner.py tests/test_alg3_crosscheck.py -q -rf -s > gpurun_out/pytest4.log 2>&1; echo "pytest rc=$?"
grep "Gauss-node\|passed\|failed\|Error" gpurun_out/pytest4.log | head -20
timeout -k 10 300 python tools/timeline.py 1000000 leg2cheb > gpurun_out/tl_cfg2.txt 2>&1; echo "tl rc=$?"
cat gpurun_out/tl_cfg2.txt
