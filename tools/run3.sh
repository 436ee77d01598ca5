mkdir -p gpurun_out
./tools/ubench_const > gpurun_out/ubench_const.txt 2>&1; cat gpurun_out/ubench_const.txt
timeout 300 python tools/timeline.py 1000000 leg2cheb > gpurun_out/tl_cfg2.txt 2>&1; echo tl rc=$?
head -14 gpurun_out/tl_cfg2.txt
