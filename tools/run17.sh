bash tools/run13.sh > gpurun_out/r13.txt 2>&1
timeout 300 python tools/timeline.py 1000000 leg2cheb > gpurun_out/tl_cfg2.txt 2>&1
