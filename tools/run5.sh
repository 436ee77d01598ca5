mkdir -p gpurun_out
timeout 300 python tools/timeline.py 1000000 leg2cheb > gpurun_out/tl_cfg2.txt 2>&1; echo tl rc=$?
head -14 gpurun_out/tl_cfg2.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lc_up_kernel" -s 2 -c 1 -o gpurun_out/up_cfg2 python tools/prof_cfg.py 1000000 1 3 > gpurun_out/ncu_up.log 2>&1; echo ncu up rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lc_stream_kernel" -s 2 -c 1 -o gpurun_out/stream_cfg2 python tools/prof_cfg.py 1000000 1 3 > gpurun_out/ncu_stream.log 2>&1; echo ncu stream rc=$?
tail -3 gpurun_out/ncu_stream.log
