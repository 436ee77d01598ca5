mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lc_stream_kernel" -s 2 -c 1 -o gpurun_out/stream_cfg2 -f python tools/prof_cfg.py 1000000 1 3 > gpurun_out/ncu_stream.log 2>&1; echo ncu stream rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lc_down_kernel" -s 2 -c 1 -o gpurun_out/down_cfg2 -f python tools/prof_cfg.py 1000000 1 3 > gpurun_out/ncu_down.log 2>&1; echo ncu down rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lc_up_kernel" -s 2 -c 1 -o gpurun_out/up_cfg2 -f python tools/prof_cfg.py 1000000 1 3 > gpurun_out/ncu_up.log 2>&1; echo ncu up rc=$?
