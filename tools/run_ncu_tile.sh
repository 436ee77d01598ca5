mkdir -p gpurun_out
python tools/prof_cfg.py 4096 4096 2 leg2cheb 0 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lc_tile_kernel" -s 1 -c 1 -o gpurun_out/prof_tile -f python tools/prof_cfg.py 4096 4096 2 leg2cheb 0 > gpurun_out/ncu_tile.log 2>&1
echo ncu rc=$?
