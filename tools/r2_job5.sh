# ncu --set full of the cfg2 up and down kernels (source-correlated) + isolated per-kernel view
mkdir -p gpurun_out
python tools/prof_cfg.py 1000000 1 3 > gpurun_out/plain5.log 2>&1 && \
timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:"lc_(up|down|stream)_kernel" -s 3 -c 3 -o gpurun_out/prof5_cfg2 -f python tools/prof_cfg.py 1000000 1 3 > gpurun_out/ncu5.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu5.log
