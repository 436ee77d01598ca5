ARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"lc_(fmm|down)_kernel" -s 4 -c 2 -o gpurun_out/prof_fmm python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo rc=$?
tail -3 gpurun_out/plain.log
