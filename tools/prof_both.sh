ARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"lc_(up|m2l|down)_kernel" -s 12 -c 3 -o gpurun_out/prof_v5 python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo rc=$?
