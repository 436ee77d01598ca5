# ncu evidence: launch lists of the bench commands (cfg2 default workload, cfg3), --set full of the kernels
mkdir -p gpurun_out
ARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3"
python bench.py $ARGS > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py $ARGS > gpurun_out/ncu_l2.log 2>&1; echo l2 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"lc_(up|stream|down)_kernel" -s 6 -c 3 -o gpurun_out/prof_cfg2 -f python bench.py $ARGS > gpurun_out/ncu_f2.log 2>&1; echo f2 rc=$?
python bench.py --config cfg3 $ARGS > gpurun_out/plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --config cfg3 $ARGS > gpurun_out/ncu_l3.log 2>&1; echo l3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"lc_tile_kernel" -s 2 -c 1 -o gpurun_out/prof_cfg3 -f python bench.py --config cfg3 $ARGS > gpurun_out/ncu_f3.log 2>&1; echo f3 rc=$?
