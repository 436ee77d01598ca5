set -x
python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err
tail -c 3000 gpurun_out/bench_default.err
ARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lc_down_kernel -s 4 -c 1 -o gpurun_out/prof_down python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo done rc=$?
