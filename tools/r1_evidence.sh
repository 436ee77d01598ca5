# Round-1 evidence: smoke, default bench line, ncu launch list, one --set full capture of the 3 kernels.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench rc=$?
tail -c 2000 gpurun_out/bench_default.err
ARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"lc_(up|stream|down)_kernel" -s 6 -c 3 -o gpurun_out/prof_r1 python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo ncu rc=$?
