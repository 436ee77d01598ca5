# Round-1 evidence: smoke, default bench line (cfg2, with cpu_baseline), reference arm, batched bench
# lines, ncu launch list of the default bench command and one --set full capture of the 3 kernels.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref rc=$?
for c in cfg3 cfg5 cfg4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?
done
ARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"lc_(up|stream|down)_kernel" -s 6 -c 3 -o gpurun_out/prof_r1 -f python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo ncu rc=$?
