# Round-2 evidence: smoke, default bench line (cfg2 + batched cfg3, cpu baselines), reference arm,
# standalone bench lines, the ncu launch list of the default bench command, ncu --set full captures
# of the dominant kernels (cfg2 engine 1, cfg3 engine 2, cfg4 engine 3), plan and NEXT-2 part times.
mkdir -p gpurun_out/ev
E=gpurun_out/ev
python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1; echo "smoke rc=$?"
LC_PARITY_LOG=$E/parity.jsonl timeout -k 10 1500 python -m pytest tests -m gpu -q -rf > $E/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $E/pytest_gpu.log
timeout -k 10 900 python bench.py > $E/bench_default.json 2> $E/bench_default.err; echo "bench rc=$?"
timeout -k 10 600 python bench.py --impl reference --steps 3 --warmup 3 > $E/bench_reference.json 2> $E/bench_reference.err; echo "ref rc=$?"
for c in cfg2b cfg3 cfg5 cfg4; do
  timeout -k 10 900 python bench.py --config $c --batched none --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 5 > $E/bench_$c.json 2> $E/bench_$c.err; echo "$c rc=$?"
done
timeout -k 10 300 python tools/part_times.py 1000000 1 2 4 8 > $E/part_times_1e6.txt 2>&1
timeout -k 10 300 python tools/part_times.py 10000000 1 2 4 8 > $E/part_times_1e7.txt 2>&1
timeout -k 10 300 python tools/part_times.py 1000000 1 2 4 8 --up > $E/part_up_1e6.txt 2>&1
timeout -k 10 300 python tools/part_times.py 10000000 1 2 4 8 --up > $E/part_up_1e7.txt 2>&1
# launch list of the default bench command (driver's K/W), then full captures of the top kernels
timeout -k 10 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $E/launches_default.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > $E/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:"lc_(up|stream|down)_kernel" -s 3 -c 3 -o $E/prof_cfg2 -f python tools/prof_cfg.py 1000000 1 3 > $E/ncu_cfg2.log 2>&1; echo "ncu cfg2 rc=$?"
timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:"lc_tile_kernel" -s 1 -c 1 -o $E/prof_cfg3 -f python tools/prof_cfg.py 4096 4096 2 > $E/ncu_cfg3.log 2>&1; echo "ncu cfg3 rc=$?"
timeout -k 10 1500 ncu --set full --clock-control none --import-source on -k regex:"lc_(up3|range)_kernel" -s 2 -c 2 -o $E/prof_cfg4 -f python tools/prof_cfg.py 10000000 64 2 > $E/ncu_cfg4.log 2>&1; echo "ncu cfg4 rc=$?"
ls -la $E
