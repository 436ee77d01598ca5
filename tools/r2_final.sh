# Final round-2 check after the down-kernel changes: smoke, the whole GPU suite (parity log), the default
# bench line and cfg2b, the ncu launch list of the default bench command and a --set full capture of cfg2.
mkdir -p gpurun_out/fin
E=gpurun_out/fin
python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1; echo "smoke rc=$?"
LC_PARITY_LOG=$E/parity.jsonl timeout -k 10 1500 python -m pytest tests -m gpu -q -rf > $E/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $E/pytest_gpu.log
timeout -k 10 900 python bench.py > $E/bench_default.json 2> $E/bench_default.err; echo "bench rc=$?"
timeout -k 10 900 python bench.py --config cfg2b --batched none --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 5 > $E/bench_cfg2b.json 2> $E/bench_cfg2b.err; echo "cfg2b rc=$?"
timeout -k 10 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $E/launches_default.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > $E/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:"lc_(up|stream|down)_kernel" -s 3 -c 3 -o $E/prof_cfg2 -f python tools/prof_cfg.py 1000000 1 3 > $E/ncu_cfg2.log 2>&1; echo "ncu cfg2 rc=$?"
