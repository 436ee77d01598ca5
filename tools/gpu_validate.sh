mkdir -p gpurun_out/v1
E=gpurun_out/v1
python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1; echo "smoke rc=$?"
LC_PARITY_LOG=$E/parity.jsonl timeout -k 10 1500 python -m pytest tests -m gpu -q -rf -x > $E/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $E/pytest_gpu.log
timeout -k 10 900 python bench.py > $E/bench_default.json 2> $E/bench_default.err; echo "bench rc=$?"; tail -c 3000 $E/bench_default.json
