# round 2, job 2: planner pin + memory-safety tests, then the new bench (default line incl. batched)
mkdir -p gpurun_out
export LC_PARITY_LOG=gpurun_out/parity2.jsonl
timeout -k 10 900 python -m pytest tests/test_gpu_planner.py tests/test_gpu_memsafety.py tests/test_gpu_parity.py tests/test_gpu_boundary.py -q -rf -s --durations=10 > gpurun_out/pytest2.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest2.log
timeout -k 10 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
tail -5 gpurun_out/bench_default.err
timeout -k 10 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
