# parity tests then one default bench line
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 2>&1 | tail -15
timeout 600 python bench.py --cpu-seconds 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
