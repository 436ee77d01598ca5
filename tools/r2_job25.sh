mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_fullsize.py tests/test_gpu_memsafety.py tests/test_gpu_engines_sweep.py tests/test_gpu_configs.py -q -x -rf > gpurun_out/pytest25.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest25.log
timeout -k 10 900 python bench.py --config cfg4 --batched none --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench25_cfg4.json 2> gpurun_out/bench25_cfg4.err; echo "cfg4 rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/bench25_cfg4.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline_transform']['frac'], d['roofline']['frac'], d['kernel_ms']['leg2cheb'], d['kernel_ms']['cheb2leg'], d['round_trip_einf'])
"
